/* helmtg_b200.h -- C-ABI of the B200-native two-grid Helmholtz hot path.
 *
 * One opaque handle owns everything the iteration needs on one GPU (the
 * equivalent of helmtg::TwoGridOperators, proj/core/include/helmtg/twogrid.hpp:92-105).
 * Vectors are complex fp64 in the reference dof order, interleaved
 * (re, im) -- layout-compatible with Eigen::VectorXcd::data(),
 * std::complex<double>[] and cuDoubleComplex[]. Unless a function says "host",
 * vector arguments are DEVICE pointers; calls are stream-ordered on the
 * handle's stream and never allocate.
 *
 * Status codes mirror the reference CLI (proj/tools/main.cpp:22-35,
 * proj/core/src/commands.cpp:156): 0 ok, 1 runtime / CUDA error,
 * 2 invalid argument (config or geometry), 3 not converged.
 * htg_last_error() returns the message of the last failure on this thread.
 */
#ifndef HELMTG_B200_H
#define HELMTG_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HTG_OK 0
#define HTG_ERR_RUNTIME 1
#define HTG_ERR_INVALID 2
#define HTG_NOT_CONVERGED 3

/* proj/core/include/helmtg/mesh.hpp:15 */
enum htg_tag { HTG_DIRICHLET = 0, HTG_NEUMANN = 1, HTG_ABSORBING = 2 };
/* proj/core/include/helmtg/twogrid.hpp:14-16 */
enum htg_coarse { HTG_COARSE_OPTIMIZED_FD = 0, HTG_COARSE_GALERKIN_P = 1, HTG_COARSE_NONE = 2 };
enum htg_smoother { HTG_SMOOTHER_CSDD = 0, HTG_SMOOTHER_EXACT_SHIFTED = 1 };
enum htg_outer { HTG_OUTER_RICHARDSON = 0, HTG_OUTER_KRYLOV = 1 };

/* A rectangle of nx x ny square cells of side h, order-p hierarchical Q_p
 * space (p in {2,4,6,8}): the mesh/space/coefficients/tags triple that
 * setup_two_grid takes (proj/core/include/helmtg/twogrid.hpp:107-108).
 * k_cells / eps_cells: per-cell values in (y, x) order, or NULL for the
 * constants. tags_*: per boundary edge (bottom/top indexed by x, left/right by
 * y), or NULL to use side_tags[] = {left, right, bottom, top}. */
typedef struct htg_problem {
    int order;
    int nx, ny;
    double h;
    double k_const, eps_const;
    const double* k_cells;
    const double* eps_cells;
    int side_tags[4];
    const int* tags_bottom;
    const int* tags_right;
    const int* tags_top;
    const int* tags_left;
    /* element kind (appended; zero = squares): HTG_ELEM_SQUARE, or HTG_ELEM_TRIANGLE
     * for cells split along the (0,0)-(1,1) diagonal (ElementKind::Triangle,
     * proj/core/include/helmtg/mesh.hpp) */
    int element_kind;
} htg_problem;
#define HTG_ELEM_SQUARE 0
#define HTG_ELEM_TRIANGLE 1

/* proj/core/include/helmtg/twogrid.hpp:18-30, same fields and defaults
 * (htg_config_default). */
typedef struct htg_config {
    double alpha_s, alpha_c;
    int n_s, n_dd;
    double omega_c;
    int l_dd;
    int coarsening, smoother, outer;
    double stop_rel_residual;
    int max_iters;
} htg_config;

typedef struct htg_handle htg_handle;

void htg_config_default(htg_config* cfg);
const char* htg_last_error(void);

/* setup_two_grid (twogrid.cpp:221-253): host setup, upload to HBM.
 *   smoother CSDD: subdomain classes and their restricted inverses / fast
 *     diagonalisation factors; ExactShifted: nested-dissection LU of the fine
 *     shifted operator A_s (u += A_s^-1 (f - A u), twogrid.cpp:257-264);
 *   coarsening OptimizedFD: the QSFEM operator (qsfem.cpp:118-149); GalerkinP:
 *     the order-p/2 Helmholtz operator with alpha_c and the inclusion IP
 *     (twogrid.cpp:189-219); both factored by nested dissection.
 * stream: the cudaStream_t every call of this handle is ordered on (NULL: the
 * legacy default stream). */
int htg_create(const htg_problem* prob, const htg_config* cfg, void* stream, htg_handle** out);
int htg_destroy(htg_handle* h);

/* out[0] ndof, [1] coarse ndof, [2] subdomains, [3] subdomain classes,
 * [4] device bytes held, [5] coarse factor bytes, [6] nx, [7] ny, [8] order,
 * [9] algorithmic flops of one sweep's subdomain solves on the path used
 * (fast diagonalisation for separable classes, 8 |U_i| |Omega_i| otherwise),
 * [10] nested-dissection levels of the coarse solver, [11] the dense-path
 * flops 8 |U_i| |Omega_i| summed, [12] subdomains solved by fast
 * diagonalisation, [13] CUDA graphs cached by the handle (bounded LRU),
 * [14] sum of |U_i| (values staged per sweep), [15] sum of |Omega_i| (values
 * gathered per sweep), [16] algorithmic bytes one coarse solve reads,
 * [17] subdomains with their own device-factored solver (no shared factor),
 * [18] bytes of those factors, [19] dense-path subdomain classes whose explicit
 * restricted inverse was computed on the device. out must hold 20 entries. */
int htg_info(const htg_handle* h, long long* out);
int htg_set_stream(htg_handle* h, void* stream);

/* K1: r = f - A u (shifted=0) or f - A_s u (shifted=1); the Eigen products
 * of twogrid.cpp:94,116,272,287. */
int htg_residual(htg_handle* h, const double* f, const double* u, double* r, int shifted);
/* ||f - A u||_2 written to *out (host); the stopping test of twogrid.cpp:287. */
int htg_residual_norm(htg_handle* h, const double* f, const double* u, double* out);
/* dd_step (twogrid.cpp:92-112): out = PoU-average of R_i u + (A_s^(i))^-1 R_i (f - A_s u).
 * dd_step and csdd_smoother need smoother = CSDD (else HTG_ERR_INVALID). */
int htg_dd_step(htg_handle* h, const double* u, const double* f, double* out);
/* csdd_smoother (twogrid.cpp:114-120), u updated in place. */
int htg_csdd_smoother(htg_handle* h, double* u, const double* f);
/* K3a: rc = IP^H r (twogrid.cpp:272); the transfers and the coarse calls
 * need coarsening != None (else HTG_ERR_INVALID). */
int htg_restrict(htg_handle* h, const double* r, double* rc);
/* K1+K3a fused: rc = IP^H (f - A u), the fine residual never materialised. */
int htg_residual_restrict(htg_handle* h, const double* f, const double* u, double* rc);
/* K3b: u += omega * IP uc (twogrid.cpp:273). */
int htg_prolong_add(htg_handle* h, double* u, const double* uc, double omega);
/* K4: y = A_c x, the QSFEM coarse stencil (qsfem.cpp:118-149), or the
 * GalerkinP coarse matrix (CSR). */
int htg_coarse_apply(htg_handle* h, const double* x, double* y);
/* uc = A_c^-1 rc by the factored coarse operator (twogrid.cpp:273). */
int htg_coarse_solve(htg_handle* h, const double* rc, double* uc);
/* two_grid_step (twogrid.cpp:268-276), u updated in place. */
int htg_two_grid_step(htg_handle* h, double* u, const double* f);
/* solve (twogrid.cpp:278-331) from u = 0: u (device, ndof) receives the
 * solution, history (host, capacity hist_cap) the relative residuals.
 * Returns HTG_NOT_CONVERGED when max_iters is reached. */
int htg_solve(htg_handle* h, const double* f, double* u, double* history, int hist_cap, int* iterations,
              int* converged);
/* Host-buffer variants: copies in/out inside the call (the end-to-end path). */
int htg_solve_host(htg_handle* h, const double* f_host, double* u_host, double* history, int hist_cap,
                   int* iterations, int* converged);
int htg_two_grid_step_host(htg_handle* h, double* u_host, const double* f_host);
int htg_csdd_smoother_host(htg_handle* h, double* u_host, const double* f_host);

/* Measured FP64 tensor-core (DMMA) throughput of this GPU, TFLOP/s (the
 * roofline denominator of the dense subdomain batch). */
int htg_measure_fp64_tensor_peak(double* tflops);
/* Per-phase device time (ms, CUDA events on the handle's stream, mean of reps;
 * every rep starts on a cold L2, a 256 MB write outside the events):
 * [0] K1 residual, [1] K2 batched subdomain GEMM, [2] K2 PoU combine,
 * [3] K1+K3a residual-restrict, [4] coarse solve, [5] K3b prolongation,
 * [6] K1 residual norm, [7] csdd_smoother sweep, [8] two_grid_step,
 * [9] K4 coarse stencil, [10] smoother sweep, [11] two_grid_step and [12]
 * coarse solve replayed as CUDA graphs (the form the public entry points use).
 * u is overwritten. ms must hold 13 entries. */
int htg_profile(htg_handle* h, double* u, const double* f, int reps, double* ms);
/* Kernel-launch accounting: launches of this library's kernels since the last reset. */
long long htg_launch_count(void);
void htg_reset_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* HELMTG_B200_H */
