// kernels.hpp -- launch interfaces of the helmtg_b200 CUDA kernels.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "common.hpp"

namespace htg {

enum K1Mode { kK1Write = 0, kK1Norm = 1, kK1Restrict = 2 };

struct K1Args {
    FineGeom g;
    const double2* __restrict__ u;
    const double2* __restrict__ f;
    double2* r;        // kK1Write
    double* partial;   // kK1Norm: one partial sum per CTA
    double2* rc;       // kK1Restrict
    int rows;          // lattice rows per CTA
    int shifted;       // use A_s (alpha_s) instead of A
};

// launch accounting (htg_launch_count)
void count_launch(int n = 1);

void upload_basis_tables(const double* M, const double* S, const double* E, int slot);

// K1: r = f - A u; returns the number of partial sums for kK1Norm
int k1_launch(int mode, const K1Args& a, cudaStream_t st);
int k1_partials(const FineGeom& g, int rows);
void reduce_partials(const double* partial, int n, double* out, cudaStream_t st);

// K1 on triangle meshes: r = f - A u (A_s when shifted) from the combined cell
// operator KMc = [K_c | M_c] ((p+1)^2 x (p+1)^2 each, lattice-node order)
void tri_residual_launch(const FineGeom& g, const double* KMc, const double2* u, const double2* f, double2* r,
                         int shifted, cudaStream_t st);
size_t tri_residual_smem(int p);

// K3b: u += omega IP uc
void prolong_add_launch(const FineGeom& g, double2* u, const double2* uc, double omega, cudaStream_t st);
// K4: y = A_c x (QSFEM)
void coarse_apply_launch(const FineGeom& g, const double4* qtab, double hc, const double2* x, double2* y,
                         cudaStream_t st);

// GalerkinP transfers (inclusion IP: coarse dof i <-> fine dof map[i], -1 for Dirichlet)
void inclusion_restrict_launch(const double2* r, const int* map, long long nc, double2* rc, cudaStream_t st);
void inclusion_prolong_launch(double2* u, const int* map, long long nc, const double2* uc, double omega,
                              cudaStream_t st);
// y = A x, complex CSR (GalerkinP coarse operator)
void csr_apply_launch(const int* rp, const int* ci, const double2* v, long long n, const double2* x, double2* y,
                      cudaStream_t st);

// timing only: read `bytes` of buf (evicts and writes back dirty L2 lines)
void l2_read(const void* buf, size_t bytes, double* sink, cudaStream_t st);

// complex CSR: mode 0 y = A x, 1 y = f - A x, 2 y += omega A x
void csr_launch(int mode, const int* rp, const int* ci, const double2* v, long long n, const double2* x,
                const double2* f, double omega, double2* y, cudaStream_t st);

// vectors
void vec_axpy(double2* y, const double2* x, double a, long long n, cudaStream_t st);  // y += a x
void vec_copy(double2* y, const double2* x, long long n, cudaStream_t st);
void vec_zero(double2* y, long long n, cudaStream_t st);
// complex dot sum conj(x) y and squared norm, deterministic two-pass
void vec_dot(const double2* x, const double2* y, long long n, double* partial, double2* out, cudaStream_t st);
// y = a*x + y with complex a read from device memory (optionally negated)
void vec_caxpy_dev(double2* y, const double2* x, const double2* a, int negate, long long n, cudaStream_t st);
void vec_scale_dev(double2* y, const double* s, int invert, long long n, cudaStream_t st);

// ---------------------------------------------------------------- K2 (DD smoother)
struct DDDevice {
    int nclass = 0, nsub = 0, nbx = 0, nby = 0, l_dd = 0;
    int nu_max = 0;           // staging stride per subdomain
    int ntiles = 0;
    // per class
    const int* cls_info;      // [nclass][8]: onx, ony, nloc, nu, kpad, (unused), loc_off, n_subdomains
    const long long* cls_boff;  // [nclass]: offset of the class's B block in Bmat (64-bit: B can exceed 2^31 entries)
    const double2* Bmat;      // all classes, [rows_pad][kpad] each
    const int* loc_g;         // per class per local dof: lgx | lgy << 16
    const int* rowmap;        // per class per local dof: U row or -1
    // per subdomain
    const int* sub_class;
    const int* sub_o;         // ox | oy << 16
    // per tile: class, m0, n0, sub list offset
    const int4* tiles;
    const int* class_subs;    // subdomains of each class, contiguous
    // partition-of-unity combine table per fine dof: >= 0: the only staged value
    // (dof in one U), < 0: -(1 + k) for shared dof k, whose staged values are
    // bsrc[bptr[k] .. bptr[k + 1]) in subdomain order
    const int* srcmap;
    const int* bptr;
    const int* bsrc;
};
void dd_gemm_launch(const FineGeom& g, const DDDevice& d, const double2* r, double2* ystage, cudaStream_t st);
// separable classes: fast-diagonalisation subdomain solves (k_fdm.cu)
struct FdmClassDev {
    const double2 *Vx, *Vy, *Dinv;
    int nx, ny, nux, nuy, ux0, uy0, onx, ony;
    const int* rowmap;  // local Omega dof -> U row
    const int* subs;    // subdomains of the class
    const int* sub_o;   // Omega origin per subdomain
    const int* goff;    // gather offsets: tile element iy * nx + ix -> dof offset from the
                        // subdomain's first dof (identical for every member), or null
    const int* gord;    // tile elements in ascending goff order (memory-order gather), or null
    // mirror-symmetric class (p = 4, 6 x 6-cell Omega, centred 4 x 4 U): parity blocks
    // Ve (13 x 13), Vo (12 x 12) per direction, Vx/Vy/Dinv in [even | odd] order and
    // mir[g] = R(g) | (s_g > 0) << 16 for g < 12 (fdm.cpp)
    int sym;
    const double2 *Vxe, *Vxo, *Vye, *Vyo;
    const int* mir;
    int nsub;
    int first;          // offset of this class in the class-sorted subdomain list
};
// the team kernel's work table as a kernel parameter (constant bank: no global round
// trip in front of the prologue) when it fits
struct FdmWorkTab {
    static constexpr int kMax = 152;
    int4 w[kMax];
};
struct FdmLaunch {
    const FdmClassDev* classes;  // device copy of the class table
    const int4* work;            // per CTA: [first, end) of the class-sorted subdomain list
    int nwork;
    int rows;                    // data rows per buffer (S = rows / max(nx, ny) subdomains per batch)
    int fac_elems;               // factor region (double2) sized for the largest class
    size_t smem;                 // dynamic shared memory per CTA
    int nwarps = 0;              // > 0: team-per-subdomain kernel with this many warps per CTA
    int team = 2;                // warps per subdomain of that kernel
    // team kernel: per class, the factor region exactly as the kernel keeps it in shared
    // memory (fac_elems double2: Vx^T, Vy^T padded, Dinv, U-row and gather tables), and
    // per position of the class-sorted list (subdomain id, Omega origin); formatted on
    // the device once (fdm_format), so a CTA's prologue is one coalesced copy
    const double2* image = nullptr;
    const int2* pos_tab = nullptr;
    FdmWorkTab tab{};            // host copy of the work table (nwork <= FdmWorkTab::kMax)
};
// fills L.image / L.pos_tab (L.classes, L.work uploaded; cls = the host copy of the table)
void fdm_format(const std::vector<FdmClassDev>& cls, int p, FdmLaunch& L, std::vector<void*>& allocs, size_t& bytes,
                cudaStream_t st);
void dd_fdm_launch(const FineGeom& g, const FdmLaunch& L, const double2* r, double2* ystage, int nu_max,
                   cudaStream_t st);
std::vector<int4> fdm_plan(std::vector<FdmClassDev>& cls, int p, int nsm, FdmLaunch& L);
// p and 1-D extents of Omega the FDM kernel takes (others use the dense path)
bool fdm_supported(int p, int nx, int ny);
// subdomains without a shared factor: device-factored per-subdomain solves (k_band.cu)
struct BandGeomDev {
    int onx, ony, NXn, NYn;  // Omega cells, lattice nodes per direction
    int ns, bw;              // skeleton dofs, half bandwidth of the skeleton matrix
    int ncell, cellstride;   // cells; factor elements per cell (A_II^-1 and W)
    int nu, nucell;          // U outputs; cells with U bubbles
    const int* node_code;    // lattice node -> skeleton index, -1 for bubbles
    const int* skel_node;    // skeleton index -> lattice node
    const int* cell_bnd;     // per cell, boundary slot -> skeleton index
    const int* uout;         // (lattice node, U row) per U member
    const int* ucells;       // cells with U bubbles
    const int* lnode;        // local reference dof -> lattice node (nloc entries)
    int nloc;
};
struct BandLaunch {
    const BandGeomDev* geoms;
    const int4* subs;        // per band subdomain: subdomain id, geometry, Omega origin (ox | oy << 16)
    const long long* foff;   // factor offset (double2) per band subdomain
    double2* pool;           // factors
    const double* khtab;     // k h per coefficient class
    const double* basis;     // 1-D M then S, (p+1)^2 each
    long long pool_elems;
    int nsub;
    // factor units (one per class, factored from its first member)
    const int4* fsubs;
    const long long* ffoff;
    int nfac;
    // explicit restricted inverses B_c = A^-1[U, :] of dense-path classes, one row per
    // item: (factor unit, geometry, U row, kpad) and the row's offset into Bmat
    const int4* inv_rows;
    const long long* inv_off;
    int ninv;
    double2* Bmat;
    int warps;               // sweep: warps (subdomains in flight) per CTA
    int warp_elems;          // sweep: shared-memory vector elements per warp
    int bw_max;              // largest half bandwidth
    size_t solve_smem;
};
struct BandSubdomain {
    int sid, ox, oy, onx, ony;
    const std::vector<int>* umem;  // U members (local reference dof order = U-row order)
    int cls;                       // subdomain class: members of a class share one factor
};
// a dense-path class whose B_c is computed on the device from its band factor
struct BandInvJob {
    int sid, ox, oy, onx, ony;      // first member
    const std::vector<int>* umem;
    int cls;
    long long boff;                 // B_c in the dense-path Bmat ([rpad][kpad])
    int kpad;
};
struct Basis1D;
BandLaunch band_setup(const FineGeom& g, const std::vector<BandSubdomain>& subs, const std::vector<BandInvJob>& jobs,
                      double2* Bmat, const Basis1D& basis, const std::vector<double>& khtab,
                      std::vector<void*>& allocs, size_t& bytes, cudaStream_t st);
void band_solve_launch(const FineGeom& g, const BandLaunch& L, const double2* r, double2* ystage, int nu_max,
                       cudaStream_t st);
// out = u + sum_i y_i / L in subdomain order (u may be null -> 0); out may alias u
void dd_combine_launch(const FineGeom& g, const DDDevice& d, const double2* ystage, const double2* u, double2* out,
                       cudaStream_t st);

}  // namespace htg
