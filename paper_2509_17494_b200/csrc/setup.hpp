// setup.hpp -- host-side setup of the two-grid operators (runs once per handle).
#pragma once

#include <array>
#include <complex>
#include <map>
#include <memory>
#include <vector>

#include "common.hpp"
#include "helmtg_b200.h"

namespace htg {

using cplx = std::complex<double>;

// 1-D hierarchical basis on [0,1]: N0 = 1-x, N1 = x, N_d (d >= 2) the
// normalised integrated Legendre functions (proj/core/src/basis.cpp:98-114).
// Every square-element matrix is a tensor product of these (p+1)x(p+1)
// factors: K_e = S (x) M + M (x) S, M_e = M (x) M, and the Robin edge mass is M
// (proj/core/src/basis.cpp:197-214,284-300).
struct Basis1D {
    int p = 0, m = 0;  // m = p/2, the coarsening factor
    double M[kMaxP + 1][kMaxP + 1] = {};
    double S[kMaxP + 1][kMaxP + 1] = {};
    // E[d][j]: coefficient of N_d in the degree-m interpolant of the values at
    // the m+1 points j/m (zero for d > m). Tensor products of E give the
    // staged interpolation of proj/core/src/fespace.cpp:260-378.
    double E[kMaxP + 1][kMaxP / 2 + 1] = {};
};
Basis1D make_basis(int p);

// Order-p triangle element of the reference's split square cell (tri.cpp):
// sub 0 lower {y <= x}, sub 1 upper {y >= x}, dofs in the reference element
// order (proj/core/src/fespace.cpp:85-108). place[i] = (dx, dy, jx, jy): element
// dof i lives in unit cell (x + dx, y + dy) at the lattice offset (jx, jy) of
// the square dof occupying the same unit-cell slot. E (n x npts) is the staged
// interpolation from the q = p/2 coarse lattice points stage_pts (offsets in
// coarse vertices from the cell origin), fespace.cpp:260-378.
struct TriElement {
    int p = 0, n = 0, npts = 0;
    std::vector<double> K, M;  // n x n, unit-cell scale (the mass scales with h^2)
    std::vector<std::array<int, 4>> place;
    std::vector<double> E;
    std::vector<std::array<int, 2>> stage_pts;
};
const TriElement& tri_element(int p, int sub);
struct HostProblem;
// IP (fine dofs x coarse vertices) of a triangle mesh as CSR (tri.cpp)
void tri_prolongation(const HostProblem& hp, std::vector<int>& rp, std::vector<int>& ci, std::vector<double>& v);

// Validated copy of the C-ABI problem plus per-cell / per-edge tables.
struct HostProblem {
    int p = 0, nx = 0, ny = 0;
    bool tri = false;  // triangle elements (each cell split along its (0,0)-(1,1) diagonal)
    double h = 0.0;
    std::vector<double> k, eps;           // per cell, (y, x) order
    std::vector<int8_t> tb, tt, tl, tr;   // tags per boundary edge
    std::vector<double> khb, kht, khl, khr;  // Robin k*h (0 unless absorbing)
    bool has_dirichlet = false;
    // unique (k, eps) coefficient classes
    std::vector<uint32_t> cls;  // per cell
    std::vector<double> cls_k, cls_eps;
    bool uniform = true;
    long long ndof() const { return (long long)(nx * p + 1) * (ny * p + 1); }
    double kc(int x, int y) const { return k[(size_t)y * nx + x]; }
    double ec(int x, int y) const { return eps[(size_t)y * nx + x]; }
    int8_t tag(char side, int i) const;
};
HostProblem make_problem(const htg_problem& prob);
void validate_config(const htg_config& cfg, const HostProblem& hp);

// ------------------------------------------------------------------ subdomains
// Non-overlapping l_dd blocks U_i grown by one cell to Omega_i
// (proj/core/src/twogrid.cpp:17-74). Subdomains whose local operator, Omega
// shape and U position coincide form one class; each class stores the
// restricted inverse B_c = (A_s^(i))^-1 [Dofs(U_i), :] (|U| x |Omega| complex).
struct DDClass {
    int onx = 0, ony = 0;       // Omega cells
    int ux = 0, uy = 0, unx = 0, uny = 0;  // U position inside Omega
    int nloc = 0, nu = 0;       // |Omega dofs|, |U dofs|
    std::vector<int> umem;      // local Omega index of each U row
    std::vector<cplx> B;        // nu x nloc, row-major
    // fast diagonalisation (separable classes): A^-1 = (Vx (x) Vy) Dinv (Vx (x) Vy)^T
    bool fdm = false;
    int fdm_nx = 0, fdm_ny = 0;    // 1-D local index ranges of Omega
    int fdm_ux0 = 0, fdm_uy0 = 0;  // first 1-D index of U
    int fdm_nux = 0, fdm_nuy = 0;  // 1-D extent of U
    std::vector<cplx> Vx, Vy;      // (nx x nx), (ny x ny) row-major, columns are eigenvectors
    std::vector<cplx> Dinv;        // nx x ny
    double fdm_err = 0.0;          // forward-error estimate of the FDM solve on probe vectors (fdm.cpp)
    // mirror-symmetric classes (an even number of Omega cells per direction, equal
    // ends, U centred): the 1-D operators commute with the reflection R (a signed
    // permutation of the hierarchical dofs), so each direction splits into an even
    // (n+1)/2 and an odd (n-1)/2 generalised eigenproblem. Vx, Vy, Dinv then hold the
    // full factors in that order ([even | odd] eigenvectors); the parity blocks are
    // V_e ((n+1)/2 square) and V_o ((n-1)/2 square) in the basis
    // e_g = (d_g + s_g d_R(g)) / sqrt 2, o_g = (d_g - s_g d_R(g)) / sqrt 2 (g < centre),
    // e_c = d_c; mirror[g] = R(g), msign[g] = s_g for g < centre.
    bool fdm_sym = false;
    std::vector<cplx> Vxe, Vxo, Vye, Vyo;
    std::vector<int> mirror, msign;
    // no shared factor (few members, coefficients varying over Omega): every
    // member is factored on the device (k_band.cu); B stays empty
    bool band = false;
    // dense path with B computed on the device from a band factor (square cells,
    // classes the fast diagonalisation cannot take): no host inverse
    bool devB = false;
};
// cheap pre-check of build_fdm's separability conditions (uniform (k, eps) over
// Omega, one non-Dirichlet tag per Omega side, p and extents the FDM kernel takes)
bool fdm_candidate(const HostProblem& hp, int ox, int oy, const DDClass& c);
// Build the FDM factors of a class whose first subdomain's Omega starts at
// cell (ox, oy); false if the class is not separable or fails validation.
// A: the assembled Omega operator (dense n x n, local dof order) the factors are checked against
bool build_fdm(const HostProblem& hp, const Basis1D& b, double alpha_s, int ox, int oy, DDClass& c,
               const std::vector<cplx>& A);
struct DDSetup {
    int l_dd = 4;
    int nbx = 0, nby = 0;  // blocks per direction
    std::vector<DDClass> classes;
    std::vector<int> sub_class;   // per subdomain (by * nbx + bx)
    std::vector<int> sub_ox, sub_oy;  // Omega origin (cells)
};
DDSetup build_dd(const HostProblem& hp, const Basis1D& b, double alpha_s, int l_dd);

// Dense complex LU with partial pivoting (setup only).
void dense_lu_solve_multi(int n, std::vector<cplx>& A, std::vector<cplx>& X, int nrhs);

}  // namespace htg
