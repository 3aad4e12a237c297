// oracle/oracle.hpp -- CPU restatement of the helmtg two-grid hot path.
//
// TEST INFRASTRUCTURE ONLY. This library is the checker that the CUDA path is
// compared against: only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it. The product library
// (paper_2509_17494_b200/) never links or calls anything in oracle/.
//
// Parity status: PINNED against the reference's own known-answer and property
// tests (proj/tests/test_{fespace,qsfem,twogrid,linalg}.cpp, acceptance C07/C11,
// README "iters=7"), ported as tests/test_oracle_*.py. The reference itself
// cannot be built here (Eigen3, doctest and CLI11 are absent), see DESIGN.md.
//
// Scope: square elements on rectangle meshes (every BASELINE config), the
// OptimizedFD (QSFEM) and GalerkinP coarse levels, CSDD and ExactShifted smoothers,
// Richardson and GMRES outer loops. Eigen's sparse products become CSR
// products, Eigen SparseLU becomes a banded LU with partial pivoting.
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

using cplx = std::complex<double>;
using cvec = std::vector<cplx>;

// proj/core/include/helmtg/mesh.hpp:15 (enum order matters for the C API)
enum class Tag : int { Dirichlet = 0, Neumann = 1, Absorbing = 2 };
// proj/core/include/helmtg/mesh.hpp:17 (Left, Right, Bottom, Top)
enum SideIdx : int { kLeft = 0, kRight = 1, kBottom = 2, kTop = 3 };

// ---------------------------------------------------------------- basis
// proj/core/src/basis.cpp:11-114
struct Poly {
    std::vector<double> c;  // monomial coefficients, lowest degree first
    double at(double x) const;
    Poly deriv() const;
};
Poly legendre(int n);
void gauss01(int n, std::vector<double>& x, std::vector<double>& w);
std::vector<Poly> hier1d(int p);

// proj/core/src/basis.cpp:148-230 (square branch only)
struct SquareElement {
    int p = 0, n = 0;
    std::vector<std::array<int, 2>> tix;  // canonical local order -> (fx, fy)
    std::vector<Poly> b, db;
    std::vector<double> K, M;  // n*n row-major
    void eval(double x, double y, double* v, double* gx, double* gy) const;
};
const SquareElement& square_element(int p);
const std::vector<double>& edge_mass(int p);  // (p+1)^2, proj/core/src/basis.cpp:284-300

// ---------------------------------------------------------------- mesh
// A rectangle of lattice cells [x0,x0+nx) x [y0,y0+ny) with spacing h
// (proj/core/src/mesh.cpp:15-51; every mesh on the hot path is a rectangle).
struct Rect {
    int x0 = 0, y0 = 0, nx = 1, ny = 1;
    double h = 1.0;
    bool has_cell(int x, int y) const { return x >= x0 && x < x0 + nx && y >= y0 && y < y0 + ny; }
};
struct Edge {
    int x, y;
    char dir;  // 'h' (x,y)->(x+1,y) or 'v' (x,y)->(x,y+1)
};
std::vector<Edge> boundary_edges(const Rect& r);  // ccw: bottom, right, top, left
bool is_boundary_edge(const Rect& r, Edge e);
std::array<int, 2> cell_adjacent(const Rect& r, Edge e);

// Per-edge tags of a rectangle's boundary (proj/core/src/mesh.cpp:136-179).
struct Tags {
    Rect r;
    std::vector<Tag> bottom, right, top, left;  // indexed by x-x0 / y-y0
    Tag get(Edge e) const;
    static Tags by_side(const Rect& r, const std::array<Tag, 4>& side);  // L,R,B,T
};

// Cell-wise k and eps over a rectangle's cells (proj/core/src/mesh.cpp:181-223).
struct Coeffs {
    Rect r;
    std::vector<double> k, eps;  // (y-y0)*nx + (x-x0)
    double kc(int x, int y) const { return k[(y - r.y0) * r.nx + (x - r.x0)]; }
    double ec(int x, int y) const { return eps[(y - r.y0) * r.nx + (x - r.x0)]; }
    Coeffs subdivided(int m, double hc) const;  // mesh.cpp:211-223
};
double layer_epsilon(double k, double depth, double width);  // mesh.cpp:225-230

// ---------------------------------------------------------------- space
// Order-p H1 space on a rectangle, dof numbering of proj/core/src/fespace.cpp:18-56:
// lattice points in (y, x) order, per point vertex, h-edge, v-edge, interior.
struct Space {
    Rect r;
    int p = 1;
    int ndof = 0;
    struct Key {
        char kind;  // 'v','h','e','c'
        int x, y, off;
    };
    std::vector<Key> keys;
    static Space build(const Rect& r, int p);
    int point_base(int X, int Y) const;  // absolute lattice coordinates
    int vertex(int X, int Y) const { return point_base(X, Y); }
    int hedge(int X, int Y) const { return point_base(X, Y) + 1; }
    int vedge(int X, int Y) const { return point_base(X, Y) + (X < r.x0 + r.nx ? p : 1); }
    int interior(int X, int Y) const { return point_base(X, Y) + 2 * p - 1; }
    void element_dofs(int cx, int cy, std::vector<int>& out) const;  // fespace.cpp:63-84
    void edge_closure(Edge e, std::vector<int>& out) const;         // fespace.cpp:130-144
    std::vector<int> dirichlet_dofs(const Tags& t) const;           // fespace.cpp:146-153
    int find(const Key& k) const;                                    // -1 if absent
};

// ---------------------------------------------------------------- sparse
struct Trip {
    int r, c;
    cplx v;
};
struct Csr {
    int n = 0, m = 0;
    std::vector<int> rp, ci;
    cvec v;
    static Csr from_triplets(int n, int m, std::vector<Trip>& t);  // sums duplicates
    void apply(const cplx* x, cplx* y) const;                      // y = A x
    void residual(const cplx* f, const cplx* x, cplx* r) const;    // r = f - A x
    void apply_adjoint(const cplx* x, cplx* y) const;              // y = A^H x
    cplx at(int i, int j) const;
    void prune_zeros();
    Csr minus(const Csr& B) const;
};
void eliminate_dirichlet(Csr& A, const std::vector<int>& dofs);  // fespace.cpp:246-258

// LU with partial pivoting on the band of A (stands in for Eigen SparseLU,
// proj/core/src/linalg.cpp:12-27). Throws std::runtime_error on a zero pivot.
struct BandLU {
    int n = 0, kl = 0, ku = 0, w = 0;
    cvec ab;
    std::vector<int> piv;
    explicit BandLU(const Csr& A);
    void solve(cplx* b) const;
};

// ---------------------------------------------------------------- assembly
// proj/core/src/fespace.cpp:181-244
Csr assemble_helmholtz(const Space& s, const Coeffs& c, const Tags& t, double alpha);
Csr assemble_mass_weighted_ieps(const Space& s, const Coeffs& c);  // weight i*eps
Csr boundary_mass(const Space& s, const Coeffs& c, const Tags& t);

// ---------------------------------------------------------------- qsfem
// proj/core/src/qsfem.cpp:8-44,118-149
struct Stencil {
    double eta, P0, P1, P2, N;
    double q(int gx, int gy) const;
};
Stencil stencil_coefficients(double eta);
double stencil_symbol(const Stencil& s, double t1, double t2);
Csr qsfem_assemble(const Space& p1, const Coeffs& c, const Tags& t);

// ---------------------------------------------------------------- two-grid
enum class Coarse : int { OptimizedFD = 0, GalerkinP = 1, None = 2 };
enum class Smoother : int { CSDD = 0, ExactShifted = 1 };
enum class Outer : int { Richardson = 0, Krylov = 1 };

// proj/core/include/helmtg/twogrid.hpp:18-30
struct Config {
    double alpha_s = 0.2, alpha_c = 0.0;
    int n_s = 1, n_dd = 1;
    double omega_c = 1.0;
    int l_dd = 4;
    Coarse coarsening = Coarse::OptimizedFD;
    Smoother smoother = Smoother::CSDD;
    Outer outer = Outer::Richardson;
    double tol = 1e-6;
    int max_iters = 200;
};

// proj/core/include/helmtg/twogrid.hpp:37-52
struct Subdomain {
    Rect u, omega;
    std::vector<int> gdofs;  // local Omega dof -> global
    std::vector<int> umem;   // local indices of Dofs(U_i)
    int factor = -1;         // index into DD::factors (identical matrices share)
};
struct DD {
    std::vector<Subdomain> subs;
    std::vector<double> mult;
    std::vector<std::unique_ptr<BandLU>> factors;
};
DD partition(const Space& s, int l_dd);                                            // twogrid.cpp:17-74
void build_subdomain_operators(const Space& s, const Coeffs& c, const Tags& t, double alpha_s,
                               DD& dd);                                              // :76-90
cvec dd_step(const cvec& u, const cvec& f, const Csr& As, const DD& dd);           // :92-112
void csdd_smoother(cvec& u, const cvec& f, const Csr& A, const Csr& As, const DD& dd, int n_dd);

struct Problem {
    Rect mesh;
    Space space;
    Coeffs coeffs;
    Tags tags;
    cvec rhs;
    double k = 0.0;
    int n_cells = 0;
};
// proj/core/src/commands.cpp:14-39 (unit square, point load at (n/2, n/2))
Problem build_problem(int order, double wavelengths, double ppw, const std::array<Tag, 4>& side,
                      unsigned layer_mask, double layer_width_dofs, double damping_D);

struct Ops {
    Space space;
    Coeffs coeffs;
    Tags tags;
    Config cfg;
    Csr A, As;
    DD dd;
    std::unique_ptr<BandLU> As_factor;
    Rect crect;
    Space cspace;
    Coeffs ccoeffs;
    Tags ctags;
    Csr Ac, IP;
    std::unique_ptr<BandLU> Ac_factor;
};
std::unique_ptr<Ops> setup_two_grid(const Space& s, const Coeffs& c, const Tags& t, const Config& cfg);

Csr build_prolongation(const Space& fine, const Space& coarse, const std::vector<int>& fdir,
                       const std::vector<int>& cdir);  // twogrid.cpp:150-187
// proj/core/src/fespace.cpp:260-378 (square, sub 0): rows = local dofs, cols = stage points
struct StageInterp {
    int n = 0, npts = 0;
    std::vector<double> E;  // n*npts
    std::vector<std::array<double, 2>> pts;
};
const StageInterp& stage_interp(int p, int q);

void two_grid_step(cvec& u, const cvec& f, const Ops& ops);  // twogrid.cpp:268-276
struct SolveResult {
    cvec u;
    int iterations = 0;
    std::vector<double> history;
    bool converged = true;
};
SolveResult solve(const cvec& f, const Ops& ops);  // twogrid.cpp:278-331

cplx evaluate(const Space& s, const cvec& u, double x, double y);  // fespace.cpp:404-424

// proj/tests/test_twogrid.cpp:15-21, with re drawn before im explicitly
cvec random_vector(int n, unsigned seed);

// proj/core/src/parallel.cpp:14-39: fresh std::threads per call, static blocks
void set_thread_count(int n);
int thread_count();
void parallel_for(std::size_t n, const std::function<void(std::size_t)>& fn);

}  // namespace orc
