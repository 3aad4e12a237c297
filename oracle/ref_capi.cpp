// oracle/ref_capi.cpp -- extern "C" driver over the REFERENCE's own hot-path
// code, compiled unmodified from /root/reference/proj/core/src/{basis,fespace,
// mesh,qsfem,twogrid,linalg,parallel}.cpp against the Eigen-subset shim in
// oracle/eigen_shim (see oracle/Makefile.ref). Output: oracle/_ref/libhelmtg_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used to validate the C++ restatement (oracle/*.cpp),
// to generate tests/golden/ref_*.npz (tools/make_ref_golden.py) and, in
// bench.py's --impl reference / cpu_baseline legs, as the CPU baseline. Never
// linked into or called by the product path.
//
// The only code here that is not the reference's is the problem construction,
// which restates build_problem (proj/core/src/commands.cpp:14-39; commands.cpp
// itself drags in the out-of-scope LFA/dispersion/CLI modules), and a
// rectangle-with-per-cell-coefficients constructor built from the reference's
// own StructuredMesh::rectangle / tag_boundary / CoefficientField::set_k|set_eps.
// Vectors cross the ABI as interleaved complex doubles (std::complex<double>[]).
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <optional>
#include <string>

#include "helmtg/parallel.hpp"
#include "helmtg/problem.hpp"
#include "helmtg/twogrid.hpp"

using namespace helmtg;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

struct Session {
    Problem pr;
    SolverConfig cfg;
    std::optional<TwoGridOperators> ops;
};

ComplexVector vin(const double* p, long n) {
    ComplexVector v(n);
    std::memcpy(v.data(), p, std::size_t(n) * sizeof(Complex));
    return v;
}
void vout(const ComplexVector& v, double* p) { std::memcpy(p, v.data(), std::size_t(v.size()) * sizeof(Complex)); }

const BoundaryTag kTag[3] = {BoundaryTag::Dirichlet, BoundaryTag::Neumann, BoundaryTag::Absorbing};
const Side kSide[4] = {Side::Left, Side::Right, Side::Bottom, Side::Top};

Session* S(void* h) { return static_cast<Session*>(h); }
const TwoGridOperators& ops_of(void* h) {
    if (!S(h)->ops) throw std::invalid_argument("session has no two-grid operators");
    return *S(h)->ops;
}
}  // namespace

extern "C" {

// Same layouts as oracle/capi.cpp's orc_spec / orc_desc / orc_cfg.
struct ref_spec {
    int order;
    double wavelengths, ppw;
    int side[4];  // L, R, B, T: 0 Dirichlet, 1 Neumann, 2 Absorbing
    unsigned layer_mask;
    double layer_width_dofs, damping_D;
    int element_kind;  // 0 Square, 1 Triangle (ElementKind)
};
struct ref_desc {
    int order, nx, ny;
    double h;
    const double* k_cells;    // nx*ny, (y,x) order
    const double* eps_cells;  // nx*ny
    int side[4];
    int element_kind;
};
struct ref_cfg {
    double alpha_s, alpha_c;
    int n_s, n_dd;
    double omega_c;
    int l_dd, coarsening, smoother, outer;
    double tol;
    int max_iters;
};

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { set_thread_count(n); }
int ref_thread_count() { return thread_count(); }

static SolverConfig to_cfg(const ref_cfg* c) {
    SolverConfig k;
    k.alpha_s = c->alpha_s;
    k.alpha_c = c->alpha_c;
    k.n_s = c->n_s;
    k.n_dd = c->n_dd;
    k.omega_c = c->omega_c;
    k.l_dd = c->l_dd;
    k.coarsening = c->coarsening == 0 ? CoarseKind::OptimizedFD
                   : c->coarsening == 1 ? CoarseKind::GalerkinP : CoarseKind::None;
    k.smoother = c->smoother == 0 ? SmootherKind::CSDD : SmootherKind::ExactShifted;
    k.outer = c->outer == 0 ? OuterKind::Richardson : OuterKind::KrylovAccelerated;
    k.stop_rel_residual = c->tol;
    k.max_iters = c->max_iters;
    return k;
}

// build_problem, restated from proj/core/src/commands.cpp:14-39 (square elements).
int ref_session_from_spec(const ref_spec* s, const ref_cfg* c, void** out) {
    return guard([&] {
        auto ses = std::make_unique<Session>();
        Problem& pr = ses->pr;
        pr.k = 2.0 * M_PI * s->wavelengths;
        pr.n_cells = static_cast<int>(std::lround(s->wavelengths * s->ppw / s->order));
        if (pr.n_cells < 2) throw std::invalid_argument("build_problem: domain under-resolved");
        pr.mesh = std::make_unique<StructuredMesh>(
            StructuredMesh::unit_square(pr.n_cells, s->element_kind ? ElementKind::Triangle : ElementKind::Square));
        pr.space = std::make_unique<FeSpace>(FeSpace::build(*pr.mesh, s->order));
        std::map<Side, BoundaryTag> sides;
        for (int i = 0; i < 4; ++i) sides[kSide[i]] = kTag[s->side[i]];
        pr.tags = tag_boundary(*pr.mesh, sides);
        std::vector<Side> layer;
        for (int i = 0; i < 4; ++i)
            if (s->layer_mask & (1u << i)) layer.push_back(kSide[i]);
        const double eps_vol = pr.k * pr.k * s->damping_D / M_PI;
        if (layer.empty()) {
            pr.coeffs = CoefficientField::constant(pr.k, eps_vol);
        } else {
            const int layer_cells = static_cast<int>(std::ceil(s->layer_width_dofs / s->order - 1e-12));
            pr.coeffs = absorbing_layer(*pr.mesh, pr.k, layer, layer_cells * pr.mesh->spacing());
            if (eps_vol > 0.0)
                for (CellIndex cc : pr.mesh->cells()) pr.coeffs.set_eps(cc, pr.coeffs.eps(cc) + eps_vol);
        }
        pr.rhs = ComplexVector::Zero(pr.space->ndof());
        const int mid = pr.n_cells / 2;
        pr.rhs(pr.space->vertex_dof(mid, mid)) = Complex(1, 0);
        for (int d : pr.space->dirichlet_dofs(pr.tags)) pr.rhs(d) = Complex(0, 0);
        if (c) {
            ses->cfg = to_cfg(c);
            ses->ops.emplace(setup_two_grid(*pr.space, pr.coeffs, pr.tags, ses->cfg));
        }
        *out = ses.release();
    });
}

// nx x ny rectangle of spacing h with per-cell k and eps and per-side tags.
int ref_session_from_desc(const ref_desc* d, const ref_cfg* c, void** out) {
    return guard([&] {
        auto ses = std::make_unique<Session>();
        Problem& pr = ses->pr;
        pr.mesh = std::make_unique<StructuredMesh>(
            StructuredMesh::rectangle(d->nx, d->ny, d->h, d->element_kind ? ElementKind::Triangle : ElementKind::Square));
        pr.space = std::make_unique<FeSpace>(FeSpace::build(*pr.mesh, d->order));
        std::map<Side, BoundaryTag> sides;
        for (int i = 0; i < 4; ++i) sides[kSide[i]] = kTag[d->side[i]];
        pr.tags = tag_boundary(*pr.mesh, sides);
        pr.coeffs = CoefficientField::constant(d->k_cells[0], 0.0);
        for (int y = 0; y < d->ny; ++y)
            for (int x = 0; x < d->nx; ++x) {
                pr.coeffs.set_k({x, y}, d->k_cells[std::size_t(y) * d->nx + x]);
                pr.coeffs.set_eps({x, y}, d->eps_cells[std::size_t(y) * d->nx + x]);
            }
        pr.k = d->k_cells[0];
        pr.n_cells = d->nx;
        pr.rhs = ComplexVector::Zero(pr.space->ndof());
        if (c) {
            ses->cfg = to_cfg(c);
            ses->ops.emplace(setup_two_grid(*pr.space, pr.coeffs, pr.tags, ses->cfg));
        }
        *out = ses.release();
    });
}

void ref_session_free(void* h) { delete S(h); }

// out: ndof, coarse ndof, nx, ny, n_subdomains, n_factors, nnz(A), nnz(Ac), nnz(IP)
int ref_info(void* h, long long* out) {
    return guard([&] {
        Session* s = S(h);
        const CellIndex hi = s->pr.mesh->cell_max();
        out[0] = s->pr.space->ndof();
        out[1] = (s->ops && s->ops->coarse_space) ? s->ops->coarse_space->ndof() : 0;
        out[2] = hi.x + 1;
        out[3] = hi.y + 1;
        out[4] = (s->ops && s->ops->dd) ? long(s->ops->dd->size()) : 0;
        out[5] = out[4];  // the reference factors every subdomain separately (twogrid.cpp:79-89)
        out[6] = s->ops ? s->ops->A.nonZeros() : 0;
        out[7] = s->ops ? s->ops->Ac.nonZeros() : 0;
        out[8] = s->ops ? s->ops->IP.nonZeros() : 0;
    });
}

int ref_rhs(void* h, double* out) {
    return guard([&] { vout(S(h)->pr.rhs, out); });
}

int ref_coeffs(void* h, double* k, double* eps) {
    return guard([&] {
        const Session* s = S(h);
        const CellIndex hi = s->pr.mesh->cell_max();
        for (int y = 0; y <= hi.y; ++y)
            for (int x = 0; x <= hi.x; ++x) {
                k[std::size_t(y) * (hi.x + 1) + x] = s->pr.coeffs.k({x, y});
                eps[std::size_t(y) * (hi.x + 1) + x] = s->pr.coeffs.eps({x, y});
            }
    });
}

// which: 0 A, 1 A_s, 2 A_c, 3 IP, 4 IP^H  (y = op x)
int ref_apply(void* h, int which, const double* x, double* y) {
    return guard([&] {
        const TwoGridOperators& o = ops_of(h);
        const SparseComplexMatrix* M = which == 0 ? &o.A : which == 1 ? &o.As : which == 2 ? &o.Ac : &o.IP;
        if (which < 0 || which > 4) throw std::invalid_argument("unknown operator id");
        if (which == 4) {
            vout(ComplexVector(o.IP.adjoint() * vin(x, o.IP.rows())), y);
        } else {
            vout(spmv(*M, vin(x, M->cols())), y);
        }
    });
}

// The OptimizedFD coarse level of setup_two_grid (proj/core/src/twogrid.cpp:235-243),
// built by the reference's own coarse_mesh_for / coarsen_* / qsfem::assemble /
// build_prolongation on a session set up with CoarseKind::None, without the
// coarse SparseLU factorization (hours at the full-size configs): A_c, IP and
// IP^H are then available through ref_apply, the coarse solve is not.
int ref_add_coarse_parts(void* h) {
    return guard([&] {
        Session* s = S(h);
        if (!s->ops) throw std::invalid_argument("session has no two-grid operators");
        TwoGridOperators& o = *s->ops;
        const FeSpace& space = *s->pr.space;
        const int m = space.order() / 2;
        o.coarse_mesh = std::make_unique<StructuredMesh>(coarse_mesh_for(space));
        o.coarse_space = std::make_unique<FeSpace>(FeSpace::build_any(*o.coarse_mesh, 1));
        const CoefficientField ccoeffs = coarsen_coefficients(s->pr.coeffs, m);
        const BoundaryTags ctags = coarsen_tags(*o.coarse_mesh, s->pr.tags, m);
        o.Ac = qsfem::assemble(*o.coarse_space, ccoeffs, ctags);
        o.IP = build_prolongation(space, *o.coarse_space, space.dirichlet_dofs(s->pr.tags),
                                  o.coarse_space->dirichlet_dofs(ctags));
    });
}

// The reference element of order p (shape 0 square, 1 lower / 2 upper triangle,
// basis.cpp:147-219): stiffness and mass (n x n row-major), n returned in *n;
// with q > 0 also the staged interpolation E (n x npts, fespace.cpp:260-378).
int ref_element(int p, int shape, int q, double* K, double* M, double* E, int* n, int* npts) {
    return guard([&] {
        const ReferenceElement& r = shape == 0 ? ReferenceElement::square(p)
                                    : shape == 1 ? ReferenceElement::triangle_lower(p)
                                                 : ReferenceElement::triangle_upper(p);
        const int nn = r.n_dofs();
        *n = nn;
        for (int i = 0; i < nn; ++i)
            for (int j = 0; j < nn; ++j) {
                K[i * nn + j] = r.stiffness()(i, j);
                M[i * nn + j] = r.mass()(i, j);
            }
        if (q > 0) {
            const StageInterp& si = stage_interp(p, shape == 0 ? ElementKind::Square : ElementKind::Triangle,
                                                 shape == 2 ? 1 : 0, q);
            *npts = int(si.points.size());
            for (int i = 0; i < nn; ++i)
                for (int j = 0; j < *npts; ++j) E[i * *npts + j] = si.E(i, j);
        }
    });
}

// r = f - A u (shifted: A_s), the expression of twogrid.cpp:116 / :94
int ref_residual(void* h, int shifted, const double* f, const double* u, double* r) {
    return guard([&] {
        const TwoGridOperators& o = ops_of(h);
        const long n = o.A.rows();
        const ComplexVector ff = vin(f, n), uu = vin(u, n);
        vout(ComplexVector(ff - (shifted ? o.As : o.A) * uu), r);
    });
}

int ref_nnz(void* h, int which) {
    try {
        const TwoGridOperators& o = ops_of(h);
        const SparseComplexMatrix* M = which == 0 ? &o.A : which == 1 ? &o.As : which == 2 ? &o.Ac : &o.IP;
        return int(M->nonZeros());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// compressed-column export: cp (cols+1), ri (nnz), v (nnz complex)
int ref_export_csc(void* h, int which, int* cp, int* ri, double* v) {
    return guard([&] {
        const TwoGridOperators& o = ops_of(h);
        const SparseComplexMatrix& M = which == 0 ? o.A : which == 1 ? o.As : which == 2 ? o.Ac : o.IP;
        std::memcpy(cp, M.outerIndexPtr(), std::size_t(M.cols() + 1) * sizeof(int));
        std::memcpy(ri, M.innerIndexPtr(), std::size_t(M.nonZeros()) * sizeof(int));
        std::memcpy(v, M.valuePtr(), std::size_t(M.nonZeros()) * sizeof(Complex));
    });
}

int ref_dd_step(void* h, const double* u, const double* f, double* out) {
    return guard([&] {
        const TwoGridOperators& o = ops_of(h);
        if (!o.dd) throw std::invalid_argument("no domain decomposition (smoother is not CSDD)");
        const long n = o.A.rows();
        vout(dd_step(vin(u, n), vin(f, n), o.As, *o.dd), out);
    });
}

int ref_csdd(void* h, double* u, const double* f) {
    return guard([&] {
        const TwoGridOperators& o = ops_of(h);
        if (!o.dd) throw std::invalid_argument("no domain decomposition (smoother is not CSDD)");
        const long n = o.A.rows();
        ComplexVector uu = vin(u, n);
        csdd_smoother(uu, vin(f, n), o.A, o.As, *o.dd, S(h)->cfg.n_dd);
        vout(uu, u);
    });
}

// u_c = A_c^{-1} r_c through the reference's SparseFactorization (twogrid.cpp:273)
int ref_coarse_solve(void* h, const double* rc, double* uc) {
    return guard([&] {
        const TwoGridOperators& o = ops_of(h);
        if (!o.Ac_factor) throw std::invalid_argument("no coarse factorization");
        vout(lu_solve(*o.Ac_factor, vin(rc, o.Ac.rows())), uc);
    });
}

// u += A_s^{-1} (f - A u): the ExactShifted smoother (twogrid.cpp:261-262)
int ref_exact_smooth(void* h, double* u, const double* f) {
    return guard([&] {
        const TwoGridOperators& o = ops_of(h);
        if (!o.As_factor) throw std::invalid_argument("no A_s factorization (smoother is not ExactShifted)");
        const long n = o.A.rows();
        ComplexVector uu = vin(u, n);
        uu += o.As_factor->solve(vin(f, n) - o.A * uu);
        vout(uu, u);
    });
}

int ref_two_grid_step(void* h, double* u, const double* f) {
    return guard([&] {
        const TwoGridOperators& o = ops_of(h);
        const long n = o.A.rows();
        ComplexVector uu = vin(u, n);
        two_grid_step(uu, vin(f, n), o, S(h)->cfg);
        vout(uu, u);
    });
}

int ref_solve(void* h, const double* f, double* u, double* hist, int hist_cap, int* iters, int* converged) {
    return guard([&] {
        const TwoGridOperators& o = ops_of(h);
        SolveResult r = solve(vin(f, o.A.rows()), o, S(h)->cfg);
        vout(r.u, u);
        for (int i = 0; i < int(r.residual_history.size()) && i < hist_cap; ++i) hist[i] = r.residual_history[i];
        *iters = r.iterations;
        *converged = r.converged ? 1 : 0;
    });
}

int ref_multiplicity(void* h, double* out) {
    return guard([&] {
        const TwoGridOperators& o = ops_of(h);
        if (!o.dd) throw std::invalid_argument("no domain decomposition");
        std::memcpy(out, o.dd->multiplicity.data(), std::size_t(o.dd->multiplicity.size()) * sizeof(double));
    });
}

// Dirichlet dofs of the fine space (coarse = 0) or of the coarse space; returns the count
int ref_dirichlet(void* h, int coarse, int* out, int cap) {
    try {
        Session* s = S(h);
        std::vector<int> d;
        if (!coarse) {
            d = s->pr.space->dirichlet_dofs(s->pr.tags);
        } else {
            const TwoGridOperators& o = ops_of(h);
            if (!o.coarse_space) throw std::invalid_argument("no coarse space");
            if (o.coarsening == CoarseKind::OptimizedFD) {
                const BoundaryTags ct = coarsen_tags(*o.coarse_mesh, s->pr.tags, s->pr.space->order() / 2);
                d = o.coarse_space->dirichlet_dofs(ct);
            } else {
                d = o.coarse_space->dirichlet_dofs(s->pr.tags);
            }
        }
        for (int i = 0; i < int(d.size()) && i < cap; ++i) out[i] = d[std::size_t(i)];
        return int(d.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// per subdomain: |Omega dofs|, |U members| (partition, twogrid.cpp:17-74)
int ref_partition_sizes(void* h, int* out) {
    return guard([&] {
        const TwoGridOperators& o = ops_of(h);
        if (!o.dd) throw std::invalid_argument("no domain decomposition");
        int k = 0;
        for (const auto& sub : o.dd->subdomains) {
            out[k++] = int(sub.global_dofs.size());
            out[k++] = int(sub.u_members.size());
        }
    });
}

// Timing loop in the style of BM_TwoGridStep (proj/benchmarks/bench_solver.cpp:9-22):
// `steps` calls of the reference's csdd_smoother on caller-owned u, f (no copies in
// the loop). Returns the wall seconds of the loop (steady_clock) in *seconds.
int ref_bench_csdd(void* h, double* u, const double* f, int steps, double* seconds) {
    return guard([&] {
        const TwoGridOperators& o = ops_of(h);
        if (!o.dd) throw std::invalid_argument("no domain decomposition (smoother is not CSDD)");
        const long n = o.A.rows();
        ComplexVector uu = vin(u, n);
        const ComplexVector ff = vin(f, n);
        const auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < steps; ++i) csdd_smoother(uu, ff, o.A, o.As, *o.dd, S(h)->cfg.n_dd);
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        vout(uu, u);
    });
}

// Same for two_grid_step (coarse solve included).
int ref_bench_two_grid(void* h, double* u, const double* f, int steps, double* seconds) {
    return guard([&] {
        const TwoGridOperators& o = ops_of(h);
        const long n = o.A.rows();
        ComplexVector uu = vin(u, n);
        const ComplexVector ff = vin(f, n);
        const auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < steps; ++i) two_grid_step(uu, ff, o, S(h)->cfg);
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        vout(uu, u);
    });
}

}  // extern "C"
