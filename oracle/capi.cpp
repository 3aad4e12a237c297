// oracle/capi.cpp -- extern "C" surface of the CPU oracle for ctypes (tests,
// smoke(), bench.py cpu_baseline). TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// Complex vectors are interleaved (re, im) doubles, i.e. std::complex<double>[].
#include <cstring>
#include <string>

#include "oracle.hpp"

using namespace orc;

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
    Problem pr;  // pr.space/coeffs/tags valid for both constructors
    std::unique_ptr<Ops> ops;
};

const cplx* C(const double* p) { return reinterpret_cast<const cplx*>(p); }
cplx* Cm(double* p) { return reinterpret_cast<cplx*>(p); }
cvec vec(const double* p, int n) { return cvec(C(p), C(p) + n); }
}  // namespace

extern "C" {

struct orc_spec {
    int order;
    double wavelengths, ppw;
    int side[4];  // L, R, B, T: 0 Dirichlet, 1 Neumann, 2 Absorbing
    unsigned layer_mask;
    double layer_width_dofs, damping_D;
};
struct orc_desc {
    int order, nx, ny;
    double h;
    const double* k_cells;    // nx*ny, (y,x) order
    const double* eps_cells;  // nx*ny
    int side[4];
};
struct orc_cfg {
    double alpha_s, alpha_c;
    int n_s, n_dd;
    double omega_c;
    int l_dd, coarsening, smoother, outer;
    double tol;
    int max_iters;
};

const char* orc_last_error() { return g_err.c_str(); }
void orc_set_threads(int n) { set_thread_count(n); }

static Config to_cfg(const orc_cfg* c) {
    Config k;
    k.alpha_s = c->alpha_s;
    k.alpha_c = c->alpha_c;
    k.n_s = c->n_s;
    k.n_dd = c->n_dd;
    k.omega_c = c->omega_c;
    k.l_dd = c->l_dd;
    k.coarsening = Coarse(c->coarsening);
    k.smoother = Smoother(c->smoother);
    k.outer = Outer(c->outer);
    k.tol = c->tol;
    k.max_iters = c->max_iters;
    return k;
}

int orc_session_from_spec(const orc_spec* s, const orc_cfg* c, void** out) {
    return guard([&] {
        auto ses = std::make_unique<Session>();
        std::array<Tag, 4> side{Tag(s->side[0]), Tag(s->side[1]), Tag(s->side[2]), Tag(s->side[3])};
        ses->pr = build_problem(s->order, s->wavelengths, s->ppw, side, s->layer_mask, s->layer_width_dofs,
                                s->damping_D);
        if (c) ses->ops = setup_two_grid(ses->pr.space, ses->pr.coeffs, ses->pr.tags, to_cfg(c));
        *out = ses.release();
    });
}

int orc_session_from_desc(const orc_desc* d, const orc_cfg* c, void** out) {
    return guard([&] {
        auto ses = std::make_unique<Session>();
        Problem& pr = ses->pr;
        pr.mesh = Rect{0, 0, d->nx, d->ny, d->h};
        pr.space = Space::build(pr.mesh, d->order);
        std::array<Tag, 4> side{Tag(d->side[0]), Tag(d->side[1]), Tag(d->side[2]), Tag(d->side[3])};
        pr.tags = Tags::by_side(pr.mesh, side);
        pr.coeffs.r = pr.mesh;
        pr.coeffs.k.assign(d->k_cells, d->k_cells + std::size_t(d->nx) * d->ny);
        pr.coeffs.eps.assign(d->eps_cells, d->eps_cells + std::size_t(d->nx) * d->ny);
        pr.rhs.assign(pr.space.ndof, cplx(0.0));
        pr.n_cells = d->nx;
        if (c) ses->ops = setup_two_grid(pr.space, pr.coeffs, pr.tags, to_cfg(c));
        *out = ses.release();
    });
}

void orc_session_free(void* h) { delete static_cast<Session*>(h); }

// out: ndof, coarse ndof, nx, ny, n_subdomains, n_factors, nnz(A), nnz(Ac), nnz(IP)
int orc_info(void* h, long long* out) {
    return guard([&] {
        Session* s = static_cast<Session*>(h);
        out[0] = s->pr.space.ndof;
        out[1] = s->ops ? s->ops->cspace.ndof : 0;
        out[2] = s->pr.mesh.nx;
        out[3] = s->pr.mesh.ny;
        out[4] = s->ops ? long(s->ops->dd.subs.size()) : 0;
        out[5] = s->ops ? long(s->ops->dd.factors.size()) : 0;
        out[6] = s->ops ? long(s->ops->A.ci.size()) : 0;
        out[7] = s->ops ? long(s->ops->Ac.ci.size()) : 0;
        out[8] = s->ops ? long(s->ops->IP.ci.size()) : 0;
    });
}

int orc_rhs(void* h, double* out) {
    return guard([&] {
        Session* s = static_cast<Session*>(h);
        std::memcpy(out, s->pr.rhs.data(), s->pr.rhs.size() * sizeof(cplx));
    });
}

int orc_coeffs(void* h, double* k, double* eps) {
    return guard([&] {
        Session* s = static_cast<Session*>(h);
        std::memcpy(k, s->pr.coeffs.k.data(), s->pr.coeffs.k.size() * sizeof(double));
        std::memcpy(eps, s->pr.coeffs.eps.data(), s->pr.coeffs.eps.size() * sizeof(double));
    });
}

static const Csr& pick(Session* s, int which) {
    if (!s->ops) throw std::invalid_argument("session has no two-grid operators");
    switch (which) {
        case 0: return s->ops->A;
        case 1: return s->ops->As;
        case 2: return s->ops->Ac;
        case 3: return s->ops->IP;
        default: throw std::invalid_argument("unknown operator id");
    }
}

// which: 0 A, 1 A_s, 2 A_c, 3 IP, 4 IP^H
int orc_apply(void* h, int which, const double* x, double* y) {
    return guard([&] {
        Session* s = static_cast<Session*>(h);
        if (which == 4)
            pick(s, 3).apply_adjoint(C(x), Cm(y));
        else
            pick(s, which).apply(C(x), Cm(y));
    });
}

int orc_residual(void* h, int shifted, const double* f, const double* u, double* r) {
    return guard([&] { pick(static_cast<Session*>(h), shifted ? 1 : 0).residual(C(f), C(u), Cm(r)); });
}

int orc_nnz(void* h, int which) {
    try {
        return int(pick(static_cast<Session*>(h), which).ci.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int orc_export_csr(void* h, int which, int* rp, int* ci, double* v) {
    return guard([&] {
        const Csr& A = pick(static_cast<Session*>(h), which);
        std::memcpy(rp, A.rp.data(), A.rp.size() * sizeof(int));
        std::memcpy(ci, A.ci.data(), A.ci.size() * sizeof(int));
        std::memcpy(v, A.v.data(), A.v.size() * sizeof(cplx));
    });
}

int orc_dd_step(void* h, const double* u, const double* f, double* out) {
    return guard([&] {
        Session* s = static_cast<Session*>(h);
        const int n = s->pr.space.ndof;
        cvec r = dd_step(vec(u, n), vec(f, n), s->ops->As, s->ops->dd);
        std::memcpy(out, r.data(), n * sizeof(cplx));
    });
}

int orc_csdd(void* h, double* u, const double* f) {
    return guard([&] {
        Session* s = static_cast<Session*>(h);
        const int n = s->pr.space.ndof;
        cvec uu = vec(u, n);
        csdd_smoother(uu, vec(f, n), s->ops->A, s->ops->As, s->ops->dd, s->ops->cfg.n_dd);
        std::memcpy(u, uu.data(), n * sizeof(cplx));
    });
}

int orc_coarse_solve(void* h, const double* rc, double* uc) {
    return guard([&] {
        Session* s = static_cast<Session*>(h);
        const int n = s->ops->cspace.ndof;
        std::memcpy(uc, rc, n * sizeof(cplx));
        if (!s->ops->Ac_factor) throw std::runtime_error("coarse operator not factored (ORC_NO_COARSE_FACTOR)");
        s->ops->Ac_factor->solve(Cm(uc));
    });
}

int orc_two_grid_step(void* h, double* u, const double* f) {
    return guard([&] {
        Session* s = static_cast<Session*>(h);
        const int n = s->pr.space.ndof;
        cvec uu = vec(u, n);
        two_grid_step(uu, vec(f, n), *s->ops);
        std::memcpy(u, uu.data(), n * sizeof(cplx));
    });
}

int orc_solve(void* h, const double* f, double* u, double* hist, int hist_cap, int* iters, int* converged) {
    return guard([&] {
        Session* s = static_cast<Session*>(h);
        const int n = s->pr.space.ndof;
        SolveResult r = solve(vec(f, n), *s->ops);
        std::memcpy(u, r.u.data(), n * sizeof(cplx));
        for (int i = 0; i < int(r.history.size()) && i < hist_cap; ++i) hist[i] = r.history[i];
        *iters = r.iterations;
        *converged = r.converged ? 1 : 0;
    });
}

// per subdomain: u(x0,y0,nx,ny), omega(x0,y0,nx,ny), |Omega dofs|, |U members|, factor id
int orc_partition_info(void* h, int* out) {
    return guard([&] {
        Session* s = static_cast<Session*>(h);
        int k = 0;
        for (const Subdomain& sub : s->ops->dd.subs) {
            const Rect* rs[2] = {&sub.u, &sub.omega};
            for (const Rect* r : rs) {
                out[k++] = r->x0;
                out[k++] = r->y0;
                out[k++] = r->nx;
                out[k++] = r->ny;
            }
            out[k++] = int(sub.gdofs.size());
            out[k++] = int(sub.umem.size());
            out[k++] = sub.factor;
        }
    });
}

int orc_subdomain_maps(void* h, int i, int* gdofs, int* umem) {
    return guard([&] {
        const Subdomain& sub = static_cast<Session*>(h)->ops->dd.subs.at(i);
        std::memcpy(gdofs, sub.gdofs.data(), sub.gdofs.size() * sizeof(int));
        std::memcpy(umem, sub.umem.data(), sub.umem.size() * sizeof(int));
    });
}

int orc_multiplicity(void* h, double* out) {
    return guard([&] {
        const auto& m = static_cast<Session*>(h)->ops->dd.mult;
        std::memcpy(out, m.data(), m.size() * sizeof(double));
    });
}

int orc_dirichlet(void* h, int coarse, int* out, int cap) {
    try {
        Session* s = static_cast<Session*>(h);
        std::vector<int> d = coarse ? s->ops->cspace.dirichlet_dofs(s->ops->ctags) : s->pr.space.dirichlet_dofs(s->pr.tags);
        for (int i = 0; i < int(d.size()) && i < cap; ++i) out[i] = d[i];
        return int(d.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int orc_find_dof(void* h, int coarse, int kind, int x, int y, int off) {
    Session* s = static_cast<Session*>(h);
    const Space& sp = coarse ? s->ops->cspace : s->pr.space;
    return sp.find(Space::Key{char(kind), x, y, off});
}

// dof keys of the fine (coarse=0) or coarse space: kind,x,y,off per dof
int orc_dof_keys(void* h, int coarse, int* out) {
    return guard([&] {
        Session* s = static_cast<Session*>(h);
        const Space& sp = coarse ? s->ops->cspace : s->pr.space;
        int k = 0;
        for (const auto& key : sp.keys) {
            out[k++] = key.kind;
            out[k++] = key.x;
            out[k++] = key.y;
            out[k++] = key.off;
        }
    });
}

int orc_evaluate(void* h, int coarse, const double* u, double x, double y, double* out) {
    return guard([&] {
        Session* s = static_cast<Session*>(h);
        const Space& sp = coarse ? s->ops->cspace : s->pr.space;
        cplx v = evaluate(sp, vec(u, sp.ndof), x, y);
        out[0] = v.real();
        out[1] = v.imag();
    });
}

int orc_element(int p, double* K, double* M) {
    return guard([&] {
        const SquareElement& e = square_element(p);
        std::memcpy(K, e.K.data(), e.K.size() * sizeof(double));
        std::memcpy(M, e.M.data(), e.M.size() * sizeof(double));
    });
}

int orc_edge_mass(int p, double* out) {
    return guard([&] {
        const auto& m = edge_mass(p);
        std::memcpy(out, m.data(), m.size() * sizeof(double));
    });
}

// out: eta, P0, P1, P2, N
int orc_stencil(double eta, double* out) {
    return guard([&] {
        Stencil s = stencil_coefficients(eta);
        out[0] = s.eta;
        out[1] = s.P0;
        out[2] = s.P1;
        out[3] = s.P2;
        out[4] = s.N;
    });
}

double orc_symbol(double eta, double t1, double t2) { return stencil_symbol(stencil_coefficients(eta), t1, t2); }

int orc_stage_interp(int p, int q, double* E, double* pts) {
    return guard([&] {
        const StageInterp& si = stage_interp(p, q);
        std::memcpy(E, si.E.data(), si.E.size() * sizeof(double));
        for (int j = 0; j < si.npts; ++j) {
            pts[2 * j] = si.pts[j][0];
            pts[2 * j + 1] = si.pts[j][1];
        }
    });
}

int orc_random_vector(int n, unsigned seed, double* out) {
    return guard([&] {
        cvec v = random_vector(n, seed);
        std::memcpy(out, v.data(), n * sizeof(cplx));
    });
}

int orc_lu_solve_csr(int n, const int* rp, const int* ci, const double* v, const double* b, double* x) {
    return guard([&] {
        Csr A;
        A.n = A.m = n;
        A.rp.assign(rp, rp + n + 1);
        A.ci.assign(ci, ci + rp[n]);
        A.v.assign(C(v), C(v) + rp[n]);
        BandLU lu(A);
        std::memcpy(x, b, n * sizeof(cplx));
        lu.solve(Cm(x));
    });
}

// Assemble one matrix on the session's space into the A slot (which=0) for export:
// kind 0 Helmholtz(alpha), 1 mass with weight (wre + i wim), 2 boundary mass, 3 QSFEM (p=1).
int orc_build_matrix(void* h, int kind, double alpha, double wre, double wim) {
    return guard([&] {
        Session* s = static_cast<Session*>(h);
        if (!s->ops) {
            s->ops = std::make_unique<Ops>();
            s->ops->space = s->pr.space;
        }
        const Space& sp = s->pr.space;
        switch (kind) {
            case 0: s->ops->A = assemble_helmholtz(sp, s->pr.coeffs, s->pr.tags, alpha); break;
            case 1: {
                Coeffs w = s->pr.coeffs;  // weight = w * 1 via the i*eps path: eps <- -i*w
                // mass with a constant complex weight: M * w = (i*eps) M with eps = -i w
                Csr Mi = assemble_mass_weighted_ieps(sp, [&] {
                    Coeffs c = w;
                    for (auto& e : c.eps) e = 1.0;
                    return c;
                }());
                for (auto& v : Mi.v) v *= cplx(wre, wim) / cplx(0.0, 1.0);
                s->ops->A = Mi;
                break;
            }
            case 2: s->ops->A = boundary_mass(sp, s->pr.coeffs, s->pr.tags); break;
            case 3: s->ops->A = qsfem_assemble(sp, s->pr.coeffs, s->pr.tags); break;
            default: throw std::invalid_argument("unknown matrix kind");
        }
    });
}

}  // extern "C"
