// setup.cpp -- host setup: 1-D basis factors, problem tables, subdomain classes.
#include "setup.hpp"
#include "kernels.hpp"
#include "coarse.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <thread>

namespace htg {

// ------------------------------------------------------------------ 1-D basis
namespace {

// Legendre P_n(s) and P_n'(s) by the three-term recurrence.
void legendre_at(int n, double s, double& pn, double& dpn) {
    double p0 = 1.0, p1 = s, d0 = 0.0, d1 = 1.0;
    if (n == 0) {
        pn = 1.0;
        dpn = 0.0;
        return;
    }
    for (int k = 1; k < n; ++k) {
        const double p2 = ((2 * k + 1) * s * p1 - k * p0) / (k + 1);
        const double d2 = d0 + (2 * k + 1) * p1;  // P'_{k+1} = P'_{k-1} + (2k+1) P_k
        p0 = p1;
        p1 = p2;
        d0 = d1;
        d1 = d2;
    }
    pn = p1;
    dpn = d1;
}

// N_d(x) and N_d'(x) on [0,1] (proj/core/src/basis.cpp:98-114).
void hier_at(int d, double x, double& v, double& dv) {
    if (d == 0) {
        v = 1.0 - x;
        dv = -1.0;
        return;
    }
    if (d == 1) {
        v = x;
        dv = 1.0;
        return;
    }
    const double s = 2.0 * x - 1.0, c = 1.0 / std::sqrt(2.0 * (2.0 * d - 1.0));
    double a, da, b, db;
    legendre_at(d, s, a, da);
    legendre_at(d - 2, s, b, db);
    v = c * (a - b);
    dv = 2.0 * c * (da - db);
}

// Gauss-Legendre nodes/weights on [0,1] by Newton iteration on P_n.
void gauss(int n, std::vector<double>& x, std::vector<double>& w) {
    x.resize(n);
    w.resize(n);
    for (int i = 0; i < n; ++i) {
        double t = std::cos(M_PI * (i + 0.75) / (n + 0.5)), pn, dp;
        for (int it = 0; it < 100; ++it) {
            legendre_at(n, t, pn, dp);
            const double step = pn / dp;
            t -= step;
            if (std::fabs(step) < 1e-16) break;
        }
        legendre_at(n, t, pn, dp);
        x[i] = 0.5 * (1.0 - t);
        w[i] = 1.0 / ((1.0 - t * t) * dp * dp);
    }
}

}  // namespace

Basis1D make_basis(int p) {
    if (p < 2 || p > kMaxP || p % 2) throw InvalidArgument("order must be even, 2 <= p <= 8");
    Basis1D b;
    b.p = p;
    b.m = p / 2;
    std::vector<double> xq, wq;
    gauss(p + 1, xq, wq);  // exact for the degree-2p products
    for (size_t q = 0; q < xq.size(); ++q) {
        double v[kMaxP + 1], dv[kMaxP + 1];
        for (int d = 0; d <= p; ++d) hier_at(d, xq[q], v[d], dv[d]);
        for (int i = 0; i <= p; ++i)
            for (int j = 0; j <= p; ++j) {
                b.M[i][j] += wq[q] * v[i] * v[j];
                b.S[i][j] += wq[q] * dv[i] * dv[j];
            }
    }
    // interpolation through j/m in the basis {N_0, N_1, N_2..N_m}: V c = values
    const int m = b.m;
    std::vector<double> V((m + 1) * (m + 1)), inv((m + 1) * (m + 1), 0.0);
    auto col_of = [](int d) { return d; };  // column d holds N_d
    for (int j = 0; j <= m; ++j)
        for (int d = 0; d <= m; ++d) {
            double v, dv;
            hier_at(d, double(j) / m, v, dv);
            V[j * (m + 1) + col_of(d)] = v;
        }
    // Gauss-Jordan inverse with partial pivoting (tiny system)
    for (int i = 0; i <= m; ++i) inv[i * (m + 1) + i] = 1.0;
    for (int k = 0; k <= m; ++k) {
        int piv = k;
        for (int i = k + 1; i <= m; ++i)
            if (std::fabs(V[i * (m + 1) + k]) > std::fabs(V[piv * (m + 1) + k])) piv = i;
        for (int j = 0; j <= m; ++j) {
            std::swap(V[k * (m + 1) + j], V[piv * (m + 1) + j]);
            std::swap(inv[k * (m + 1) + j], inv[piv * (m + 1) + j]);
        }
        const double d = V[k * (m + 1) + k];
        for (int j = 0; j <= m; ++j) {
            V[k * (m + 1) + j] /= d;
            inv[k * (m + 1) + j] /= d;
        }
        for (int i = 0; i <= m; ++i) {
            if (i == k) continue;
            const double f = V[i * (m + 1) + k];
            for (int j = 0; j <= m; ++j) {
                V[i * (m + 1) + j] -= f * V[k * (m + 1) + j];
                inv[i * (m + 1) + j] -= f * inv[k * (m + 1) + j];
            }
        }
    }
    // vertex coefficients are exactly the end values (bubbles vanish at 0 and 1)
    for (int d = 0; d <= m; ++d)
        for (int j = 0; j <= m; ++j) b.E[d][j] = inv[d * (m + 1) + j];
    for (int j = 0; j <= m; ++j) {
        b.E[0][j] = (j == 0) ? 1.0 : 0.0;
        b.E[1][j] = (j == m) ? 1.0 : 0.0;
    }
    return b;
}

// ------------------------------------------------------------------ problem
int8_t HostProblem::tag(char side, int i) const {
    switch (side) {
        case 'b': return tb[i];
        case 't': return tt[i];
        case 'l': return tl[i];
        default: return tr[i];
    }
}

HostProblem make_problem(const htg_problem& pr) {
    HostProblem hp;
    if (pr.order < 2 || pr.order > kMaxP || pr.order % 2)
        throw InvalidArgument("build_space: order must be even, 2 <= p <= 8 (coarsening requires p/2 integral)");
    if (pr.nx < 1 || pr.ny < 1) throw InvalidArgument("rectangle: cell counts must be >= 1");
    if (!(pr.h > 0.0)) throw InvalidArgument("rectangle: spacing must be positive");
    hp.p = pr.order;
    if (pr.element_kind != HTG_ELEM_SQUARE && pr.element_kind != HTG_ELEM_TRIANGLE)
        throw InvalidArgument("unknown element kind");
    hp.tri = pr.element_kind == HTG_ELEM_TRIANGLE;
    hp.nx = pr.nx;
    hp.ny = pr.ny;
    hp.h = pr.h;
    const size_t nc = size_t(pr.nx) * pr.ny;
    hp.k.resize(nc);
    hp.eps.resize(nc);
    for (size_t c = 0; c < nc; ++c) {
        hp.k[c] = pr.k_cells ? pr.k_cells[c] : pr.k_const;
        hp.eps[c] = pr.eps_cells ? pr.eps_cells[c] : pr.eps_const;
        if (!(hp.k[c] > 0.0)) throw InvalidArgument("CoefficientField: k must be positive");
        if (hp.eps[c] < 0.0) throw InvalidArgument("CoefficientField: eps must be nonnegative");
    }
    auto fill = [&](std::vector<int8_t>& dst, const int* src, int n, int side) {
        dst.resize(n);
        for (int i = 0; i < n; ++i) {
            const int t = src ? src[i] : pr.side_tags[side];
            if (t < 0 || t > 2) throw InvalidArgument("unknown boundary tag");
            dst[i] = int8_t(t);
        }
    };
    fill(hp.tl, pr.tags_left, pr.ny, 0);
    fill(hp.tr, pr.tags_right, pr.ny, 1);
    fill(hp.tb, pr.tags_bottom, pr.nx, 2);
    fill(hp.tt, pr.tags_top, pr.nx, 3);
    auto robin = [&](std::vector<double>& kh, const std::vector<int8_t>& tg, bool horiz, bool lo) {
        const int n = int(tg.size());
        kh.assign(n, 0.0);
        for (int i = 0; i < n; ++i) {
            if (tg[i] != kAbsorbing) continue;
            const int cx = horiz ? i : (lo ? 0 : pr.nx - 1);
            const int cy = horiz ? (lo ? 0 : pr.ny - 1) : i;
            kh[i] = hp.kc(cx, cy) * pr.h;  // k of the adjacent cell (fespace.cpp:198-203)
        }
    };
    robin(hp.khb, hp.tb, true, true);
    robin(hp.kht, hp.tt, true, false);
    robin(hp.khl, hp.tl, false, true);
    robin(hp.khr, hp.tr, false, false);
    for (auto* v : {&hp.tb, &hp.tt, &hp.tl, &hp.tr})
        for (int8_t t : *v) hp.has_dirichlet |= (t == kDirichlet);
    // coefficient classes
    std::map<std::pair<double, double>, int> ids;
    hp.cls.resize(nc);
    for (size_t c = 0; c < nc; ++c) {
        auto key = std::make_pair(hp.k[c], hp.eps[c]);
        auto it = ids.find(key);
        if (it == ids.end()) {
            it = ids.emplace(key, int(ids.size())).first;
            hp.cls_k.push_back(key.first);
            hp.cls_eps.push_back(key.second);
        }
        hp.cls[c] = uint32_t(it->second);
    }
    hp.uniform = ids.size() == 1;
    return hp;
}

void validate_config(const htg_config& c, const HostProblem& hp) {
    if (c.n_s < 0 || c.n_dd < 1 || c.max_iters < 0) throw InvalidArgument("invalid iteration counts");
    if (c.smoother == HTG_SMOOTHER_CSDD && c.l_dd < 2) throw InvalidArgument("partition: l_dd must be >= 2");
    if (c.coarsening != HTG_COARSE_OPTIMIZED_FD && c.coarsening != HTG_COARSE_GALERKIN_P &&
        c.coarsening != HTG_COARSE_NONE)
        throw InvalidArgument("unknown coarsening");
    if (c.smoother != HTG_SMOOTHER_CSDD && c.smoother != HTG_SMOOTHER_EXACT_SHIFTED)
        throw InvalidArgument("unknown smoother");
    if (c.outer != HTG_OUTER_RICHARDSON && c.outer != HTG_OUTER_KRYLOV) throw InvalidArgument("unknown outer iteration");
    if (c.coarsening == HTG_COARSE_OPTIMIZED_FD) {
        const double hc = 2.0 * hp.h / hp.p;
        for (double k : hp.cls_k) {
            const double eta = hc * k;
            if (!(eta > 0.0) || !(eta < M_PI))
                throw InvalidArgument("qsfem: eta = k*h_c must lie in (0, pi) (at least two coarse points per wavelength)");
        }
    }
}

// ------------------------------------------------------------------ dense LU
void dense_lu_solve_multi(int n, std::vector<cplx>& A, std::vector<cplx>& X, int nrhs) {
    std::vector<int> piv(n);
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = std::abs(A[size_t(k) * n + k]);
        for (int i = k + 1; i < n; ++i) {
            const double a = std::abs(A[size_t(i) * n + k]);
            if (a > best) {
                best = a;
                p = i;
            }
        }
        if (best == 0.0) throw RuntimeError("subdomain LU: singular matrix");
        piv[k] = p;
        if (p != k) {
            std::swap_ranges(A.begin() + size_t(k) * n, A.begin() + size_t(k + 1) * n, A.begin() + size_t(p) * n);
            std::swap_ranges(X.begin() + size_t(k) * nrhs, X.begin() + size_t(k + 1) * nrhs,
                             X.begin() + size_t(p) * nrhs);
        }
        const cplx inv = 1.0 / A[size_t(k) * n + k];
        const cplx* rk = &A[size_t(k) * n];
        const cplx* xk = &X[size_t(k) * nrhs];
        for (int i = k + 1; i < n; ++i) {
            cplx* ri = &A[size_t(i) * n];
            if (ri[k] == cplx(0.0)) continue;
            const cplx l = ri[k] * inv;
            ri[k] = l;
            for (int j = k + 1; j < n; ++j) ri[j] -= l * rk[j];
            cplx* xi = &X[size_t(i) * nrhs];
            for (int j = 0; j < nrhs; ++j) xi[j] -= l * xk[j];
        }
    }
    for (int k = n - 1; k >= 0; --k) {
        cplx* xk = &X[size_t(k) * nrhs];
        const cplx* rk = &A[size_t(k) * n];
        for (int c = k + 1; c < n; ++c) {
            const cplx a = rk[c];
            if (a == cplx(0.0)) continue;
            const cplx* xc = &X[size_t(c) * nrhs];
            for (int j = 0; j < nrhs; ++j) xk[j] -= a * xc[j];
        }
        const cplx inv = 1.0 / rk[k];
        for (int j = 0; j < nrhs; ++j) xk[j] *= inv;
    }
}

// ------------------------------------------------------------------ subdomains
namespace {

struct ClassKey {
    std::vector<double> v;
    bool operator<(const ClassKey& o) const { return v < o.v; }
};

// Assemble A_s on the Omega rectangle [ox, ox+onx) x [oy, oy+ony) in the local
// reference numbering: element tensor products, Robin on absorbing Omega edges
// (internal edges are absorbing, outer edges inherit; twogrid.cpp:80-86),
// Dirichlet rows/columns -> identity (fespace.cpp:246-258).
void assemble_omega_tri(const HostProblem& hp, const Basis1D& b, double alpha, int ox, int oy, int onx, int ony,
                        std::vector<cplx>& A, int& n);

void assemble_omega(const HostProblem& hp, const Basis1D& b, double alpha, int ox, int oy, int onx, int ony,
                    std::vector<cplx>& A, int& n) {
    if (hp.tri) {
        assemble_omega_tri(hp, b, alpha, ox, oy, onx, ony, A, n);
        return;
    }
    const int p = hp.p;
    n = int(dof_index(onx, ony, p, onx * p, ony * p)) + 1;
    A.assign(size_t(n) * n, cplx(0.0));
    auto li = [&](int cx, int a) { return a == 0 ? cx * p : (a == 1 ? (cx + 1) * p : cx * p + a - 1); };
    const double h2 = hp.h * hp.h;
    for (int cy = 0; cy < ony; ++cy)
        for (int cx = 0; cx < onx; ++cx) {
            const double k = hp.kc(ox + cx, oy + cy), e = hp.ec(ox + cx, oy + cy);
            const cplx m = cplx(k * k, k * k * alpha + e) * h2;
            for (int a = 0; a <= p; ++a)
                for (int bb = 0; bb <= p; ++bb) {
                    const long long r = dof_index(onx, ony, p, li(cx, a), li(cy, bb));
                    for (int c = 0; c <= p; ++c)
                        for (int d = 0; d <= p; ++d) {
                            const double sm = b.S[a][c] * b.M[bb][d] + b.M[a][c] * b.S[bb][d];
                            const double mm = b.M[a][c] * b.M[bb][d];
                            if (sm == 0.0 && mm == 0.0) continue;
                            const long long col = dof_index(onx, ony, p, li(cx, c), li(cy, d));
                            A[size_t(r) * n + col] += sm - m * mm;
                        }
                }
        }
    // boundary edges of Omega: tag and k h of the adjacent cell
    auto edge_tag = [&](char side, int i) -> int8_t {
        // global boundary edge -> inherited tag, otherwise absorbing
        switch (side) {
            case 'b': return oy == 0 ? hp.tb[ox + i] : kAbsorbing;
            case 't': return oy + ony == hp.ny ? hp.tt[ox + i] : kAbsorbing;
            case 'l': return ox == 0 ? hp.tl[oy + i] : kAbsorbing;
            default: return ox + onx == hp.nx ? hp.tr[oy + i] : kAbsorbing;
        }
    };
    std::vector<char> dir(n, 0);
    for (int side = 0; side < 4; ++side) {
        const char s = "btlr"[side];
        const bool horiz = side < 2;
        const int cnt = horiz ? onx : ony;
        for (int i = 0; i < cnt; ++i) {
            const int8_t t = edge_tag(s, i);
            const int cx = horiz ? i : (s == 'l' ? 0 : onx - 1);
            const int cy = horiz ? (s == 'b' ? 0 : ony - 1) : i;
            const int fixed = (s == 'b') ? 0 : (s == 't' ? ony * p : (s == 'l' ? 0 : onx * p));
            // closure dofs of this edge in 1-D local index order a = 0..p along the edge
            auto dof = [&](int a) {
                const int g = horiz ? li(cx, a) : li(cy, a);
                return horiz ? dof_index(onx, ony, p, g, fixed) : dof_index(onx, ony, p, fixed, g);
            };
            if (t == kAbsorbing) {
                const double kh = hp.kc(ox + cx, oy + cy) * hp.h;
                for (int a = 0; a <= p; ++a)
                    for (int c = 0; c <= p; ++c)
                        if (b.M[a][c] != 0.0) A[size_t(dof(a)) * n + dof(c)] += cplx(0.0, -kh * b.M[a][c]);
            } else if (t == kDirichlet) {
                for (int a = 0; a <= p; ++a) dir[dof(a)] = 1;
            }
        }
    }
    for (int i = 0; i < n; ++i) {
        if (!dir[i]) continue;
        for (int j = 0; j < n; ++j) {
            A[size_t(i) * n + j] = 0.0;
            A[size_t(j) * n + i] = 0.0;
        }
        A[size_t(i) * n + i] = 1.0;
    }
}

// Triangle meshes: A_s on Omega is the FE matrix of the Omega rectangle as a
// problem of its own (fe_lattice, triangle branch): its cells' k and eps,
// outer edges inheriting the global tags and k h, internal Omega edges
// absorbing with the k of the Omega cell on them (twogrid.cpp:80-86).
void assemble_omega_tri(const HostProblem& hp, const Basis1D& b, double alpha, int ox, int oy, int onx, int ony,
                        std::vector<cplx>& A, int& n) {
    HostProblem s;
    s.p = hp.p;
    s.tri = true;
    s.nx = onx;
    s.ny = ony;
    s.h = hp.h;
    for (int y = 0; y < ony; ++y)
        for (int x = 0; x < onx; ++x) {
            s.k.push_back(hp.kc(ox + x, oy + y));
            s.eps.push_back(hp.ec(ox + x, oy + y));
        }
    auto side = [&](bool outer, int8_t tg, double khg, double kcell, std::vector<int8_t>& T, std::vector<double>& K) {
        const int8_t t = outer ? tg : kAbsorbing;
        T.push_back(t);
        K.push_back(t == kAbsorbing ? (outer ? khg : kcell * hp.h) : 0.0);
        s.has_dirichlet |= t == kDirichlet;
    };
    for (int i = 0; i < onx; ++i) {
        side(oy == 0, oy == 0 ? hp.tb[ox + i] : kAbsorbing, oy == 0 ? hp.khb[ox + i] : 0.0, hp.kc(ox + i, oy), s.tb, s.khb);
        const bool top = oy + ony == hp.ny;
        side(top, top ? hp.tt[ox + i] : kAbsorbing, top ? hp.kht[ox + i] : 0.0, hp.kc(ox + i, oy + ony - 1), s.tt, s.kht);
    }
    for (int i = 0; i < ony; ++i) {
        side(ox == 0, ox == 0 ? hp.tl[oy + i] : kAbsorbing, ox == 0 ? hp.khl[oy + i] : 0.0, hp.kc(ox, oy + i), s.tl, s.khl);
        const bool right = ox + onx == hp.nx;
        side(right, right ? hp.tr[oy + i] : kAbsorbing, right ? hp.khr[oy + i] : 0.0, hp.kc(ox + onx - 1, oy + i), s.tr,
             s.khr);
    }
    const LatticeMatrix L = fe_lattice(s, b, hp.p, alpha);
    n = int(s.ndof());
    A.assign(size_t(n) * n, cplx(0.0));
    for (int i = 0; i < n; ++i)
        for (int k = L.rp[i]; k < L.rp[i + 1]; ++k) A[size_t(i) * n + L.ci[k]] = L.v[k];
}

}  // namespace

DDSetup build_dd(const HostProblem& hp, const Basis1D& b, double alpha_s, int l_dd) {
    DDSetup dd;
    dd.l_dd = l_dd;
    dd.nbx = (hp.nx + l_dd - 1) / l_dd;
    dd.nby = (hp.ny + l_dd - 1) / l_dd;
    const int nsub = dd.nbx * dd.nby;
    dd.sub_class.resize(nsub);
    dd.sub_ox.resize(nsub);
    dd.sub_oy.resize(nsub);
    std::map<ClassKey, int> ids;
    struct Pending {
        int ox, oy;
    };
    std::vector<Pending> first;
    for (int by = 0; by < dd.nby; ++by)
        for (int bx = 0; bx < dd.nbx; ++bx) {
            const int s = by * dd.nbx + bx;
            const int ux0 = bx * l_dd, uy0 = by * l_dd;
            const int ux1 = std::min(ux0 + l_dd, hp.nx), uy1 = std::min(uy0 + l_dd, hp.ny);
            const int ox0 = std::max(ux0 - 1, 0), oy0 = std::max(uy0 - 1, 0);
            const int ox1 = std::min(ux1 + 1, hp.nx), oy1 = std::min(uy1 + 1, hp.ny);
            ClassKey key;
            key.v = {double(ox1 - ox0), double(oy1 - oy0), double(ux0 - ox0), double(uy0 - oy0),
                     double(ux1 - ux0), double(uy1 - uy0)};
            // boundary situation of Omega (inherited tags) and coefficients in Omega
            key.v.push_back(oy0 == 0 ? 1 : 0);
            key.v.push_back(oy1 == hp.ny ? 1 : 0);
            key.v.push_back(ox0 == 0 ? 1 : 0);
            key.v.push_back(ox1 == hp.nx ? 1 : 0);
            for (int x = ox0; x < ox1; ++x) {
                key.v.push_back(oy0 == 0 ? hp.tb[x] : -1);
                key.v.push_back(oy1 == hp.ny ? hp.tt[x] : -1);
            }
            for (int y = oy0; y < oy1; ++y) {
                key.v.push_back(ox0 == 0 ? hp.tl[y] : -1);
                key.v.push_back(ox1 == hp.nx ? hp.tr[y] : -1);
            }
            for (int y = oy0; y < oy1; ++y)
                for (int x = ox0; x < ox1; ++x) {
                    key.v.push_back(hp.kc(x, y));
                    key.v.push_back(hp.ec(x, y));
                }
            auto it = ids.find(key);
            if (it == ids.end()) {
                it = ids.emplace(key, int(first.size())).first;
                first.push_back({ox0, oy0});
                DDClass c;
                c.onx = ox1 - ox0;
                c.ony = oy1 - oy0;
                c.ux = ux0 - ox0;
                c.uy = uy0 - oy0;
                c.unx = ux1 - ux0;
                c.uny = uy1 - uy0;
                dd.classes.push_back(c);
            }
            dd.sub_class[s] = it->second;
            dd.sub_ox[s] = ox0;
            dd.sub_oy[s] = oy0;
        }
    // classes without a shared factor: few members (HTG_BAND_MAX, default 8) and
    // coefficients that vary over Omega (not separable); HTG_BAND=0 keeps every
    // class on the dense path
    const int nc = int(dd.classes.size());
    {
        const char* be = std::getenv("HTG_BAND");
        const char* bm = std::getenv("HTG_BAND_MAX");
        const int band_max = bm ? std::atoi(bm) : 8;
        std::vector<int> members(nc, 0);
        for (int c : dd.sub_class) ++members[c];
        if (!(be && be[0] == '0'))
            for (int ci = 0; ci < nc; ++ci) {
                const DDClass& c = dd.classes[ci];
                const int ox = first[ci].ox, oy = first[ci].oy;
                bool varies = false;
                for (int y = oy; y < oy + c.ony && !varies; ++y)
                    for (int x = ox; x < ox + c.onx; ++x)
                        if (hp.kc(x, y) != hp.kc(ox, oy) || hp.ec(x, y) != hp.ec(ox, oy)) {
                            varies = true;
                            break;
                        }
                // device factors (square cells): unique coefficient patterns, and every
                // class at p >= 6, where a host dense inverse of |Omega| = 1369..2401 dofs
                // costs seconds and the shared class factor stays L2-resident
                dd.classes[ci].band = !hp.tri && varies && members[ci] <= band_max;
                // the other square-cell classes the fast diagonalisation cannot take get
                // their B_c from a device band factor (HTG_DEVB=0: host dense inverse)
                const char* db = std::getenv("HTG_DEVB");
                dd.classes[ci].devB = !(db && db[0] == '0') && !hp.tri && !dd.classes[ci].band &&
                                      !fdm_candidate(hp, ox, oy, c);
            }
    }
    // restricted inverses, one per class (threads over classes)
    std::vector<std::exception_ptr> errs(nc);
    auto work = [&](int ci) {
        try {
            DDClass& c = dd.classes[ci];
            std::vector<cplx> A;
            const int p = hp.p;
            if (c.band || c.devB) c.nloc = int(dof_index(c.onx, c.ony, p, c.onx * p, c.ony * p)) + 1;
            else assemble_omega(hp, b, alpha_s, first[ci].ox, first[ci].oy, c.onx, c.ony, A, c.nloc);
            const int n = c.nloc;
            // U members: local dofs whose support touches a U cell (twogrid.cpp:46-62)
            const int NG_x = c.onx * p + 1, NG_y = c.ony * p + 1;
            std::vector<int> isU(n, 0);
            for (int gy = 0; gy < NG_y; ++gy)
                for (int gx = 0; gx < NG_x; ++gx) {
                    const int x = gx / p, jx = gx % p, y = gy / p, jy = gy % p;
                    const int xlo = jx ? x : x - 1, ylo = jy ? y : y - 1;
                    bool in = false;
                    for (int cy = ylo; cy <= y; ++cy)
                        for (int cx = xlo; cx <= x; ++cx)
                            in |= cx >= c.ux && cx < c.ux + c.unx && cy >= c.uy && cy < c.uy + c.uny;
                    isU[dof_index(c.onx, c.ony, p, gx, gy)] = in;
                }
            for (int l = 0; l < n; ++l)
                if (isU[l]) c.umem.push_back(l);
            c.nu = int(c.umem.size());
            if (c.band || c.devB) return;  // factored on the device
            // fast diagonalisation where the FDM kernel takes the class: its factors are
            // checked against A by probing, and no dense inverse is formed
            const char* fdm_env = std::getenv("HTG_FDM");
            if (!(fdm_env && fdm_env[0] == '0') && fdm_supported(p, c.onx * p + 1, c.ony * p + 1)) {
                c.fdm = build_fdm(hp, b, alpha_s, first[ci].ox, first[ci].oy, c, A);
                if (c.fdm) return;
            }
            // B = A^-1 [U, :] = (A^-T [:, U])^T: solve A^T X = E_U
            std::vector<cplx> At(size_t(n) * n);
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) At[size_t(j) * n + i] = A[size_t(i) * n + j];
            std::vector<cplx> X(size_t(n) * c.nu, cplx(0.0));
            for (int r = 0; r < c.nu; ++r) X[size_t(c.umem[r]) * c.nu + r] = 1.0;
            dense_lu_solve_multi(n, At, X, c.nu);
            c.B.resize(size_t(c.nu) * n);
            for (int r = 0; r < c.nu; ++r)
                for (int l = 0; l < n; ++l) c.B[size_t(r) * n + l] = X[size_t(l) * c.nu + r];
        } catch (...) {
            errs[ci] = std::current_exception();
        }
    };
    const int nthr = std::max(1, std::min<int>(nc, int(std::thread::hardware_concurrency())));
    std::vector<std::thread> pool;
    for (int t = 0; t < nthr; ++t)
        pool.emplace_back([&, t] {
            for (int ci = t; ci < nc; ci += nthr) work(ci);
        });
    for (auto& th : pool) th.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    return dd;
}

}  // namespace htg
