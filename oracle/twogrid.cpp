// oracle/twogrid.cpp -- partition, CSDD smoother, transfers, two-grid step, solve.
// TEST INFRASTRUCTURE ONLY (see oracle.hpp).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <unordered_map>

#include "oracle.hpp"

#include <cstdlib>

namespace orc {

static int floordiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// ---------------------------------------------------------------- partition
// proj/core/src/twogrid.cpp:17-74
DD partition(const Space& s, int l_dd) {
    if (l_dd < 2) throw std::invalid_argument("partition: l_dd must be >= 2");
    const Rect& r = s.r;
    const int xe = r.x0 + r.nx, ye = r.y0 + r.ny;
    DD dd;
    for (int by = r.y0; by < ye; by += l_dd)
        for (int bx = r.x0; bx < xe; bx += l_dd) {
            Subdomain sub;
            sub.u = Rect{bx, by, std::min(bx + l_dd, xe) - bx, std::min(by + l_dd, ye) - by, r.h};
            const int ox0 = std::max(bx - 1, r.x0), oy0 = std::max(by - 1, r.y0);
            const int ox1 = std::min(sub.u.x0 + sub.u.nx + 1, xe), oy1 = std::min(sub.u.y0 + sub.u.ny + 1, ye);
            sub.omega = Rect{ox0, oy0, ox1 - ox0, oy1 - oy0, r.h};
            Space os = Space::build(sub.omega, s.p);
            sub.gdofs.resize(os.ndof);
            for (int i = 0; i < os.ndof; ++i) {
                const Space::Key& k = os.keys[i];
                sub.gdofs[i] = s.find(k);
                auto inU = [&](int x, int y) { return sub.u.has_cell(x, y); };
                bool in_u;
                switch (k.kind) {
                    case 'v': in_u = inU(k.x - 1, k.y - 1) || inU(k.x, k.y - 1) || inU(k.x - 1, k.y) || inU(k.x, k.y); break;
                    case 'h': in_u = inU(k.x, k.y) || inU(k.x, k.y - 1); break;
                    case 'e': in_u = inU(k.x, k.y) || inU(k.x - 1, k.y); break;
                    default: in_u = inU(k.x, k.y); break;
                }
                if (in_u) sub.umem.push_back(i);
            }
            dd.subs.push_back(std::move(sub));
        }
    dd.mult.assign(s.ndof, 0.0);
    for (const auto& sub : dd.subs)
        for (int li : sub.umem) dd.mult[sub.gdofs[li]] += 1.0;
    for (double m : dd.mult)
        if (m < 1.0) throw std::logic_error("partition: some dof belongs to no subdomain");
    return dd;
}

// Omega tags: outer edges inherit, internal edges absorbing (twogrid.cpp:80-86).
static Tags omega_tags(const Rect& global, const Tags& gt, const Rect& om) {
    Tags t;
    t.r = om;
    auto pick = [&](Edge e) { return is_boundary_edge(global, e) ? gt.get(e) : Tag::Absorbing; };
    for (int x = om.x0; x < om.x0 + om.nx; ++x) {
        t.bottom.push_back(pick({x, om.y0, 'h'}));
        t.top.push_back(pick({x, om.y0 + om.ny, 'h'}));
    }
    for (int y = om.y0; y < om.y0 + om.ny; ++y) {
        t.left.push_back(pick({om.x0, y, 'v'}));
        t.right.push_back(pick({om.x0 + om.nx, y, 'v'}));
    }
    return t;
}

static std::size_t hash_csr(const Csr& A) {
    std::size_t h = std::hash<int>()(A.n) ^ (A.ci.size() * 1315423911u);
    auto mix = [&h](const void* p, std::size_t nb) {
        const unsigned char* c = static_cast<const unsigned char*>(p);
        for (std::size_t i = 0; i < nb; ++i) h = h * 1099511628211ull ^ c[i];
    };
    mix(A.rp.data(), A.rp.size() * sizeof(int));
    mix(A.ci.data(), A.ci.size() * sizeof(int));
    mix(A.v.data(), A.v.size() * sizeof(cplx));
    return h;
}

static bool same_csr(const Csr& A, const Csr& B) {
    return A.n == B.n && A.rp == B.rp && A.ci == B.ci &&
           std::memcmp(A.v.data(), B.v.data(), A.v.size() * sizeof(cplx)) == 0;
}

// proj/core/src/twogrid.cpp:76-90. Bit-identical subdomain matrices share one
// factorization (the reference factors each; identical inputs give identical factors).
void build_subdomain_operators(const Space& s, const Coeffs& c, const Tags& t, double alpha_s, DD& dd) {
    std::vector<Csr> mats(dd.subs.size());
    parallel_for(dd.subs.size(), [&](std::size_t i) {
        const Rect& om = dd.subs[i].omega;
        Space os = Space::build(om, s.p);
        mats[i] = assemble_helmholtz(os, c, omega_tags(s.r, t, om), alpha_s);
    });
    std::unordered_multimap<std::size_t, int> seen;
    std::vector<int> uniq;
    for (std::size_t i = 0; i < mats.size(); ++i) {
        const std::size_t h = hash_csr(mats[i]);
        int found = -1;
        auto range = seen.equal_range(h);
        for (auto it = range.first; it != range.second; ++it)
            if (same_csr(mats[uniq[it->second]], mats[i])) {
                found = it->second;
                break;
            }
        if (found < 0) {
            found = int(uniq.size());
            uniq.push_back(int(i));
            seen.emplace(h, found);
        }
        dd.subs[i].factor = found;
    }
    dd.factors.resize(uniq.size());
    parallel_for(uniq.size(), [&](std::size_t u) { dd.factors[u] = std::make_unique<BandLU>(mats[uniq[u]]); });
}

// w_i = R_i u + (A_s^(i))^{-1} R_i (f - A_s u); out_j = sum_{i: j in U_i} w_i(j) / L_j
// (proj/core/src/twogrid.cpp:92-112)
cvec dd_step(const cvec& u, const cvec& f, const Csr& As, const DD& dd) {
    const std::size_t n = u.size();
    cvec g(n);
    As.residual(f.data(), u.data(), g.data());
    std::vector<cvec> w(dd.subs.size());
    parallel_for(dd.subs.size(), [&](std::size_t i) {
        const Subdomain& sub = dd.subs[i];
        const std::size_t nl = sub.gdofs.size();
        cvec gl(nl);
        for (std::size_t j = 0; j < nl; ++j) gl[j] = g[sub.gdofs[j]];
        dd.factors[sub.factor]->solve(gl.data());
        for (std::size_t j = 0; j < nl; ++j) gl[j] += u[sub.gdofs[j]];
        w[i] = std::move(gl);
    });
    cvec out(n, cplx(0.0));
    for (std::size_t i = 0; i < dd.subs.size(); ++i)
        for (int li : dd.subs[i].umem) out[dd.subs[i].gdofs[li]] += w[i][li];
    for (std::size_t j = 0; j < n; ++j) out[j] /= dd.mult[j];
    return out;
}

// r = f - A u; v = 0; n_dd x v = dd_step(v, r); u += v (proj/core/src/twogrid.cpp:114-120)
void csdd_smoother(cvec& u, const cvec& f, const Csr& A, const Csr& As, const DD& dd, int n_dd) {
    cvec r(u.size());
    A.residual(f.data(), u.data(), r.data());
    cvec v(u.size(), cplx(0.0));
    for (int i = 0; i < n_dd; ++i) v = dd_step(v, r, As, dd);
    for (std::size_t j = 0; j < u.size(); ++j) u[j] += v[j];
}

// ---------------------------------------------------------------- stage interpolation
static void dense_solve_real(int n, std::vector<double> B, std::vector<double>& R, int nrhs) {
    // partial-pivoting LU of B (n x n), solve B X = R in place (R is n x nrhs)
    std::vector<int> piv(n);
    for (int k = 0; k < n; ++k) {
        int p = k;
        for (int i = k + 1; i < n; ++i)
            if (std::abs(B[i * n + k]) > std::abs(B[p * n + k])) p = i;
        if (B[p * n + k] == 0.0) throw std::runtime_error("stage_interp: singular interpolation system");
        if (p != k) {
            for (int j = 0; j < n; ++j) std::swap(B[k * n + j], B[p * n + j]);
            for (int j = 0; j < nrhs; ++j) std::swap(R[k * nrhs + j], R[p * nrhs + j]);
        }
        for (int i = k + 1; i < n; ++i) {
            const double l = B[i * n + k] / B[k * n + k];
            for (int j = k; j < n; ++j) B[i * n + j] -= l * B[k * n + j];
            for (int j = 0; j < nrhs; ++j) R[i * nrhs + j] -= l * R[k * nrhs + j];
        }
    }
    for (int k = n - 1; k >= 0; --k)
        for (int j = 0; j < nrhs; ++j) {
            double s = R[k * nrhs + j];
            for (int c = k + 1; c < n; ++c) s -= B[k * n + c] * R[c * nrhs + j];
            R[k * nrhs + j] = s / B[k * n + k];
        }
}

// Staged hierarchical interpolation on the reference square: vertices, then
// the degree<=q edge coefficients from the q-lattice edge points, then the
// degree<=q interior coefficients (proj/core/src/fespace.cpp:260-378).
const StageInterp& stage_interp(int p, int q) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, StageInterp> cache;
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find({p, q});
    if (it != cache.end()) return it->second;
    if (q < 1 || q > p) throw std::invalid_argument("stage_interp: need 1 <= q <= p");
    const SquareElement& el = square_element(p);
    StageInterp si;
    si.n = el.n;
    const double V[4][2] = {{0, 0}, {1, 0}, {0, 1}, {1, 1}};
    const double EA[4][2] = {{0, 0}, {0, 1}, {0, 0}, {1, 0}};
    const double EB[4][2] = {{1, 0}, {1, 1}, {0, 1}, {1, 1}};
    for (auto& v : V) si.pts.push_back({v[0], v[1]});
    for (int e = 0; e < 4; ++e)
        for (int a = 1; a < q; ++a)
            si.pts.push_back({EA[e][0] + (EB[e][0] - EA[e][0]) * a / q, EA[e][1] + (EB[e][1] - EA[e][1]) * a / q});
    for (int bx = 1; bx < q; ++bx)
        for (int by = 1; by < q; ++by) si.pts.push_back({double(bx) / q, double(by) / q});
    si.npts = int(si.pts.size());
    const int n = el.n, np = si.npts, ne = p - 1, neq = q - 1;
    si.E.assign(std::size_t(n) * np, 0.0);
    std::vector<double> v(n), gx(n), gy(n);
    auto residual_row = [&](int pt, double* row) {
        el.eval(si.pts[pt][0], si.pts[pt][1], v.data(), gx.data(), gy.data());
        for (int j = 0; j < np; ++j) {
            double s = 0.0;
            for (int i = 0; i < n; ++i) s += v[i] * si.E[i * np + j];
            row[j] = -s;
        }
        row[pt] += 1.0;
    };
    for (int vtx = 0; vtx < 4; ++vtx) si.E[vtx * np + vtx] = 1.0;
    int pt = 4;
    for (int e = 0; e < 4 && neq > 0; ++e) {
        std::vector<int> rows;
        for (int d = 2; d <= q; ++d) rows.push_back(4 + e * ne + (d - 2));
        std::vector<double> B(neq * neq), R(std::size_t(neq) * np);
        for (int a = 0; a < neq; ++a) {
            residual_row(pt + a, &R[std::size_t(a) * np]);  // evaluates v at the point
            for (int d = 0; d < neq; ++d) B[a * neq + d] = v[rows[d]];
        }
        dense_solve_real(neq, B, R, np);
        for (int d = 0; d < neq; ++d)
            for (int j = 0; j < np; ++j) si.E[rows[d] * np + j] = R[std::size_t(d) * np + j];
        pt += neq;
    }
    std::vector<int> irows;
    for (int dx = 2; dx <= q; ++dx)
        for (int dy = 2; dy <= q; ++dy) irows.push_back(4 + 4 * ne + (dx - 2) * ne + (dy - 2));
    const int ni = int(irows.size());
    if (ni > 0) {
        std::vector<double> B(ni * ni), R(std::size_t(ni) * np);
        for (int a = 0; a < ni; ++a) {
            residual_row(pt + a, &R[std::size_t(a) * np]);
            for (int d = 0; d < ni; ++d) B[a * ni + d] = v[irows[d]];
        }
        dense_solve_real(ni, B, R, np);
        for (int d = 0; d < ni; ++d)
            for (int j = 0; j < np; ++j) si.E[irows[d] * np + j] = R[std::size_t(d) * np + j];
    }
    return cache.emplace(std::make_pair(p, q), std::move(si)).first->second;
}

// proj/core/src/twogrid.cpp:150-187: each fine row written once, by the first
// cell (in (y,x) order) that contains it; Dirichlet rows/columns dropped.
Csr build_prolongation(const Space& fine, const Space& coarse, const std::vector<int>& fdir,
                       const std::vector<int>& cdir) {
    const int p = fine.p, m = p / 2;
    std::vector<char> fd(fine.ndof, 0), cd(coarse.ndof, 0), written(fine.ndof, 0);
    for (int d : fdir) fd[d] = 1;
    for (int d : cdir) cd[d] = 1;
    const StageInterp& si = stage_interp(p, m);
    std::vector<Trip> trips;
    std::vector<int> dofs, cdofs(si.npts);
    for (int cy = fine.r.y0; cy < fine.r.y0 + fine.r.ny; ++cy)
        for (int cx = fine.r.x0; cx < fine.r.x0 + fine.r.nx; ++cx) {
            fine.element_dofs(cx, cy, dofs);
            for (int j = 0; j < si.npts; ++j)
                cdofs[j] = coarse.vertex(cx * m + int(std::lround(si.pts[j][0] * m)),
                                         cy * m + int(std::lround(si.pts[j][1] * m)));
            for (std::size_t i = 0; i < dofs.size(); ++i) {
                if (written[dofs[i]]) continue;
                written[dofs[i]] = 1;
                if (fd[dofs[i]]) continue;
                for (int j = 0; j < si.npts; ++j) {
                    const double val = si.E[i * si.npts + j];
                    if (val != 0.0 && !cd[cdofs[j]]) trips.push_back({dofs[i], cdofs[j], cplx(val, 0)});
                }
            }
        }
    return Csr::from_triplets(fine.ndof, coarse.ndof, trips);
}

// ---------------------------------------------------------------- setup
// proj/core/src/twogrid.cpp:221-253
std::unique_ptr<Ops> setup_two_grid(const Space& s, const Coeffs& c, const Tags& t, const Config& cfg) {
    auto ops = std::make_unique<Ops>();
    ops->space = s;
    ops->coeffs = c;
    ops->tags = t;
    ops->cfg = cfg;
    ops->A = assemble_helmholtz(s, c, t, 0.0);
    ops->As = assemble_helmholtz(s, c, t, cfg.alpha_s);
    if (cfg.smoother == Smoother::CSDD) {
        ops->dd = partition(s, cfg.l_dd);
        build_subdomain_operators(s, c, t, cfg.alpha_s, ops->dd);
    } else {
        ops->As_factor = std::make_unique<BandLU>(ops->As);
    }
    if (cfg.coarsening == Coarse::OptimizedFD) {
        const int m = s.p / 2;
        if (m < 1) throw std::invalid_argument("coarse_mesh_for: order must be even >= 2");
        const double hc = 2.0 * s.r.h / s.p;
        ops->crect = Rect{s.r.x0 * m, s.r.y0 * m, s.r.nx * m, s.r.ny * m, hc};
        ops->cspace = Space::build(ops->crect, 1);
        ops->ccoeffs = c.subdivided(m, hc);
        // coarse boundary edges take the tag of their parent fine edge (twogrid.cpp:140-148)
        Tags ct;
        ct.r = ops->crect;
        for (int X = ops->crect.x0; X < ops->crect.x0 + ops->crect.nx; ++X) {
            ct.bottom.push_back(t.get({floordiv(X, m), floordiv(ops->crect.y0, m), 'h'}));
            ct.top.push_back(t.get({floordiv(X, m), floordiv(ops->crect.y0 + ops->crect.ny, m), 'h'}));
        }
        for (int Y = ops->crect.y0; Y < ops->crect.y0 + ops->crect.ny; ++Y) {
            ct.left.push_back(t.get({floordiv(ops->crect.x0, m), floordiv(Y, m), 'v'}));
            ct.right.push_back(t.get({floordiv(ops->crect.x0 + ops->crect.nx, m), floordiv(Y, m), 'v'}));
        }
        ops->ctags = ct;
        ops->Ac = qsfem_assemble(ops->cspace, ops->ccoeffs, ct);
        ops->IP = build_prolongation(s, ops->cspace, s.dirichlet_dofs(t), ops->cspace.dirichlet_dofs(ct));
        // ORC_NO_COARSE_FACTOR: leave A_c unfactored (full-size checks factor it with
        // another direct solver, e.g. SuperLU from the exported CSR); coarse_solve
        // and two_grid_step then raise
        if (!std::getenv("ORC_NO_COARSE_FACTOR")) ops->Ac_factor = std::make_unique<BandLU>(ops->Ac);
    } else if (cfg.coarsening == Coarse::GalerkinP) {
        // proj/core/src/twogrid.cpp:189-219 (galerkin_p_coarse): the order-p/2 space on
        // the same mesh, its Helmholtz matrix with alpha_c, and IP = the inclusion of the
        // hierarchical order-p/2 functions among the order-p ones
        const int p = s.p;
        if (p % 2 != 0) throw std::invalid_argument("galerkin_p_coarse: order must be even");
        const int pc = p / 2;
        ops->crect = s.r;
        ops->cspace = Space::build(s.r, pc);
        ops->ccoeffs = c;
        ops->ctags = t;
        ops->Ac = assemble_helmholtz(ops->cspace, c, t, cfg.alpha_c);
        std::vector<char> fdir(s.ndof, 0), cdir(ops->cspace.ndof, 0);
        for (int d : s.dirichlet_dofs(t)) fdir[d] = 1;
        for (int d : ops->cspace.dirichlet_dofs(t)) cdir[d] = 1;
        std::vector<Trip> trips;
        for (int ci = 0; ci < ops->cspace.ndof; ++ci) {
            Space::Key k = ops->cspace.keys[ci];
            if (k.kind == 'c') {  // interior index (dx-2)(pc-1)+(dy-2) -> (dx-2)(p-1)+(dy-2)
                const int dx = k.off / std::max(pc - 1, 1), dy = k.off % std::max(pc - 1, 1);
                k.off = dx * (p - 1) + dy;
            }
            const int fi = s.find(k);  // edge offsets carry over as-is
            if (fi < 0) throw std::logic_error("galerkin_p_coarse: missing fine dof for inclusion");
            if (!fdir[fi] && !cdir[ci]) trips.push_back({fi, ci, cplx(1.0, 0.0)});
        }
        ops->IP = Csr::from_triplets(s.ndof, ops->cspace.ndof, trips);
        ops->Ac_factor = std::make_unique<BandLU>(ops->Ac);
    }
    return ops;
}

// ---------------------------------------------------------------- iteration
static void smooth(cvec& u, const cvec& f, const Ops& ops) {
    if (ops.cfg.smoother == Smoother::CSDD) {
        csdd_smoother(u, f, ops.A, ops.As, ops.dd, ops.cfg.n_dd);
    } else {
        cvec r(u.size());
        ops.A.residual(f.data(), u.data(), r.data());
        ops.As_factor->solve(r.data());
        for (std::size_t j = 0; j < u.size(); ++j) u[j] += r[j];
    }
}

// proj/core/src/twogrid.cpp:268-276
void two_grid_step(cvec& u, const cvec& f, const Ops& ops) {
    for (int i = 0; i < ops.cfg.n_s; ++i) smooth(u, f, ops);
    if (ops.cfg.coarsening != Coarse::None) {
        cvec r(u.size()), rc(ops.cspace.ndof), t(u.size());
        ops.A.residual(f.data(), u.data(), r.data());
        ops.IP.apply_adjoint(r.data(), rc.data());
        if (!ops.Ac_factor) throw std::runtime_error("coarse operator not factored (ORC_NO_COARSE_FACTOR)");
        ops.Ac_factor->solve(rc.data());
        ops.IP.apply(rc.data(), t.data());
        for (std::size_t j = 0; j < u.size(); ++j) u[j] += ops.cfg.omega_c * t[j];
    }
    for (int i = 0; i < ops.cfg.n_s; ++i) smooth(u, f, ops);
}

static double norm2(const cvec& v) {
    double s = 0.0;
    for (const cplx& z : v) s += std::norm(z);
    return std::sqrt(s);
}

// Householder QR least squares min ||H y - beta e1|| for an (m+1) x m matrix
// (stands in for colPivHouseholderQr, proj/core/src/twogrid.cpp:318-320).
static cvec small_lstsq(std::vector<cvec> H /* columns */, int rows, cplx beta) {
    const int cols = int(H.size());
    cvec b(rows, cplx(0.0));
    b[0] = beta;
    for (int k = 0; k < cols; ++k) {
        double nrm = 0.0;
        for (int i = k; i < rows; ++i) nrm += std::norm(H[k][i]);
        nrm = std::sqrt(nrm);
        if (nrm == 0.0) continue;
        const cplx a = H[k][k];
        const cplx alpha = (std::abs(a) > 0 ? -a / std::abs(a) : cplx(-1.0)) * nrm;
        cvec vh(rows, cplx(0.0));
        for (int i = k; i < rows; ++i) vh[i] = H[k][i];
        vh[k] -= alpha;
        double vn = 0.0;
        for (int i = k; i < rows; ++i) vn += std::norm(vh[i]);
        if (vn == 0.0) continue;
        auto reflect = [&](cvec& x) {
            cplx d = 0.0;
            for (int i = k; i < rows; ++i) d += std::conj(vh[i]) * x[i];
            d *= 2.0 / vn;
            for (int i = k; i < rows; ++i) x[i] -= d * vh[i];
        };
        for (int j = k; j < cols; ++j) reflect(H[j]);
        reflect(b);
    }
    cvec y(cols, cplx(0.0));
    for (int k = cols - 1; k >= 0; --k) {
        cplx s = b[k];
        for (int j = k + 1; j < cols; ++j) s -= H[j][k] * y[j];
        y[k] = (H[k][k] != cplx(0.0)) ? s / H[k][k] : cplx(0.0);
    }
    return y;
}

// proj/core/src/twogrid.cpp:278-331
SolveResult solve(const cvec& f, const Ops& ops) {
    SolveResult res;
    const std::size_t n = f.size();
    res.u.assign(n, cplx(0.0));
    const double nf = norm2(f);
    if (nf == 0.0) return res;
    const Config& cfg = ops.cfg;
    cvec r(n);
    if (cfg.outer == Outer::Richardson) {
        for (int it = 1; it <= cfg.max_iters; ++it) {
            two_grid_step(res.u, f, ops);
            ops.A.residual(f.data(), res.u.data(), r.data());
            const double rr = norm2(r) / nf;
            res.history.push_back(rr);
            res.iterations = it;
            if (rr <= cfg.tol) return res;
        }
        res.converged = false;
        return res;
    }
    // GMRES on M A u = M f, M = two-grid step from zero (left preconditioner)
    auto precond = [&](const cvec& rhs) {
        cvec z(n, cplx(0.0));
        two_grid_step(z, rhs, ops);
        return z;
    };
    const int mmax = cfg.max_iters;
    cvec b = precond(f);
    const double beta = norm2(b);
    std::vector<cvec> Q;
    Q.push_back(b);
    for (auto& z : Q.back()) z /= beta;
    std::vector<cvec> Hcols;  // column it-1 has it+1 entries (padded as needed)
    cvec Aq(n);
    for (int it = 1; it <= mmax; ++it) {
        ops.A.apply(Q.back().data(), Aq.data());
        cvec w = precond(Aq);
        cvec hcol(mmax + 1, cplx(0.0));
        for (int i = 0; i < it; ++i) {
            cplx d = 0.0;
            for (std::size_t j = 0; j < n; ++j) d += std::conj(Q[i][j]) * w[j];
            hcol[i] = d;
            for (std::size_t j = 0; j < n; ++j) w[j] -= d * Q[i][j];
        }
        const double hn = norm2(w);
        hcol[it] = hn;
        if (hn > 1e-300)
            for (auto& z : w) z /= hn;
        else
            std::fill(w.begin(), w.end(), cplx(0.0));
        Q.push_back(std::move(w));
        Hcols.push_back(hcol);
        std::vector<cvec> Hs;
        for (int c = 0; c < it; ++c) Hs.push_back(cvec(Hcols[c].begin(), Hcols[c].begin() + it + 1));
        cvec y = small_lstsq(Hs, it + 1, cplx(beta, 0.0));
        cvec u(n, cplx(0.0));
        for (int i = 0; i < it; ++i)
            for (std::size_t j = 0; j < n; ++j) u[j] += y[i] * Q[i][j];
        ops.A.residual(f.data(), u.data(), r.data());
        const double rr = norm2(r) / nf;
        res.history.push_back(rr);
        res.iterations = it;
        if (rr <= cfg.tol || it == mmax) {
            res.u = u;
            res.converged = rr <= cfg.tol;
            return res;
        }
    }
    res.converged = false;
    return res;
}

// ---------------------------------------------------------------- problem
// proj/core/src/commands.cpp:14-39 and proj/core/src/mesh.cpp:232-261
Problem build_problem(int order, double wavelengths, double ppw, const std::array<Tag, 4>& side,
                      unsigned layer_mask, double layer_width_dofs, double damping_D) {
    Problem pr;
    pr.k = 2.0 * M_PI * wavelengths;
    pr.n_cells = int(std::lround(wavelengths * ppw / order));
    if (pr.n_cells < 2) throw std::invalid_argument("build_problem: domain under-resolved");
    if (order < 2 || order > 8 || order % 2 != 0)
        throw std::invalid_argument("build_space: order must be even, 2 <= p <= 8");
    const int n = pr.n_cells;
    pr.mesh = Rect{0, 0, n, n, 1.0 / n};
    pr.space = Space::build(pr.mesh, order);
    pr.tags = Tags::by_side(pr.mesh, side);
    const double eps_vol = pr.k * pr.k * damping_D / M_PI;
    if (!(pr.k > 0.0)) throw std::invalid_argument("CoefficientField: k must be positive");
    if (eps_vol < 0.0) throw std::invalid_argument("CoefficientField: eps must be nonnegative");
    pr.coeffs.r = pr.mesh;
    pr.coeffs.k.assign(std::size_t(n) * n, pr.k);
    pr.coeffs.eps.assign(std::size_t(n) * n, layer_mask ? 0.0 : eps_vol);
    if (layer_mask) {
        const int layer_cells = int(std::ceil(layer_width_dofs / order - 1e-12));
        const double h = pr.mesh.h, width = layer_cells * h;
        if (width > n * h) throw std::invalid_argument("absorbing_layer: layer wider than domain");
        for (int y = 0; y < n; ++y)
            for (int x = 0; x < n; ++x) {
                double d = 0.0;
                for (int sd = 0; sd < 4; ++sd) {
                    if (!(layer_mask & (1u << sd))) continue;
                    double dist;
                    switch (sd) {
                        case kLeft: dist = (x + 0.5) * h; break;
                        case kRight: dist = (n - 1 - x + 0.5) * h; break;
                        case kBottom: dist = (y + 0.5) * h; break;
                        default: dist = (n - 1 - y + 0.5) * h; break;
                    }
                    d = std::max(d, width - dist);
                }
                double e = d > 0.0 ? layer_epsilon(pr.k, d, width) : 0.0;
                if (eps_vol > 0.0) e += eps_vol;
                pr.coeffs.eps[y * n + x] = e;
            }
    }
    pr.rhs.assign(pr.space.ndof, cplx(0.0));
    pr.rhs[pr.space.vertex(n / 2, n / 2)] = cplx(1.0, 0.0);
    for (int d : pr.space.dirichlet_dofs(pr.tags)) pr.rhs[d] = cplx(0.0);
    return pr;
}

cvec random_vector(int n, unsigned seed) {
    std::mt19937 rng(seed);
    std::normal_distribution<double> g;
    cvec v(n);
    for (int i = 0; i < n; ++i) {
        const double re = g(rng);
        const double im = g(rng);
        v[i] = cplx(re, im);
    }
    return v;
}

}  // namespace orc
