// tri.cpp -- order-p triangle elements (host setup).
//
// The reference's triangle meshes split every square cell along the diagonal
// (0,0)-(1,1) into a lower {y <= x} and an upper {y >= x} triangle with the
// hierarchical P_p basis of proj/core/src/basis.cpp:147-252: barycentric
// vertex functions, edge functions lam_a lam_b K_d(lam_b - lam_a) oriented by
// the global rule (h edges left->right, v edges bottom->top, diagonals
// lower-left->upper-right), bubbles lam_0 lam_1 lam_2 P_i(lam_1 - lam_0)
// P_j(2 lam_2 - 1) degree-major; element matrices by the collapsed Gauss rule
// of basis.cpp:134-146. The dofs of a unit cell are vertex, h-edge, v-edge,
// diagonal edge, lower interior, upper interior (fespace.cpp:37-54), p^2 in all
// -- the same count and the same unit-cell layout as a square cell, so every
// triangle dof gets the lattice position of the square dof that occupies its
// slot: the vertex / edge positions coincide and the diagonal and interior dofs
// fill the square's interior block. Element rows then address the same lattice
// and global numbering as the square path (fe_lattice, the partition, the
// gather / combine tables).
#include <algorithm>
#include <array>
#include <cmath>
#include <mutex>
#include <utility>
#include <vector>

#include "coarse.hpp"
#include "setup.hpp"

namespace htg {

namespace {

using Poly = std::vector<double>;  // coefficients, lowest degree first

double peval(const Poly& c, double x) {
    double v = 0.0;
    for (int i = int(c.size()) - 1; i >= 0; --i) v = v * x + c[i];
    return v;
}
Poly pder(const Poly& c) {
    if (c.size() <= 1) return Poly{0.0};
    Poly d(c.size() - 1);
    for (size_t i = 1; i < c.size(); ++i) d[i - 1] = c[i] * double(i);
    return d;
}
Poly legendre(int n) {  // (m+1) P_{m+1} = (2m+1) x P_m - m P_{m-1}
    Poly pm{1.0};
    if (n == 0) return pm;
    Poly pc{0.0, 1.0};
    for (int m = 1; m < n; ++m) {
        Poly pn(m + 2, 0.0);
        for (size_t i = 0; i < pc.size(); ++i) pn[i + 1] += (2.0 * m + 1.0) * pc[i];
        for (size_t i = 0; i < pm.size(); ++i) pn[i] -= double(m) * pm[i];
        for (double& v : pn) v /= (m + 1.0);
        pm = pc;
        pc = pn;
    }
    return pc;
}
// Gauss-Legendre on [0, 1] (basis.cpp:62-92)
void gauss01(int n, std::vector<double>& x, std::vector<double>& w) {
    x.assign(n, 0.0);
    w.assign(n, 0.0);
    for (int i = 0; i < n; ++i) {
        double t = std::cos(M_PI * (i + 0.75) / (n + 0.5));
        for (int it = 0; it < 100; ++it) {
            double pm = 1.0, pc = t;
            if (n == 0) pc = 1.0;
            for (int m = 1; m < n; ++m) {
                const double pn = ((2.0 * m + 1.0) * t * pc - m * pm) / (m + 1.0);
                pm = pc;
                pc = pn;
            }
            const double dp = n * (t * pc - pm) / (t * t - 1.0), dt = pc / dp;
            t -= dt;
            if (std::abs(dt) < 1e-15) break;
        }
        x[i] = 0.5 * (1.0 - t);
        double pm = 1.0, pc = t;
        for (int m = 1; m < n; ++m) {
            const double pn = ((2.0 * m + 1.0) * t * pc - m * pm) / (m + 1.0);
            pm = pc;
            pc = pn;
        }
        const double dp = n * (t * pc - pm) / (t * t - 1.0);
        w[i] = 1.0 / ((1.0 - t * t) * dp * dp);
    }
}

// dense solve with partial pivoting (tiny stage-interpolation systems)
void lu_solve(int n, std::vector<double> A, std::vector<double>& X, int nrhs) {
    std::vector<int> piv(n);
    for (int k = 0; k < n; ++k) {
        int p = k;
        for (int i = k + 1; i < n; ++i)
            if (std::abs(A[size_t(i) * n + k]) > std::abs(A[size_t(p) * n + k])) p = i;
        if (A[size_t(p) * n + k] == 0.0) throw RuntimeError("stage_interp: singular interpolation system");
        if (p != k) {
            for (int j = 0; j < n; ++j) std::swap(A[size_t(k) * n + j], A[size_t(p) * n + j]);
            for (int j = 0; j < nrhs; ++j) std::swap(X[size_t(k) * nrhs + j], X[size_t(p) * nrhs + j]);
        }
        for (int i = k + 1; i < n; ++i) {
            const double f = A[size_t(i) * n + k] / A[size_t(k) * n + k];
            for (int j = k; j < n; ++j) A[size_t(i) * n + j] -= f * A[size_t(k) * n + j];
            for (int j = 0; j < nrhs; ++j) X[size_t(i) * nrhs + j] -= f * X[size_t(k) * nrhs + j];
        }
    }
    for (int i = n - 1; i >= 0; --i)
        for (int j = 0; j < nrhs; ++j) {
            double s = X[size_t(i) * nrhs + j];
            for (int k = i + 1; k < n; ++k) s -= A[size_t(i) * n + k] * X[size_t(k) * nrhs + j];
            X[size_t(i) * nrhs + j] = s / A[size_t(i) * n + i];
        }
}

struct TriBasis {
    int p = 0, sub = 0, n = 0, nint = 0;
    double bary[3][3];  // lam_i = bary[0][i] + bary[1][i] x + bary[2][i] y
    std::vector<std::array<int, 2>> epairs;
    std::vector<Poly> kern, kern_der, leg, leg_der;
    std::vector<std::array<int, 2>> bubbles;

    TriBasis(int p_, int sub_) : p(p_), sub(sub_) {
        double verts[3][2];
        if (sub == 0) {  // lower: (0,0),(1,0),(1,1); edges bottom, right-v, diagonal
            const double v[3][2] = {{0, 0}, {1, 0}, {1, 1}};
            std::copy(&v[0][0], &v[0][0] + 6, &verts[0][0]);
            epairs = {{0, 1}, {1, 2}, {0, 2}};
        } else {  // upper: (0,0),(1,1),(0,1); edges top-h, left-v, diagonal
            const double v[3][2] = {{0, 0}, {1, 1}, {0, 1}};
            std::copy(&v[0][0], &v[0][0] + 6, &verts[0][0]);
            epairs = {{2, 1}, {0, 2}, {0, 1}};
        }
        // inverse of V = [1 x y] rows (basis.cpp: bary_coef_ = V.inverse())
        double V[3][3];
        for (int i = 0; i < 3; ++i) V[i][0] = 1.0, V[i][1] = verts[i][0], V[i][2] = verts[i][1];
        const double det = V[0][0] * (V[1][1] * V[2][2] - V[1][2] * V[2][1]) -
                           V[0][1] * (V[1][0] * V[2][2] - V[1][2] * V[2][0]) +
                           V[0][2] * (V[1][0] * V[2][1] - V[1][1] * V[2][0]);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                const int i1 = (j + 1) % 3, i2 = (j + 2) % 3, j1 = (i + 1) % 3, j2 = (i + 2) % 3;
                bary[i][j] = (V[i1][j1] * V[i2][j2] - V[i1][j2] * V[i2][j1]) / det;  // inverse(i, j)
            }
        for (int d = 2; d <= p; ++d) {
            Poly k = pder(legendre(d - 1));
            const double s = -4.0 * std::sqrt((2.0 * d - 1.0) / 2.0) / (d * (d - 1.0));
            for (double& v : k) v *= s;
            kern.push_back(k);
            kern_der.push_back(pder(k));
        }
        for (int d = 3; d <= p; ++d)
            for (int i = 0; i <= d - 3; ++i) bubbles.push_back({i, d - 3 - i});
        for (int m = 0; m <= p; ++m) {
            leg.push_back(legendre(m));
            leg_der.push_back(pder(leg.back()));
        }
        nint = int(bubbles.size());
        n = 3 + 3 * (p - 1) + nint;
    }

    void eval(double x, double y, std::vector<double>& val, std::vector<std::array<double, 2>>& grad) const {
        val.assign(n, 0.0);
        grad.assign(n, {0.0, 0.0});
        double lam[3], dl[3][2];
        for (int i = 0; i < 3; ++i) {
            lam[i] = bary[0][i] + bary[1][i] * x + bary[2][i] * y;
            dl[i][0] = bary[1][i];
            dl[i][1] = bary[2][i];
        }
        int idx = 0;
        for (int i = 0; i < 3; ++i, ++idx) {
            val[idx] = lam[i];
            grad[idx] = {dl[i][0], dl[i][1]};
        }
        for (const auto& e : epairs) {
            const int a = e[0], b = e[1];
            for (int d = 2; d <= p; ++d, ++idx) {
                const double s = lam[b] - lam[a];
                const double Kv = peval(kern[d - 2], s), Kd = peval(kern_der[d - 2], s);
                val[idx] = lam[a] * lam[b] * Kv;
                for (int c = 0; c < 2; ++c)
                    grad[idx][c] = (dl[a][c] * lam[b] + lam[a] * dl[b][c]) * Kv + lam[a] * lam[b] * Kd * (dl[b][c] - dl[a][c]);
            }
        }
        const double bub = lam[0] * lam[1] * lam[2];
        double db[2];
        for (int c = 0; c < 2; ++c) db[c] = dl[0][c] * lam[1] * lam[2] + lam[0] * dl[1][c] * lam[2] + lam[0] * lam[1] * dl[2][c];
        for (const auto& bb : bubbles) {
            const double u = lam[1] - lam[0], v = 2.0 * lam[2] - 1.0;
            const double Pi = peval(leg[bb[0]], u), Pj = peval(leg[bb[1]], v);
            const double dPi = peval(leg_der[bb[0]], u), dPj = peval(leg_der[bb[1]], v);
            val[idx] = bub * Pi * Pj;
            for (int c = 0; c < 2; ++c)
                grad[idx][c] = db[c] * Pi * Pj + bub * (dPi * (dl[1][c] - dl[0][c]) * Pj + Pi * dPj * 2.0 * dl[2][c]);
            ++idx;
        }
    }
};

TriElement build_tri_element(int p, int sub) {
    TriBasis tb(p, sub);
    TriElement T;
    T.p = p;
    T.n = tb.n;
    T.K.assign(size_t(T.n) * T.n, 0.0);
    T.M.assign(size_t(T.n) * T.n, 0.0);
    // collapsed Gauss rule on the element's triangle (basis.cpp:134-146)
    const double a[2] = {0, 0};
    const double b[2] = {sub == 0 ? 1.0 : 1.0, sub == 0 ? 0.0 : 1.0};
    const double c[2] = {sub == 0 ? 1.0 : 0.0, 1.0};
    std::vector<double> xu, wu, xv, wv;
    gauss01(p + 1, xu, wu);
    gauss01(p + 2, xv, wv);
    const double detJ = std::abs((b[0] - a[0]) * (c[1] - a[1]) - (c[0] - a[0]) * (b[1] - a[1]));
    std::vector<double> val;
    std::vector<std::array<double, 2>> grad;
    for (size_t i = 0; i < xu.size(); ++i)
        for (size_t j = 0; j < xv.size(); ++j) {
            const double r = xu[i] * (1.0 - xv[j]), s = xv[j];
            const double x = a[0] + r * (b[0] - a[0]) + s * (c[0] - a[0]);
            const double y = a[1] + r * (b[1] - a[1]) + s * (c[1] - a[1]);
            const double w = wu[i] * wv[j] * (1.0 - xv[j]) * detJ;
            tb.eval(x, y, val, grad);
            for (int r2 = 0; r2 < T.n; ++r2)
                for (int c2 = 0; c2 < T.n; ++c2) {
                    T.K[size_t(r2) * T.n + c2] += w * (grad[r2][0] * grad[c2][0] + grad[r2][1] * grad[c2][1]);
                    T.M[size_t(r2) * T.n + c2] += w * val[r2] * val[c2];
                }
        }
    // lattice placement of the element dofs (fespace.cpp:85-108 element_dofs)
    const int ne = p - 1, ni = (p - 1) * (p - 2) / 2;
    auto slot_int = [&](int i) {  // square interior slot i -> pseudo (jx, jy)
        return std::array<int, 2>{1 + i / ne, 1 + i % ne};
    };
    auto add = [&](int dx, int dy, int jx, int jy) { T.place.push_back({dx, dy, jx, jy}); };
    if (sub == 0) {
        add(0, 0, 0, 0);
        add(1, 0, 0, 0);
        add(1, 1, 0, 0);
        for (int d = 0; d < ne; ++d) add(0, 0, 1 + d, 0);  // bottom h edge
        for (int d = 0; d < ne; ++d) add(1, 0, 0, 1 + d);  // right v edge
        for (int d = 0; d < ne; ++d) {                     // diagonal
            const auto s = slot_int(d);
            add(0, 0, s[0], s[1]);
        }
        for (int i = 0; i < ni; ++i) {
            const auto s = slot_int(ne + i);
            add(0, 0, s[0], s[1]);
        }
    } else {
        add(0, 0, 0, 0);
        add(1, 1, 0, 0);
        add(0, 1, 0, 0);
        for (int d = 0; d < ne; ++d) add(0, 1, 1 + d, 0);  // top h edge
        for (int d = 0; d < ne; ++d) add(0, 0, 0, 1 + d);  // left v edge
        for (int d = 0; d < ne; ++d) {                     // diagonal
            const auto s = slot_int(d);
            add(0, 0, s[0], s[1]);
        }
        for (int i = 0; i < ni; ++i) {
            const auto s = slot_int(ne + ni + i);
            add(0, 0, s[0], s[1]);
        }
    }
    // staged interpolation from the q = p/2 coarse lattice (fespace.cpp:260-378)
    const int q = p / 2;
    std::vector<std::array<double, 2>> pts;
    std::vector<std::array<double, 2>> verts;
    std::vector<std::array<std::array<double, 2>, 2>> edges;
    if (sub == 0) {
        verts = {{{0, 0}}, {{1, 0}}, {{1, 1}}};
        edges = {{{{0, 0}, {1, 0}}}, {{{1, 0}, {1, 1}}}, {{{0, 0}, {1, 1}}}};
    } else {
        verts = {{{0, 0}}, {{1, 1}}, {{0, 1}}};
        edges = {{{{0, 1}, {1, 1}}}, {{{0, 0}, {0, 1}}}, {{{0, 0}, {1, 1}}}};
    }
    for (auto v : verts) pts.push_back(v);
    for (auto e : edges)
        for (int s = 1; s < q; ++s)
            pts.push_back({e[0][0] + (e[1][0] - e[0][0]) * s / q, e[0][1] + (e[1][1] - e[0][1]) * s / q});
    if (sub == 0) {
        for (int s = 1; s < q; ++s)
            for (int t = 1; t < s; ++t) pts.push_back({double(s) / q, double(t) / q});
    } else {
        for (int s = 1; s < q; ++s)
            for (int t = s + 1; t < q; ++t) pts.push_back({double(s) / q, double(t) / q});
    }
    const int npts = int(pts.size()), nv = 3, neq = q - 1;
    std::vector<std::vector<int>> erows(3);
    for (int e = 0; e < 3; ++e)
        for (int d = 2; d <= q; ++d) erows[e].push_back(nv + e * ne + (d - 2));
    std::vector<int> irows;
    const int ib = nv + 3 * ne, nbq = (q - 1) * (q - 2) / 2;
    for (int i = 0; i < nbq; ++i) irows.push_back(ib + i);
    std::vector<double> E(size_t(T.n) * npts, 0.0);
    for (int v = 0; v < nv; ++v) E[size_t(v) * npts + v] = 1.0;
    auto stage = [&](const std::vector<int>& rows, int pt0) {
        const int k = int(rows.size());
        if (k == 0) return;
        std::vector<double> B(size_t(k) * k), R(size_t(k) * npts, 0.0);
        for (int a2 = 0; a2 < k; ++a2) {
            tb.eval(pts[pt0 + a2][0], pts[pt0 + a2][1], val, grad);
            for (int d = 0; d < k; ++d) B[size_t(a2) * k + d] = val[rows[d]];
            for (int j = 0; j < npts; ++j) {  // minus the current interpolant
                double s = 0.0;
                for (int i = 0; i < T.n; ++i) s += val[i] * E[size_t(i) * npts + j];
                R[size_t(a2) * npts + j] = -s;
            }
            R[size_t(a2) * npts + pt0 + a2] += 1.0;
        }
        lu_solve(k, B, R, npts);
        for (int d = 0; d < k; ++d)
            for (int j = 0; j < npts; ++j) E[size_t(rows[d]) * npts + j] = R[size_t(d) * npts + j];
    };
    int pt = nv;
    for (int e = 0; e < 3; ++e) {
        if (neq == 0) break;
        stage(erows[e], pt);
        pt += neq;
    }
    stage(irows, pt);
    T.E = E;
    T.npts = npts;
    for (auto& p2 : pts) T.stage_pts.push_back({int(std::lround(p2[0] * q)), int(std::lround(p2[1] * q))});
    return T;
}

}  // namespace

// IP for triangle meshes, build_prolongation (proj/core/src/twogrid.cpp:150-187)
// restated: cells in mesh order, lower then upper triangle; each fine row is
// written by the first element holding the dof; rows of fine Dirichlet dofs and
// columns of coarse Dirichlet vertices are zero. CSR over fine dofs.
void tri_prolongation(const HostProblem& hp, std::vector<int>& rp, std::vector<int>& ci, std::vector<double>& v) {
    const int p = hp.p, m = p / 2, CX = hp.nx * m, CY = hp.ny * m;
    const long long nf = hp.ndof();
    const std::vector<char> fd = fe_dirichlet(hp, p);
    const int W = hp.nx * p + 1;
    std::vector<char> fdir(size_t(nf), 0), written(size_t(nf), 0);
    for (int gy = 0; gy <= hp.ny * p; ++gy)
        for (int gx = 0; gx < W; ++gx)
            if (fd[size_t(gy) * W + gx]) fdir[size_t(dof_index(hp.nx, hp.ny, p, gx, gy))] = 1;
    auto cdir = [&](int X, int Y) {
        if (!hp.has_dirichlet) return false;
        bool d = false;
        if (X == 0 || X == CX) {
            const auto& tg = X == 0 ? hp.tl : hp.tr;
            d |= (Y > 0 && tg[(Y - 1) / m] == kDirichlet) || (Y < CY && tg[Y / m] == kDirichlet);
        }
        if (Y == 0 || Y == CY) {
            const auto& tg = Y == 0 ? hp.tb : hp.tt;
            d |= (X > 0 && tg[(X - 1) / m] == kDirichlet) || (X < CX && tg[X / m] == kDirichlet);
        }
        return d;
    };
    std::vector<std::vector<std::pair<int, double>>> rows(static_cast<size_t>(nf));
    for (int cy = 0; cy < hp.ny; ++cy)
        for (int cx = 0; cx < hp.nx; ++cx)
            for (int sub = 0; sub < 2; ++sub) {
                const TriElement& T = tri_element(p, sub);
                for (int i = 0; i < T.n; ++i) {
                    const auto& pl = T.place[i];
                    const long long d = dof_index(hp.nx, hp.ny, p, (cx + pl[0]) * p + pl[2], (cy + pl[1]) * p + pl[3]);
                    if (written[size_t(d)]) continue;
                    written[size_t(d)] = 1;
                    if (fdir[size_t(d)]) continue;
                    for (int j = 0; j < T.npts; ++j) {
                        const double val = T.E[size_t(i) * T.npts + j];
                        const int X = cx * m + T.stage_pts[j][0], Y = cy * m + T.stage_pts[j][1];
                        if (val != 0.0 && !cdir(X, Y)) rows[size_t(d)].push_back({Y * (CX + 1) + X, val});
                    }
                }
            }
    rp.assign(size_t(nf) + 1, 0);
    ci.clear();
    v.clear();
    for (long long r = 0; r < nf; ++r) {
        auto& rr = rows[size_t(r)];
        std::sort(rr.begin(), rr.end());
        for (auto& e : rr) {
            if (!ci.empty() && int(ci.size()) > rp[size_t(r)] && ci.back() == e.first) v.back() += e.second;
            else ci.push_back(e.first), v.push_back(e.second);
        }
        rp[size_t(r) + 1] = int(ci.size());
    }
}

const TriElement& tri_element(int p, int sub) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, TriElement> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(p, sub);
    auto it = cache.find(key);
    if (it == cache.end()) it = cache.emplace(key, build_tri_element(p, sub)).first;
    return it->second;
}

}  // namespace htg
