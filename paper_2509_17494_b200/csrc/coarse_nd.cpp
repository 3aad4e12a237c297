// coarse_nd.cpp -- QSFEM coarse matrix and its nested-dissection multifrontal
// LU, factored once on the host at setup (coarse.cu uploads the factors and
// runs the level-batched solves on the GPU).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <map>
#include <thread>

#include "coarse.hpp"

// host AVX2 + FMA kernel of the trailing update (the product build passes
// -march=x86-64-v3; HTG_ND_NOAVX keeps the scalar form; never in device code)
#if defined(__AVX2__) && defined(__FMA__) && !defined(__CUDA_ARCH__) && !defined(HTG_ND_NOAVX)
#include <immintrin.h>
#define HTG_ND_AVX2 1
#else
#define HTG_ND_AVX2 0
#endif

namespace htg {

// ------------------------------------------------------------------ QSFEM
QsfemWeights qsfem_weights(double eta) {
    if (!(eta > 0.0) || !(eta < M_PI))
        throw InvalidArgument("qsfem: eta = k*h_c must lie in (0, pi) (at least two coarse points per wavelength)");
    // zero set of the symbol interpolated in the directions pi/16 and 3pi/16
    const double a1 = std::cos(eta * std::cos(M_PI / 16.0)), b1 = std::cos(eta * std::sin(M_PI / 16.0));
    const double a2 = std::cos(eta * std::cos(3.0 * M_PI / 16.0)), b2 = std::cos(eta * std::sin(3.0 * M_PI / 16.0));
    const double den = a2 * b2 * (a1 + b1) - a1 * b1 * (a2 + b2);
    if (std::fabs(den) < 1e-14) throw RuntimeError("qsfem: degenerate stencil (denominator ~ 0)");
    QsfemWeights w;
    w.eta = eta;
    w.P0 = 4.0;
    w.P1 = 2.0 * (a1 * b1 - a2 * b2) / den;
    w.P2 = (a2 + b2 - a1 - b1) / den;
    const double sigma0 = w.P0 + 4.0 * w.P1 + 4.0 * w.P2;  // symbol at the origin
    if (sigma0 == 0.0) throw RuntimeError("qsfem: sigma_P(0) = 0, scaling undefined");
    w.N = -eta * eta / sigma0;
    w.q0 = w.N * w.P0 / 4.0;
    w.q1 = w.N * w.P1 / 2.0;
    w.q2 = w.N * w.P2;
    return w;
}

std::vector<cplx> coarse_stencil(const HostProblem& hp) {
    const int m = hp.p / 2, CX = hp.nx * m, CY = hp.ny * m;
    const double hc = 2.0 * hp.h / hp.p;
    const size_t nv = size_t(CX + 1) * (CY + 1);
    std::vector<cplx> A9(nv * 9, cplx(0.0));
    std::vector<QsfemWeights> qw(hp.cls_k.size());
    for (size_t c = 0; c < qw.size(); ++c) qw[c] = qsfem_weights(hc * hp.cls_k[c]);
    auto cellcls = [&](int cx, int cy) { return hp.cls[size_t(cy / m) * hp.nx + cx / m]; };
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
    auto rows_of = [&](int Y0, int Y1) {
    for (int Y = Y0; Y < Y1; ++Y)
        for (int X = 0; X <= CX; ++X) {
            cplx* row = &A9[(size_t(Y) * (CX + 1) + X) * 9];
            if (cdir(X, Y)) {
                row[4] = 1.0;
                continue;
            }
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int WX = X + dx, WY = Y + dy;
                    if (WX < 0 || WX > CX || WY < 0 || WY > CY || cdir(WX, WY)) continue;
                    cplx s = 0.0;
                    for (int cy = std::max(std::max(Y, WY) - 1, 0); cy <= std::min(std::min(Y, WY), CY - 1); ++cy)
                        for (int cx = std::max(std::max(X, WX) - 1, 0); cx <= std::min(std::min(X, WX), CX - 1); ++cx) {
                            const int c = cellcls(cx, cy);
                            const QsfemWeights& q = qw[c];
                            const int md = std::abs(dx) + std::abs(dy);
                            const double qv = md == 0 ? q.q0 : (md == 1 ? q.q1 : q.q2);
                            const double mass = double((dx == 0 ? 2 : 1) * (dy == 0 ? 2 : 1)) / 36.0;
                            s += cplx(qv, -hp.cls_eps[c] * hc * hc * mass);
                        }
                    // absorbing coarse boundary edges containing both vertices
                    auto robin = [&](const std::vector<double>& kh, int e) {
                        const double khc = kh[e / m] / m;
                        s += cplx(0.0, -khc * ((dx == 0 && dy == 0) ? 1.0 / 3.0 : 1.0 / 6.0));
                    };
                    if (dy == 0 && (Y == 0 || Y == CY)) {
                        const auto& kh = Y == 0 ? hp.khb : hp.kht;
                        if (dx <= 0 && X > 0) robin(kh, X - 1);
                        if (dx >= 0 && X < CX) robin(kh, X);
                    }
                    if (dx == 0 && (X == 0 || X == CX)) {
                        const auto& kh = X == 0 ? hp.khl : hp.khr;
                        if (dy <= 0 && Y > 0) robin(kh, Y - 1);
                        if (dy >= 0 && Y < CY) robin(kh, Y);
                    }
                    row[(dy + 1) * 3 + (dx + 1)] = s;
                }
        }
    };
    // lattice rows are independent: split them over the host threads
    const int nthr = nv < 100000 ? 1 : std::max(1, std::min(int(std::thread::hardware_concurrency()), CY + 1));
    if (nthr == 1) {
        rows_of(0, CY + 1);
    } else {
        std::vector<std::thread> th;
        for (int w = 0; w < nthr; ++w) th.emplace_back(rows_of, (CY + 1) * w / nthr, (CY + 1) * (w + 1) / nthr);
        for (auto& x : th) x.join();
    }
    return A9;
}

// ------------------------------------------------------------------ lattice matrices
cplx LatticeMatrix::at(int i, int j) const {
    const auto b = ci.begin() + rp[i], e = ci.begin() + rp[i + 1];
    const auto it = std::lower_bound(b, e, j);
    return (it != e && *it == j) ? v[size_t(it - ci.begin())] : cplx(0.0);
}

namespace {
// CSR from per-row (col, value) lists: sort, sum duplicates
void finish_csr(LatticeMatrix& L, std::vector<std::vector<std::pair<int, cplx>>>& rows) {
    const int n = int(rows.size());
    L.rp.assign(n + 1, 0);
    L.ci.clear();
    L.v.clear();
    for (int i = 0; i < n; ++i) {
        auto& r = rows[i];
        std::sort(r.begin(), r.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        for (size_t k = 0; k < r.size(); ++k) {
            if (!L.ci.empty() && int(L.ci.size()) > L.rp[i] && L.ci.back() == r[k].first) {
                L.v.back() += r[k].second;
            } else {
                L.ci.push_back(r[k].first);
                L.v.push_back(r[k].second);
            }
        }
        L.rp[i + 1] = int(L.ci.size());
        std::vector<std::pair<int, cplx>>().swap(r);
    }
}
}  // namespace

LatticeMatrix qsfem_lattice(const HostProblem& hp) {
    const int m = hp.p / 2;
    LatticeMatrix L;
    L.W = hp.nx * m + 1;
    L.H = hp.ny * m + 1;
    L.q = 1;
    const int nv = L.W * L.H;
    L.id.resize(nv);
    for (int i = 0; i < nv; ++i) L.id[i] = i;
    const std::vector<cplx> A9 = coarse_stencil(hp);
    // CSR straight from the stencil: (dy, dx) ascending is column-ascending
    L.rp.assign(size_t(nv) + 1, 0);
    L.ci.reserve(size_t(nv) * 9);
    L.v.reserve(size_t(nv) * 9);
    for (int Y = 0; Y < L.H; ++Y)
        for (int X = 0; X < L.W; ++X) {
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int WX = X + dx, WY = Y + dy;
                    if (WX < 0 || WX >= L.W || WY < 0 || WY >= L.H) continue;
                    const cplx a = A9[(size_t(Y) * L.W + X) * 9 + (dy + 1) * 3 + (dx + 1)];
                    if (a != cplx(0.0)) {
                        L.ci.push_back(WY * L.W + WX);
                        L.v.push_back(a);
                    }
                }
            L.rp[size_t(Y) * L.W + X + 1] = int(L.ci.size());
        }
    return L;
}

std::vector<char> fe_dirichlet(const HostProblem& hp, int q) {
    const int W = hp.nx * q + 1, H = hp.ny * q + 1;
    std::vector<char> d(size_t(W) * H, 0);
    if (!hp.has_dirichlet) return d;
    for (int cx = 0; cx < hp.nx; ++cx)
        for (int j = 0; j <= q; ++j) {
            if (hp.tb[cx] == kDirichlet) d[cx * q + j] = 1;
            if (hp.tt[cx] == kDirichlet) d[size_t(H - 1) * W + cx * q + j] = 1;
        }
    for (int cy = 0; cy < hp.ny; ++cy)
        for (int j = 0; j <= q; ++j) {
            if (hp.tl[cy] == kDirichlet) d[size_t(cy * q + j) * W] = 1;
            if (hp.tr[cy] == kDirichlet) d[size_t(cy * q + j) * W + W - 1] = 1;
        }
    return d;
}

LatticeMatrix fe_lattice(const HostProblem& hp, const Basis1D& b, int q, double alpha) {
    if (q < 1 || q > hp.p) throw InvalidArgument("fe_lattice: order must lie in [1, p]");
    LatticeMatrix L;
    L.W = hp.nx * q + 1;
    L.H = hp.ny * q + 1;
    L.q = q;
    const int nv = L.W * L.H;
    L.id.resize(nv);
    for (int Y = 0; Y < L.H; ++Y)
        for (int X = 0; X < L.W; ++X) L.id[Y * L.W + X] = int(dof_index(hp.nx, hp.ny, q, X, Y));
    // 1-D local index a (0, 1: vertices, >= 2: bubble of degree a) -> lattice offset in the cell
    auto off = [&](int a) { return a == 0 ? 0 : (a == 1 ? q : a - 1); };
    const int B = q + 1;
    std::vector<std::vector<std::pair<int, cplx>>> rows(nv);
    auto dof = [&](int cx, int cy, int a, int c) { return L.id[(cy * q + off(c)) * L.W + cx * q + off(a)]; };
    const double h2 = hp.h * hp.h;
    if (hp.tri) {  // two order-q triangles per cell (tri.cpp), rows in the same lattice numbering
        for (int sub = 0; sub < 2; ++sub) {
            const TriElement& T = tri_element(q, sub);
            for (int cy = 0; cy < hp.ny; ++cy)
                for (int cx = 0; cx < hp.nx; ++cx) {
                    const double k = hp.kc(cx, cy), e = hp.ec(cx, cy);
                    const cplx m = cplx(k * k, k * k * alpha + e) * h2;
                    std::vector<int> gd(T.n);
                    for (int i = 0; i < T.n; ++i) {
                        const auto& pl = T.place[i];
                        gd[i] = L.id[((cy + pl[1]) * q + pl[3]) * L.W + (cx + pl[0]) * q + pl[2]];
                    }
                    for (int i = 0; i < T.n; ++i) {
                        auto& row = rows[gd[i]];
                        for (int j = 0; j < T.n; ++j) {
                            const cplx a = T.K[size_t(i) * T.n + j] - m * T.M[size_t(i) * T.n + j];
                            if (a != cplx(0.0)) row.push_back({gd[j], a});
                        }
                    }
                }
        }
    }
    for (int cy = 0; cy < (hp.tri ? 0 : hp.ny); ++cy)
        for (int cx = 0; cx < hp.nx; ++cx) {
            const double k = hp.kc(cx, cy), e = hp.ec(cx, cy);
            const cplx m = cplx(k * k, k * k * alpha + e) * h2;
            for (int ay = 0; ay < B; ++ay)
                for (int ax = 0; ax < B; ++ax) {
                    auto& row = rows[dof(cx, cy, ax, ay)];
                    for (int cy2 = 0; cy2 < B; ++cy2)
                        for (int cx2 = 0; cx2 < B; ++cx2) {
                            const double mm = b.M[ax][cx2] * b.M[ay][cy2];
                            const double kk = b.S[ax][cx2] * b.M[ay][cy2] + b.M[ax][cx2] * b.S[ay][cy2];
                            const cplx a = kk - m * mm;
                            if (a != cplx(0.0)) row.push_back({dof(cx, cy, cx2, cy2), a});
                        }
                }
        }
    // Robin edges: - i k h times the 1-D mass along the edge
    auto robin = [&](int cx, int cy, bool horiz, int side_local, double kh) {
        if (kh == 0.0) return;
        for (int a = 0; a < B; ++a)
            for (int c = 0; c < B; ++c) {
                const cplx val(0.0, -kh * b.M[a][c]);
                if (horiz) rows[dof(cx, cy, a, side_local)].push_back({dof(cx, cy, c, side_local), val});
                else rows[dof(cx, cy, side_local, a)].push_back({dof(cx, cy, side_local, c), val});
            }
    };
    for (int cx = 0; cx < hp.nx; ++cx) {
        robin(cx, 0, true, 0, hp.khb[cx]);
        robin(cx, hp.ny - 1, true, 1, hp.kht[cx]);
    }
    for (int cy = 0; cy < hp.ny; ++cy) {
        robin(0, cy, false, 0, hp.khl[cy]);
        robin(hp.nx - 1, cy, false, 1, hp.khr[cy]);
    }
    finish_csr(L, rows);
    if (hp.has_dirichlet) {  // closures of Dirichlet edges -> identity rows and columns
        const std::vector<char> dn = fe_dirichlet(hp, q);
        std::vector<char> dir(nv, 0);
        for (int i = 0; i < nv; ++i) dir[L.id[i]] = dn[i];
        for (int i = 0; i < nv; ++i)
            for (int k = L.rp[i]; k < L.rp[i + 1]; ++k)
                if (dir[i] || dir[L.ci[k]]) L.v[k] = L.ci[k] == i ? cplx(1.0) : cplx(0.0);
    }
    return L;
}

// ------------------------------------------------------------------ nested dissection
namespace {

// a separator line strictly inside [a0, a1] on the stride-q grid, nearest the middle, or -1
int pick_line(int a0, int a1, int q) {
    const int mid = (a0 + a1) / 2;
    int best = -1;
    for (int c = (a0 / q + 1) * q; c < a1; c += q)
        if (c > a0 && (best < 0 || std::abs(c - mid) < std::abs(best - mid))) best = c;
    return best;
}

int build_nd(NDTree& t, const LatticeMatrix& A, int x0, int x1, int y0, int y1, int depth, int leaf_max) {
    NDNode n;
    n.x0 = x0;
    n.x1 = x1;
    n.y0 = y0;
    n.y1 = y1;
    n.depth = depth;
    const int w = x1 - x0 + 1, h = y1 - y0 + 1;
    const auto node = [&](int x, int y) { return A.id[y * A.W + x]; };
    std::vector<int> kids;
    const int xl = pick_line(x0, x1, A.q), yl = pick_line(y0, y1, A.q);
    const bool sx = xl >= 0 && (w >= h || yl < 0), sy = !sx && yl >= 0;  // cut the longer side if it can be cut
    const int xm = sx ? xl : -1, ym = sy ? yl : -1;
    if (w * h <= leaf_max || (!sx && !sy)) {
        n.leaf = true;
        for (int y = y0; y <= y1; ++y)
            for (int x = x0; x <= x1; ++x) n.vars.push_back(node(x, y));
    } else if (xm >= 0) {
        kids.push_back(build_nd(t, A, x0, xm - 1, y0, y1, depth + 1, leaf_max));
        kids.push_back(build_nd(t, A, xm + 1, x1, y0, y1, depth + 1, leaf_max));
        for (int y = y0; y <= y1; ++y) n.vars.push_back(node(xm, y));
    } else {
        kids.push_back(build_nd(t, A, x0, x1, y0, ym - 1, depth + 1, leaf_max));
        kids.push_back(build_nd(t, A, x0, x1, ym + 1, y1, depth + 1, leaf_max));
        for (int x = x0; x <= x1; ++x) n.vars.push_back(node(x, ym));
    }
    // box edges lie next to separator lines (or the domain boundary), so every
    // coupling of the box leaves it through the one-node frame
    for (int y = y0 - 1; y <= y1 + 1; ++y)
        for (int x = x0 - 1; x <= x1 + 1; ++x) {
            if (x < 0 || y < 0 || x >= A.W || y >= A.H) continue;
            if (x >= x0 && x <= x1 && y >= y0 && y <= y1) continue;
            n.ring.push_back(node(x, y));
        }
    n.children = kids;
    t.max_depth = std::max(t.max_depth, depth);
    t.nodes.push_back(std::move(n));
    const int id = int(t.nodes.size()) - 1;
    for (int k : kids) t.nodes[k].parent = id;
    return id;
}

// C[rows i0..i1) -= A (m x k) * B (k x n), row-major, parallel over rows
void gemm_sub(int m, int n, int k, const cplx* A, const cplx* B, cplx* C, int nthreads) {
    auto body = [&](int i0, int i1) {
        for (int i = i0; i < i1; ++i) {
            cplx* ci = C + size_t(i) * n;
            const cplx* ai = A + size_t(i) * k;
            for (int kk = 0; kk < k; ++kk) {
                const cplx a = ai[kk];
                if (a == cplx(0.0)) continue;
                const cplx* bk = B + size_t(kk) * n;
                for (int j = 0; j < n; ++j) ci[j] -= a * bk[j];
            }
        }
    };
    if (nthreads <= 1 || size_t(m) * n * k < 2000000) {
        body(0, m);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t) th.emplace_back(body, m * t / nthreads, m * (t + 1) / nthreads);
    for (auto& x : th) x.join();
}


// Factor one front (children already factored). rpos/cpos: scratch
// global -> front row / column maps (all -1 on entry and exit).
//
// Front rows are [own separator vars | rows delayed by the children | ring],
// columns [own vars | columns delayed by the children | ring]. LU with
// threshold partial pivoting over the pivot block (the first sN rows and
// columns): column k is eliminated only if its best pivot candidate is at
// least pivtol times the largest entry of that column in the ring rows, which
// bounds the multipliers L21 by 1/pivtol. A column that fails is delayed: it
// is swapped to the end of the pivot block and, with the same number of
// unpivoted rows, handed to the parent as part of the contribution block.
// Pivoting restricted to one front cannot otherwise cope with the nearly
// singular pivot blocks of boxes close to a Dirichlet resonance (Helmholtz),
// and the growth it lets through costs ~cond * eps in backward error.
// key of a front for sharing: two independent 64-bit mixes of (F, sN, nown) and the
// bits of the assembled front matrix
struct FrontKey {
    unsigned long long a = 0, b = 0;
    bool operator<(const FrontKey& o) const { return a != o.a ? a < o.a : b < o.b; }
};

// key != nullptr: assemble the front and return its key only (no elimination).
// A sharer (n.rep >= 0) takes the representative's pivot order instead of factoring.
void factor_node(NDTree& t, int id, const LatticeMatrix& A, std::vector<int>& rpos, std::vector<int>& cpos,
                 double pivtol, int nthreads, FrontKey* key = nullptr) {
    NDNode& n = t.nodes[id];
    std::vector<int> rows = n.vars, cols = n.vars;
    for (int c : n.children) {
        const NDNode& ch = t.nodes[c];
        rows.insert(rows.end(), ch.rows.begin() + ch.ke, ch.rows.begin() + ch.sN);
        cols.insert(cols.end(), ch.cols.begin() + ch.ke, ch.cols.begin() + ch.sN);
    }
    const int nown = int(n.vars.size()), sN = int(rows.size()), u = int(n.ring.size()), F = sN + u;
    rows.insert(rows.end(), n.ring.begin(), n.ring.end());
    cols.insert(cols.end(), n.ring.begin(), n.ring.end());
    if (!key && n.rep >= 0) {  // sharer: the representative's pivot order on this node's labels
        const NDNode& rp = t.nodes[size_t(n.rep)];
        n.sN = sN;
        n.F = F;
        n.ke = rp.ke;
        n.rows.resize(F);
        n.cols.resize(F);
        for (int i = 0; i < F; ++i) {
            n.rows[i] = rows[size_t(rp.perm_r[i])];
            n.cols[i] = cols[size_t(rp.perm_c[i])];
        }
        n.rc.assign(F, -1);
        for (int v : n.vars) cpos[v] = 0;
        for (int i = 0; i < F; ++i)
            if (cpos[n.rows[i]] == 0) n.rc[i] = n.rows[i];
        for (int v : n.vars) cpos[v] = -1;
        return;
    }
    for (int i = 0; i < F; ++i) {
        rpos[rows[i]] = i;
        cpos[cols[i]] = i;
    }
    std::vector<int> prow(F), pcol(F);  // initial position of each front row / column
    for (int i = 0; i < F; ++i) prow[i] = pcol[i] = i;
    std::vector<cplx> Fm(size_t(F) * F, cplx(0.0));
    // original entries not assembled below: own-var rows against own and ring
    // columns, and ring rows against own columns (a delayed variable's
    // couplings already sit in the child's contribution block)
    auto fresh = [&](int p) { return p >= 0 && (p < nown || p >= sN); };
    for (int i = 0; i < nown; ++i) {
        const int v = n.vars[i];
        for (int k = A.rp[v]; k < A.rp[v + 1]; ++k) {
            const int w = A.ci[k], pw = cpos[w];
            if (!fresh(pw)) continue;
            Fm[size_t(i) * F + pw] += A.v[k];
            if (pw >= sN) Fm[size_t(rpos[w]) * F + i] += A.at(w, v);
        }
    }
    for (int c : n.children) {
        NDNode& ch = t.nodes[c];
        const std::vector<cplx>& chS = nd_blocks(t.nodes, ch).S;
        const int uc = ch.F - ch.ke;
        std::vector<int> rm(uc), cm(uc);
        for (int a = 0; a < uc; ++a) {
            rm[a] = rpos[ch.rows[ch.ke + a]];
            cm[a] = cpos[ch.cols[ch.ke + a]];
        }
        for (int a = 0; a < uc; ++a)
            for (int b = 0; b < uc; ++b) Fm[size_t(rm[a]) * F + cm[b]] += chS[size_t(a) * uc + b];
    }
    for (int i = 0; i < F; ++i) {
        rpos[rows[i]] = -1;
        cpos[cols[i]] = -1;
    }
    if (key) {
        unsigned long long h1 = 0x9E3779B97F4A7C15ull ^ (unsigned long long)F, h2 = 0xC2B2AE3D27D4EB4Full + (unsigned long long)sN;
        auto mix = [&](unsigned long long x) {
            h1 = (h1 ^ x) * 0x9E3779B97F4A7C15ull;
            h1 ^= h1 >> 29;
            h2 = (h2 + x) * 0xC2B2AE3D27D4EB4Full;
            h2 ^= h2 >> 31;
        };
        mix((unsigned long long)nown);
        const unsigned long long* w = reinterpret_cast<const unsigned long long*>(Fm.data());
        for (size_t i = 0; i < Fm.size() * 2; ++i) mix(w[i]);
        key->a = h1;
        key->b = h2;
        return;
    }

    // Elimination, right-looking by panels of kPanel pivot columns. Inside a panel
    // a pivot's rank-1 update is applied at once to the panel's columns only (all
    // rows below, so the next column's pivot test sees up-to-date entries); the
    // columns right of the panel get the whole panel's update in one pass per row
    // (the row segment stays in L1 over the panel's pivots; with one pivot at a
    // time the trailing matrix of a 1200-row front streamed through memory once
    // per pivot). A column that fails the pivot test ends its panel early: after
    // the trailing update every column right of it is current, and it is swapped
    // with the last candidate column. Large fronts use a team of threads that
    // lives for the whole front: thread 0 factors the panel, every thread updates
    // its share of the trailing rows; two spin barriers per panel.
    constexpr int kPanel = 32;
    int k = 0, last = sN;  // columns [k, last) are still candidates
    const int team = (nthreads > 1 && F >= 192) ? nthreads : 1;
    std::atomic<int> bar_count{0}, bar_gen{0};
    auto barrier = [&]() {
        const int g = bar_gen.load(std::memory_order_acquire);
        if (bar_count.fetch_add(1, std::memory_order_acq_rel) == team - 1) {
            bar_count.store(0, std::memory_order_relaxed);
            bar_gen.store(g + 1, std::memory_order_release);
        } else {
            while (bar_gen.load(std::memory_order_acquire) == g) std::this_thread::yield();
        }
    };
    // pivot test of column k (current for all rows >= k): the row of the largest
    // candidate, or -1 when the column has to be delayed
    auto find_pivot = [&]() -> int {
        // squared moduli: the same decisions as on |.| (std::abs of a complex is a hypot call)
        int p = k;
        double best = std::norm(Fm[size_t(k) * F + k]);
        for (int i = k + 1; i < sN; ++i) {
            const double a = std::norm(Fm[size_t(i) * F + k]);
            if (a > best) {
                best = a;
                p = i;
            }
        }
        double ringmax = 0.0;
        for (int i = sN; i < F; ++i) ringmax = std::max(ringmax, std::norm(Fm[size_t(i) * F + k]));
        if (best == 0.0 || best < pivtol * pivtol * ringmax) return -1;
        return p;
    };
    auto delay_column = [&]() {
        if (u == 0) throw RuntimeError("coarse LU: singular root front (zero pivot)");
        --last;  // delay column k
        if (last != k)
            for (int i = 0; i < F; ++i) std::swap(Fm[size_t(i) * F + k], Fm[size_t(i) * F + last]);
        std::swap(cols[k], cols[last]);
        std::swap(pcol[k], pcol[last]);
    };
    int k0 = 0, kend = 0;  // the open panel: pivots [k0, k), columns [k0, kend)
    // thread 0: pivots of one panel; returns true when a column failed its test
    auto panel = [&]() -> bool {
        k0 = k;
        kend = std::min(k0 + kPanel, last);
        while (k < kend) {
            const int p = find_pivot();
            if (p < 0) return true;
            if (p != k) {
                std::swap_ranges(Fm.begin() + size_t(k) * F, Fm.begin() + size_t(k) * F + F, Fm.begin() + size_t(p) * F);
                std::swap(rows[k], rows[p]);
                std::swap(prow[k], prow[p]);
            }
            const cplx inv = 1.0 / Fm[size_t(k) * F + k];
            const cplx* rk = &Fm[size_t(k) * F];
            for (int i = k + 1; i < F; ++i) {
                cplx* ri = &Fm[size_t(i) * F];
                if (ri[k] == cplx(0.0)) continue;
                const cplx l = ri[k] * inv;
                ri[k] = l;
                for (int j = k + 1; j < kend; ++j) ri[j] -= l * rk[j];
            }
            ++k;
        }
        return false;
    };
    // thread 0: the panel's own rows right of the panel (U12 of the panel), in pivot order
    auto panel_rows = [&]() {
        for (int q = k0 + 1; q < k; ++q) {
            cplx* rq = &Fm[size_t(q) * F];
            for (int q2 = k0; q2 < q; ++q2) {
                const cplx l = rq[q2];
                if (l == cplx(0.0)) continue;
                const cplx* r2 = &Fm[size_t(q2) * F];
                for (int j = kend; j < F; ++j) rq[j] -= l * r2[j];
            }
        }
    };
    // rows k + [i0, i1): minus the panel's multipliers times the panel's rows, columns [kend, F)
    auto trailing = [&](int i0, int i1) {
        int i = k + i0;
        const int iend = k + i1;
#if HTG_ND_AVX2
        // register-blocked form for wide updates: 2 rows x 8 columns of complex
        // accumulators held over the panel's pivots (the row segments are loaded and
        // stored once per panel instead of once per pivot, every panel row segment once
        // per row pair), fused multiply-adds
        if (F - kend >= 64) {
            const double* base = reinterpret_cast<const double*>(Fm.data());
            for (; i + 2 <= iend; i += 2) {
                double* ra = reinterpret_cast<double*>(&Fm[size_t(i) * F]);
                double* rb = reinterpret_cast<double*>(&Fm[size_t(i + 1) * F]);
                int j = kend;
                for (; j + 8 <= F; j += 8) {
                    __m256d a0 = _mm256_loadu_pd(ra + 2 * j), a1 = _mm256_loadu_pd(ra + 2 * j + 4),
                            a2 = _mm256_loadu_pd(ra + 2 * j + 8), a3 = _mm256_loadu_pd(ra + 2 * j + 12);
                    __m256d b0 = _mm256_loadu_pd(rb + 2 * j), b1 = _mm256_loadu_pd(rb + 2 * j + 4),
                            b2 = _mm256_loadu_pd(rb + 2 * j + 8), b3 = _mm256_loadu_pd(rb + 2 * j + 12);
                    for (int q = k0; q < k; ++q) {
                        const double* rq = base + 2 * (size_t(q) * F + j);
                        const __m256d lar = _mm256_set1_pd(ra[2 * q]), lbr = _mm256_set1_pd(rb[2 * q]);
                        const double ai = ra[2 * q + 1], bi = rb[2 * q + 1];
                        const __m256d lai = _mm256_set_pd(-ai, ai, -ai, ai), lbi = _mm256_set_pd(-bi, bi, -bi, bi);
                        __m256d v = _mm256_loadu_pd(rq), w = _mm256_permute_pd(v, 5);
                        a0 = _mm256_fmadd_pd(lai, w, _mm256_fnmadd_pd(lar, v, a0));
                        b0 = _mm256_fmadd_pd(lbi, w, _mm256_fnmadd_pd(lbr, v, b0));
                        v = _mm256_loadu_pd(rq + 4), w = _mm256_permute_pd(v, 5);
                        a1 = _mm256_fmadd_pd(lai, w, _mm256_fnmadd_pd(lar, v, a1));
                        b1 = _mm256_fmadd_pd(lbi, w, _mm256_fnmadd_pd(lbr, v, b1));
                        v = _mm256_loadu_pd(rq + 8), w = _mm256_permute_pd(v, 5);
                        a2 = _mm256_fmadd_pd(lai, w, _mm256_fnmadd_pd(lar, v, a2));
                        b2 = _mm256_fmadd_pd(lbi, w, _mm256_fnmadd_pd(lbr, v, b2));
                        v = _mm256_loadu_pd(rq + 12), w = _mm256_permute_pd(v, 5);
                        a3 = _mm256_fmadd_pd(lai, w, _mm256_fnmadd_pd(lar, v, a3));
                        b3 = _mm256_fmadd_pd(lbi, w, _mm256_fnmadd_pd(lbr, v, b3));
                    }
                    _mm256_storeu_pd(ra + 2 * j, a0);
                    _mm256_storeu_pd(ra + 2 * j + 4, a1);
                    _mm256_storeu_pd(ra + 2 * j + 8, a2);
                    _mm256_storeu_pd(ra + 2 * j + 12, a3);
                    _mm256_storeu_pd(rb + 2 * j, b0);
                    _mm256_storeu_pd(rb + 2 * j + 4, b1);
                    _mm256_storeu_pd(rb + 2 * j + 8, b2);
                    _mm256_storeu_pd(rb + 2 * j + 12, b3);
                }
                for (int r2 = 0; r2 < 2; ++r2) {  // columns left over
                    cplx* ri = &Fm[size_t(i + r2) * F];
                    for (int q = k0; q < k; ++q) {
                        const cplx l = ri[q];
                        const cplx* rq = &Fm[size_t(q) * F];
                        for (int jj = j; jj < F; ++jj) ri[jj] -= l * rq[jj];
                    }
                }
            }
        }
#endif
        for (; i < iend; ++i) {
            cplx* ri = &Fm[size_t(i) * F];
            for (int q = k0; q < k; ++q) {
                const cplx l = ri[q];
                if (l == cplx(0.0)) continue;
                const cplx* rq = &Fm[size_t(q) * F];
                for (int j = kend; j < F; ++j) ri[j] -= l * rq[j];
            }
        }
    };
    if (team == 1) {
        while (k < last) {
            const bool failed = panel();
            if (k > k0 && kend < F) {
                panel_rows();
                trailing(0, F - k);
            }
            if (failed) delay_column();
        }
    } else {
        bool done = false, failed = false;
        std::exception_ptr err;
        auto worker = [&](int w) {
            for (;;) {
                if (w == 0) {
                    try {
                        failed = panel();
                        if (k > k0 && kend < F) panel_rows();
                    } catch (...) {
                        err = std::current_exception();
                        done = true;
                    }
                }
                barrier();
                if (done) return;
                if (k > k0 && kend < F) {
                    const int nrows = F - k;
                    trailing(nrows * w / team, nrows * (w + 1) / team);
                }
                barrier();
                if (w == 0) {
                    try {
                        if (failed) delay_column();
                    } catch (...) {
                        err = std::current_exception();
                        done = true;
                    }
                    if (k >= last) done = true;
                }
                barrier();
                if (done) return;
            }
        };
        if (k >= last) done = true;
        if (!done) {
            std::vector<std::thread> th;
            for (int w = 1; w < team; ++w) th.emplace_back(worker, w);
            worker(0);
            for (auto& x : th) x.join();
        }
        if (err) std::rethrow_exception(err);
    }
    const int ke = k, r = F - ke;  // eliminated here / handed to the parent
    n.sN = sN;
    n.F = F;
    n.ke = ke;
    n.rc.assign(F, -1);  // right-hand side entries injected at this front: own-var rows
    {  // own variables marked in the (idle) column scratch map
        for (int v : n.vars) cpos[v] = 0;
        for (int i = 0; i < F; ++i)
            if (cpos[rows[i]] == 0) n.rc[i] = rows[i];
        for (int v : n.vars) cpos[v] = -1;
    }
    // Now rows [0, ke): unit L11 (cols < ke), U11 (cols >= row, < ke), U12 (cols >= ke);
    //     rows [ke, F): L21 (cols < ke), S (cols >= ke) -- the contribution block.
    n.S.assign(size_t(r) * r, cplx(0.0));
    for (int i = 0; i < r; ++i)
        for (int j = 0; j < r; ++j) n.S[size_t(i) * r + j] = Fm[size_t(ke + i) * F + ke + j];
    n.L21.assign(size_t(r) * ke, cplx(0.0));
    for (int i = 0; i < r; ++i)
        for (int j = 0; j < ke; ++j) n.L21[size_t(i) * ke + j] = Fm[size_t(ke + i) * F + j];
    // Finv = L11^-1 (the row permutation is folded into the front's row order) and
    // Uinv = U11^-1, by rows: row i of the inverse is e_i minus a combination of the
    // rows already computed (contiguous axpys); column blocks are independent, so a
    // large front splits them over its thread team.
    n.Finv.assign(size_t(ke) * ke, cplx(0.0));
    n.Uinv.assign(size_t(ke) * ke, cplx(0.0));
    auto inv_cols = [&](int c0, int c1) {
        for (int i = 0; i < ke; ++i) {  // unit lower: X[i][c] = [i == c] - sum_{k2 < i} L[i][k2] X[k2][c], c <= i
            cplx* xi = &n.Finv[size_t(i) * ke];
            const int ce = std::min(c1, i);
            for (int k2 = c0; k2 < i; ++k2) {
                const cplx l = Fm[size_t(i) * F + k2];
                if (l == cplx(0.0)) continue;
                const cplx* xk = &n.Finv[size_t(k2) * ke];
                const int cb = std::min(ce, k2 + 1);  // row k2 is zero right of its diagonal
                for (int c = c0; c < cb; ++c) xi[c] -= l * xk[c];
            }
            if (i >= c0 && i < c1) xi[i] = 1.0;
        }
        for (int i = ke - 1; i >= 0; --i) {  // upper: X[i][c] = ([i == c] - sum_{k2 > i} U[i][k2] X[k2][c]) / U[i][i], c >= i
            cplx* xi = &n.Uinv[size_t(i) * ke];
            const int cs = std::max(c0, i);
            for (int k2 = i + 1; k2 < c1; ++k2) {
                const cplx uu = Fm[size_t(i) * F + k2];
                if (uu == cplx(0.0)) continue;
                const cplx* xk = &n.Uinv[size_t(k2) * ke];
                for (int c = std::max(cs, k2); c < c1; ++c) xi[c] -= uu * xk[c];
            }
            if (i >= c0 && i < c1) xi[i] += 1.0;
            const cplx dinv = 1.0 / Fm[size_t(i) * F + i];
            for (int c = cs; c < c1; ++c) xi[c] *= dinv;
        }
    };
    if (team > 1 && ke >= 128) {
        std::vector<std::thread> th;
        for (int w = 0; w < team; ++w) th.emplace_back(inv_cols, ke * w / team, ke * (w + 1) / team);
        for (auto& x : th) x.join();
    } else {
        inv_cols(0, ke);
    }
    // Z = Uinv U12
    n.Z.assign(size_t(ke) * r, cplx(0.0));
    if (r > 0 && ke > 0) {
        std::vector<cplx> U12(size_t(ke) * r);
        for (int i = 0; i < ke; ++i)
            for (int j = 0; j < r; ++j) U12[size_t(i) * r + j] = Fm[size_t(i) * F + ke + j];
        std::vector<cplx> negZ(size_t(ke) * r, cplx(0.0));
        gemm_sub(ke, r, ke, n.Uinv.data(), U12.data(), negZ.data(), nthreads);
        for (size_t i = 0; i < negZ.size(); ++i) n.Z[i] = -negZ[i];
    }
    n.rows.swap(rows);
    n.cols.swap(cols);
    n.perm_r.swap(prow);
    n.perm_c.swap(pcol);
}

}  // namespace

void nd_factor(const LatticeMatrix& A, NDTree& t, int leaf_max, double pivtol) {
    t.W = A.W;
    t.H = A.H;
    t.q = A.q;
    t.nv = A.W * A.H;
    const int nv = t.nv;
    build_nd(t, A, 0, A.W - 1, 0, A.H - 1, 0, leaf_max);
    // factor bottom-up by depth; nodes of one depth in parallel
    const int nthr = std::max(1, int(std::thread::hardware_concurrency()));
    std::vector<std::vector<int>> bydepth(t.max_depth + 1);
    for (int i = 0; i < int(t.nodes.size()); ++i) bydepth[t.nodes[i].depth].push_back(i);
    const bool times = std::getenv("HTG_ND_TIMES") != nullptr;
    const char* share_env = std::getenv("HTG_ND_SHARE");
    const bool share = !(share_env && share_env[0] == '0');
    for (int d = t.max_depth; d >= 0; --d) {
        const auto& ids = bydepth[d];
        const auto td0 = std::chrono::steady_clock::now();
        if (int(ids.size()) >= nthr) {
            // every thread takes fronts off a shared counter; fn(front index in list, scratch maps)
            auto for_fronts = [&](const std::vector<int>& list, auto&& fn) {
                std::vector<std::thread> th;
                std::vector<std::exception_ptr> errs(nthr);
                std::atomic<int> next{0};
                for (int w = 0; w < nthr; ++w)
                    th.emplace_back([&, w] {
                        try {
                            std::vector<int> rpos(nv, -1), cpos(nv, -1);
                            for (int i; (i = next++) < int(list.size());) fn(i, rpos, cpos);
                        } catch (...) {
                            errs[w] = std::current_exception();
                        }
                    });
                for (auto& x : th) x.join();
                for (auto& e : errs)
                    if (e) std::rethrow_exception(e);
            };
            // Fronts with bit-identical assembled matrices (same size, same pivot block)
            // have identical factors: key every front, factor the first of each key,
            // give the others its pivot order (HTG_ND_SHARE=0: factor every front).
            std::vector<int> reps, sharers;
            if (share) {
                std::vector<FrontKey> keys(ids.size());
                for_fronts(ids, [&](int i, std::vector<int>& rpos, std::vector<int>& cpos) {
                    factor_node(t, ids[i], A, rpos, cpos, pivtol, 1, &keys[i]);
                });
                std::map<FrontKey, int> first;
                for (size_t i = 0; i < ids.size(); ++i) {
                    auto it = first.find(keys[i]);
                    if (it == first.end()) {
                        first.emplace(keys[i], ids[i]);
                        reps.push_back(ids[i]);
                    } else {
                        t.nodes[size_t(ids[i])].rep = it->second;
                        sharers.push_back(ids[i]);
                    }
                }
                t.shared += (long long)sharers.size();
            } else {
                reps = ids;
            }
            for_fronts(reps, [&](int i, std::vector<int>& rpos, std::vector<int>& cpos) {
                factor_node(t, reps[i], A, rpos, cpos, pivtol, 1);
            });
            if (!sharers.empty())
                for_fronts(sharers, [&](int i, std::vector<int>& rpos, std::vector<int>& cpos) {
                    factor_node(t, sharers[i], A, rpos, cpos, pivtol, 1);
                });
        } else {  // fewer fronts than threads: all fronts at once, a thread team each
            const int per = std::max(1, nthr / std::max(1, int(ids.size())));
            std::vector<std::thread> th;
            std::vector<std::exception_ptr> errs(ids.size());
            for (size_t q = 0; q < ids.size(); ++q)
                th.emplace_back([&, q] {
                    try {
                        std::vector<int> rpos(nv, -1), cpos(nv, -1);
                        factor_node(t, ids[q], A, rpos, cpos, pivtol, per);
                    } catch (...) {
                        errs[q] = std::current_exception();
                    }
                });
            for (auto& x : th) x.join();
            for (auto& e : errs)
                if (e) std::rethrow_exception(e);
        }
        if (times) {
            int fmax = 0;
            for (int id : ids) fmax = std::max(fmax, t.nodes[id].F);
            int nshare = 0;
            for (int id : ids) nshare += t.nodes[id].rep >= 0;
            std::fprintf(stderr, "htg nd: depth %2d fronts %6d (%6d shared) max F %5d  %.3f s\n", d, int(ids.size()), nshare, fmax,
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - td0).count());
        }
        for (int id : ids) {
            const NDNode& n = t.nodes[id];
            t.delayed += n.sN - n.ke;
            t.max_front = std::max(t.max_front, n.F);
            for (int c : n.children) std::vector<cplx>().swap(t.nodes[c].S);
        }
    }
}

}  // namespace htg
