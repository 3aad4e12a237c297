// coarse.cu -- QSFEM coarse matrix, nested-dissection multifrontal LU (host)
// and the level-batched GPU triangular solves.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <functional>
#include <thread>

#include "coarse.hpp"
#include "kernels.hpp"

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
    for (int Y = 0; Y <= CY; ++Y)
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
    return A9;
}

// ------------------------------------------------------------------ nested dissection
namespace {

struct NDNode {
    int x0, x1, y0, y1;  // box of the subtree (inclusive vertex coordinates)
    int depth = 0;
    bool leaf = false;
    std::vector<int> vars, ring, children;
    // factor blocks (host, freed after upload)
    std::vector<cplx> Finv, L21, Uinv, Z, S;
    std::vector<int> cmap;  // this node's ring -> parent's front positions
};

struct NDTree {
    int CX, CY;
    std::vector<NDNode> nodes;  // postorder: children before parents, root last
    int max_depth = 0;
};

int build_nd(NDTree& t, int x0, int x1, int y0, int y1, int depth, int leaf_max) {
    NDNode n;
    n.x0 = x0;
    n.x1 = x1;
    n.y0 = y0;
    n.y1 = y1;
    n.depth = depth;
    const int w = x1 - x0 + 1, h = y1 - y0 + 1;
    std::vector<int> kids;
    if (w * h <= leaf_max || std::max(w, h) < 3) {
        n.leaf = true;
        for (int y = y0; y <= y1; ++y)
            for (int x = x0; x <= x1; ++x) n.vars.push_back(y * (t.CX + 1) + x);
    } else if (w >= h) {
        const int xm = (x0 + x1) / 2;
        kids.push_back(build_nd(t, x0, xm - 1, y0, y1, depth + 1, leaf_max));
        kids.push_back(build_nd(t, xm + 1, x1, y0, y1, depth + 1, leaf_max));
        for (int y = y0; y <= y1; ++y) n.vars.push_back(y * (t.CX + 1) + xm);
    } else {
        const int ym = (y0 + y1) / 2;
        kids.push_back(build_nd(t, x0, x1, y0, ym - 1, depth + 1, leaf_max));
        kids.push_back(build_nd(t, x0, x1, ym + 1, y1, depth + 1, leaf_max));
        for (int x = x0; x <= x1; ++x) n.vars.push_back(ym * (t.CX + 1) + x);
    }
    for (int y = y0 - 1; y <= y1 + 1; ++y)
        for (int x = x0 - 1; x <= x1 + 1; ++x) {
            if (x < 0 || y < 0 || x > t.CX || y > t.CY) continue;
            if (x >= x0 && x <= x1 && y >= y0 && y <= y1) continue;
            n.ring.push_back(y * (t.CX + 1) + x);
        }
    n.children = kids;
    t.max_depth = std::max(t.max_depth, depth);
    t.nodes.push_back(std::move(n));
    return int(t.nodes.size()) - 1;
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

void parallel_rows(int m, int nthreads, const std::function<void(int, int)>& body, size_t work) {
    if (nthreads <= 1 || work < 2000000) {
        body(0, m);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t) th.emplace_back(body, m * t / nthreads, m * (t + 1) / nthreads);
    for (auto& x : th) x.join();
}

// Factor one front (children already factored). pos: scratch global->front map.
void factor_node(NDTree& t, int id, const std::vector<cplx>& A9, std::vector<int>& pos, int nthreads) {
    NDNode& n = t.nodes[id];
    const int s = int(n.vars.size()), u = int(n.ring.size()), F = s + u;
    for (int i = 0; i < s; ++i) pos[n.vars[i]] = i;
    for (int i = 0; i < u; ++i) pos[n.ring[i]] = s + i;
    std::vector<cplx> Fm(size_t(F) * F, cplx(0.0));
    const int W = t.CX + 1;
    for (int i = 0; i < s; ++i) {
        const int v = n.vars[i], X = v % W, Y = v / W;
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int WX = X + dx, WY = Y + dy;
                if (WX < 0 || WX > t.CX || WY < 0 || WY > t.CY) continue;
                const int w = WY * W + WX, pw = pos[w];
                if (pw < 0) continue;
                Fm[size_t(i) * F + pw] += A9[size_t(v) * 9 + (dy + 1) * 3 + (dx + 1)];
                if (pw >= s) Fm[size_t(pw) * F + i] += A9[size_t(w) * 9 + (1 - dy) * 3 + (1 - dx)];
            }
    }
    for (int c : n.children) {
        NDNode& ch = t.nodes[c];
        const int uc = int(ch.ring.size());
        ch.cmap.resize(uc);
        for (int a = 0; a < uc; ++a) ch.cmap[a] = pos[ch.ring[a]];
        for (int a = 0; a < uc; ++a) {
            const int pa = ch.cmap[a];
            for (int b = 0; b < uc; ++b) Fm[size_t(pa) * F + ch.cmap[b]] += ch.S[size_t(a) * uc + b];
        }
        std::vector<cplx>().swap(ch.S);
    }
    for (int i = 0; i < s; ++i) pos[n.vars[i]] = -1;
    for (int i = 0; i < u; ++i) pos[n.ring[i]] = -1;

    // LU of F11 with partial pivoting restricted to the front's pivot rows;
    // row swaps applied to the whole front row (F11 and F12 parts)
    std::vector<int> perm(s);
    for (int i = 0; i < s; ++i) perm[i] = i;
    for (int k = 0; k < s; ++k) {
        int p = k;
        double best = std::abs(Fm[size_t(k) * F + k]);
        for (int i = k + 1; i < s; ++i) {
            const double a = std::abs(Fm[size_t(i) * F + k]);
            if (a > best) {
                best = a;
                p = i;
            }
        }
        if (best == 0.0) throw RuntimeError("coarse LU: singular front (zero pivot)");
        if (p != k) {
            std::swap_ranges(Fm.begin() + size_t(k) * F, Fm.begin() + size_t(k) * F + F, Fm.begin() + size_t(p) * F);
            std::swap(perm[k], perm[p]);
        }
        const cplx inv = 1.0 / Fm[size_t(k) * F + k];
        const cplx* rk = &Fm[size_t(k) * F];
        // eliminate below in the pivot block and in the F21 block (rows s..F-1 are
        // the L21 computation: L21 = F21 U^-1 falls out of the same elimination)
        auto elim = [&](int i0, int i1) {
            for (int i = i0; i < i1; ++i) {
                const int row = i < s - k - 1 ? k + 1 + i : s + (i - (s - k - 1));
                cplx* ri = &Fm[size_t(row) * F];
                if (ri[k] == cplx(0.0)) continue;
                const cplx l = ri[k] * inv;
                ri[k] = l;
                for (int j = k + 1; j < F; ++j) ri[j] -= l * rk[j];
            }
        };
        const int nrows = (s - k - 1) + u;
        parallel_rows(nrows, nthreads, elim, size_t(nrows) * (F - k));
    }
    // Now: rows 0..s-1: L (unit, strict lower of cols < s), U (upper of cols < s), U12 (cols >= s)
    //      rows s..F-1: L21 (cols < s), S (cols >= s) -- the Schur complement
    n.S.assign(size_t(u) * u, cplx(0.0));
    for (int i = 0; i < u; ++i)
        for (int j = 0; j < u; ++j) n.S[size_t(i) * u + j] = Fm[size_t(s + i) * F + s + j];
    n.L21.assign(size_t(u) * s, cplx(0.0));
    for (int i = 0; i < u; ++i)
        for (int j = 0; j < s; ++j) n.L21[size_t(i) * s + j] = Fm[size_t(s + i) * F + j];
    // Finv = L^-1 P : column perm[k] of Finv is column k of L^-1
    std::vector<cplx> Linv(size_t(s) * s, cplx(0.0));
    for (int c = 0; c < s; ++c) {
        Linv[size_t(c) * s + c] = 1.0;
        for (int i = c + 1; i < s; ++i) {
            cplx acc = 0.0;
            for (int k2 = c; k2 < i; ++k2) acc += Fm[size_t(i) * F + k2] * Linv[size_t(k2) * s + c];
            Linv[size_t(i) * s + c] = -acc;
        }
    }
    n.Finv.assign(size_t(s) * s, cplx(0.0));
    for (int i = 0; i < s; ++i)
        for (int k2 = 0; k2 < s; ++k2) n.Finv[size_t(i) * s + perm[k2]] = Linv[size_t(i) * s + k2];
    // Uinv (upper triangular inverse)
    n.Uinv.assign(size_t(s) * s, cplx(0.0));
    for (int c = s - 1; c >= 0; --c) {
        n.Uinv[size_t(c) * s + c] = 1.0 / Fm[size_t(c) * F + c];
        for (int i = c - 1; i >= 0; --i) {
            cplx acc = 0.0;
            for (int k2 = i + 1; k2 <= c; ++k2) acc += Fm[size_t(i) * F + k2] * n.Uinv[size_t(k2) * s + c];
            n.Uinv[size_t(i) * s + c] = -acc / Fm[size_t(i) * F + i];
        }
    }
    // Z = Uinv U12
    n.Z.assign(size_t(s) * u, cplx(0.0));
    if (u > 0) {
        std::vector<cplx> U12(size_t(s) * u);
        for (int i = 0; i < s; ++i)
            for (int j = 0; j < u; ++j) U12[size_t(i) * u + j] = Fm[size_t(i) * F + s + j];
        std::vector<cplx> negZ(size_t(s) * u, cplx(0.0));
        gemm_sub(s, u, s, n.Uinv.data(), U12.data(), negZ.data(), nthreads);
        for (size_t i = 0; i < negZ.size(); ++i) n.Z[i] = -negZ[i];
    }
}

// ------------------------------------------------------------------ GPU solve
struct NodeDev {
    int s, u;
    long long off_F, off_L, off_U, off_Z;  // into the factor buffer (row-major blocks)
    int off_var, off_ring;                 // into idx
    int off_front;                         // front scratch (s+u)
    int off_contrib;                       // contribution vector (u)
    int off_gsrc;                          // per front position: <= 2 child contribution indices
    int pad;
};
// a launch's work item carries its front descriptor (no dependent load at start)
struct Task {
    NodeDev nd;
    int r0, nr;
};

constexpr int kCT = 256;     // threads per CTA (8 warps)
constexpr int kWarpFMax = 128;  // warp-tier shared buffers (fronts with s + u <= g_warpF)
static int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}
// tier thresholds (overridable for tuning: HTG_ND_LEAF, HTG_ND_WARPF, HTG_ND_MIDDATA, HTG_ND_RPT)

__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

struct NDArgs {
    const int* idx;
    const int2* gsrc;
    const double2* fac;
    const double2* rc;
    double2* contrib;
    double2* front;
    double2* Y;
    double2* X;
};

// Rows [r0, r1) of a row-major (rows x len) complex block times v, by lane
// groups of G lanes (G = power of two >= min(len, 32)): consecutive lanes read
// consecutive entries of a row and consecutive groups consecutive rows, so a
// warp's loads are contiguous even for short rows. out(r, value) on the
// group's first lane. warps/nw: this warp's index among the nw warps sharing the rows.
template <class Out>
__device__ __forceinline__ void rows_dot(const double2* __restrict__ M, int len, const double2* v, int r0, int r1,
                                         int warp, int nw, int lane, Out&& out) {
    int G = 32;
    if (len <= 4) G = 4;
    else if (len <= 8) G = 8;
    else if (len <= 16) G = 16;
    const int rpw = 32 / G, gl = lane & (G - 1), gi = lane / G;
    constexpr int U = 4;  // independent rows in flight per lane group
    const int step = nw * rpw;
    for (int rb = r0 + warp * rpw; rb < r1; rb += U * step) {
        double2 acc[U];
        int rr[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            acc[q] = make_double2(0.0, 0.0);
            rr[q] = rb + q * step + gi;
        }
        for (int k = gl; k < len; k += G) {
            const double2 vk = v[k];
#pragma unroll
            for (int q = 0; q < U; ++q)
                if (rr[q] < r1) acc[q] = cfma(M[(size_t)rr[q] * len + k], vk, acc[q]);
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
            for (int o = G >> 1; o > 0; o >>= 1) {
                acc[q].x += __shfl_xor_sync(0xffffffffu, acc[q].x, o);
                acc[q].y += __shfl_xor_sync(0xffffffffu, acc[q].y, o);
            }
            if (gl == 0 && rr[q] < r1) out(rr[q], acc[q]);
        }
    }
}

// front vector v = [rc(vars); 0] + the children's contribution vectors (each
// position has at most two, added in child order), one pass, no barrier inside
template <int STRIDE, class Sync>
__device__ void gather_front(const NDArgs& a, const NodeDev& nd, double2* sv, int t, Sync&& sync) {
    const int F = nd.s + nd.u;
    for (int i = t; i < F; i += STRIDE) {
        double2 v = i < nd.s ? a.rc[a.idx[nd.off_var + i]] : make_double2(0.0, 0.0);
        const int2 src = a.gsrc[nd.off_gsrc + i];
        if (src.x >= 0) {
            const double2 c = a.contrib[src.x];
            v.x += c.x;
            v.y += c.y;
        }
        if (src.y >= 0) {
            const double2 c = a.contrib[src.y];
            v.x += c.x;
            v.y += c.y;
        }
        sv[i] = v;
    }
    sync();
}

// forward: y1 = (L^-1 P) v1, c = v2 - L21 y1. Warp tier: one warp per front.
__global__ void __launch_bounds__(kCT) k_nd_fwd_warp(const NodeDev* __restrict__ list, int n, NDArgs a) {
    __shared__ double2 sv[kCT / 32][kWarpFMax];
    __shared__ double2 sy[kCT / 32][kWarpFMax];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int id = blockIdx.x * (kCT / 32) + w;
    if (id >= n) return;
    const NodeDev nd = list[id];
    double2* v = sv[w];
    double2* y = sy[w];
    gather_front<32>(a, nd, v, lane, [] { __syncwarp(); });
    rows_dot(a.fac + nd.off_F, nd.s, v, 0, nd.s, 0, 1, lane, [&](int r, double2 acc) {
        y[r] = acc;
        a.Y[a.idx[nd.off_var + r]] = acc;
    });
    __syncwarp();
    rows_dot(a.fac + nd.off_L, nd.s, y, 0, nd.u, 0, 1, lane, [&](int r, double2 acc) {
        const double2 v2 = v[nd.s + r];
        a.contrib[nd.off_contrib + r] = make_double2(v2.x - acc.x, v2.y - acc.y);
    });
}

// forward, CTA tier: one CTA per front, both phases
__global__ void __launch_bounds__(kCT) k_nd_fwd_mid(const NodeDev* __restrict__ list, NDArgs a) {
    extern __shared__ double2 smem[];
    const NodeDev nd = list[blockIdx.x];
    double2* v = smem;
    double2* y = smem + nd.s + nd.u;
    gather_front<kCT>(a, nd, v, threadIdx.x, [] { __syncthreads(); });
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    rows_dot(a.fac + nd.off_F, nd.s, v, 0, nd.s, warp, kCT / 32, lane, [&](int r, double2 acc) {
        y[r] = acc;
        a.Y[a.idx[nd.off_var + r]] = acc;
    });
    __syncthreads();
    rows_dot(a.fac + nd.off_L, nd.s, y, 0, nd.u, warp, kCT / 32, lane, [&](int r, double2 acc) {
        const double2 v2 = v[nd.s + r];
        a.contrib[nd.off_contrib + r] = make_double2(v2.x - acc.x, v2.y - acc.y);
    });
}

// forward, large tier phase 1: y1 rows of a task (v2 stashed by the r0 == 0 task)
__global__ void __launch_bounds__(kCT) k_nd_fwd1(const Task* tasks, NDArgs a) {
    extern __shared__ double2 smem[];
    const Task tk = tasks[blockIdx.x];
    const NodeDev nd = tk.nd;
    gather_front<kCT>(a, nd, smem, threadIdx.x, [] { __syncthreads(); });
    if (tk.r0 == 0)
        for (int i = nd.s + threadIdx.x; i < nd.s + nd.u; i += kCT) a.front[nd.off_front + i] = smem[i];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    rows_dot(a.fac + nd.off_F, nd.s, smem, tk.r0, tk.r0 + tk.nr, warp, kCT / 32, lane,
             [&](int r, double2 acc) { a.Y[a.idx[nd.off_var + r]] = acc; });
}

// forward, large tier phase 2: contribution rows c = v2 - L21 y1
__global__ void __launch_bounds__(kCT) k_nd_fwd2(const Task* tasks, NDArgs a) {
    extern __shared__ double2 smem[];
    const Task tk = tasks[blockIdx.x];
    const NodeDev nd = tk.nd;
    for (int i = threadIdx.x; i < nd.s; i += kCT) smem[i] = a.Y[a.idx[nd.off_var + i]];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    rows_dot(a.fac + nd.off_L, nd.s, smem, tk.r0, tk.r0 + tk.nr, warp, kCT / 32, lane, [&](int r, double2 acc) {
        const double2 v2 = a.front[nd.off_front + nd.s + r];
        a.contrib[nd.off_contrib + r] = make_double2(v2.x - acc.x, v2.y - acc.y);
    });
}

// backward: x1 = U^-1 y1 - (U^-1 U12) x2. Z rows are computed into sz first.
__device__ __forceinline__ void bwd_rows(const NDArgs& a, const NodeDev& nd, const double2* y1, const double2* x2,
                                         double2* sz, int r0, int r1, int warp, int nw, int lane,
                                         void (*sync)()) {
    if (nd.u > 0) {
        rows_dot(a.fac + nd.off_Z, nd.u, x2, r0, r1, warp, nw, lane, [&](int r, double2 acc) { sz[r - r0] = acc; });
        sync();
    }
    rows_dot(a.fac + nd.off_U, nd.s, y1, r0, r1, warp, nw, lane, [&](int r, double2 acc) {
        if (nd.u > 0) {
            acc.x -= sz[r - r0].x;
            acc.y -= sz[r - r0].y;
        }
        a.X[a.idx[nd.off_var + r]] = acc;
    });
}
__device__ void sync_warp_fn() { __syncwarp(); }
__device__ void sync_cta_fn() { __syncthreads(); }

__global__ void __launch_bounds__(kCT) k_nd_bwd_warp(const NodeDev* __restrict__ list, int n, NDArgs a) {
    __shared__ double2 sv[kCT / 32][kWarpFMax];
    __shared__ double2 sz[kCT / 32][kWarpFMax];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int id = blockIdx.x * (kCT / 32) + w;
    if (id >= n) return;
    const NodeDev nd = list[id];
    double2* v = sv[w];
    for (int i = lane; i < nd.s; i += 32) v[i] = a.Y[a.idx[nd.off_var + i]];
    for (int i = lane; i < nd.u; i += 32) v[nd.s + i] = a.X[a.idx[nd.off_ring + i]];
    __syncwarp();
    bwd_rows(a, nd, v, v + nd.s, sz[w], 0, nd.s, 0, 1, lane, sync_warp_fn);
}

// backward, CTA tasks (whole front for the CTA tier, row blocks for the large tier)
__global__ void __launch_bounds__(kCT) k_nd_bwd(const Task* tasks, NDArgs a) {
    extern __shared__ double2 smem[];
    const Task tk = tasks[blockIdx.x];
    const NodeDev nd = tk.nd;
    double2* y1 = smem;
    double2* x2 = smem + nd.s;
    double2* sz = smem + nd.s + nd.u;
    for (int i = threadIdx.x; i < nd.s; i += kCT) y1[i] = a.Y[a.idx[nd.off_var + i]];
    for (int i = threadIdx.x; i < nd.u; i += kCT) x2[i] = a.X[a.idx[nd.off_ring + i]];
    __syncthreads();
    bwd_rows(a, nd, y1, x2, sz, tk.r0, tk.r0 + tk.nr, threadIdx.x >> 5, kCT / 32, threadIdx.x & 31, sync_cta_fn);
}

class NDSolver : public CoarseSolver {
  public:
    NDSolver(const HostProblem& hp, cudaStream_t st) {
        const int m = hp.p / 2;
        NDTree t;
        t.CX = hp.nx * m;
        t.CY = hp.ny * m;
        const int nv = (t.CX + 1) * (t.CY + 1);
        nv_ = nv;
        build_nd(t, 0, t.CX, 0, t.CY, 0, env_int("HTG_ND_LEAF", 16));
        const std::vector<cplx> A9 = coarse_stencil(hp);
        // factor bottom-up by depth; nodes of one depth in parallel
        const int nthr = std::max(1, int(std::thread::hardware_concurrency()));
        std::vector<std::vector<int>> bydepth(t.max_depth + 1);
        for (int i = 0; i < int(t.nodes.size()); ++i) bydepth[t.nodes[i].depth].push_back(i);
        for (int d = t.max_depth; d >= 0; --d) {
            const auto& ids = bydepth[d];
            if (int(ids.size()) >= nthr) {
                std::vector<std::thread> th;
                std::vector<std::exception_ptr> errs(nthr);
                std::atomic<int> next{0};
                for (int w = 0; w < nthr; ++w)
                    th.emplace_back([&, w] {
                        try {
                            std::vector<int> pos(nv, -1);
                            for (int i; (i = next++) < int(ids.size());) factor_node(t, ids[i], A9, pos, 1);
                        } catch (...) {
                            errs[w] = std::current_exception();
                        }
                    });
                for (auto& x : th) x.join();
                for (auto& e : errs)
                    if (e) std::rethrow_exception(e);
            } else {
                std::vector<int> pos(nv, -1);
                for (int id : ids) factor_node(t, id, A9, pos, nthr);
            }
        }
        upload(t, st);
    }
    ~NDSolver() override {
        for (void* p : allocs_) cudaFree(p);
    }
    size_t device_bytes() const override { return bytes_; }
    int levels() const override { return int(levels_.size()); }

    void solve(const double2* rc, double2* uc, cudaStream_t st) override {
        NDArgs a = args_;
        a.rc = rc;
        a.X = uc;
        for (int L = int(levels_.size()) - 1; L >= 0; --L) {  // forward: deepest level first
            const Level& lv = levels_[L];
            if (lv.nwarp) {
                k_nd_fwd_warp<<<(lv.nwarp + 7) / 8, kCT, 0, st>>>(lv.warp, lv.nwarp, a);
                count_launch();
            }
            if (lv.nmid) {
                k_nd_fwd_mid<<<lv.nmid, kCT, lv.smem_mid, st>>>(lv.mid, a);
                count_launch();
            }
            if (lv.nf1) {
                k_nd_fwd1<<<lv.nf1, kCT, lv.smem_big, st>>>(lv.f1, a);
                count_launch();
            }
            if (lv.nf2) {
                k_nd_fwd2<<<lv.nf2, kCT, lv.smem_big, st>>>(lv.f2, a);
                count_launch();
            }
        }
        for (int L = 0; L < int(levels_.size()); ++L) {  // backward: root first
            const Level& lv = levels_[L];
            if (lv.nb) {
                k_nd_bwd<<<lv.nb, kCT, lv.smem_b, st>>>(lv.b, a);
                count_launch();
            }
            if (lv.nwarp) {
                k_nd_bwd_warp<<<(lv.nwarp + 7) / 8, kCT, 0, st>>>(lv.warp, lv.nwarp, a);
                count_launch();
            }
        }
        HTG_CUDA(cudaGetLastError());
    }

  private:
    struct Level {
        const NodeDev *warp = nullptr, *mid = nullptr;
        const Task *f1 = nullptr, *f2 = nullptr, *b = nullptr;
        int nwarp = 0, nmid = 0, nf1 = 0, nf2 = 0, nb = 0;
        size_t smem_mid = 0, smem_big = 0, smem_b = 0;
    };
    std::vector<Level> levels_;
    std::vector<void*> allocs_;
    size_t bytes_ = 0;
    int nv_ = 0;
    NDArgs args_{};

    template <class T>
    T* up(const std::vector<T>& v, cudaStream_t st) {
        void* p = nullptr;
        HTG_CUDA(cudaMalloc(&p, std::max<size_t>(1, v.size()) * sizeof(T)));
        allocs_.push_back(p);
        bytes_ += v.size() * sizeof(T);
        if (!v.empty()) HTG_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
        HTG_CUDA(cudaStreamSynchronize(st));
        return static_cast<T*>(p);
    }

    void upload(NDTree& t, cudaStream_t st) {
        const int nn = int(t.nodes.size());
        std::vector<NodeDev> nd(nn);
        std::vector<int> idx;
        long long fac_total = 0;
        int front_total = 0, contrib_total = 0, gsrc_total = 0;
        for (int i = 0; i < nn; ++i) {
            const NDNode& n = t.nodes[i];
            NodeDev& d = nd[i];
            d.s = int(n.vars.size());
            d.u = int(n.ring.size());
            d.off_F = fac_total;
            fac_total += (long long)d.s * d.s;
            d.off_L = fac_total;
            fac_total += (long long)d.u * d.s;
            d.off_U = fac_total;
            fac_total += (long long)d.s * d.s;
            d.off_Z = fac_total;
            fac_total += (long long)d.s * d.u;
            d.off_var = int(idx.size());
            idx.insert(idx.end(), n.vars.begin(), n.vars.end());
            d.off_ring = int(idx.size());
            idx.insert(idx.end(), n.ring.begin(), n.ring.end());
            d.off_front = front_total;
            front_total += d.s + d.u;
            d.off_contrib = contrib_total;
            contrib_total += d.u;
            d.off_gsrc = gsrc_total;
            gsrc_total += d.s + d.u;
        }
        // gather plan: front position <- contribution entries of the children (child order)
        std::vector<int2> gsrc(std::max(gsrc_total, 1), make_int2(-1, -1));
        for (int i = 0; i < nn; ++i) {
            for (int c : t.nodes[i].children) {
                const NDNode& ch = t.nodes[c];
                for (int k = 0; k < int(ch.cmap.size()); ++k) {
                    int2& e = gsrc[nd[i].off_gsrc + ch.cmap[k]];
                    const int src = nd[c].off_contrib + k;
                    if (e.x < 0) e.x = src;
                    else if (e.y < 0) e.y = src;
                    else throw RuntimeError("coarse solve: more than two contributions to a front position");
                }
            }
        }
        void* facp = nullptr;
        HTG_CUDA(cudaMalloc(&facp, std::max<long long>(1, fac_total) * sizeof(double2)));
        allocs_.push_back(facp);
        bytes_ += fac_total * sizeof(double2);
        for (int i = 0; i < nn; ++i) {
            NDNode& n = t.nodes[i];
            const NodeDev& d = nd[i];
            auto put = [&](std::vector<cplx>& v, long long off) {
                if (v.empty()) return;
                HTG_CUDA(cudaMemcpy(static_cast<double2*>(facp) + off, v.data(), v.size() * sizeof(cplx),
                                    cudaMemcpyHostToDevice));
                std::vector<cplx>().swap(v);
            };
            put(n.Finv, d.off_F);
            put(n.L21, d.off_L);
            put(n.Uinv, d.off_U);
            put(n.Z, d.off_Z);
        }
        args_.fac = static_cast<const double2*>(facp);
        args_.idx = up(idx, st);
        args_.gsrc = up(gsrc, st);
        args_.contrib = up(std::vector<double2>(std::max(contrib_total, 1)), st);
        args_.front = up(std::vector<double2>(std::max(front_total, 1)), st);
        args_.Y = up(std::vector<double2>(nv_), st);
        // per depth: warp tier, CTA tier, large tier (8 rows per CTA task)
        const int D = t.max_depth + 1;
        levels_.resize(D);
        std::vector<std::vector<NodeDev>> wp(D), md(D);
        std::vector<std::vector<Task>> f1(D), f2(D), bw(D);
        size_t max_smem = 0;
        const int warpF = std::min(kWarpFMax, env_int("HTG_ND_WARPF", 64));
        const long long midData = env_int("HTG_ND_MIDDATA", 16384);
        for (int i = 0; i < nn; ++i) {
            const int dep = t.nodes[i].depth;
            const NodeDev& d = nd[i];
            Level& lv = levels_[dep];
            const int F = d.s + d.u;
            if (F <= warpF) {
                wp[dep].push_back(d);
            } else if ((long long)d.s * F <= midData) {
                md[dep].push_back(d);
                bw[dep].push_back({d, 0, d.s});
                lv.smem_mid = std::max(lv.smem_mid, size_t(F + d.s) * sizeof(double2));
                lv.smem_b = std::max(lv.smem_b, size_t(F + d.s) * sizeof(double2));
            } else {
                const int rpt = env_int("HTG_ND_RPT", 8);
                for (int r = 0; r < d.s; r += rpt) {
                    f1[dep].push_back({d, r, std::min(rpt, d.s - r)});
                    bw[dep].push_back({d, r, std::min(rpt, d.s - r)});
                }
                for (int r = 0; r < d.u; r += rpt) f2[dep].push_back({d, r, std::min(rpt, d.u - r)});
                lv.smem_big = std::max(lv.smem_big, size_t(F) * sizeof(double2));
                lv.smem_b = std::max(lv.smem_b, size_t(F + rpt) * sizeof(double2));
            }
        }
        for (int L = 0; L < D; ++L) {
            Level& lv = levels_[L];
            lv.nwarp = int(wp[L].size());
            lv.nmid = int(md[L].size());
            lv.nf1 = int(f1[L].size());
            lv.nf2 = int(f2[L].size());
            lv.nb = int(bw[L].size());
            lv.warp = up(wp[L], st);
            lv.mid = up(md[L], st);
            lv.f1 = up(f1[L], st);
            lv.f2 = up(f2[L], st);
            lv.b = up(bw[L], st);
            max_smem = std::max({max_smem, lv.smem_mid, lv.smem_big, lv.smem_b});
        }
        if (max_smem > 227 * 1024) throw InvalidArgument("coarse front too large for shared memory");
        if (max_smem > 48 * 1024) {
            HTG_CUDA(cudaFuncSetAttribute(k_nd_fwd_mid, cudaFuncAttributeMaxDynamicSharedMemorySize, int(max_smem)));
            HTG_CUDA(cudaFuncSetAttribute(k_nd_fwd1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(max_smem)));
            HTG_CUDA(cudaFuncSetAttribute(k_nd_fwd2, cudaFuncAttributeMaxDynamicSharedMemorySize, int(max_smem)));
            HTG_CUDA(cudaFuncSetAttribute(k_nd_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, int(max_smem)));
        }
    }
};

}  // namespace

std::unique_ptr<CoarseSolver> make_coarse_solver(const HostProblem& hp, cudaStream_t st) {
    return std::make_unique<NDSolver>(hp, st);
}

}  // namespace htg
