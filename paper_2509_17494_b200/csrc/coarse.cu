// coarse.cu -- level-batched GPU solves with the nested-dissection multifrontal
// factors of the QSFEM coarse matrix (factored on the host in coarse_nd.cpp).
#include <mutex>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <functional>
#include <thread>
#include <utility>

#include <cooperative_groups.h>

#include "coarse.hpp"
#include "kernels.hpp"

namespace cg = cooperative_groups;

namespace htg {

namespace {

// ------------------------------------------------------------------ GPU solve
struct NodeDev {
    int s, u;                              // eliminated here / contribution rows (delayed + ring)
    long long off_F, off_L, off_U, off_Z;  // into the factor buffer (row-major blocks)
    int off_var, off_ring;                 // into idx: eliminated / remaining column labels
    int off_front;                         // front scratch (s+u)
    int off_contrib;                       // contribution vector (u)
    int off_gsrc;                          // per front position: <= 4 child contribution indices
    int off_rc;                            // into idx: per front row, rhs entry injected here or -1
};
// a launch's work item carries its front descriptor (no dependent load at start)
struct Task {
    NodeDev nd;
    int r0, nr;
};

constexpr int kCT = 256;     // threads per CTA (8 warps)
#ifndef HTG_ND_KU
#define HTG_ND_KU 4
#endif
constexpr int kWarpFMax = 128;  // warp-tier shared buffers (fronts with s + u <= g_warpF)
#ifndef HTG_ND_MERGED
#define HTG_ND_MERGED 0
#endif
constexpr bool kMergedLevels = HTG_ND_MERGED != 0;  // one launch per (branch, level) for all tiers
static int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}
// tier thresholds (overridable for tuning: HTG_ND_LEAF, HTG_ND_WARPF, HTG_ND_MIDDATA, HTG_ND_RPT)

// programmatic dependent launch (HTG_ND_PDL=1; off: measured 1.01 vs 0.84 ms at cfg4, the
// early-scheduled dependent CTAs hold SM slots the other branches need): a level kernel lets the
// next one in its stream be scheduled at once and waits for its predecessor only
// before touching solve data, so the ~30 dependent launches of a subtree branch
// overlap their launch latency with the previous level's tail
#ifndef HTG_ND_PDL
#define HTG_ND_PDL 0
#endif
constexpr bool kPdl = HTG_ND_PDL != 0;
__device__ __forceinline__ void pdl_begin() {
    if constexpr (kPdl) {
        asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
        asm volatile("griddepcontrol.wait;\n" ::: "memory");
    }
}

__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

struct NDArgs {
    const int* idx;
    const int4* gsrc;
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
// TRI: 0 dense; 1 lower triangular (row r has nonzeros k <= r: L^-1 P); 2 upper
// triangular (k >= r: U^-1). The zero half of a triangular block is neither read
// nor multiplied.
template <int TRI = 0, class Out>
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
        // KU k-steps per trip with their loads issued together: a warp often owns a
        // single long row (large-tier tasks), so the loop must keep several
        // DRAM loads in flight per lane
        constexpr int KU = HTG_ND_KU;
        const int rlast = min(rr[U - 1], r1 - 1);
        const int kend = TRI == 1 ? min(len, rlast + 1) : len;
        int k = TRI == 2 ? (rr[0] / G) * G + gl : gl;
        auto live = [&](int q, int kk) { return rr[q] < r1 && (TRI != 1 || kk <= rr[q]) && (TRI != 2 || kk >= rr[q]); };
        for (; k + (KU - 1) * G < kend; k += KU * G) {
            double2 m[U][KU], vk[KU];
#pragma unroll
            for (int j = 0; j < KU; ++j) vk[j] = v[k + j * G];
#pragma unroll
            for (int q = 0; q < U; ++q)
#pragma unroll
                for (int j = 0; j < KU; ++j)
                    m[q][j] = live(q, k + j * G) ? M[(size_t)rr[q] * len + k + j * G] : make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < U; ++q)
#pragma unroll
                for (int j = 0; j < KU; ++j) acc[q] = cfma(m[q][j], vk[j], acc[q]);
        }
        for (; k < kend; k += G) {
            const double2 vk = v[k];
#pragma unroll
            for (int q = 0; q < U; ++q)
                if (live(q, k)) acc[q] = cfma(M[(size_t)rr[q] * len + k], vk, acc[q]);
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

// Warp tier (small fronts): blocks are stored column-major, one lane group per
// row: lanes (i, part) with i = lane % R accumulate the k = part (mod S) terms
// of row i, S = 32 / R parts combined with S - 1 shuffles. Column reads are
// coalesced and there is no per-row reduction tree (short rows).
template <int TRI = 0, class Out>
__device__ __forceinline__ void cols_dot(const double2* __restrict__ M, int rows, int len, const double2* v, int lane,
                                         Out&& out) {
    int R = 32;
    if (rows <= 4) R = 4;
    else if (rows <= 8) R = 8;
    else if (rows <= 16) R = 16;
    const int S = 32 / R, i0 = lane % R, part = lane / R;
    for (int rb = 0; rb < rows; rb += R) {
        const int i = rb + i0;
        double2 acc = make_double2(0.0, 0.0);
        if (i < rows) {
            // triangular blocks: lane row i only walks its nonzero columns
            const int kb = TRI == 2 ? part + ((max(i - part, 0) + S - 1) / S) * S : part;
            const int ke = TRI == 1 ? min(len, i + 1) : len;
#pragma unroll 4
            for (int k = kb; k < ke; k += S) acc = cfma(M[(size_t)k * rows + i], v[k], acc);
        }
        for (int o = R; o < 32; o <<= 1) {
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        }
        if (part == 0 && i < rows) out(i, acc);
    }
}

// front vector v = [rc(vars); 0] + the children's contribution vectors (each
// position has at most two, added in child order), one pass, no barrier inside
template <int STRIDE, class Sync>
__device__ void gather_front(const NDArgs& a, const NodeDev& nd, double2* sv, int t, Sync&& sync, int gend = -1) {
    const int F = gend >= 0 ? gend : nd.s + nd.u;  // positions [0, gend) only, when given
#pragma unroll 4
    for (int i = t; i < F; i += STRIDE) {
        const int ri = a.idx[nd.off_rc + i];
        double2 v = ri >= 0 ? a.rc[ri] : make_double2(0.0, 0.0);
        const int4 src = a.gsrc[nd.off_gsrc + i];
        const int sx[4] = {src.x, src.y, src.z, src.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (sx[q] < 0) break;
            const double2 c = a.contrib[sx[q]];
            v.x += c.x;
            v.y += c.y;
        }
        sv[i] = v;
    }
    sync();
}

// forward: y1 = (L^-1 P) v1, c = v2 - L21 y1. Warp tier: one warp per front,
// front item * 8 + warp of the list; ws: 2 x 8 x kWarpFMax shared entries.
__device__ __forceinline__ void dev_fwd_warp(const NodeDev* __restrict__ list, int n, const NDArgs& a, int item,
                                             double2* ws) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int id = item * (kCT / 32) + w;
    if (id >= n) return;
    const NodeDev nd = list[id];
    double2* v = ws + w * 2 * kWarpFMax;
    double2* y = v + kWarpFMax;
    gather_front<32>(a, nd, v, lane, [] { __syncwarp(); });
    cols_dot<1>(a.fac + nd.off_F, nd.s, nd.s, v, lane, [&](int r, double2 acc) {
        y[r] = acc;
        a.Y[a.idx[nd.off_var + r]] = acc;
    });
    __syncwarp();
    cols_dot(a.fac + nd.off_L, nd.u, nd.s, y, lane, [&](int r, double2 acc) {
        const double2 v2 = v[nd.s + r];
        a.contrib[nd.off_contrib + r] = make_double2(v2.x - acc.x, v2.y - acc.y);
    });
}
__global__ void __launch_bounds__(kCT) k_nd_fwd_warp(const NodeDev* __restrict__ list, int n, NDArgs a) {
    pdl_begin();
    __shared__ double2 ws[(kCT / 32) * 2 * kWarpFMax];
    dev_fwd_warp(list, n, a, blockIdx.x, ws);
}

// forward, CTA tier: one CTA per front, both phases
__device__ __forceinline__ void dev_fwd_mid(const NodeDev& nd, const NDArgs& a, double2* smem) {
    double2* v = smem;
    double2* y = smem + nd.s + nd.u;
    gather_front<kCT>(a, nd, v, threadIdx.x, [] { __syncthreads(); });
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    rows_dot<1>(a.fac + nd.off_F, nd.s, v, 0, nd.s, warp, kCT / 32, lane, [&](int r, double2 acc) {
        y[r] = acc;
        a.front[nd.off_front + r] = acc;  // y1, contiguous, for the backward pass
    });
    __syncthreads();
    rows_dot(a.fac + nd.off_L, nd.s, y, 0, nd.u, warp, kCT / 32, lane, [&](int r, double2 acc) {
        const double2 v2 = v[nd.s + r];
        a.contrib[nd.off_contrib + r] = make_double2(v2.x - acc.x, v2.y - acc.y);
    });
}
__global__ void __launch_bounds__(kCT) k_nd_fwd_mid(const NodeDev* __restrict__ list, NDArgs a) {
    pdl_begin();
    extern __shared__ double2 smem[];
    dev_fwd_mid(list[blockIdx.x], a, smem);
}

// forward, large tier phase 1: y1 rows of a task (v2 stashed by the r0 == 0 task)
__device__ __forceinline__ void dev_fwd1(const Task& tk, const NDArgs& a, double2* smem) {
    const NodeDev& nd = tk.nd;
    // rows [r0, r0 + nr) of the lower-triangular L^-1 P read v[0, r0 + nr) only; the
    // r0 == 0 task also stashes v2 for the contribution tasks
    gather_front<kCT>(a, nd, smem, threadIdx.x, [] { __syncthreads(); },
                      tk.r0 == 0 ? nd.s + nd.u : min(nd.s, tk.r0 + tk.nr));
    if (tk.r0 == 0)
        for (int i = nd.s + threadIdx.x; i < nd.s + nd.u; i += kCT) a.front[nd.off_front + i] = smem[i];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    rows_dot<1>(a.fac + nd.off_F, nd.s, smem, tk.r0, tk.r0 + tk.nr, warp, kCT / 32, lane,
             [&](int r, double2 acc) { a.front[nd.off_front + r] = acc; });
}
__global__ void __launch_bounds__(kCT) k_nd_fwd1(const Task* tasks, NDArgs a) {
    pdl_begin();
    extern __shared__ double2 smem[];
    dev_fwd1(tasks[blockIdx.x], a, smem);
}

// forward, large tier phase 2: contribution rows c = v2 - L21 y1
__device__ __forceinline__ void dev_fwd2(const Task& tk, const NDArgs& a, double2* smem) {
    const NodeDev& nd = tk.nd;
#pragma unroll 4
    for (int i = threadIdx.x; i < nd.s; i += kCT) smem[i] = a.front[nd.off_front + i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    rows_dot(a.fac + nd.off_L, nd.s, smem, tk.r0, tk.r0 + tk.nr, warp, kCT / 32, lane, [&](int r, double2 acc) {
        const double2 v2 = a.front[nd.off_front + nd.s + r];
        a.contrib[nd.off_contrib + r] = make_double2(v2.x - acc.x, v2.y - acc.y);
    });
}
__global__ void __launch_bounds__(kCT) k_nd_fwd2(const Task* tasks, NDArgs a) {
    pdl_begin();
    extern __shared__ double2 smem[];
    dev_fwd2(tasks[blockIdx.x], a, smem);
}

// backward: x1 = U^-1 y1 - (U^-1 U12) x2. Z rows are computed into sz first.
__device__ __forceinline__ void bwd_rows(const NDArgs& a, const NodeDev& nd, const double2* y1, const double2* x2,
                                         double2* sz, int r0, int r1, int warp, int nw, int lane,
                                         void (*sync)()) {
    if (nd.u > 0) {
        rows_dot(a.fac + nd.off_Z, nd.u, x2, r0, r1, warp, nw, lane, [&](int r, double2 acc) { sz[r - r0] = acc; });
        sync();
    }
    rows_dot<2>(a.fac + nd.off_U, nd.s, y1, r0, r1, warp, nw, lane, [&](int r, double2 acc) {
        if (nd.u > 0) {
            acc.x -= sz[r - r0].x;
            acc.y -= sz[r - r0].y;
        }
        a.X[a.idx[nd.off_var + r]] = acc;
    });
}
__device__ void sync_cta_fn() { __syncthreads(); }

__device__ __forceinline__ void dev_bwd_warp(const NodeDev* __restrict__ list, int n, const NDArgs& a, int item,
                                             double2* ws) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int id = item * (kCT / 32) + w;
    if (id >= n) return;
    const NodeDev nd = list[id];
    double2* v = ws + w * 2 * kWarpFMax;
#pragma unroll 4
    for (int i = lane; i < nd.s; i += 32) v[i] = a.Y[a.idx[nd.off_var + i]];
#pragma unroll 4
    for (int i = lane; i < nd.u; i += 32) v[nd.s + i] = a.X[a.idx[nd.off_ring + i]];
    __syncwarp();
    // x1 = U^-1 y1 - Z x2 (column-major blocks)
    double2* z = v + kWarpFMax;
    if (nd.u > 0) {
        cols_dot(a.fac + nd.off_Z, nd.s, nd.u, v + nd.s, lane, [&](int r, double2 acc) { z[r] = acc; });
        __syncwarp();
    }
    cols_dot<2>(a.fac + nd.off_U, nd.s, nd.s, v, lane, [&](int r, double2 acc) {
        if (nd.u > 0) {
            acc.x -= z[r].x;
            acc.y -= z[r].y;
        }
        a.X[a.idx[nd.off_var + r]] = acc;
    });
}
__global__ void __launch_bounds__(kCT) k_nd_bwd_warp(const NodeDev* __restrict__ list, int n, NDArgs a) {
    pdl_begin();
    __shared__ double2 ws[(kCT / 32) * 2 * kWarpFMax];
    dev_bwd_warp(list, n, a, blockIdx.x, ws);
}

// The warp-tier bottom of a subtree branch in one launch per direction: a CTA owns the
// sub-subtree below one front of the first all-warp-tier level and walks its levels
// itself (deepest first going forward, root first going backward), a block barrier
// between levels: the contributions / solution entries a level reads were written by
// this CTA's previous level. Replaces one launch per level (HTG_ND_SUBTREE).
constexpr int kSubLevels = 8;
struct WarpSub {
    int off[kSubLevels];  // per level below the root (0 = root level): first front of this CTA's list
    int cnt[kSubLevels];
    int nlev;
};
__global__ void __launch_bounds__(kCT) k_nd_fwd_sub(const NodeDev* __restrict__ list, const WarpSub* __restrict__ subs,
                                                   NDArgs a) {
    __shared__ double2 ws[(kCT / 32) * 2 * kWarpFMax];
    const WarpSub s = subs[blockIdx.x];
    for (int L = s.nlev - 1; L >= 0; --L) {
        for (int it = 0; it * (kCT / 32) < s.cnt[L]; ++it) {
            dev_fwd_warp(list + s.off[L], s.cnt[L], a, it, ws);
            __syncwarp();
        }
        __threadfence_block();
        __syncthreads();
    }
}
__global__ void __launch_bounds__(kCT) k_nd_bwd_sub(const NodeDev* __restrict__ list, const WarpSub* __restrict__ subs,
                                                   NDArgs a) {
    __shared__ double2 ws[(kCT / 32) * 2 * kWarpFMax];
    const WarpSub s = subs[blockIdx.x];
    for (int L = 0; L < s.nlev; ++L) {
        for (int it = 0; it * (kCT / 32) < s.cnt[L]; ++it) {
            dev_bwd_warp(list + s.off[L], s.cnt[L], a, it, ws);
            __syncwarp();
        }
        __threadfence_block();
        __syncthreads();
    }
}

// backward, CTA tasks (whole front for the CTA tier, row blocks for the large tier)
__device__ __forceinline__ void dev_bwd(const Task& tk, const NDArgs& a, double2* smem) {
    const NodeDev& nd = tk.nd;
    double2* y1 = smem;
    double2* x2 = smem + nd.s;
    double2* sz = smem + nd.s + nd.u;
    // the upper-triangular U^-1 rows [r0, ..) read y1[k >= r0] (from the 32-aligned
    // block the row dots start at)
#pragma unroll 4
    for (int i = (tk.r0 & ~31) + threadIdx.x; i < nd.s; i += kCT) y1[i] = a.front[nd.off_front + i];
#pragma unroll 4
    for (int i = threadIdx.x; i < nd.u; i += kCT) x2[i] = a.X[a.idx[nd.off_ring + i]];
    __syncthreads();
    bwd_rows(a, nd, y1, x2, sz, tk.r0, tk.r0 + tk.nr, threadIdx.x >> 5, kCT / 32, threadIdx.x & 31, sync_cta_fn);
}
__global__ void __launch_bounds__(kCT) k_nd_bwd(const Task* tasks, NDArgs a) {
    pdl_begin();
    extern __shared__ double2 smem[];
    dev_bwd(tasks[blockIdx.x], a, smem);
}

// ------------------------------------------------------------------ persistent solve
// The whole solve as ONE cooperative launch: the phases (per depth, deepest
// first: warp-tier fronts + CTA-tier fronts + large-tier y1 tasks, then the
// large-tier contribution tasks; backward per depth, top first) are walked by
// every CTA of a co-resident grid, items grid-strided, with a grid barrier
// between phases. Replaces ~250 dependent launches (16 subtree branches on
// forked streams) whose launch latencies dominated the solve.
struct NDPhase {
    const Task* tasks;    // fwd: y1 tasks (kind 0) or contribution tasks (kind 1); bwd: CTA / row-block tasks
    const NodeDev* mid;   // fwd CTA-tier fronts
    const NodeDev* warp;  // warp-tier fronts (8 per item)
    int ntask, nmid, nwarp, kind;  // kind 0 fwd, 1 fwd contributions, 2 bwd
};
__device__ __forceinline__ int phase_items(const NDPhase& P) {
    return P.ntask + P.nmid + (P.nwarp + kCT / 32 - 1) / (kCT / 32);
}
__device__ __forceinline__ void phase_item(const NDPhase& P, int it, const NDArgs& a, double2* smem) {
    if (it < P.ntask) {
        const Task tk = P.tasks[it];
        if (P.kind == 0) dev_fwd1(tk, a, smem);
        else if (P.kind == 1) dev_fwd2(tk, a, smem);
        else dev_bwd(tk, a, smem);
    } else if (it < P.ntask + P.nmid) {
        const NodeDev nd = P.mid[it - P.ntask];
        dev_fwd_mid(nd, a, smem);
    } else {
        const int wi = it - P.ntask - P.nmid;
        if (P.kind == 2) dev_bwd_warp(P.warp, P.nwarp, a, wi, smem);
        else dev_fwd_warp(P.warp, P.nwarp, a, wi, smem);
    }
}
__global__ void __launch_bounds__(kCT) k_nd_persist(const NDPhase* __restrict__ ph, int nph, NDArgs a) {
    extern __shared__ double2 smem[];
    cg::grid_group grid = cg::this_grid();
    for (int p = 0; p < nph; ++p) {
        const NDPhase P = ph[p];
        const int total = phase_items(P);
        for (int it = blockIdx.x; it < total; it += gridDim.x) {
            phase_item(P, it, a, smem);
            __syncthreads();  // shared memory reuse by the next item
        }
        if (p + 1 < nph) grid.sync();
    }
}
// one level of one subtree branch, every tier in ONE launch (item = block)
__global__ void __launch_bounds__(kCT) k_nd_level(NDPhase P, NDArgs a) {
    extern __shared__ double2 smem[];
    phase_item(P, blockIdx.x, a, smem);
}

class NDSolver : public CoarseSolver {
  public:
    NDSolver(const LatticeMatrix& A, cudaStream_t st) {
        NDTree t;
        const char* pt = std::getenv("HTG_ND_PIVTOL");
        const auto t0 = std::chrono::steady_clock::now();
        nd_factor(A, t, env_int("HTG_ND_LEAF", 36), pt ? std::atof(pt) : 0.3);
        if (std::getenv("HTG_SETUP_TIMES"))
            std::fprintf(stderr, "htg setup:   nested-dissection factor %8.3f s (%d fronts, %lld sharing factors, max front %d)\n",
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(),
                         int(t.nodes.size()), t.shared, t.max_front);
        nv_ = t.nv;
        delayed_ = t.delayed;
        const auto t1 = std::chrono::steady_clock::now();
        upload(t, st);
        if (std::getenv("HTG_SETUP_TIMES"))
            std::fprintf(stderr, "htg setup:   factor upload + solve plan %8.3f s\n",
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count());
    }
    ~NDSolver() override {
        for (void* p : allocs_) cudaFree(p);
        for (cudaStream_t x : bst_) cudaStreamDestroy(x);
        for (cudaEvent_t e : ev_join_) cudaEventDestroy(e);
        if (ev_fork_) cudaEventDestroy(ev_fork_);
    }
    size_t device_bytes() const override { return bytes_; }
    int levels() const override { return nlevels_; }
    size_t solve_read_bytes() const override { return read_bytes_; }

    // Forward: the subtrees below the split depth run on forked streams (in a
    // CUDA graph: parallel branches), deepest level first, then the top levels;
    // backward in the reverse order. Levels with few fronts are latency-bound
    // launches, so independent subtrees overlap them.
    void solve(const double2* rc, double2* uc, cudaStream_t st) override {
        NDArgs a = args_;
        a.rc = rc;
        a.X = uc;
        if (nph_ > 0) {  // one cooperative launch walks every level (k_nd_persist)
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(pgrid_);
            cfg.blockDim = dim3(kCT);
            cfg.dynamicSmemBytes = psmem_;
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeCooperative;
            at[0].val.cooperative = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            HTG_CUDA(cudaLaunchKernelEx(&cfg, k_nd_persist, static_cast<const NDPhase*>(phases_), nph_, a));
            count_launch();
            return;
        }
        const int nb = int(br_.size()) - 1;  // branch 0: the top levels
#ifdef HTG_ND_TIMING_SKIP
        static const int skip = env_int("HTG_ND_SKIP", 0);  // timing experiments only: 1 branches, 2 top
#else
        constexpr int skip = 0;
#endif
        HTG_CUDA(cudaEventRecord(ev_fork_, st));
        for (int b = 1; b <= nb; ++b) {
            HTG_CUDA(cudaStreamWaitEvent(bst_[b - 1], ev_fork_, 0));
            if (skip != 1) {
                const SubFused& sf = sub_[b];
                int Ltop = int(br_[b].size());
                if (sf.nroots > 0) {
                    launch(k_nd_fwd_sub, sf.nroots, 0, bst_[b - 1], sf.list, sf.subs, a);
                    Ltop = sf.Lw;
                }
                for (int L = Ltop - 1; L >= 0; --L) fwd_level(br_[b][L], a, bst_[b - 1]);
            }
            HTG_CUDA(cudaEventRecord(ev_join_[b - 1], bst_[b - 1]));
        }
        for (int b = 1; b <= nb; ++b) HTG_CUDA(cudaStreamWaitEvent(st, ev_join_[b - 1], 0));
        if (skip != 2) {
            for (int L = int(br_[0].size()) - 1; L >= 0; --L) fwd_level(br_[0][L], a, st);
            for (int L = 0; L < int(br_[0].size()); ++L) bwd_level(br_[0][L], a, st);
        }
        HTG_CUDA(cudaEventRecord(ev_fork_, st));
        for (int b = 1; b <= nb; ++b) {
            HTG_CUDA(cudaStreamWaitEvent(bst_[b - 1], ev_fork_, 0));
            if (skip != 1) {
                const SubFused& sf = sub_[b];
                const int Ltop = sf.nroots > 0 ? sf.Lw : int(br_[b].size());
                for (int L = 0; L < Ltop; ++L) bwd_level(br_[b][L], a, bst_[b - 1]);
                if (sf.nroots > 0) launch(k_nd_bwd_sub, sf.nroots, 0, bst_[b - 1], sf.list, sf.subs, a);
            }
            HTG_CUDA(cudaEventRecord(ev_join_[b - 1], bst_[b - 1]));
        }
        for (int b = 1; b <= nb; ++b) HTG_CUDA(cudaStreamWaitEvent(st, ev_join_[b - 1], 0));
        HTG_CUDA(cudaGetLastError());
    }

  private:
    struct Level {
        const NodeDev *warp = nullptr, *mid = nullptr;
        const Task *f1 = nullptr, *f2 = nullptr, *b = nullptr;
        int nwarp = 0, nmid = 0, nf1 = 0, nf2 = 0, nb = 0;
        size_t smem_mid = 0, smem_big = 0, smem_b = 0;
    };
    template <class... KArgs, class... Args>
    static void launch(void (*kern)(KArgs...), int grid, size_t smem, cudaStream_t st, Args&&... args) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(unsigned(grid));
        cfg.blockDim = dim3(kCT);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = kPdl ? 1 : 0;
        HTG_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
        count_launch();
    }
    static void fwd_level(const Level& lv, const NDArgs& a, cudaStream_t st) {
        if (kMergedLevels) {  // warp + CTA + large-tier y1 items in one launch, then the contributions
            const NDPhase p0{lv.f1, lv.mid, lv.warp, lv.nf1, lv.nmid, lv.nwarp, 0};
            const int n0 = lv.nf1 + lv.nmid + (lv.nwarp + 7) / 8;
            if (n0) {
                const size_t sm = std::max({lv.nwarp ? size_t(2 * (kCT / 32) * kWarpFMax) * sizeof(double2) : size_t(0),
                                            lv.smem_mid, lv.smem_big});
                k_nd_level<<<n0, kCT, sm, st>>>(p0, a);
                count_launch();
            }
            if (lv.nf2) {
                k_nd_level<<<lv.nf2, kCT, lv.smem_big, st>>>(NDPhase{lv.f2, nullptr, nullptr, lv.nf2, 0, 0, 1}, a);
                count_launch();
            }
            return;
        }
        if (lv.nwarp) launch(k_nd_fwd_warp, (lv.nwarp + 7) / 8, 0, st, lv.warp, lv.nwarp, a);
        if (lv.nmid) launch(k_nd_fwd_mid, lv.nmid, lv.smem_mid, st, lv.mid, a);
        if (lv.nf1) launch(k_nd_fwd1, lv.nf1, lv.smem_big, st, lv.f1, a);
        if (lv.nf2) launch(k_nd_fwd2, lv.nf2, lv.smem_big, st, lv.f2, a);
    }
    static void bwd_level(const Level& lv, const NDArgs& a, cudaStream_t st) {
        if (kMergedLevels) {
            const int n = lv.nb + (lv.nwarp + 7) / 8;
            if (n) {
                const size_t sm = std::max(lv.nwarp ? size_t(2 * (kCT / 32) * kWarpFMax) * sizeof(double2) : size_t(0),
                                           lv.smem_b);
                k_nd_level<<<n, kCT, sm, st>>>(NDPhase{lv.b, nullptr, lv.warp, lv.nb, 0, lv.nwarp, 2}, a);
                count_launch();
            }
            return;
        }
        if (lv.nb) launch(k_nd_bwd, lv.nb, lv.smem_b, st, lv.b, a);
        if (lv.nwarp) launch(k_nd_bwd_warp, (lv.nwarp + 7) / 8, 0, st, lv.warp, lv.nwarp, a);
    }
    // br_[0]: levels 0 .. split-1 (the top); br_[b]: the subtree of the b-th node at
    // the split depth, indexed by depth - split
    // per branch: the fused warp-tier bottom (levels >= Lw of the branch), or nroots == 0
    struct SubFused {
        const NodeDev* list = nullptr;
        const WarpSub* subs = nullptr;
        int nroots = 0, Lw = 0;
    };
    std::vector<SubFused> sub_;
    std::vector<std::vector<Level>> br_;
    std::vector<cudaStream_t> bst_;
    std::vector<cudaEvent_t> ev_join_;
    cudaEvent_t ev_fork_ = nullptr;
    int nlevels_ = 0;
    std::vector<void*> allocs_;
    size_t bytes_ = 0;
    size_t read_bytes_ = 0;
    const NDPhase* phases_ = nullptr;  // persistent solve (HTG_ND_PERSIST, default on)
    int nph_ = 0, pgrid_ = 0;
    size_t psmem_ = 0;
    int nv_ = 0;
    long long delayed_ = 0;
    NDArgs args_{};

    template <class T>
    T* up(const std::vector<T>& v, cudaStream_t st) {
        if (v.empty()) return nullptr;  // empty per-(branch, level) lists: nothing to launch
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
        std::vector<int> idx, owners;  // owners: nodes holding their own factor blocks
        long long fac_total = 0;
        int front_total = 0, contrib_total = 0, gsrc_total = 0;
        for (int i = 0; i < nn; ++i) {
            const NDNode& n = t.nodes[i];
            NodeDev& d = nd[i];
            d.s = n.ke;
            d.u = n.F - n.ke;
            if (n.rep >= 0) {  // the representative's blocks (an earlier node)
                const NodeDev& r = nd[size_t(n.rep)];
                if (n.rep >= i || r.s != d.s || r.u != d.u) throw RuntimeError("coarse solve: bad shared front");
                d.off_F = r.off_F;
                d.off_L = r.off_L;
                d.off_U = r.off_U;
                d.off_Z = r.off_Z;
            } else {
                owners.push_back(i);
                d.off_F = fac_total;
                fac_total += (long long)d.s * d.s;
                d.off_L = fac_total;
                fac_total += (long long)d.u * d.s;
                d.off_U = fac_total;
                fac_total += (long long)d.s * d.s;
                d.off_Z = fac_total;
                fac_total += (long long)d.s * d.u;
            }
            d.off_var = int(idx.size());
            idx.insert(idx.end(), n.cols.begin(), n.cols.begin() + n.ke);
            d.off_ring = int(idx.size());
            idx.insert(idx.end(), n.cols.begin() + n.ke, n.cols.end());
            d.off_rc = int(idx.size());
            idx.insert(idx.end(), n.rc.begin(), n.rc.end());
            d.off_front = front_total;
            front_total += d.s + d.u;
            d.off_contrib = contrib_total;
            contrib_total += d.u;
            d.off_gsrc = gsrc_total;
            gsrc_total += d.s + d.u;
        }
        // gather plan: front position <- contribution entries of the children (child order)
        std::vector<int4> gsrc(std::max(gsrc_total, 1), make_int4(-1, -1, -1, -1));
        std::vector<int> rpos(nv_, -1);
        for (int i = 0; i < nn; ++i) {
            const NDNode& n = t.nodes[i];
            for (int k = 0; k < n.F; ++k) rpos[n.rows[k]] = k;
            for (int c : n.children) {
                const NDNode& ch = t.nodes[c];
                for (int k = 0; k < ch.F - ch.ke; ++k) {
                    int4& e = gsrc[nd[i].off_gsrc + rpos[ch.rows[ch.ke + k]]];
                    const int src = nd[c].off_contrib + k;
                    if (e.x < 0) e.x = src;
                    else if (e.y < 0) e.y = src;
                    else if (e.z < 0) e.z = src;
                    else if (e.w < 0) e.w = src;
                    else throw RuntimeError("coarse solve: more than four contributions to a front position");
                }
            }
            for (int k = 0; k < n.F; ++k) rpos[n.rows[k]] = -1;
        }
        const int warpF = std::min(kWarpFMax, env_int("HTG_ND_WARPF", 96));
        void* facp = nullptr;
        HTG_CUDA(cudaMalloc(&facp, std::max<long long>(1, fac_total) * sizeof(double2)));
        allocs_.push_back(facp);
        bytes_ += fac_total * sizeof(double2);
        // The factor blocks are laid out back to back in node order (off_F, off_L, off_U,
        // off_Z). Runs of nodes of up to 64 MB are packed by all host threads into one of
        // two pinned staging buffers (warp-tier blocks transposed on the way: column-major
        // for cols_dot) and copied asynchronously, so packing overlaps the transfer
        // (one cudaMemcpy per block took seconds at cfg4: 4 blocks x 68k fronts; one
        // thread packing through one buffer 0.5 s).
        // (on its own thread and stream: the solve plan below is built meanwhile)
        std::exception_ptr pack_err;
        int pack_dev = 0;
        HTG_CUDA(cudaGetDevice(&pack_dev));
        auto pack_all = [&]() {
          try {
            HTG_CUDA(cudaSetDevice(pack_dev));
            cudaStream_t st = nullptr;  // shadows the caller's stream inside this thread
            HTG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            const auto tp0 = std::chrono::steady_clock::now();
            const size_t chunk = size_t(64) << 20;  // bytes
            cplx* stage[2] = {nullptr, nullptr};
            cudaEvent_t done[2];
            for (int b = 0; b < 2; ++b) {
                HTG_CUDA(cudaMallocHost(&stage[b], chunk));
                HTG_CUDA(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
            }
            auto node_end = [&](int i) { return nd[i].off_Z + (long long)nd[i].s * nd[i].u; };
            const int nthr = std::max(1, int(std::thread::hardware_concurrency()));
            int buf = 0;
            const int no = int(owners.size());
            for (int i0 = 0; i0 < no;) {
                const long long base = nd[owners[i0]].off_F;
                int i1 = i0 + 1;
                while (i1 < no && size_t(node_end(owners[i1]) - base) * sizeof(cplx) <= chunk) ++i1;
                const size_t bytes = size_t(node_end(owners[i1 - 1]) - base) * sizeof(cplx);
                if (bytes > chunk) throw RuntimeError("coarse solve: a front's factors exceed the staging buffer");
                HTG_CUDA(cudaEventSynchronize(done[buf]));  // the buffer's previous copy
                cplx* dst = stage[buf];
                std::atomic<int> next{i0};
                auto pack = [&]() {
                    for (int oi; (oi = next++) < i1;) {
                        const int i = owners[oi];
                        NDNode& n = t.nodes[i];
                        const NodeDev& d = nd[i];
                        const bool colmajor = d.s + d.u <= warpF;
                        auto put = [&](std::vector<cplx>& v, long long off, int rows, int cols) {
                            cplx* o = dst + (off - base);
                            if (colmajor) {
                                for (int r = 0; r < rows; ++r)
                                    for (int k = 0; k < cols; ++k) o[size_t(k) * rows + r] = v[size_t(r) * cols + k];
                            } else if (!v.empty()) {
                                std::memcpy(o, v.data(), v.size() * sizeof(cplx));
                            }
                            std::vector<cplx>().swap(v);
                        };
                        put(n.Finv, d.off_F, d.s, d.s);
                        put(n.L21, d.off_L, d.u, d.s);
                        put(n.Uinv, d.off_U, d.s, d.s);
                        put(n.Z, d.off_Z, d.s, d.u);
                    }
                };
                const int nt = std::min(nthr, i1 - i0);
                std::vector<std::thread> th;
                for (int w = 1; w < nt; ++w) th.emplace_back(pack);
                pack();
                for (auto& x : th) x.join();
                if (bytes)
                    HTG_CUDA(cudaMemcpyAsync(static_cast<double2*>(facp) + base, dst, bytes, cudaMemcpyHostToDevice, st));
                HTG_CUDA(cudaEventRecord(done[buf], st));
                buf ^= 1;
                i0 = i1;
            }
            for (int b = 0; b < 2; ++b) {
                HTG_CUDA(cudaEventSynchronize(done[b]));
                HTG_CUDA(cudaEventDestroy(done[b]));
                HTG_CUDA(cudaFreeHost(stage[b]));
            }
            HTG_CUDA(cudaStreamSynchronize(st));
            cudaStreamDestroy(st);
            if (std::getenv("HTG_SETUP_TIMES"))
                std::fprintf(stderr, "htg setup:     factor pack + copy       %8.3f s\n",
                             std::chrono::duration<double>(std::chrono::steady_clock::now() - tp0).count());
          } catch (...) {
            pack_err = std::current_exception();
          }
        };
        std::thread pack_thread(pack_all);
        struct PackJoin {  // joined on every path out of upload()
            std::thread& t;
            ~PackJoin() {
                if (t.joinable()) t.join();
            }
        } pack_join{pack_thread};
        args_.fac = static_cast<const double2*>(facp);
        args_.idx = up(idx, st);
        args_.gsrc = up(gsrc, st);
        args_.contrib = up(std::vector<double2>(std::max(contrib_total, 1)), st);
        args_.front = up(std::vector<double2>(std::max(front_total, 1)), st);
        args_.Y = up(std::vector<double2>(nv_), st);
        // Branches: the subtrees rooted at the nodes of depth `split` (env
        // HTG_ND_SPLIT, default 4: sixteen subtrees) run on their own streams; the
        // levels above them are branch 0. Per (branch, depth): warp tier, CTA
        // tier, large tier (8 rows per CTA task).
        const int split = std::max(0, env_int("HTG_ND_SPLIT", 4));
        std::vector<int> branch(nn, 0);
        int nbranch = 0;
        {
            std::vector<int> bid(nn, -1);
            for (int i = nn - 1; i >= 0; --i)  // postorder reversed: parents before children
                if (t.nodes[i].depth == split && split > 0) bid[i] = ++nbranch;
            for (int i = nn - 1; i >= 0; --i) {
                const int par = t.nodes[i].parent;
                if (bid[i] < 0) bid[i] = (par >= 0 && t.nodes[i].depth > split) ? bid[par] : 0;
                branch[i] = std::max(bid[i], 0);
            }
        }
        const int D = t.max_depth + 1;
        nlevels_ = D;
        br_.assign(nbranch + 1, {});
        for (int b = 0; b <= nbranch; ++b) br_[b].resize(b == 0 ? std::min(split > 0 ? split : D, D) : std::max(D - split, 0));
        const int NL = D * (nbranch + 1);
        auto li = [&](int b, int dep) { return b * D + dep; };
        std::vector<Level> lvs(NL);
        std::vector<std::vector<NodeDev>> wp(NL), md(NL);
        std::vector<std::vector<Task>> f1(NL), f2(NL), bw(NL);
        size_t max_smem = 0;
        const long long midData = env_int("HTG_ND_MIDDATA", 16384);
        for (int i = 0; i < nn; ++i) {
            const int dep = t.nodes[i].depth, k = li(branch[i], dep);
            const NodeDev& d = nd[i];
            Level& lv = lvs[k];
            const int F = d.s + d.u;
            // bytes one solve has to fetch from HBM: shared blocks once (their owner's)
            if (t.nodes[i].rep < 0) read_bytes_ += sizeof(double2) * (size_t(d.s) * (d.s + 1) + 2 * size_t(d.s) * d.u);
            if (F <= warpF) {
                wp[k].push_back(d);
            } else if ((long long)d.s * F <= midData) {
                md[k].push_back(d);
                bw[k].push_back({d, 0, d.s});
                lv.smem_mid = std::max(lv.smem_mid, size_t(F + d.s) * sizeof(double2));
                lv.smem_b = std::max(lv.smem_b, size_t(F + d.s) * sizeof(double2));
            } else {
                const int rpt = branch[i] == 0 ? env_int("HTG_ND_RPT_TOP", 8) : env_int("HTG_ND_RPT", 8);
                for (int r = 0; r < d.s; r += rpt) {
                    f1[k].push_back({d, r, std::min(rpt, d.s - r)});
                    bw[k].push_back({d, r, std::min(rpt, d.s - r)});
                }
                for (int r = 0; r < d.u; r += rpt) f2[k].push_back({d, r, std::min(rpt, d.u - r)});
                lv.smem_big = std::max(lv.smem_big, size_t(F) * sizeof(double2));
                lv.smem_b = std::max(lv.smem_b, size_t(F + rpt) * sizeof(double2));
            }
        }
        for (int b = 0; b <= nbranch; ++b)
            for (int dep = 0; dep < D; ++dep) {
                const int k = li(b, dep);
                const int L = b == 0 ? dep : dep - split;  // level index inside the branch
                if (L < 0 || L >= int(br_[b].size())) {
                    if (!wp[k].empty() || !md[k].empty() || !f1[k].empty() || !bw[k].empty())
                        throw RuntimeError("coarse solve: front outside its branch's level range");
                    continue;
                }
                Level& lv = lvs[k];
                lv.nwarp = int(wp[k].size());
                lv.nmid = int(md[k].size());
                lv.nf1 = int(f1[k].size());
                lv.nf2 = int(f2[k].size());
                lv.nb = int(bw[k].size());
                lv.warp = up(wp[k], st);
                lv.mid = up(md[k], st);
                lv.f1 = up(f1[k], st);
                lv.f2 = up(f2[k], st);
                lv.b = up(bw[k], st);
                max_smem = std::max({max_smem, lv.smem_mid, lv.smem_big, lv.smem_b});
                br_[b][L] = lv;
            }
        // fused warp-tier bottoms: per branch the first level from which every deeper level
        // holds warp-tier fronts only; one CTA per front of that level
        sub_.assign(size_t(nbranch) + 1, SubFused{});
        if (env_int("HTG_ND_SUBTREE", 0) && split > 0) {
            for (int b = 1; b <= nbranch; ++b) {
                const int NLb = int(br_[b].size());
                int Lw = NLb;
                while (Lw > 0 && br_[b][Lw - 1].nmid == 0 && br_[b][Lw - 1].nf1 == 0 && br_[b][Lw - 1].nb == 0 &&
                       br_[b][Lw - 1].nwarp > 0)
                    --Lw;
                Lw = std::max(Lw, NLb - std::min(kSubLevels, env_int("HTG_ND_SUBLEVELS", kSubLevels)));
                if (NLb - Lw < 2) continue;
                const int dep0 = split + Lw;
                std::vector<NodeDev> list;
                std::vector<WarpSub> subs;
                for (int i = 0; i < nn; ++i) {
                    if (branch[i] != b || t.nodes[i].depth != dep0) continue;
                    WarpSub ws{};
                    std::vector<int> cur{i};
                    int L = 0;
                    while (!cur.empty() && L < kSubLevels) {
                        ws.off[L] = int(list.size());
                        ws.cnt[L] = int(cur.size());
                        std::vector<int> next;
                        for (int id : cur) {
                            list.push_back(nd[id]);
                            next.insert(next.end(), t.nodes[id].children.begin(), t.nodes[id].children.end());
                        }
                        cur.swap(next);
                        ++L;
                    }
                    if (!cur.empty()) throw RuntimeError("coarse solve: fused subtree deeper than expected");
                    ws.nlev = L;
                    subs.push_back(ws);
                }
                if (subs.empty()) continue;
                sub_[b].list = up(list, st);
                sub_[b].subs = up(subs, st);
                sub_[b].nroots = int(subs.size());
                sub_[b].Lw = Lw;
            }
        }
        // persistent solve: the same work lists merged over the branches, per depth
        if (env_int("HTG_ND_PERSIST", 0)) {
            std::vector<NDPhase> ph;
            auto mergedT = [&](std::vector<std::vector<Task>>& lists, int dep) {
                std::vector<Task> out;
                for (int b = 0; b <= nbranch; ++b) out.insert(out.end(), lists[li(b, dep)].begin(), lists[li(b, dep)].end());
                return out;
            };
            auto mergedN = [&](std::vector<std::vector<NodeDev>>& lists, int dep) {
                std::vector<NodeDev> out;
                for (int b = 0; b <= nbranch; ++b) out.insert(out.end(), lists[li(b, dep)].begin(), lists[li(b, dep)].end());
                return out;
            };
            for (int dep = D - 1; dep >= 0; --dep) {
                auto t1 = mergedT(f1, dep), t2 = mergedT(f2, dep);
                auto m = mergedN(md, dep), w = mergedN(wp, dep);
                if (!t1.empty() || !m.empty() || !w.empty())
                    ph.push_back({up(t1, st), up(m, st), up(w, st), int(t1.size()), int(m.size()), int(w.size()), 0});
                if (!t2.empty()) ph.push_back({up(t2, st), nullptr, nullptr, int(t2.size()), 0, 0, 1});
            }
            for (int dep = 0; dep < D; ++dep) {
                auto tb = mergedT(bw, dep);
                auto w = mergedN(wp, dep);
                if (!tb.empty() || !w.empty())
                    ph.push_back({up(tb, st), nullptr, up(w, st), int(tb.size()), 0, int(w.size()), 2});
            }
            psmem_ = std::max(max_smem, size_t(2 * (kCT / 32) * kWarpFMax) * sizeof(double2));
            if (psmem_ > 227 * 1024) throw InvalidArgument("coarse front too large for shared memory");
            static std::once_flag pers_once;
            std::call_once(pers_once, [] {
                HTG_CUDA(cudaFuncSetAttribute(k_nd_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
            });
            int per_sm = 0;
            HTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_nd_persist, kCT, psmem_));
            pgrid_ = std::max(1, per_sm) * current_sm_count();
            phases_ = up(ph, st);
            nph_ = int(ph.size());
        }
        for (int b = 0; b < nbranch; ++b) {
            cudaStream_t x;
            cudaEvent_t e;
            HTG_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
            HTG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            bst_.push_back(x);
            ev_join_.push_back(e);
        }
        HTG_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
        pack_thread.join();
        if (pack_err) std::rethrow_exception(pack_err);
        if (max_smem > 227 * 1024) throw InvalidArgument("coarse front too large for shared memory");
        // The attribute is process-global: always grant the opt-in maximum (it is a
        // permission, not a reservation), so handles of different sizes never lower
        // each other's limit.
        static std::once_flag smem_once;
        std::call_once(smem_once, [] {
            const int kOptIn = 227 * 1024;
            HTG_CUDA(cudaFuncSetAttribute(k_nd_fwd_mid, cudaFuncAttributeMaxDynamicSharedMemorySize, kOptIn));
            HTG_CUDA(cudaFuncSetAttribute(k_nd_fwd1, cudaFuncAttributeMaxDynamicSharedMemorySize, kOptIn));
            HTG_CUDA(cudaFuncSetAttribute(k_nd_fwd2, cudaFuncAttributeMaxDynamicSharedMemorySize, kOptIn));
            HTG_CUDA(cudaFuncSetAttribute(k_nd_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, kOptIn));
            HTG_CUDA(cudaFuncSetAttribute(k_nd_level, cudaFuncAttributeMaxDynamicSharedMemorySize, kOptIn));
        });
    }
};

}  // namespace

std::unique_ptr<CoarseSolver> make_nd_solver(const LatticeMatrix& A, cudaStream_t st) {
    return std::make_unique<NDSolver>(A, st);
}

std::unique_ptr<CoarseSolver> make_coarse_solver(const HostProblem& hp, cudaStream_t st) {
    const auto t0 = std::chrono::steady_clock::now();
    const LatticeMatrix A = qsfem_lattice(hp);
    if (std::getenv("HTG_SETUP_TIMES"))
        std::fprintf(stderr, "htg setup:   coarse stencil matrix      %8.3f s\n",
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    return make_nd_solver(A, st);
}

}  // namespace htg
