// k_fdm.cu -- K2 for separable subdomain classes: fast diagonalisation on DMMA.
//
// For a class with A_s^(Omega) = Kx (x) My + Mx (x) Ky (fdm.cpp) the U rows of
// A^-1 g are, with the gathered residual as a tensor tile G[ix][iy],
//   Y_U = Vx_U [ (Vx^T G Vy) o Dinv ] Vy_U^T,
// four small complex products per subdomain (8 (nx^2 ny + nx ny^2 + nux nx ny + nux ny nuy)
// flop, 3.7x fewer than the dense |U| x |Omega| product at p = 4).
//
// Batching: the four products share their class factor, so a group of 4 warps
// solves S subdomains of one class at once, stacked along the data dimension
// of every product (S = 2 at p = 4 with 4 groups: 50 data rows instead of
// 2 x 25 padded to 2 x 32). Only the factor dimension is padded to the m8/n8
// tile, and the contraction to the k4 step: 13% fewer DMMAs than one
// subdomain per product. The factor is the stationary operand (its fragments
// stay in registers across the data tiles); a factor dimension of 8 t + 1 or
// 8 t + 2 (25 and 17 at p = 4) runs its last rows as DFMA dot products on the
// CUDA cores instead of a DMMA tile that is 7/8 zeros (-28% DMMAs). Four groups per CTA (one CTA per SM, 16 warps, the
// whole 227 KB of shared memory) alternate batches of the CTA's range; measured
// at cfg4: 2 groups x S=4 0.265 ms, 3 x S=2 0.259 ms, 4 x S=2 0.242 ms.
// Every product is mma.sync.m8n8k4.f64 in the Gauss (3M) form: three real
// DMMAs per complex k-step and tile.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.hpp"
#include "kernels.hpp"

namespace htg {

namespace {

#ifndef HTG_FDM_GROUPS
#define HTG_FDM_GROUPS 4
#endif
constexpr int kFGroups = HTG_FDM_GROUPS, kFThreads = kFGroups * 128;
constexpr int kSmemMax = 232448;  // opt-in dynamic shared memory per block (227 KB)

// Row pitch of every operand (double2). An odd pitch puts the 8 rows x 4 k of a
// 128-bit fragment load, the 8 rows x 2 columns of an epilogue store (row-major
// and transposed) and 8 consecutive rows of a remainder dot on distinct bank
// groups (a pitch of 4 mod 8 left the epilogue stores and the dots two-way
// conflicted); k steps cover [0, 4 KS).
#ifndef HTG_FDM_ODD_LD
#define HTG_FDM_ODD_LD 1
#endif
template <int P> struct FdmDims;
template <> struct FdmDims<2> { static constexpr int LD = HTG_FDM_ODD_LD ? 17 : 20, KS = 4; };  // extents <= 16
template <> struct FdmDims<4> { static constexpr int LD = HTG_FDM_ODD_LD ? 29 : 28, KS = 7; };  // extents <= 28
constexpr bool kSkew = !HTG_FDM_ODD_LD;  // xor-skew the k of remainder dots (even pitch only)
// Fragment row r of every tile maps to tile row pi(r) = (r >> 1) | (r & 1) << 2: a
// 128-bit fragment load's quarter-warp (rows 2p, 2p+1 x 4 k) then covers all 8
// bank groups with the odd pitch (pi(2p+1) - pi(2p) = 4, 5 * 4 = 4 mod 8), and so
// do the row-major and transposed epilogue stores; without it every fragment
// load is two-way conflicted (8 wavefronts instead of 4, 31% of the kernel's
// shared-memory traffic)
#ifndef HTG_FDM_PERM
#define HTG_FDM_PERM 1
#endif
__device__ __forceinline__ int frow_perm(int r) { return HTG_FDM_PERM ? ((r >> 1) | ((r & 1) << 2)) : r; }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ void group_sync(int g) {
    asm volatile("bar.sync %0, 128;\n" ::"r"(g + 1) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
// exact floor(n / d) for 0 <= n < 2^16 and small d (margin 0.5 / n >> fp32 rounding)
__device__ __forceinline__ int fdiv(int n, float inv) { return __float2int_rz((float(n) + 0.5f) * inv); }

// One stage C[m][n] = sum_k A[m][k] B[n][k], A rows [0, am), B rows [0, bn),
// MT x NT tiles of 8 x 8, KS k steps of 4. Rows past am / bn are clamped (their
// outputs are discarded); the k padding of one operand is zero, so the
// padded k columns contribute exactly zero.
//
// Tile order per warp q of the group:
//   MT % 4 == 0: A-stationary, the warp owns m-tiles q, q+4, .., its A
//                fragments stay in registers over all n-tiles (1 load per tile-step);
//   NT % 4 == 0: B-stationary, likewise;
//   otherwise:   tiles q, q+4, q+8, .. of the flattened list, 4 in flight.
// The tile count of a group of tiles is a template argument, so the DMMAs are
// straight-line code without predicates.
#ifndef HTG_FDM_KSPLIT
#define HTG_FDM_KSPLIT 1
#endif
constexpr int kKP = HTG_FDM_KSPLIT;  // independent accumulator chains per product (k steps interleaved)
#ifndef HTG_FDM_TG
#define HTG_FDM_TG 4
#endif
constexpr int kTG = HTG_FDM_TG;  // moving tiles in flight per warp (one stationary fragment set)
#ifndef HTG_FDM_DR
#define HTG_FDM_DR 0
#endif
constexpr bool kDataRem = HTG_FDM_DR != 0;  // data-row remainders on the CUDA cores (group kernel)

// Complex products on the real DMMA: 3M (default: t1 = Re a Re b, t2 = Im a Im b,
// t3 = (Re a + Im a)(Re b + Im b); re = t1 - t2, im = t3 - t1 - t2) or, with
// HTG_FDM_4M, four products into two accumulators (re += Re a Re b + (-Im a) Im b,
// im += Re a Im b + Im a Re b): a third more DMMAs, but no pre-sum of the moving
// operand in front of every third DMMA and no post-combination.
#ifndef HTG_FDM_4M
#define HTG_FDM_4M 0
#endif
constexpr bool kF4M = HTG_FDM_4M != 0;
// HTG_FDM_SWAPB: products whose factor is the B operand (C[data][factor]) are issued
// as the transposed product with the factor as A (C'[factor][data]); only the
// epilogue's index interpretation changes
#ifndef HTG_FDM_SWAPB
#define HTG_FDM_SWAPB 1
#endif
constexpr bool kSwapB = HTG_FDM_SWAPB != 0;
// the stationary operand's auxiliary value: Re + Im (3M) or -Im (4M, a sign flip
// on the integer pipe)
__device__ __forceinline__ double stat_aux(double2 v) {
    if constexpr (kF4M) return __longlong_as_double(__double_as_longlong(v.y) ^ (1ll << 63));
    else return v.x + v.y;
}

template <int LD, int KS, bool FTR = false>
struct Stage {
    const double2* fac;  // factor operand [F][LD] (zero k padding)
    int F;               // factor rows (the padded output dimension)
    const double2* dat;  // data operand [nd][LD]
    int nd;              // data rows of the batch
    bool sa;             // the factor is the A operand (C[factor][data]); else B (C[data][factor])
    int q, lane;
    int fo = 0;          // FTR (transposed factor): row f, k at fac[k * LD + fo + f]

    __device__ __forceinline__ double2 fval(int f, int k) const { return FTR ? fac[k * LD + fo + f] : fac[f * LD + k]; }

    using Acc = double[kKP][kTG][2];
    template <int NTL, bool SA, class Epi>
    __device__ __forceinline__ void finish(Acc& t1, Acc& t2, Acc& t3, const int* tm, const int* tn, Epi& epi) const {
        const int r = lane >> 2, kq = lane & 3;
#pragma unroll
        for (int j = 0; j < NTL; ++j)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                double a1 = t1[0][j][i], a2 = t2[0][j][i], a3 = t3[0][j][i];
#pragma unroll
                for (int h = 1; h < kKP; ++h) {
                    a1 += t1[h][j][i];
                    a2 += t2[h][j][i];
                    a3 += t3[h][j][i];
                }
                if (kSwapB && !SA)
                    epi(tm[j] * 8 + frow_perm(2 * kq + i), tn[j] * 8 + frow_perm(r), make_double2(a1 - a2, a3 - a1 - a2));
                else
                    epi(tm[j] * 8 + frow_perm(r), tn[j] * 8 + frow_perm(2 * kq + i), make_double2(a1 - a2, a3 - a1 - a2));
            }
    }
    template <int NTL>
    __device__ __forceinline__ static void zero(Acc& t1, Acc& t2, Acc& t3) {
#pragma unroll
        for (int h = 0; h < kKP; ++h)
#pragma unroll
            for (int j = 0; j < NTL; ++j)
                t1[h][j][0] = t1[h][j][1] = t2[h][j][0] = t2[h][j][1] = t3[h][j][0] = t3[h][j][1] = 0.0;
    }

    // stationary fragments sf/ss (all k), moving operand rows mv + mrow[j]
    template <int NTL, bool SA, class Epi>
    __device__ __forceinline__ void run_stat(const double2 (&sf)[KS], const double (&ss)[KS], const double2* mv,
                                             const int* mrow, const int* tm, const int* tn, Epi& epi) const {
        Acc t1, t2, t3;
        zero<NTL>(t1, t2, t3);
        if constexpr (kF4M) {  // t1: re, t2: im (ss = -Im of the stationary fragment)
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const int h = ks % kKP;
                double2 v[kTG];
#pragma unroll
                for (int j = 0; j < NTL; ++j) v[j] = mv[mrow[j] + ks * 4];
#pragma unroll
                for (int j = 0; j < NTL; ++j) {
                    if (SA) dmma(t1[h][j][0], t1[h][j][1], sf[ks].x, v[j].x);
                    else dmma(t1[h][j][0], t1[h][j][1], v[j].x, sf[ks].x);
                }
#pragma unroll
                for (int j = 0; j < NTL; ++j) {
                    if (SA) dmma(t2[h][j][0], t2[h][j][1], sf[ks].x, v[j].y);
                    else dmma(t2[h][j][0], t2[h][j][1], v[j].x, sf[ks].y);
                }
#pragma unroll
                for (int j = 0; j < NTL; ++j) {
                    if (SA) dmma(t1[h][j][0], t1[h][j][1], ss[ks], v[j].y);
                    else dmma(t1[h][j][0], t1[h][j][1], v[j].y, ss[ks]);
                }
#pragma unroll
                for (int j = 0; j < NTL; ++j) {
                    if (SA) dmma(t2[h][j][0], t2[h][j][1], sf[ks].y, v[j].x);
                    else dmma(t2[h][j][0], t2[h][j][1], v[j].y, sf[ks].x);
                }
            }
            const int r = lane >> 2, kq = lane & 3;
#pragma unroll
            for (int j = 0; j < NTL; ++j)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    double re = t1[0][j][i], im = t2[0][j][i];
#pragma unroll
                    for (int hh = 1; hh < kKP; ++hh) re += t1[hh][j][i], im += t2[hh][j][i];
                    epi(tm[j] * 8 + frow_perm(r), tn[j] * 8 + frow_perm(2 * kq + i), make_double2(re, im));
                }
            return;
        }
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const int h = ks % kKP;
            double2 v[kTG];
            double vs[kTG];
#pragma unroll
            for (int j = 0; j < NTL; ++j) {
                v[j] = mv[mrow[j] + ks * 4];
                vs[j] = v[j].x + v[j].y;
            }
#pragma unroll
            for (int j = 0; j < NTL; ++j) {
                if (SA || kSwapB) dmma(t1[h][j][0], t1[h][j][1], sf[ks].x, v[j].x);
                else dmma(t1[h][j][0], t1[h][j][1], v[j].x, sf[ks].x);
            }
#pragma unroll
            for (int j = 0; j < NTL; ++j) {
                if (SA || kSwapB) dmma(t2[h][j][0], t2[h][j][1], sf[ks].y, v[j].y);
                else dmma(t2[h][j][0], t2[h][j][1], v[j].y, sf[ks].y);
            }
#pragma unroll
            for (int j = 0; j < NTL; ++j) {
                if (SA || kSwapB) dmma(t3[h][j][0], t3[h][j][1], ss[ks], vs[j]);
                else dmma(t3[h][j][0], t3[h][j][1], vs[j], ss[ks]);
            }
        }
        finish<NTL, SA>(t1, t2, t3, tm, tn, epi);
    }

    // run_stat for the tile count nt <= N (compile-time tile counts)
    template <int N, class Epi>
    __device__ __forceinline__ void dispatch(int nt, const double2 (&sf)[KS], const double (&ss)[KS], const int* mrow,
                                             const int* tm, const int* tn, Epi& epi) const {
        if constexpr (N >= 1) {
            if (nt == N) {
                if (sa) run_stat<N, true>(sf, ss, dat, mrow, tm, tn, epi);
                else run_stat<N, false>(sf, ss, dat, mrow, tm, tn, epi);
            } else {
                dispatch<N - 1>(nt, sf, ss, mrow, tm, tn, epi);
            }
        }
    }

    // dispatch with the operand role a compile-time constant
    template <int N, bool SA, class Epi>
    __device__ __forceinline__ void dispatch_sa(int nt, const double2 (&sf)[KS], const double (&ss)[KS], const int* mrow,
                                                const int* tm, const int* tn, Epi& epi) const {
        if constexpr (N >= 1) {
            if (nt == N) run_stat<N, SA>(sf, ss, dat, mrow, tm, tn, epi);
            else dispatch_sa<N - 1, SA>(nt, sf, ss, mrow, tm, tn, epi);
        }
    }

    // full 8-row tiles ST of the factor on DMMA, the last FR <= 2 factor rows
    // on the CUDA cores (a padded tile would be 7/8 or 6/8 zeros); likewise the
    // last DR <= 2 data rows (HTG_FDM_DR, default on: 50 = 6 x 8 + 2 data rows
    // of a two-subdomain batch at p = 4)
    template <class Epi>
    __device__ __forceinline__ void operator()(Epi&& epi) const {
        const int r = lane >> 2, kq = lane & 3;
        const int FR = (F & 7) <= 2 ? (F & 7) : 0;
        const int DR = kDataRem && (nd & 7) <= 2 ? (nd & 7) : 0;
        const int ST = (F - FR + 7) >> 3, OT = (nd - DR + 7) >> 3;
        const int FT = F - FR, n1 = FR * nd, n2 = DR * FT;
        // warp q: stationary tiles st0, st0 + sstep, ..; moving tiles [o_lo, o_hi);
        // remainder items [i_lo, i_hi) of the n1 + n2 dot products
        int st0 = q, sstep = 4, o_lo = 0, o_hi = OT, nrem = n1 + n2, i_lo = 0, i_hi = 0;
        if (ST == 3) {
            if (q == 3) st0 = ST, i_hi = nrem;
        } else if (ST == 2) {
            const int h = (OT + 1) >> 1;
            st0 = q & 1;
            sstep = 2;
            o_lo = (q >> 1) ? h : 0;
            o_hi = (q >> 1) ? OT : h;
            if (q >= 2) i_lo = (q - 2) * nrem / 2, i_hi = (q - 1) * nrem / 2;
        } else if (ST == 1) {
            st0 = 0;
            sstep = 1 << 30;
            o_lo = q * OT / 4;
            o_hi = (q + 1) * OT / 4;
            i_lo = q * nrem / 4, i_hi = (q + 1) * nrem / 4;
        } else {
            i_lo = q * nrem / 4, i_hi = (q + 1) * nrem / 4;
        }
        const int flim = FT - 1, dlim = nd - DR - 1;
        for (int st = st0; st < ST; st += sstep) {
            double2 sf[KS];
            double ss[KS];
            const int frow = min(st * 8 + frow_perm(r), flim);
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                sf[ks] = fval(frow, ks * 4 + kq);
                ss[ks] = stat_aux(sf[ks]);
            }
            for (int o0 = o_lo; o0 < o_hi; o0 += kTG) {
                const int nt = min(kTG, o_hi - o0);
                int mrow[kTG], tm[kTG], tn[kTG];
#pragma unroll
                for (int j = 0; j < kTG; ++j) {
                    mrow[j] = min((o0 + j) * 8 + frow_perm(r), dlim) * LD + kq;
                    tm[j] = sa ? st : o0 + j;
                    tn[j] = sa ? o0 + j : st;
                }
                dispatch<kTG>(nt, sf, ss, mrow, tm, tn, epi);
            }
        }
        // remainder: one complex dot product of a factor row and a data row per
        // lane; k is xor-skewed by the data row so 8 lanes hit distinct banks
        for (int it = i_lo + lane; it < i_hi; it += 32) {
            int f, d;
            if (it < n1) {
                const int a = it / nd;
                f = FT + a;
                d = it - a * nd;
            } else {
                const int j = it - n1, a = j / FT;
                d = nd - DR + a;
                f = j - a * FT;
            }
            const double2* dr = dat + d * LD;
            const int sk = kSkew ? ((lane >> 1) & 3) : 0;  // consecutive lanes: consecutive rows
            // 8 independent accumulator chains (4 terms x k parity): the dot is
            // DFMA-latency bound otherwise
            double acc[2][4] = {};
#pragma unroll
            for (int kk = 0; kk < 4 * KS; ++kk) {
                const double2 a = fval(f, kk ^ sk), b = dr[kk ^ sk];
                double* c = acc[kk & 1];
                c[0] = fma(a.x, b.x, c[0]);
                c[1] = fma(a.y, b.y, c[1]);
                c[2] = fma(a.x, b.y, c[2]);
                c[3] = fma(a.y, b.x, c[3]);
            }
            const double re = (acc[0][0] + acc[1][0]) - (acc[0][1] + acc[1][1]);
            const double im = (acc[0][2] + acc[1][2]) + (acc[0][3] + acc[1][3]);
            if (sa) epi(f, d, make_double2(re, im));
            else epi(d, f, make_double2(re, im));
        }
    }
};

template <int P>
__global__ void __launch_bounds__(kFThreads, 1) k_dd_fdm(FineGeom g, const FdmClassDev* __restrict__ classes,
                                                         const int4* __restrict__ work, const double2* __restrict__ r,
                                                         double2* __restrict__ ystage, int nu_max, int rows,
                                                         int fac_elems) {
    constexpr int LD = FdmDims<P>::LD, KS = FdmDims<P>::KS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* fac = reinterpret_cast<double2*>(smem_raw);
    const int tid = threadIdx.x;
    const int grp = tid >> 7, gt = tid & 127, lane = tid & 31;
    // role of this warp inside its group, rotated by group: warp q of every group
    // runs on SM sub-partition q, so the rotation spreads the CUDA-core remainder
    // rows (one role) over the four sub-partitions' FP64 pipes
    const int q = ((gt >> 5) + grp) & 3;
    double2* X = fac + fac_elems + size_t(grp) * 2 * rows * LD;  // gathered tile, then Q o Dinv
    double2* W = X + rows * LD;                                  // stage 1 / stage 3 products
    {  // the k padding of the data buffers must be finite: zero them once
        double2* data = fac + fac_elems;
        for (int i = tid; i < kFGroups * 2 * rows * LD; i += kFThreads) data[i] = make_double2(0.0, 0.0);
    }
#ifdef HTG_FDM_CLOCKS
    long long clk_acc[6] = {0, 0, 0, 0, 0, 0}, clk_prev = 0;
#define HTG_CLK(i)                                  \
    do {                                            \
        const long long t_ = clock64();             \
        if (i > 0) clk_acc[i - 1] += t_ - clk_prev; \
        clk_prev = t_;                              \
    } while (0)
#else
#define HTG_CLK(i) \
    do {           \
    } while (0)
#endif
    const int4 wk = work[blockIdx.x];  // [first, end) of the class-sorted subdomain list
    int pos = wk.x;
    while (pos < wk.y) {
        int ci = 0;
        while (classes[ci].first + classes[ci].nsub <= pos) ++ci;
        const FdmClassDev c = classes[ci];
        const int seg_end = min(wk.y, c.first + c.nsub);
        const int nx = c.nx, ny = c.ny, nux = c.nux, nuy = c.nuy;
        constexpr int KP = 4 * KS;
        double2* V1T = fac;            // [ix'][ix] = Vx[ix][ix'], KP rows (rows >= nx zero); the U-row
        double2* V2T = V1T + KP * LD;  // factor Vx[ux0 + ixu][ix'] of stage 3 is V1T[ix'][ux0 + ixu]
        double2* D = V2T + KP * LD;    // Dinv[ix'][iy']
        __syncthreads();  // previous segment finished with the factors
        const double2 z = make_double2(0.0, 0.0);
        for (int i = tid; i < 2 * KP * LD; i += kFThreads) {
            const int a = i / LD, b = i - a * LD;
            double2 v = z;
            if (a < KP) v = (a < nx && b < nx) ? c.Vx[b * nx + a] : z;
            else v = (a - KP < ny && b < ny) ? c.Vy[b * ny + (a - KP)] : z;
            fac[i] = v;
        }
        for (int i = tid; i < nx * ny; i += kFThreads) D[i] = c.Dinv[i];
        // U row of each (ixu, iyu) of U, and the class's relative gather offsets
        int* urow = reinterpret_cast<int*>(D + nx * ny) + kFGroups * 32;
        for (int i = tid; i < nux * nuy; i += kFThreads) {
            const int ixu = i / nuy, iyu = i - ixu * nuy;
            urow[i] = c.rowmap[dof_index(c.onx, c.ony, P, c.ux0 + ixu, c.uy0 + iyu)];
        }
        int* gofs = urow + nux * nuy;
        if (c.goff)
            for (int i = tid; i < nx * ny; i += kFThreads) gofs[i] = c.goff[i];
        __syncthreads();
        const int S = min(8, rows / max(nx, ny));  // subdomains per batch
        const int nxy = nx * ny;
        const float inv_nx = 1.0f / nx, inv_ny = 1.0f / ny, inv_nux = 1.0f / nux;
        // subdomain ids and origins of the group's batches, double-buffered by batch
        // parity: the next batch's are loaded into registers under stages 1-3 and
        // published before the stage-3 barrier, its tile is gathered under stage 4
        // while stage 4 of the current batch still stores with the current ids
        int* meta = reinterpret_cast<int*>(D + nx * ny) + grp * 32;  // [parity][sid 8 | origin 8]
        int* sid = meta;  // sid[parity * 16 + s]
        int par = 0;
        auto gather = [&](int nb, int pr) {
            // roles 2 and 3 issue the gather (roles 0 and 1 carry the larger share
            // of stage 4's DMMA tiles; measured 0.216 -> 0.211 ms at cfg4)
            if (q < 2) {
                asm volatile("cp.async.commit_group;\n" ::: "memory");
                return;
            }
            const int gt = (q - 2) * 32 + lane;
            constexpr int kGS = 64;
            for (int s = 0; s < nb; ++s) {
                const int so = meta[pr * 16 + 8 + s];
                const int ox = (so & 0xffff) * P, oy = (so >> 16) * P;
                double2* xs = X + s * ny * LD;
                if (c.goff) {
                    const double2* rb = r + dof_index(g.nx, g.ny, P, ox, oy);
                    for (int l = gt; l < nxy; l += kGS) {
                        const int iy = fdiv(l, inv_nx), ix = l - iy * nx;
                        cp_async16(&xs[iy * LD + ix], rb + gofs[l]);
                    }
                } else {
                    for (int l = gt; l < nxy; l += kGS) {
                        const int iy = fdiv(l, inv_nx), ix = l - iy * nx;
                        cp_async16(&xs[iy * LD + ix], r + dof_index(g.nx, g.ny, P, ox + ix, oy + iy));
                    }
                }
            }
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        };
        // this group's batches of the segment: full rounds of S subdomains per
        // group, then the remainder (< groups x S) split evenly, so the groups of
        // a CTA finish within one subdomain of each other
        const int nseg = seg_end - pos, R = nseg / (kFGroups * S), rem = nseg - R * kFGroups * S;
        const int tail_n = rem / kFGroups + (grp < rem % kFGroups ? 1 : 0);
        const int tail_b = pos + R * kFGroups * S + grp * (rem / kFGroups) + min(grp, rem % kFGroups);
        const int nbatch = R + (tail_n > 0 ? 1 : 0);
        auto bstart = [&](int i) { return i < R ? pos + (i * kFGroups + grp) * S : tail_b; };
        auto bsize = [&](int i) { return i < R ? S : tail_n; };
        if (nbatch > 0) {
            if (gt < bsize(0)) {
                const int id = c.subs[bstart(0) - c.first + gt];
                meta[gt] = id;
                meta[8 + gt] = c.sub_o[id];
            }
            group_sync(grp);
            gather(bsize(0), 0);
        }
        for (int bi = 0; bi < nbatch; ++bi, par ^= 1) {
            const int nb = bsize(bi);
            HTG_CLK(0);
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            group_sync(grp);
            HTG_CLK(1);
            int nid = -1, nso = 0;  // next batch, one subdomain per lane gt < its size
            if (bi + 1 < nbatch && gt < bsize(bi + 1)) {
                nid = c.subs[bstart(bi + 1) - c.first + gt];
                nso = c.sub_o[nid];
            }
            // 1: P[ix'][(s,iy)] = sum_ix Vx[ix][ix'] G_s[ix][iy]  -> W[(s,ix')][iy]
            Stage<LD, KS>{V1T, nx, X, nb * ny, true, q, lane}([&](int m, int n, double2 v) {
                if (m < nx && n < nb * ny) {
                    const int s = fdiv(n, inv_ny);
                    W[(s * nx + m) * LD + n - s * ny] = v;
                }
            });
            group_sync(grp);
            HTG_CLK(2);
            // 2: Q[(s,ix')][iy'] = (sum_iy P[(s,ix')][iy] Vy[iy][iy']) Dinv[ix'][iy']  -> X[(s,iy')][ix']
            Stage<LD, KS>{V2T, ny, W, nb * nx, false, q, lane}([&](int m, int n, double2 v) {
                if (m < nb * nx && n < ny) {
                    const int s = fdiv(m, inv_nx), ix = m - s * nx;
                    const double2 d = D[ix * ny + n];
                    X[(s * ny + n) * LD + ix] = make_double2(v.x * d.x - v.y * d.y, v.x * d.y + v.y * d.x);
                }
            });
            group_sync(grp);
            HTG_CLK(3);
            // 3: R[ixu][(s,iy')] = sum_ix' Vx[ux0 + ixu][ix'] Q[(s,iy')][ix']  -> W[(s,ixu)][iy']
            Stage<LD, KS, true>{V1T, nux, X, nb * ny, true, q, lane, c.ux0}([&](int m, int n, double2 v) {
                if (m < nux && n < nb * ny) {
                    const int s = fdiv(n, inv_ny);
                    W[(s * nux + m) * LD + n - s * ny] = v;
                }
            });
            if (nid >= 0) {
                meta[(par ^ 1) * 16 + gt] = nid;
                meta[(par ^ 1) * 16 + 8 + gt] = nso;
            }
            group_sync(grp);
            HTG_CLK(4);
            // the gathered tile is free: fetch the group's next batch under stage 4
            if (bi + 1 < nbatch) gather(bsize(bi + 1), par ^ 1);
            HTG_CLK(5);
            // 4: Y[(s,ixu)][iyu] = sum_iy' R[(s,ixu)][iy'] Vy[uy0 + iyu][iy']  -> staging rows
            Stage<LD, KS, true>{V2T, nuy, W, nb * nux, false, q, lane, c.uy0}(
                [&](int m, int n, double2 v) {
                    if (m < nb * nux && n < nuy) {
                        const int s = fdiv(m, inv_nux), ixu = m - s * nux;
                        ystage[(size_t)sid[par * 16 + s] * nu_max + urow[ixu * nuy + n]] = v;
                    }
                });
            // (no barrier here: the next batch's first barrier also orders this
            // stage's reads of W before that batch's stage-1 writes)
            HTG_CLK(6);
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        pos = seg_end;
    }
#ifdef HTG_FDM_CLOCKS
    if (lane == 0 && blockIdx.x < 2)
        printf("fdm clk cta %d grp %d role %d: top %lld s1 %lld s2 %lld s3 %lld gather %lld s4 %lld\n", blockIdx.x, grp,
               q, clk_acc[0], clk_acc[1], clk_acc[2], clk_acc[3], clk_acc[4], clk_acc[5]);
#endif
}

template <int P>
int fdm_rows(int fac_elems) {
    return (kSmemMax / int(sizeof(double2)) - fac_elems) / (kFGroups * 2 * FdmDims<P>::LD);
}

// ---------------------------------------------------------------- team per subdomain
// A team of NP warps (NP = 1 or 2) runs all four products of one subdomain,
// synchronised only by a team barrier between stages, so the DMMA pipe of an
// SM sub-partition is fed by independent teams instead of 4-warp groups
// waiting on each other's stage tails. The tiles of a product are split
// evenly over the team (the odd tile alternates between the warps from stage
// to stage); factor rows 8t + FR and data rows 8t + DR with FR, DR <= 2 run
// their last rows as DFMA dot products spread over the team's lanes (25 = 3 x
// 8 + 1 and 17 = 2 x 8 + 1 at p = 4: 588 DMMAs per subdomain against 693 for
// the batched 4-warp form). The U-row factors of stages 3 and 4 are read
// transposed out of Vx^T, Vy^T (their rows are columns there), which leaves
// shared memory for 8 teams of two 25-row buffers each at p = 4.
#ifndef HTG_FDM_TGW
#define HTG_FDM_TGW 1  // cfg4 (with HTG_FDM_SWAPB): 1 tile 172.7 us, 2 tiles 176.6, 3 tiles 181.9
#endif
constexpr int kTGW = HTG_FDM_TGW < kTG ? HTG_FDM_TGW : kTG;  // moving tiles in flight (team kernel)
#ifndef HTG_FDM_PADF
#define HTG_FDM_PADF 0
#endif
#ifndef HTG_FDM_PADD
#define HTG_FDM_PADD 0
#endif
constexpr bool kPadF = HTG_FDM_PADF != 0, kPadD = HTG_FDM_PADD != 0;

#ifndef HTG_FDM_DOT_UNROLL
#define HTG_FDM_DOT_UNROLL 28
#endif
constexpr int kDotUnroll = HTG_FDM_DOT_UNROLL;  // unrolling of the remainder dot products (code size)

// (the operand role as a template argument halves the product bodies per call site
// but measured slower: 196.3 vs 185.8 us at cfg4)
template <int LD, int KS, bool FTR>
struct WStage {
    const double2* fac;  // FTR: factor row f, k at fac[k * LD + fo + f]; else fac[f * LD + k]
    int F, fo;
    const double2* dat;  // data rows [0, nd), [row][k]
    int nd;
    bool sa;             // C[factor][data] (else C[data][factor])
    int lane;
    int part, np;        // this warp's share of the team's tiles and dot products

    __device__ __forceinline__ double2 fval(int f, int k) const {
        return FTR ? fac[k * LD + fo + f] : fac[f * LD + k];
    }

    template <class Epi>
    __device__ __forceinline__ void operator()(Epi&& epi) const {
        const Stage<LD, KS> b{fac, F, dat, nd, sa, 0, lane};
        const int r = lane >> 2, kq = lane & 3;
        // remainder rows of 8t + 1 / 8t + 2 extents run as DFMA dots unless padded
        // into a tile (HTG_FDM_PADF / HTG_FDM_PADD: padded rows repeat the last row,
        // so their fragment loads are broadcasts, and their outputs are dropped)
        const int FR = (!kPadF && (F & 7) <= 2) ? (F & 7) : 0, DR = (!kPadD && (nd & 7) <= 2) ? (nd & 7) : 0;
        const int ST = (F - FR + 7) >> 3, OT = (nd - DR + 7) >> 3;
        const int flim = F - FR - 1, dlim = nd - DR - 1;
        // tiles (st, ot) flattened st-major; this warp takes [t0, t1)
        const int T = ST * OT, t0 = T * part / np, t1 = T * (part + 1) / np;
        for (int t = t0; t < t1;) {
            const int st = t / OT, o_lo = t - st * OT, o_hi = min(OT, o_lo + (t1 - t));
            double2 sf[KS];
            double ss[KS];
            const int fr = min(st * 8 + frow_perm(r), flim);
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                sf[ks] = fval(fr, ks * 4 + kq);
                ss[ks] = stat_aux(sf[ks]);
            }
            for (int o0 = o_lo; o0 < o_hi; o0 += kTGW) {
                const int nt = min(kTGW, o_hi - o0);
                int mrow[kTG], tm[kTG], tn[kTG];
#pragma unroll
                for (int j = 0; j < kTG; ++j) {
                    mrow[j] = min((o0 + j) * 8 + frow_perm(r), dlim) * LD + kq;
                    tm[j] = sa ? st : o0 + j;
                    tn[j] = sa ? o0 + j : st;
                }
                b.template dispatch<kTGW>(nt, sf, ss, mrow, tm, tn, epi);
            }
            t += o_hi - o_lo;
        }
        // remainder rows: factor rows [F - FR, F) x all data rows, then data rows
        // [nd - DR, nd) x the tiled factor rows; one complex dot per lane
        const int FT = F - FR, n1 = FR * nd, n2 = DR * FT;
        for (int it = part * 32 + lane; it < n1 + n2; it += np * 32) {
            int f, d;
            if (it < n1) {
                const int a = it / nd;
                f = FT + a;
                d = it - a * nd;
            } else {
                const int j = it - n1, a = j / FT;
                d = nd - DR + a;
                f = j - a * FT;
            }
            const double2* dr = dat + d * LD;
            const int sk = kSkew ? ((lane >> 1) & 3) : 0;  // consecutive lanes: consecutive rows
            double acc[2][4] = {};  // independent chains, as in Stage
#pragma unroll kDotUnroll
            for (int kk = 0; kk < 4 * KS; ++kk) {
                const double2 a = fval(f, kk ^ sk), bb = dr[kk ^ sk];
                double* c = acc[kk & 1];
                c[0] = fma(a.x, bb.x, c[0]);
                c[1] = fma(a.y, bb.y, c[1]);
                c[2] = fma(a.x, bb.y, c[2]);
                c[3] = fma(a.y, bb.x, c[3]);
            }
            const double re = (acc[0][0] + acc[1][0]) - (acc[0][1] + acc[1][1]);
            const double im = (acc[0][2] + acc[1][2]) + (acc[0][3] + acc[1][3]);
            if (sa) epi(f, d, make_double2(re, im));
            else epi(d, f, make_double2(re, im));
        }
    }
};

// WStage with every extent a compile-time constant (the interior class of a
// uniform medium: 96% of the subdomains at cfg4): factor rows F and data rows ND
// of the form 8 t + 1 (full tiles only: no clamps, no output guards), contraction
// length K, this warp's share PART of NP. After unrolling, the tile list of a warp
// is straight-line code whose shared-memory addresses are a per-lane base plus
// immediates, which frees the registers and integer work of the generic path.
template <int N>
struct IntC {
    static constexpr int value = N;
};
template <int NP, class Fn>
__device__ __forceinline__ void for_part(int part, Fn&& fn) {
    if constexpr (NP == 1) {
        fn(IntC<0>{});
    } else if constexpr (NP == 2) {
        if (part == 0) fn(IntC<0>{});
        else fn(IntC<1>{});
    } else if constexpr (NP == 3) {
        if (part == 0) fn(IntC<0>{});
        else if (part == 1) fn(IntC<1>{});
        else fn(IntC<2>{});
    } else {
        if (part == 0) fn(IntC<0>{});
        else if (part == 1) fn(IntC<1>{});
        else if (part == 2) fn(IntC<2>{});
        else fn(IntC<3>{});
    }
}

// Merged last round (teams join on the R < nteam subdomains left): measured without
// gain (cfg3 59.5 vs 59.0 us, cfg4 175.6 vs 172.6): a team's subdomain takes ~19,000
// cycles alone and ~44,000 beside seven others, the merged round ~10,000 plus an
// unprefetched gather, and the extra code slows the main rounds.
#ifndef HTG_FDM_MERGE
#define HTG_FDM_MERGE 0
#endif
constexpr bool kFdmMerge = HTG_FDM_MERGE != 0;
#ifndef HTG_FDM_DOTBAL
#define HTG_FDM_DOTBAL 1
#endif
template <int LD, int KS, bool FTR, int F, int ND, int K, bool SA, int NP>
struct CStage {
    const double2* fac;  // FTR: factor row f, k at fac[k * LD + fo + f]; else fac[f * LD + k]
    int fo;
    const double2* dat;  // data rows [0, ND), [row][k]
    int lane;

    __device__ __forceinline__ double2 fval(int f, int k) const {
        return FTR ? fac[k * LD + fo + f] : fac[f * LD + k];
    }

    // Lean form for the 24-warp CTA (eight 3-warp teams, 80 registers): one tile at a
    // time, the factor fragment re-read from shared memory at every k step instead of
    // held in 42 registers across the tiles of a factor tile.
    template <bool RSV, int PART, class Epi>
    __device__ __forceinline__ void go(Epi&& epi) const {
        if constexpr (RSV) run_rs<PART>(epi);
        else run<PART>(epi);
    }
    template <int PART, class Epi>
    __device__ __forceinline__ void run_rs(Epi&& epi) const {
        constexpr int FR = F & 7, DR = ND & 7, FT = F - FR, DT = ND - DR;
        constexpr int ST = FT / 8, OT = DT / 8, T = ST * OT, t0 = T * PART / NP, t1 = T * (PART + 1) / NP;
        const int r = lane >> 2, kq = lane & 3, pr = frow_perm(r);
        const double2* sp0 = FTR ? fac + kq * LD + fo + pr : fac + pr * LD + kq;
        const double2* mp0 = dat + pr * LD + kq;
        constexpr int SSTEP = FTR ? 4 * LD : 4, STILE = FTR ? 8 : 8 * LD;
#pragma unroll
        for (int t = t0; t < t1; ++t) {
            const int st = t / OT, o = t - st * OT;
            const double2* sp = sp0 + st * STILE;
            const double2* mp = mp0 + o * 8 * LD;
            double a1[2] = {0.0, 0.0}, a2[2] = {0.0, 0.0}, a3[2] = {0.0, 0.0};
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const double2 sv = sp[ks * SSTEP], v = mp[ks * 4];
                dmma(a1[0], a1[1], sv.x, v.x);
                dmma(a2[0], a2[1], sv.y, v.y);
                dmma(a3[0], a3[1], sv.x + sv.y, v.x + v.y);
            }
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int f = st * 8 + pr, d = o * 8 + frow_perm(2 * kq + i);
                const double2 val = make_double2(a1[i] - a2[i], a3[i] - a1[i] - a2[i]);
                if (SA) epi(f, d, val);
                else epi(d, f, val);
            }
        }
        dots<PART, T, t0, t1>(epi);
    }

    template <int PART, class Epi>
    __device__ __forceinline__ void run(Epi&& epi) const {
        constexpr int FR = F & 7, DR = ND & 7, FT = F - FR, DT = ND - DR;
        static_assert(FR <= 2 && DR <= 2 && K <= 4 * KS, "CStage: extents 8 t + {0, 1, 2}");
        constexpr int ST = FT / 8, OT = DT / 8, T = ST * OT, t0 = T * PART / NP, t1 = T * (PART + 1) / NP;
        const Stage<LD, KS> b{fac, F, dat, ND, SA, 0, lane};
        const int r = lane >> 2, kq = lane & 3;
        const int pr = frow_perm(r);
#pragma unroll
        for (int st = 0; st < ST; ++st) {
            const int lo = t0 - st * OT > 0 ? t0 - st * OT : 0, hi = t1 - st * OT < OT ? t1 - st * OT : OT;
            if (lo < hi) {
                double2 sf[KS];
                double ss[KS];
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    sf[ks] = fval(st * 8 + pr, ks * 4 + kq);
                    ss[ks] = stat_aux(sf[ks]);
                }
#pragma unroll
                for (int o0 = lo; o0 < hi; o0 += kTGW) {
                    const int nt = hi - o0 < kTGW ? hi - o0 : kTGW;
                    int mrow[kTG], tm[kTG], tn[kTG];
#pragma unroll
                    for (int j = 0; j < kTG; ++j) {
                        mrow[j] = ((o0 + j) * 8 + pr) * LD + kq;
                        tm[j] = SA ? st : o0 + j;
                        tn[j] = SA ? o0 + j : st;
                    }
                    b.template dispatch<kTGW>(nt, sf, ss, mrow, tm, tn, epi);
                }
            }
        }
        dots<PART, T, t0, t1>(epi);
    }

    template <int PART, int T, int t0, int t1, class Epi>
    __device__ __forceinline__ void dots(Epi&& epi) const {
        constexpr int FR = F & 7, DR = ND & 7, FT = F - FR, DT = ND - DR;
        // remainder rows: factor rows [FT, F) x all data rows, then data rows [DT, ND) x
        // the tiled factor rows; one complex dot of length K per lane
        // With two warps and an odd tile count (9 = 4 + 5) the warp with fewer tiles takes
        // every dot product (a pass of 32 dots costs about 0.6 tiles of FP64 pipe time).
        constexpr int n1 = FR * ND, n2 = DR * FT;
        constexpr bool kUneven = HTG_FDM_DOTBAL && NP == 2 && (T & 1);
        constexpr bool kLight = (t1 - t0) * 2 < T;
        constexpr int it_first = kUneven ? (kLight ? 0 : n1 + n2) : PART * 32, it_step = kUneven ? 32 : NP * 32;
#pragma unroll
        for (int it0 = it_first; it0 < n1 + n2; it0 += it_step) {
            const int it = it0 + lane;
            if (it < n1 + n2) {
                int f, d;
                if (it < n1) {
                    const int a = it / ND;
                    f = FT + a;
                    d = it - a * ND;
                } else {
                    const int j = it - n1, a = j / FT;
                    d = DT + a;
                    f = j - a * FT;
                }
                const double2* dr = dat + d * LD;
                double acc[2][4] = {};
#pragma unroll
                for (int kk = 0; kk < K; ++kk) {
                    const double2 a = fval(f, kk), bb = dr[kk];
                    double* c = acc[kk & 1];
                    c[0] = fma(a.x, bb.x, c[0]);
                    c[1] = fma(a.y, bb.y, c[1]);
                    c[2] = fma(a.x, bb.y, c[2]);
                    c[3] = fma(a.y, bb.x, c[3]);
                }
                const double re = (acc[0][0] + acc[1][0]) - (acc[0][1] + acc[1][1]);
                const double im = (acc[0][2] + acc[1][2]) + (acc[0][3] + acc[1][3]);
                if (SA) epi(f, d, make_double2(re, im));
                else epi(d, f, make_double2(re, im));
            }
        }
    }
};

// CTA size the kernel is compiled for: NP = 1 at p = 4 runs 8 warps (shared
// memory holds 8 buffer pairs), so the register budget is the full 255 per thread
#ifndef HTG_FDM_TTHREADS
#define HTG_FDM_TTHREADS 512
#endif
// CTA sizes the team kernel is instantiated for, per team size (the launch picks the
// smallest one that holds the planned warps; the register budget follows the size)
constexpr int kWSizes[5][2] = {{0, 0}, {256, 512}, {384, 512}, {480, 576}, {512, 512}};
constexpr int kWLean = 768;  // eight 3-warp teams, 80 registers (CStage::run_rs)

#ifndef HTG_FDM_TEAM4_BELOW
#define HTG_FDM_TEAM4_BELOW 40
#endif
constexpr int kFdmTeam4Below = HTG_FDM_TEAM4_BELOW;  // subdomains per SM below which teams are 4 warps

template <int NP>
__device__ __forceinline__ void team_sync(int team) {
    if constexpr (NP == 1) __syncwarp();
    else asm volatile("bar.sync %0, %1;\n" ::"r"(team + 1), "r"(NP * 32) : "memory");
}

// One class's factor region in the layout the team kernel keeps in shared memory
// (generic: Vx^T, Vy^T; mirror-symmetric classes: the parity blocks and mirror tables).
template <int P>
__global__ void __launch_bounds__(256) k_fdm_format(const FdmClassDev* __restrict__ classes, double2* __restrict__ image,
                                                   int2* __restrict__ pos_tab, int fac_elems) {
    constexpr int LD = FdmDims<P>::LD, KS = FdmDims<P>::KS, KP = 4 * KS;
    const FdmClassDev c = classes[blockIdx.x];
    double2* fac = image + size_t(blockIdx.x) * fac_elems;
    const int tid = threadIdx.x, nthr = blockDim.x;
    double2* V1T = fac;
    double2* V2T = V1T + KP * LD;
    double2* D = V2T + KP * LD;
    const int nx = c.nx, ny = c.ny, nux = c.nux, nuy = c.nuy;
    int* urow = reinterpret_cast<int*>(D + nx * ny);
    int* gofs = urow + nux * nuy;
    int* gpos = gofs + nx * ny;
    (void)V1T;
    const double2 z = make_double2(0.0, 0.0);
    const bool sym = HTG_FDM_SYM_CODE && (P == 4) && c.sym;
    // mirror tables of a symmetric class (after the gather tables):
    // bfn[r]: natural rows of reordered row r; ubn[n]: reordered rows of natural row n
    int* bfn = gpos + nx * ny;
    int* ubn = bfn + 32;
    if (sym) {
        // V1T: rows [0, 16) Ve^T (13 x 13), rows [16, 28) Vo^T (12 x 12); same for V2T
        for (int i = tid; i < 2 * KP * LD; i += nthr) {
            const int a0 = i / LD, b = i - a0 * LD, dir = a0 / KP, a = a0 - dir * KP;
            const double2* Ve = dir ? c.Vye : c.Vxe;
            const double2* Vo = dir ? c.Vyo : c.Vxo;
            double2 v = z;
            if (a < 16) v = (a < 13 && b < 13) ? Ve[b * 13 + a] : z;
            else v = (a - 16 < 12 && b < 12) ? Vo[b * 12 + (a - 16)] : z;
            fac[i] = v;
        }
        if (tid < 25) {
            // reordered r -> natural: r < 12 pair g = r (n1 = g, n2 = R(g), +s); r = 12 centre;
            // r >= 13 odd pair g = r - 13 (-s). packed n1 | n2 << 8 | sign bit << 16 (bit set: -)
            const int r = tid;
            int code;
            if (r == 12) code = 12 | (255 << 8);
            else {
                const int gg = r < 12 ? r : r - 13, m = c.mir[gg];
                const bool spos = (m >> 16) & 1;
                const bool neg = r < 12 ? !spos : spos;
                code = gg | ((m & 0xffff) << 8) | (neg ? 1 << 16 : 0);
            }
            bfn[r] = code;
            // natural n -> (pair g, form): n < 12: (e_g + o_g)/r2; n = 12: e_c; n > 12:
            // s_g (e_g - o_g)/r2 with R(g) = n. packed g | form << 8 (0 plus, 1 centre, 2 s>0, 3 s<0)
            const int n = tid;
            int ucode = 12 | (1 << 8);
            if (n < 12) ucode = n;
            else if (n > 12)
                for (int gg = 0; gg < 12; ++gg)
                    if ((c.mir[gg] & 0xffff) == n) ucode = gg | ((((c.mir[gg] >> 16) & 1) ? 2 : 3) << 8);
            ubn[n] = ucode;
        }
    } else {
        for (int i = tid; i < 2 * KP * LD; i += nthr) {
            const int a = i / LD, b = i - a * LD;
            double2 v = z;
            if (a < KP) v = (a < nx && b < nx) ? c.Vx[b * nx + a] : z;
            else v = (a - KP < ny && b < ny) ? c.Vy[b * ny + (a - KP)] : z;
            fac[i] = v;
        }
    }
    for (int i = tid; i < nx * ny; i += nthr) D[i] = c.Dinv[i];
    for (int i = tid; i < nux * nuy; i += nthr) {
        const int ixu = i / nuy, iyu = i - ixu * nuy;
        urow[i] = c.rowmap[dof_index(c.onx, c.ony, P, c.ux0 + ixu, c.uy0 + iyu)];
    }
    if (c.goff)
        for (int i = tid; i < nx * ny; i += nthr) {
            const int e = c.gord[i], iy = e / nx;
            gofs[i] = c.goff[e];
            gpos[i] = iy * LD + (e - iy * nx);
        }
    for (int j = tid; j < c.nsub; j += nthr) {
        const int id = c.subs[j];
        pos_tab[c.first + j] = make_int2(id, c.sub_o[id]);
    }
}

// HTG_FDM_TRACE: per-team clock64 accounting of the generic path (CTAs 0 and 1 print)
#ifdef HTG_FDM_TRACE
#define HTG_TR(i)                                  \
    do {                                           \
        const long long t_ = clock64();            \
        tr_acc[i] += t_ - tr_last;                 \
        tr_last = t_;                              \
    } while (0)
#else
#define HTG_TR(i) \
    do {          \
    } while (0)
#endif

template <int P, int NP, int NT>
__global__ void __launch_bounds__(NT, 1)
    k_dd_fdm_w(FineGeom g, const FdmClassDev* __restrict__ classes, const int4* __restrict__ work,
               const __grid_constant__ FdmWorkTab wtab, const double2* __restrict__ image,
               const int2* __restrict__ pos_tab, const double2* __restrict__ r, double2* __restrict__ ystage, int nu_max,
               int rows, int fac_elems) {
    constexpr int LD = FdmDims<P>::LD, KS = FdmDims<P>::KS, KP = 4 * KS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* fac = reinterpret_cast<double2*>(smem_raw);
    const int tid = threadIdx.x, nthr = blockDim.x, nteam = nthr / (32 * NP);
    const int warp = tid >> 5, lane = tid & 31, team = warp / NP, part = warp - team * NP;
    const int tl = part * 32 + lane;                               // lane within the team
#ifdef HTG_FDM_TRACE
    long long tr_acc[8] = {}, tr_last = clock64();
    const long long tr_t0 = tr_last;
    int tr_n = 0;
#endif
    double2* X = fac + fac_elems + size_t(team) * 2 * rows * LD;  // gathered tile, then Q o Dinv
    double2* W = X + rows * LD;                                   // stage 1 / stage 3 products
    double2* V1T = fac;            // [ix'][ix] = Vx[ix][ix'], KP rows (rows >= nx zero)
    double2* V2T = V1T + KP * LD;  // [iy'][iy] = Vy[iy][iy']
    double2* D = V2T + KP * LD;    // Dinv[ix'][iy']
    // [first, end) of the class-sorted list, class of first (parameter copy unless the table is too long)
    const int4 wk = work ? work[blockIdx.x] : wtab.w[blockIdx.x];
    int pos = wk.x, ci = wk.z;
    // the class's factor region (formatted once by k_fdm_format) -> shared memory, asynchronously
    auto copy_image = [&](int cls) {
        const double2* src = image + size_t(cls) * fac_elems;
        for (int i = tid; i < fac_elems; i += nthr) cp_async16(&fac[i], src + i);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    copy_image(ci);
    {  // the k padding of the data buffers must be finite: zero them once (under the copy)
        double2* data = fac + fac_elems;
        for (int i = tid; i < nteam * 2 * rows * LD; i += nthr) data[i] = make_double2(0.0, 0.0);
    }
    while (pos < wk.y) {
        const FdmClassDev c = classes[ci];  // holds pos (work table; ++ci at the segment's end)
        const int seg_end = min(wk.y, c.first + c.nsub);
        const int nx = c.nx, ny = c.ny, nux = c.nux, nuy = c.nuy;
        int* urow = reinterpret_cast<int*>(D + nx * ny);
        int* gofs = urow + nux * nuy;  // gather: dof offsets in memory order ...
        int* gpos = gofs + nx * ny;    // ... and the tile slot each one lands in
        const bool sym = HTG_FDM_SYM_CODE && (P == 4) && c.sym;
        // mirror tables of a symmetric class (after the gather tables):
        // bfn[r]: natural rows of reordered row r; ubn[n]: reordered rows of natural row n
        int* bfn = gpos + nx * ny;
        int* ubn = bfn + 32;
        // Last round of the CTA's last segment with R < nteam subdomains left: the teams
        // merge, g = nteam / R of them per subdomain (cfg3: 17 subdomains per SM are two
        // rounds of eight 2-warp teams and one subdomain solved by all 16 warps instead of
        // a third round run by one team), HTG_FDM_MERGE
        const int nseg = seg_end - pos, full = nseg / nteam * nteam, Rl = nseg - full;
        const int mg = (kFdmMerge && NP >= 2 && nteam <= 8 && !sym && Rl > 0 && seg_end == wk.y) ? nteam / Rl : 1;
        const bool merge = mg >= 2;
        const int main_end = merge ? pos + full : seg_end;  // subdomains of the team-per-subdomain rounds
        int cur = pos + team;
        int2 pt = cur < main_end ? pos_tab[cur] : make_int2(0, 0);  // (subdomain id, Omega origin)
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        const int nxy = nx * ny;
        const float inv_nx = 1.0f / nx;
        auto gather = [&](int so) {
            const int ox = (so & 0xffff) * P, oy = (so >> 16) * P;
            if (c.goff) {
                const double2* rb = r + dof_index(g.nx, g.ny, P, ox, oy);
                for (int l = tl; l < nxy; l += NP * 32) cp_async16(&X[gpos[l]], rb + gofs[l]);
            } else {
                for (int l = tl; l < nxy; l += NP * 32) {
                    const int iy = fdiv(l, inv_nx), ix = l - iy * nx;
                    cp_async16(&X[iy * LD + ix], r + dof_index(g.nx, g.ny, P, ox + ix, oy + iy));
                }
            }
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        };
        HTG_TR(0);  // segment setup (factor image)
        if (cur < main_end) gather(pt.y);
        if constexpr (P == 4) {
            if (sym) {
                constexpr double r2 = 0.70710678118654752440;
                for (; cur < main_end; cur += nteam) {
                    const int id = pt.x;
                    const bool more = cur + nteam < main_end;
                    if (more) pt = pos_tab[cur + nteam];
                    asm volatile("cp.async.wait_all;\n" ::: "memory");
                    team_sync<NP>(team);
                    // mirror butterflies in x and y: G[iy][ix] (natural) -> W[iy_r][ix_r]
                    for (int e = tl; e < 625; e += NP * 32) {
                        const int ry = e / 25, rx = e - ry * 25;
                        const int by = bfn[ry], bx = bfn[rx];
                        const int y1 = by & 255, y2 = (by >> 8) & 255, x1 = bx & 255, x2 = (bx >> 8) & 255;
                        const double cy2 = (by >> 16) ? -r2 : r2, cx2 = (bx >> 16) ? -r2 : r2;
                        const double cy1 = y2 == 255 ? 1.0 : r2, cx1 = x2 == 255 ? 1.0 : r2;
                        const double2 a = X[y1 * LD + x1];
                        double2 s = make_double2(cy1 * cx1 * a.x, cy1 * cx1 * a.y);
                        if (x2 != 255) {
                            const double2 b = X[y1 * LD + x2];
                            s.x = fma(cy1 * cx2, b.x, s.x);
                            s.y = fma(cy1 * cx2, b.y, s.y);
                        }
                        if (y2 != 255) {
                            const double2 b = X[y2 * LD + x1];
                            s.x = fma(cy2 * cx1, b.x, s.x);
                            s.y = fma(cy2 * cx1, b.y, s.y);
                            if (x2 != 255) {
                                const double2 d2 = X[y2 * LD + x2];
                                s.x = fma(cy2 * cx2, d2.x, s.x);
                                s.y = fma(cy2 * cx2, d2.y, s.y);
                            }
                        }
                        W[ry * LD + rx] = s;
                    }
                    team_sync<NP>(team);
                    // 1: per x-parity P_p[ix'][iy] = sum_{ix in p} V_p[ix][ix'] G[iy][ix] -> X[ix'_r][iy]
                    WStage<LD, 4, false>{V1T, 13, 0, W, 25, true, lane, part, NP}([&](int m, int n, double2 v) {
                        if (m < 13 && n < 25) X[m * LD + n] = v;
                    });
                    WStage<LD, 3, false>{V1T + 16 * LD, 12, 0, W + 13, 25, true, lane, NP - 1 - part, NP}(
                        [&](int m, int n, double2 v) {
                            if (m < 12 && n < 25) X[(m + 13) * LD + n] = v;
                        });
                    team_sync<NP>(team);
                    // 2: per y-parity, times Dinv -> W[iy'_r][ix'_r]
                    WStage<LD, 4, false>{V2T, 13, 0, X, 25, false, lane, part, NP}([&](int m, int n, double2 v) {
                        if (m < 25 && n < 13) {
                            const double2 d = D[m * 25 + n];
                            W[n * LD + m] = make_double2(v.x * d.x - v.y * d.y, v.x * d.y + v.y * d.x);
                        }
                    });
                    WStage<LD, 3, false>{V2T + 16 * LD, 12, 0, X + 13, 25, false, lane, NP - 1 - part, NP}(
                        [&](int m, int n, double2 v) {
                            if (m < 25 && n < 12) {
                                const double2 d = D[m * 25 + n + 13];
                                W[(n + 13) * LD + m] = make_double2(v.x * d.x - v.y * d.y, v.x * d.y + v.y * d.x);
                            }
                        });
                    team_sync<NP>(team);
                    // 3: U rows per x-parity (pairs 4..12 even, 4..11 odd) -> X[u_r][iy'_r]
                    WStage<LD, 4, true>{V1T, 9, 4, W, 25, true, lane, part, NP}([&](int m, int n, double2 v) {
                        if (m < 9 && n < 25) X[m * LD + n] = v;
                    });
                    WStage<LD, 3, true>{V1T + 16 * LD, 8, 4, W + 13, 25, true, lane, NP - 1 - part, NP}(
                        [&](int m, int n, double2 v) {
                            if (m < 8 && n < 25) X[(m + 9) * LD + n] = v;
                        });
                    team_sync<NP>(team);
                    // 4: U columns per y-parity -> W[u_r][v_r]
                    WStage<LD, 4, true>{V2T, 9, 4, X, 17, false, lane, part, NP}([&](int m, int n, double2 v) {
                        if (m < 17 && n < 9) W[m * LD + n] = v;
                    });
                    WStage<LD, 3, true>{V2T + 16 * LD, 8, 4, X + 13, 17, false, lane, NP - 1 - part, NP}(
                        [&](int m, int n, double2 v) {
                            if (m < 17 && n < 8) W[m * LD + n + 9] = v;
                        });
                    team_sync<NP>(team);
                    // the gathered tile is free: fetch the team's next subdomain under the unbutterfly
                    if (more) gather(pt.y);
                    // inverse butterflies on the U block -> staging row of the subdomain
                    double2* yrow = ystage + (size_t)id * nu_max;
                    for (int e = tl; e < 289; e += NP * 32) {
                        const int ixu = e / 17, iyu = e - ixu * 17;
                        int rx[2], ry[2];
                        double cx[2], cy[2];
                        auto coef = [&](int nat, int* rr, double* cc) {
                            const int u = ubn[nat], gg = u & 255, form = u >> 8;
                            rr[0] = gg - 4;
                            rr[1] = 9 + gg - 4;
                            if (form == 1) cc[0] = 1.0, cc[1] = 0.0, rr[1] = rr[0];
                            else if (form == 0) cc[0] = r2, cc[1] = r2;
                            else if (form == 2) cc[0] = r2, cc[1] = -r2;
                            else cc[0] = -r2, cc[1] = r2;
                        };
                        coef(4 + ixu, rx, cx);
                        coef(4 + iyu, ry, cy);
                        double2 s = make_double2(0.0, 0.0);
#pragma unroll
                        for (int a = 0; a < 2; ++a)
#pragma unroll
                            for (int b = 0; b < 2; ++b) {
                                const double w = cx[a] * cy[b];
                                const double2 v = W[rx[a] * LD + ry[b]];
                                s.x = fma(w, v.x, s.x);
                                s.y = fma(w, v.y, s.y);
                            }
                        yrow[urow[ixu * 17 + iyu]] = s;
                    }
                }
                asm volatile("cp.async.wait_all;\n" ::: "memory");
                pos = seg_end;
                ++ci;
                if (pos < wk.y) {
                    __syncthreads();  // every team finished with the factors
                    copy_image(ci);
                }
                continue;
            }
        }
#ifndef HTG_FDM_CONST
#define HTG_FDM_CONST 1  // compile-time path (2-warp teams only: cfg4 187.5 -> 181.9 us; with the 3-warp
                         // teams of cfg3 it is slower, 63.5 vs 61.4 us) for the 6 x 6-cell Omega / 4 x 4-cell U class at p = 4
#endif
        constexpr bool RS = NT > 576;  // 24 warps: 80 registers per thread
#ifndef HTG_FDM_CONST3
#define HTG_FDM_CONST3 0  // compile-time path also for 3-warp teams
#endif
        if constexpr (P == 4 && (NP == 2 || RS || (NP == 3 && HTG_FDM_CONST3)) && HTG_FDM_CONST) {
            if (nx == 25 && ny == 25 && nux == 17 && nuy == 17) {
                const int ux0 = c.ux0, uy0 = c.uy0;
                for (; cur < main_end; cur += nteam) {
                    const int id = pt.x;
                    const bool more = cur + nteam < main_end;
                    if (more) pt = pos_tab[cur + nteam];
                    asm volatile("cp.async.wait_all;\n" ::: "memory");
                    team_sync<NP>(team);
                    for_part<NP>(part, [&](auto pc) {
                        CStage<LD, KS, false, 25, 25, 25, true, NP>{V1T, 0, X, lane}.template go<RS, decltype(pc)::value>(
                            [&](int m, int n, double2 v) { W[m * LD + n] = v; });
                    });
                    team_sync<NP>(team);
                    for_part<NP>(NP - 1 - part, [&](auto pc) {
                        CStage<LD, KS, false, 25, 25, 25, false, NP>{V2T, 0, W, lane}.template go<RS, decltype(pc)::value>(
                            [&](int m, int n, double2 v) {
                                const double2 d = D[m * 25 + n];
                                X[n * LD + m] = make_double2(v.x * d.x - v.y * d.y, v.x * d.y + v.y * d.x);
                            });
                    });
                    team_sync<NP>(team);
                    for_part<NP>(part, [&](auto pc) {
                        CStage<LD, KS, true, 17, 25, 25, true, NP>{V1T, ux0, X, lane}.template go<RS, decltype(pc)::value>(
                            [&](int m, int n, double2 v) { W[m * LD + n] = v; });
                    });
                    team_sync<NP>(team);
                    if (more) gather(pt.y);
                    double2* yrow = ystage + (size_t)id * nu_max;
                    for_part<NP>(NP - 1 - part, [&](auto pc) {
                        CStage<LD, KS, true, 17, 17, 25, false, NP>{V2T, uy0, W, lane}.template go<RS, decltype(pc)::value>(
                            [&](int m, int n, double2 v) { yrow[urow[m * 17 + n]] = v; });
                    });
                }
            }
        }
        for (; cur < main_end; cur += nteam) {
            const int id = pt.x;
            const bool more = cur + nteam < main_end;
            if (more) pt = pos_tab[cur + nteam];  // next subdomain of the team, used at stage 4
            HTG_TR(1);
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            team_sync<NP>(team);
            HTG_TR(2);  // gather wait
#ifdef HTG_FDM_TRACE
            ++tr_n;
#endif
            // 1: P[ix'][iy] = sum_ix Vx[ix][ix'] G[iy][ix]  -> W[ix'][iy]
            WStage<LD, KS, false>{V1T, nx, 0, X, ny, true, lane, part, NP}([&](int m, int n, double2 v) {
                if (m < nx && n < ny) W[m * LD + n] = v;
            });
            team_sync<NP>(team);
            HTG_TR(3);
            // 2: Q[ix'][iy'] = (sum_iy P[ix'][iy] Vy[iy][iy']) Dinv[ix'][iy']  -> X[iy'][ix']
#ifndef HTG_FDM_EXP
#define HTG_FDM_EXP 0  // timing experiments only (wrong results): 1 no Dinv, 2 no part flip, 3 untransposed store
#endif
            WStage<LD, KS, false>{V2T, ny, 0, W, nx, false, lane, HTG_FDM_EXP == 2 ? part : NP - 1 - part, NP}([&](int m, int n, double2 v) {
                if (m < nx && n < ny) {
                    if (HTG_FDM_EXP == 1) {
                        X[n * LD + m] = v;
                    } else {
                        const double2 d = D[m * ny + n];
                        const double2 o = make_double2(v.x * d.x - v.y * d.y, v.x * d.y + v.y * d.x);
                        if (HTG_FDM_EXP == 3) X[m * LD + n] = o;
                        else X[n * LD + m] = o;
                    }
                }
            });
            team_sync<NP>(team);
            HTG_TR(4);
            // 3: R[ixu][iy'] = sum_ix' Vx[ux0 + ixu][ix'] Q[iy'][ix']  -> W[ixu][iy']
            WStage<LD, KS, true>{V1T, nux, c.ux0, X, ny, true, lane, part, NP}([&](int m, int n, double2 v) {
                if (m < nux && n < ny) W[m * LD + n] = v;
            });
            team_sync<NP>(team);
            HTG_TR(5);
            // the gathered tile is free: fetch the team's next subdomain under stage 4
            if (more) gather(pt.y);
            // 4: Y[ixu][iyu] = sum_iy' R[ixu][iy'] Vy[uy0 + iyu][iy']  -> staging row of the subdomain
            double2* yrow = ystage + (size_t)id * nu_max;
            WStage<LD, KS, true>{V2T, nuy, c.uy0, W, nux, false, lane, NP - 1 - part, NP}(
                [&](int m, int n, double2 v) {
                    if (m < nux && n < nuy) yrow[urow[m * nuy + n]] = v;
                });
            HTG_TR(6);
        }
        if (merge) {
            const int st = team / mg;  // merged team; works in the buffers of its first team
            if (st < Rl) {
                const int prt = (team - st * mg) * NP + part, npp = mg * NP;
                double2* Xs = fac + fac_elems + size_t(st * mg) * 2 * rows * LD;
                double2* Ws = Xs + rows * LD;
                auto sbar = [&]() { asm volatile("bar.sync %0, %1;\n" ::"r"(9 + st), "r"(npp * 32) : "memory"); };
                const int2 p2 = pos_tab[pos + full + st];
                sbar();  // every member team is through its own rounds: the buffers are free
                {
                    const int ox = (p2.y & 0xffff) * P, oy = (p2.y >> 16) * P;
                    if (c.goff) {
                        const double2* rb = r + dof_index(g.nx, g.ny, P, ox, oy);
                        for (int l = prt * 32 + lane; l < nxy; l += npp * 32) cp_async16(&Xs[gpos[l]], rb + gofs[l]);
                    } else {
                        for (int l = prt * 32 + lane; l < nxy; l += npp * 32) {
                            const int iy = fdiv(l, inv_nx), ix = l - iy * nx;
                            cp_async16(&Xs[iy * LD + ix], r + dof_index(g.nx, g.ny, P, ox + ix, oy + iy));
                        }
                    }
                    asm volatile("cp.async.commit_group;\n" ::: "memory");
                }
                asm volatile("cp.async.wait_all;\n" ::: "memory");
                sbar();
                WStage<LD, KS, false>{V1T, nx, 0, Xs, ny, true, lane, prt, npp}([&](int m, int n, double2 v) {
                    if (m < nx && n < ny) Ws[m * LD + n] = v;
                });
                sbar();
                WStage<LD, KS, false>{V2T, ny, 0, Ws, nx, false, lane, npp - 1 - prt, npp}([&](int m, int n, double2 v) {
                    if (m < nx && n < ny) {
                        const double2 d = D[m * ny + n];
                        Xs[n * LD + m] = make_double2(v.x * d.x - v.y * d.y, v.x * d.y + v.y * d.x);
                    }
                });
                sbar();
                WStage<LD, KS, true>{V1T, nux, c.ux0, Xs, ny, true, lane, prt, npp}([&](int m, int n, double2 v) {
                    if (m < nux && n < ny) Ws[m * LD + n] = v;
                });
                sbar();
                double2* yrow = ystage + (size_t)p2.x * nu_max;
                WStage<LD, KS, true>{V2T, nuy, c.uy0, Ws, nux, false, lane, npp - 1 - prt, npp}(
                    [&](int m, int n, double2 v) {
                        if (m < nux && n < nuy) yrow[urow[m * nuy + n]] = v;
                    });
            }
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        pos = seg_end;
        ++ci;
        if (pos < wk.y) {
            __syncthreads();  // every team finished with the factors
            copy_image(ci);
        }
    }
#ifdef HTG_FDM_TRACE
    if (lane == 0 && (blockIdx.x == 0 || blockIdx.x == 70))
        printf("fdm trace cta %d team %d part %d: n %d total %lld | setup %lld loop %lld wait %lld s1 %lld s2 %lld s3 %lld s4 %lld\n",
               blockIdx.x, team, part, tr_n, clock64() - tr_t0, tr_acc[0], tr_acc[1], tr_acc[2], tr_acc[3], tr_acc[4],
               tr_acc[5], tr_acc[6]);
#endif
}

}  // namespace

// fdm_supported (fdm.cpp) admits 1-D extents up to 4 KS
static_assert(4 * FdmDims<2>::KS == 16 && 4 * FdmDims<4>::KS == 28, "fdm_supported limits out of date");

// One launch for every separable class: CTAs take contiguous ranges of the
// class-sorted subdomain list (work table built once, fdm_plan).
void dd_fdm_launch(const FineGeom& g, const FdmLaunch& L, const double2* r, double2* ystage, int nu_max,
                   cudaStream_t st) {
    if (L.nwork == 0) return;
    static bool attr[9] = {};
    static bool attr_w[12] = {};
    auto go = [&](auto kern, int p) {
        if (!attr[p]) {
            HTG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax));
            attr[p] = true;
        }
        kern<<<L.nwork, kFThreads, L.smem, st>>>(g, L.classes, L.work, r, ystage, nu_max, L.rows, L.fac_elems);
    };
    auto go_w = [&](auto kern, int slot) {
        if (!attr_w[slot]) {
            HTG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax));
            attr_w[slot] = true;
        }
        kern<<<L.nwork, L.nwarps * 32, L.smem, st>>>(g, L.classes, L.nwork <= FdmWorkTab::kMax ? nullptr : L.work, L.tab,
                                                     L.image, L.pos_tab, r, ystage, nu_max, L.rows, L.fac_elems);
    };
    if (L.nwarps > 0) {
        const bool small = L.nwarps * 32 <= kWSizes[L.team][0];
        switch (g.p * 8 + L.team) {
            case 17: go_w(k_dd_fdm_w<2, 1, 512>, 1); break;
            case 18: go_w(k_dd_fdm_w<2, 2, 512>, 0); break;
            case 19: go_w(k_dd_fdm_w<2, 3, 576>, 6); break;
            case 20: go_w(k_dd_fdm_w<2, 4, 512>, 4); break;
            case 33:
                if (small) go_w(k_dd_fdm_w<4, 1, kWSizes[1][0]>, 3);
                else go_w(k_dd_fdm_w<4, 1, kWSizes[1][1]>, 7);
                break;
            case 34:
                if (small) go_w(k_dd_fdm_w<4, 2, kWSizes[2][0]>, 8);
                else go_w(k_dd_fdm_w<4, 2, kWSizes[2][1]>, 2);
                break;
            case 35:
                if (small) go_w(k_dd_fdm_w<4, 3, kWSizes[3][0]>, 9);
                else if (L.nwarps * 32 <= kWSizes[3][1]) go_w(k_dd_fdm_w<4, 3, kWSizes[3][1]>, 10);
                else go_w(k_dd_fdm_w<4, 3, kWLean>, 11);
                break;
            case 36: go_w(k_dd_fdm_w<4, 4, 512>, 5); break;
            default: throw InvalidArgument("FDM subdomain kernel: p must be 2 or 4");
        }
    } else {
        switch (g.p) {
            case 2: go(k_dd_fdm<2>, 2); break;
            case 4: go(k_dd_fdm<4>, 4); break;
            default: throw InvalidArgument("FDM subdomain kernel: p must be 2 or 4");
        }
    }
    HTG_CUDA(cudaGetLastError());
    count_launch();
}

// Shared-memory layout (factor region sized for the largest class, two data
// buffers per group) and contiguous, equal ranges of the class-sorted
// subdomain list, one per SM.
std::vector<int4> fdm_plan(std::vector<FdmClassDev>& cls, int p, int nsm, FdmLaunch& L) {
    const int LD = p == 2 ? FdmDims<2>::LD : FdmDims<4>::LD;
    int total = 0, fac = 0, ext = 0;
    for (auto& c : cls) {
        c.first = total;
        total += c.nsub;
        fac = std::max(fac, 2 * (p == 2 ? 4 * FdmDims<2>::KS : 4 * FdmDims<4>::KS) * LD + c.nx * c.ny +
                                (kFGroups * 32 + c.nux * c.nuy + c.nx * c.ny + 3) / 4);
        ext = std::max({ext, c.nx, c.ny});
    }
    // team-per-subdomain kernel (default: 2-warp teams; HTG_FDM_TEAM=1 one warp per
    // subdomain; HTG_FDM_GROUPK=1 selects the batched 4-warp-group kernel)
    const char* gk = std::getenv("HTG_FDM_GROUPK");
    const char* tk = std::getenv("HTG_FDM_TEAM");
    L.nwarps = 0;
    // team size: 2 warps (8 teams at p = 4); when an SM gets few subdomains (cfg3: 17
    // per SM) the time is the latency of a team's chain of subdomains, not the DMMA
    // pipe: five 3-warp teams (a product's 9 / 6 tiles split evenly over 3 warps)
    // take 75.8 us at cfg3 against 80.2 (four 4-warp teams) and 82.3 (eight 2-warp
    // teams). HTG_FDM_TEAM=1..4 / HTG_FDM_NTEAMS force the shape.
    const int per_sm = (total + std::max(nsm, 1) - 1) / std::max(nsm, 1);
    const bool few = per_sm < kFdmTeam4Below;
    L.team = few ? (p == 4 ? 3 : 4) : 2;
    if (tk && tk[0] >= '1' && tk[0] <= '4') L.team = tk[0] - '0';
    const char* ntk = std::getenv("HTG_FDM_NTEAMS");  // teams per CTA (default: as many as fit)
    const int nt_default = (few && p == 4 && L.team == 3) ? 5 : 1 << 20;  // 480 threads: 128 registers
    if (!(gk && gk[0] == '1')) {
        const int KP = p == 2 ? 4 * FdmDims<2>::KS : 4 * FdmDims<4>::KS;
        int wfac = 0;
        for (auto& c : cls)
            wfac = std::max(wfac, 2 * KP * LD + c.nx * c.ny + (c.nux * c.nuy + 2 * c.nx * c.ny + 64 + 3) / 4);
        wfac = (wfac + 7) / 8 * 8;
        const int per_warp = 2 * ext * LD;
        int nt = (kSmemMax / int(sizeof(double2)) - wfac) / per_warp;  // teams (buffer pairs)
        nt = std::min(nt, (p == 4 ? (L.team == 3 ? kWLean : kWSizes[L.team][1]) : (L.team == 3 ? 576 : 512)) / (32 * L.team));
        if (L.team != 3 && nt * L.team >= 8) nt = (nt * L.team) / 4 * 4 / L.team;  // whole warps per SM sub-partition
        nt = std::min(nt, (ntk && std::atoi(ntk) >= 1) ? std::atoi(ntk) : nt_default);
        if (nt >= 1) {
            L.nwarps = nt * L.team;
            L.fac_elems = wfac;
            L.rows = ext;
            L.smem = size_t(wfac + nt * per_warp) * sizeof(double2);
        }
    }
    if (L.nwarps == 0) {
        fac = (fac + 7) / 8 * 8;
        L.fac_elems = fac;
        L.rows = p == 2 ? fdm_rows<2>(fac) : fdm_rows<4>(fac);
        if (L.rows < ext) throw RuntimeError("FDM subdomain kernel: shared memory too small for the class extents");
        L.smem = size_t(fac + kFGroups * 2 * L.rows * LD) * sizeof(double2);
    }
    std::vector<int4> work;
    if (total == 0) return work;
    const int ctas = std::min(nsm, total);
    for (int i = 0; i < ctas; ++i) {
        const int a = int((long long)total * i / ctas), b = int((long long)total * (i + 1) / ctas);
        if (b > a) {
            int ci = 0;
            while (cls[ci].first + cls[ci].nsub <= a) ++ci;
            work.push_back(make_int4(a, b, ci, 0));
        }
    }
    for (size_t i = 0; i < work.size() && i < size_t(FdmWorkTab::kMax); ++i) L.tab.w[i] = work[i];
    return work;
}

void fdm_format(const std::vector<FdmClassDev>& cls, int p, FdmLaunch& L, std::vector<void*>& allocs, size_t& bytes,
                cudaStream_t st) {
    if (cls.empty() || L.nwarps == 0) return;
    for (const FdmClassDev& c : cls)
        if (c.nsub == 0) throw RuntimeError("FDM subdomain kernel: empty class");
    int total = 0;
    for (const FdmClassDev& c : cls) total += c.nsub;
    void *img = nullptr, *pt = nullptr;
    const size_t ib = cls.size() * size_t(L.fac_elems) * sizeof(double2), pb = size_t(total) * sizeof(int2);
    HTG_CUDA(cudaMalloc(&img, ib));
    allocs.push_back(img);
    HTG_CUDA(cudaMalloc(&pt, pb));
    allocs.push_back(pt);
    bytes += ib + pb;
    HTG_CUDA(cudaMemsetAsync(img, 0, ib, st));
    if (p == 2) k_fdm_format<2><<<unsigned(cls.size()), 256, 0, st>>>(L.classes, static_cast<double2*>(img), static_cast<int2*>(pt), L.fac_elems);
    else k_fdm_format<4><<<unsigned(cls.size()), 256, 0, st>>>(L.classes, static_cast<double2*>(img), static_cast<int2*>(pt), L.fac_elems);
    HTG_CUDA(cudaGetLastError());
    L.image = static_cast<const double2*>(img);
    L.pos_tab = static_cast<const int2*>(pt);
}

}  // namespace htg
