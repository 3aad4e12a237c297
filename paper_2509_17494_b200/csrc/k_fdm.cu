// k_fdm.cu -- K2 for separable subdomain classes: fast diagonalisation on DMMA.
//
// For a class with A_s^(Omega) = Kx (x) My + Mx (x) Ky (fdm.cpp) the U rows of
// A^-1 g are, with the gathered residual as a tensor tile G[ix][iy],
//   Y_U = Vx_U [ (Vx^T G Vy) o Dinv ] Vy_U^T,
// four small complex products per subdomain (8 (2 nx^2 ny + nux nx ny + nux ny nuy)
// flop, 3.7x fewer than the dense |U| x |Omega| product at p = 4).
// A CTA runs kGroups groups of 4 warps; a group takes one subdomain at a time
// (named barrier per group), the class factors sit in shared memory, every
// stage is mma.sync.m8n8k4.f64 on tiles padded to 32 with k steps of 4.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.hpp"
#include "kernels.hpp"

namespace htg {

namespace {

// rows padded to 32 (m8/n8 tiles), k to 28 (k4 steps); LD = 28 = 4 mod 8 keeps the
// 128-bit fragment loads of 8 lanes (2 rows x 4 k) on distinct banks
constexpr int kNP = 32, kLDF = 28;
#ifndef HTG_FDM_GROUPS
#define HTG_FDM_GROUPS 4
#endif
constexpr int kGroups = HTG_FDM_GROUPS, kFThreads = kGroups * 128;
constexpr int kXBuf = kGroups <= 3 ? 2 : 1;  // prefetch the next tile when shared memory allows

struct FdmSmem {
    double2 V1T[kNP][kLDF];  // A of stage 1: [ix'][ix] = Vx[ix][ix']
    double2 V2T[kNP][kLDF];  // B of stage 2: [iy'][iy] = Vy[iy][iy']
    double2 V1U[kNP][kLDF];  // A of stage 3: [ixu][ix'] = Vx[ux0 + ixu][ix']
    double2 V2U[kNP][kLDF];  // B of stage 4: [iyu][iy'] = Vy[uy0 + iyu][iy']
    double2 D[kNP][kNP + 1]; // Dinv[ix'][iy']
    double2 X[kGroups][kXBuf][kNP][kLDF];  // gathered tile (ping-pong when prefetching)
    double2 W[kGroups][kNP][kLDF];
};

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
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

// C[m][n] = sum_k A[m][k] B[n][k] over MT x NT 8x8 tiles, KS k-steps of 4; the
// group's warp q owns tiles q, q+4, q+8, q+12 (all in flight together).
// epi(m, n, value) is called for every element of the warp's tiles.
template <class Epi>
__device__ __forceinline__ void stage(const double2 (*A)[kLDF], const double2 (*B)[kLDF], int MT, int NT, int KS,
                                      int q, int lane, Epi&& epi) {
    const int nt_all = MT * NT;
    // Gauss / 3M complex product: t1 = ar br, t2 = ai bi, t3 = (ar + ai)(br + bi);
    // re = t1 - t2, im = t3 - t1 - t2 -- three DMMAs per k-step and tile instead of four
    double t1[4][2], t2[4][2], t3[4][2];
    int tm[4], tn[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        t1[j][0] = t1[j][1] = t2[j][0] = t2[j][1] = t3[j][0] = t3[j][1] = 0.0;
        const int t = q + 4 * j;
        tm[j] = t < nt_all ? t / NT : -1;
        tn[j] = t < nt_all ? t % NT : 0;
    }
    const int r = lane >> 2, kq = lane & 3;
    const int ntile = max(0, min(4, (nt_all - q + 3) / 4));
    for (int ks = 0; ks < KS; ++ks) {
        const int k = ks * 4 + kq;
        double2 a[4], b[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int m = j < ntile ? tm[j] : 0, n = j < ntile ? tn[j] : 0;
            a[j] = A[m * 8 + r][k];
            b[j] = B[n * 8 + r][k];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (j < ntile) dmma(t1[j][0], t1[j][1], a[j].x, b[j].x);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (j < ntile) dmma(t2[j][0], t2[j][1], a[j].y, b[j].y);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (j < ntile) dmma(t3[j][0], t3[j][1], a[j].x + a[j].y, b[j].x + b[j].y);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (tm[j] < 0) break;
#pragma unroll
        for (int i = 0; i < 2; ++i)
            epi(tm[j] * 8 + r, tn[j] * 8 + 2 * kq + i,
                make_double2(t1[j][i] - t2[j][i], t3[j][i] - t1[j][i] - t2[j][i]));
    }
}

template <int P>
__global__ void __launch_bounds__(kFThreads, 1) k_dd_fdm(FineGeom g, const FdmClassDev* __restrict__ classes,
                                                         const int4* __restrict__ work, const double2* __restrict__ r,
                                                         double2* __restrict__ ystage, int nu_max) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FdmSmem& sm = *reinterpret_cast<FdmSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const int4 wk = work[blockIdx.x];  // first, end index into the class-sorted subdomain list
    const int grp = tid >> 7, gt = tid & 127, q = gt >> 5, lane = tid & 31;
    double2 (*W)[kLDF] = sm.W[grp];
    // segments of one class inside this CTA's range: reload the factors per segment
    int pos = wk.x;
    while (pos < wk.y) {
        int ci = 0;
        while (classes[ci].first + classes[ci].nsub <= pos) ++ci;
        const FdmClassDev c = classes[ci];
        const int seg_end = min(wk.y, c.first + c.nsub);
        __syncthreads();  // previous segment finished with the factors
        for (int i = tid; i < kNP * kLDF; i += kFThreads) {
            const int a = i / kLDF, b = i % kLDF;
            const double2 z = make_double2(0.0, 0.0);
            sm.V1T[a][b] = (a < c.nx && b < c.nx) ? c.Vx[b * c.nx + a] : z;
            sm.V2T[a][b] = (a < c.ny && b < c.ny) ? c.Vy[b * c.ny + a] : z;
            sm.V1U[a][b] = (a < c.nux && b < c.nx) ? c.Vx[(c.ux0 + a) * c.nx + b] : z;
            sm.V2U[a][b] = (a < c.nuy && b < c.ny) ? c.Vy[(c.uy0 + a) * c.ny + b] : z;
        }
        for (int i = tid; i < kNP * kNP; i += kFThreads) {
            const int a = i / kNP, b = i % kNP;
            sm.D[a][b] = (a < c.nx && b < c.ny) ? c.Dinv[a * c.ny + b] : make_double2(0.0, 0.0);
        }
        // work buffers: padding must be zero for this class's extents
        for (int i = gt; i < kNP * kLDF; i += 128) {
            for (int b2 = 0; b2 < kXBuf; ++b2) (&sm.X[grp][b2][0][0])[i] = make_double2(0.0, 0.0);
            (&W[0][0])[i] = make_double2(0.0, 0.0);
        }
        __syncthreads();
        const int MTx = (c.nx + 7) / 8, MTy = (c.ny + 7) / 8, MTux = (c.nux + 7) / 8, MTuy = (c.nuy + 7) / 8;
        const int KSx = (c.nx + 3) / 4, KSy = (c.ny + 3) / 4;
        const int nloc = c.nx * c.ny;
        auto gather = [&](int sp, double2 (*X)[kLDF]) {
            const int s = c.subs[sp - c.first];
            const int so = c.sub_o[s];
            const int ox = (so & 0xffff) * P, oy = (so >> 16) * P;
            for (int l = gt; l < nloc; l += 128) {
                const int iy = l / c.nx, ix = l - iy * c.nx;
                cp_async16(&X[iy][ix], r + dof_index(g.nx, g.ny, P, ox + ix, oy + iy));
            }
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        };
        int cur = 0;
        if (pos + grp < seg_end) gather(pos + grp, sm.X[grp][0]);
        for (int sp = pos + grp; sp < seg_end; sp += kGroups, cur ^= (kXBuf - 1)) {
            double2 (*X)[kLDF] = sm.X[grp][cur];
            const int s = c.subs[sp - c.first];
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            group_sync(grp);
            if (kXBuf == 2 && sp + kGroups < seg_end) gather(sp + kGroups, sm.X[grp][cur ^ 1]);  // prefetch
            // 1: P[ix'][iy] = sum_ix Vx[ix][ix'] G[ix][iy]  -> W[ix'][iy]
            stage(sm.V1T, X, MTx, MTy, KSx, q, lane, [&](int m, int n, double2 v) {
                if (m < c.nx && n < c.ny) W[m][n] = v;
            });
            group_sync(grp);
            // 2: Q[ix'][iy'] = (sum_iy P[ix'][iy] Vy[iy][iy']) Dinv[ix'][iy']  -> X[iy'][ix']
            stage(W, sm.V2T, MTx, MTy, KSy, q, lane, [&](int m, int n, double2 v) {
                if (m < c.nx && n < c.ny) {
                    const double2 d = sm.D[m][n];
                    X[n][m] = make_double2(v.x * d.x - v.y * d.y, v.x * d.y + v.y * d.x);
                }
            });
            group_sync(grp);
            // 3: R[ixu][iy'] = sum_ix' Vx[ux0 + ixu][ix'] Q[ix'][iy']  -> W[ixu][iy']
            stage(sm.V1U, X, MTux, MTy, KSx, q, lane, [&](int m, int n, double2 v) {
                if (m < c.nux && n < c.ny) W[m][n] = v;
            });
            group_sync(grp);
            // 4: Y[ixu][iyu] = sum_iy' R[ixu][iy'] Vy[uy0 + iyu][iy']  -> staging rows
            stage(W, sm.V2U, MTux, MTuy, KSy, q, lane, [&](int m, int n, double2 v) {
                if (m < c.nux && n < c.nuy) {
                    const int li = int(dof_index(c.onx, c.ony, P, c.ux0 + m, c.uy0 + n));
                    ystage[(size_t)s * nu_max + c.rowmap[li]] = v;
                }
            });
            group_sync(grp);
            if (kXBuf == 1 && sp + kGroups < seg_end) gather(sp + kGroups, X);
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        pos = seg_end;
    }
}

}  // namespace

// One launch for every separable class: CTAs are split over the classes in
// proportion to their subdomain counts (work table built once, on first use).
void dd_fdm_launch(const FineGeom& g, const FdmLaunch& L, const double2* r, double2* ystage, int nu_max,
                   cudaStream_t st) {
    if (L.nwork == 0) return;
    const size_t smem = sizeof(FdmSmem);
    static bool attr[9] = {};
    auto go = [&](auto kern, int p) {
        if (!attr[p]) {
            HTG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            attr[p] = true;
        }
        kern<<<L.nwork, kFThreads, smem, st>>>(g, L.classes, L.work, r, ystage, nu_max);
    };
    switch (g.p) {
        case 2: go(k_dd_fdm<2>, 2); break;
        case 4: go(k_dd_fdm<4>, 4); break;
        default: throw InvalidArgument("FDM subdomain kernel: p > 4 not supported (1-D extent > 32)");
    }
    HTG_CUDA(cudaGetLastError());
    count_launch();
}

// Contiguous ranges of the class-sorted subdomain list, one per SM (a CTA may
// span a class boundary; it reloads the factors per class segment).
std::vector<int4> fdm_work_table(std::vector<FdmClassDev>& cls, int nsm) {
    int total = 0;
    for (auto& c : cls) {
        c.first = total;
        total += c.nsub;
    }
    std::vector<int4> work;
    if (total == 0) return work;
    const int ctas = std::min(nsm, (total + kGroups - 1) / kGroups);
    const int per = ((total + ctas - 1) / ctas + kGroups - 1) / kGroups * kGroups;
    for (int s0 = 0; s0 < total; s0 += per) work.push_back(make_int4(s0, std::min(total, s0 + per), 0, 0));
    return work;
}

}  // namespace htg
