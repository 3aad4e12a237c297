// k_band.cu -- K2 for subdomains that share no factor: per-subdomain direct
// solves factored on the device (north star "otherwise as
// batched banded/LU solves").
//
// The reference factors every subdomain operator A_s^(i) with its own SparseLU
// (proj/core/src/twogrid.cpp:76-90) and solves with it in dd_step (:92-112).
// Subdomains whose local operator is shared by a class use the FDM or dense
// class kernels; a subdomain with its own coefficients (a heterogeneous medium
// makes every subdomain unique) gets its own factor here:
//
//  * static condensation: the (p-1)^2 bubble dofs of each cell couple only
//    inside the cell, so per cell A_II^-1 and W = A_II^-1 A_IB are stored and
//    the cell's Schur complement A_BB - A_BI W is added into the skeleton
//    matrix (vertex + edge dofs, 301 of 625 at p = 4 for a 6 x 6-cell Omega);
//  * the skeleton matrix, ordered by lattice rows, is banded (half bandwidth
//    one cell row of skeleton dofs, 50 at p = 4) and complex symmetric with a
//    negative definite imaginary part (alpha_s > 0 and the Robin terms), so
//    every leading minor is nonsingular and it is factored as L D L^T without
//    pivoting (Dirichlet rows / columns are identity);
//  * setup: one CTA per subdomain assembles its cells from the 1-D factors
//    (K_e = S (x) M + M (x) S - m M (x) M, Robin -i k h M on absorbing Omega
//    edges, proj/core/src/fespace.cpp:181-210, twogrid.cpp:80-86), condenses
//    and factors in device memory: no host factorization;
//  * sweep: one warp per subdomain gathers g = r on Omega, condenses, runs the
//    banded forward / backward substitution and back-substitutes the bubbles
//    of the U cells; the U values go to the same staging rows as the other
//    subdomain kernels (the PoU combine is shared).
// Factor storage per subdomain at p = 4, l_dd = 4: 36 cells x 225 + 301 x 51
// complex = 375 KB (3.7 GB for the 10,000 subdomains of cfg4).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <vector>

#include "common.hpp"
#include "kernels.hpp"
#include "setup.hpp"

namespace htg {

namespace {

__device__ __forceinline__ double2 cmulb(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ void cfma(double2& c, double2 a, double2 b) {  // c += a b
    c.x = fma(a.x, b.x, fma(-a.y, b.y, c.x));
    c.y = fma(a.x, b.y, fma(a.y, b.x, c.y));
}
__device__ __forceinline__ void cfms(double2& c, double2 a, double2 b) {  // c -= a b
    c.x = fma(-a.x, b.x, fma(a.y, b.y, c.x));
    c.y = fma(-a.x, b.y, fma(-a.y, b.x, c.y));
}
__device__ __forceinline__ double2 crecip(double2 a) {
    const double d = a.x * a.x + a.y * a.y;
    return make_double2(a.x / d, -a.y / d);
}

// 1-D basis index of lattice position t in [0, p] of a cell: 0 left vertex, 1
// right vertex, d >= 2 the bubble of degree d at position d - 1
__host__ __device__ __forceinline__ int basis_of(int t, int p) { return t == 0 ? 0 : (t == p ? 1 : t + 1); }

// cell-local node (a, b), a, b in [0, p]: boundary nodes (a or b in {0, p}) in
// (b, a) order get slots [0, 4p), interior nodes slots [0, (p-1)^2)
template <int P>
__device__ __forceinline__ int bnd_node(int k) {  // boundary slot -> node index b (P+1) + a
    constexpr int NE1 = P + 1;
    if (k < NE1) return k;                              // b = 0
    if (k >= 4 * P - NE1) return P * NE1 + (k - (4 * P - NE1));  // b = P
    const int r = k - NE1, b = 1 + r / 2;               // b in [1, P-1]: a = 0 or P
    return b * NE1 + ((r & 1) ? P : 0);
}
template <int P>
__device__ __forceinline__ int int_node(int i) {  // interior slot -> node index
    return (1 + i / (P - 1)) * (P + 1) + 1 + i % (P - 1);
}

__device__ __forceinline__ int8_t omega_edge(const FineGeom& g, const double* khtab, int side, int ox, int oy,
                                             int onx, int ony, int i, double& kh) {
    // perimeter edge i of Omega (side 0 bottom, 1 top, 2 left, 3 right): the
    // global tag and k h on the global boundary, else absorbing with the k h of
    // the Omega cell on it (twogrid.cpp:80-86)
    int cx, cy;
    bool outer;
    const int8_t* tg;
    const double* khg;
    if (side == 0) cx = ox + i, cy = oy, outer = oy == 0, tg = g.tg_b, khg = g.kh_b;
    else if (side == 1) cx = ox + i, cy = oy + ony - 1, outer = oy + ony == g.ny, tg = g.tg_t, khg = g.kh_t;
    else if (side == 2) cx = ox, cy = oy + i, outer = ox == 0, tg = g.tg_l, khg = g.kh_l;
    else cx = ox + onx - 1, cy = oy + i, outer = ox + onx == g.nx, tg = g.tg_r, khg = g.kh_r;
    if (outer) {
        const int e = side < 2 ? cx : cy;
        kh = khg[e];
        return tg[e];
    }
    kh = khtab[g.cls ? g.cls[(size_t)cy * g.nx + cx] : 0];
    return kAbsorbing;
}

// ------------------------------------------------------------------ setup
template <int P>
__global__ void __launch_bounds__(256) k_band_factor(FineGeom g, BandLaunch L) {
    constexpr int NE1 = P + 1, NE = NE1 * NE1, NB = 4 * P, NI = (P - 1) * (P - 1);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* Ae = reinterpret_cast<double2*>(smem_raw);  // NE x NE element matrix
    double2* Ai = Ae + NE * NE;                          // NI x NI: A_II, inverted in place
    double2* Wm = Ai + NI * NI;                          // NI x NB: W = A_II^-1 A_IB
    double2* colk = Wm + NI * NB;                        // NI: pivot column of a Gauss-Jordan step
    int* dsk = reinterpret_cast<int*>(colk + NI);        // Dirichlet flag per skeleton dof
    __shared__ double Ms[NE1][NE1], Ss[NE1][NE1];
    __shared__ int dirn[NE];  // Dirichlet flag per cell node
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < NE1 * NE1; i += nt) {
        Ms[i / NE1][i % NE1] = L.basis[i];
        Ss[i / NE1][i % NE1] = L.basis[NE1 * NE1 + i];
    }
    for (int bs = blockIdx.x; bs < L.nfac; bs += gridDim.x) {
        const int4 sd = L.fsubs[bs];
        const BandGeomDev G = L.geoms[sd.y];
        const int ox = sd.z & 0xffff, oy = sd.z >> 16;
        double2* F = L.pool + L.ffoff[bs];
        double2* band = F + (size_t)G.ncell * G.cellstride;
        const int ns = G.ns, bw = G.bw, LDB = bw + 1;
        for (size_t i = tid; i < (size_t)ns * LDB; i += nt) band[i] = make_double2(0.0, 0.0);
        for (int i = tid; i < ns; i += nt) dsk[i] = 0;
        __syncthreads();
        // Dirichlet dofs of Omega: the closures of its Dirichlet perimeter edges
        // (a vertex shared with a non-Dirichlet edge is Dirichlet too)
        for (int side = 0; side < 4; ++side) {
            const int cnt = side < 2 ? G.onx : G.ony;
            for (int i = tid; i < cnt; i += nt) {
                double kh;
                if (omega_edge(g, L.khtab, side, ox, oy, G.onx, G.ony, i, kh) != kDirichlet) continue;
                for (int s = 0; s <= P; ++s) {
                    const int gx = side < 2 ? i * P + s : (side == 2 ? 0 : G.onx * P);
                    const int gy = side >= 2 ? i * P + s : (side == 0 ? 0 : G.ony * P);
                    dsk[G.node_code[gy * G.NXn + gx]] = 1;
                }
            }
        }
        __syncthreads();
        for (int cell = 0; cell < G.ncell; ++cell) {
            const int cx = cell % G.onx, cy = cell / G.onx;
            const double2 m = g.mtabS[g.cls ? g.cls[(size_t)(oy + cy) * g.nx + ox + cx] : 0];
            // element matrix in lattice-position order: K_e - m M_e (fespace.cpp:181-210)
            for (int e = tid; e < NE * NE; e += nt) {
                const int r = e / NE, c = e % NE;
                const int ba = basis_of(r % NE1, P), bb = basis_of(r / NE1, P);
                const int bc = basis_of(c % NE1, P), bd = basis_of(c / NE1, P);
                const double sm = Ss[ba][bc] * Ms[bb][bd] + Ms[ba][bc] * Ss[bb][bd];
                const double mm = Ms[ba][bc] * Ms[bb][bd];
                Ae[e] = make_double2(sm - m.x * mm, -m.y * mm);
            }
            for (int i = tid; i < NE; i += nt) {
                const int a = i % NE1, b = i / NE1;
                const int code = G.node_code[(cy * P + b) * G.NXn + cx * P + a];
                dirn[i] = code >= 0 ? dsk[code] : 0;
            }
            __syncthreads();
            // Robin on the cell's edges that lie on Omega's absorbing perimeter
            // (one thread: at most 4 edges of (p+1)^2 entries)
            if (tid == 0) {
                for (int side = 0; side < 4; ++side) {
                    const bool on = side == 0 ? cy == 0 : side == 1 ? cy == G.ony - 1 : side == 2 ? cx == 0 : cx == G.onx - 1;
                    if (!on) continue;
                    double kh = 0.0;
                    const int8_t t = omega_edge(g, L.khtab, side, ox, oy, G.onx, G.ony, side < 2 ? cx : cy, kh);
                    // edge closure nodes in 1-D position order along the edge
                    auto node = [&](int s) {
                        return side == 0 ? s : side == 1 ? P * NE1 + s : side == 2 ? s * NE1 : s * NE1 + P;
                    };
                    if (t == kAbsorbing) {
                        for (int s = 0; s <= P; ++s)
                            for (int u = 0; u <= P; ++u) {
                                const double mv = Ms[basis_of(s, P)][basis_of(u, P)];
                                if (mv != 0.0) Ae[node(s) * NE + node(u)].y -= kh * mv;
                            }
                    }
                }
            }
            __syncthreads();
            // Dirichlet nodes: rows and columns out of the cell matrix (identity set on the skeleton)
            for (int e = tid; e < NE * NE; e += nt)
                if (dirn[e / NE] || dirn[e % NE]) Ae[e] = make_double2(0.0, 0.0);
            __syncthreads();
            // A_II, inverted in place (Gauss-Jordan without pivoting: a principal
            // submatrix of a matrix with definite imaginary part is nonsingular)
            for (int e = tid; e < NI * NI; e += nt) Ai[e] = Ae[int_node<P>(e / NI) * NE + int_node<P>(e % NI)];
            __syncthreads();
            for (int k = 0; k < NI; ++k) {
                const double2 piv = crecip(Ai[k * NI + k]);
                for (int i = tid; i < NI; i += nt) colk[i] = Ai[i * NI + k];  // multipliers, before any update
                __syncthreads();
                // row k scaled (the pivot entry becomes 1 / pivot)
                for (int j = tid; j < NI; j += nt) Ai[k * NI + j] = j == k ? piv : cmulb(Ai[k * NI + j], piv);
                __syncthreads();
                for (int e = tid; e < NI * NI; e += nt) {
                    const int i = e / NI, j = e % NI;
                    if (i == k) continue;
                    const double2 f = colk[i];
                    if (j == k) Ai[e] = make_double2(-(f.x * piv.x - f.y * piv.y), -(f.x * piv.y + f.y * piv.x));
                    else cfms(Ai[e], f, Ai[k * NI + j]);
                }
                __syncthreads();
            }
            // W = A_II^-1 A_IB
            for (int e = tid; e < NI * NB; e += nt) {
                const int i = e / NB, k = e % NB;
                double2 s = make_double2(0.0, 0.0);
                for (int j = 0; j < NI; ++j) cfma(s, Ai[i * NI + j], Ae[int_node<P>(j) * NE + bnd_node<P>(k)]);
                Wm[e] = s;
            }
            __syncthreads();
            // store A_II^-1 and W; Schur complement A_BB - A_BI W into the band (lower triangle)
            // cell block [j][o], o < NI: (A_II^-1)[o][j] (symmetric), o >= NI: W[j][o - NI]; for a
            // fixed j the lanes of the sweep read consecutive entries (coalesced)
            double2* Fc = F + (size_t)cell * G.cellstride;
            for (int e = tid; e < NI * (NI + NB); e += nt) {
                const int j = e / (NI + NB), o = e % (NI + NB);
                Fc[e] = o < NI ? Ai[o * NI + j] : Wm[j * NB + (o - NI)];
            }
            const int* cb = G.cell_bnd + (size_t)cell * NB;
            for (int e = tid; e < NB * NB; e += nt) {
                const int a = e / NB, b = e % NB;
                const int sa = cb[a], sb = cb[b];
                if (sa < sb) continue;  // lower triangle (sa >= sb): column sb, offset sa - sb
                double2 s = Ae[bnd_node<P>(a) * NE + bnd_node<P>(b)];
                for (int j = 0; j < NI; ++j) cfms(s, Ae[bnd_node<P>(a) * NE + int_node<P>(j)], Wm[j * NB + b]);
                double2& t = band[(size_t)sb * LDB + (sa - sb)];
                t.x += s.x;
                t.y += s.y;
            }
            __syncthreads();
        }
        // Dirichlet skeleton dofs: identity (their rows / columns are already zero)
        for (int i = tid; i < ns; i += nt)
            if (dsk[i]) band[(size_t)i * LDB] = make_double2(1.0, 0.0);
        __syncthreads();
        // banded L D L^T, right-looking; column j holds 1/d_j and L[j+i][j]
        for (int j = 0; j < ns; ++j) {
            double2* cj = band + (size_t)j * LDB;
            const double2 dinv = crecip(cj[0]);
            const int nb = min(bw, ns - 1 - j);
            __syncthreads();
            // trailing update A[j+i][j+k] -= l_i d l_k = c_i c_k / d  (c = column j before scaling)
            for (int e = tid; e < nb * nb; e += nt) {
                const int i = 1 + e / nb, k = 1 + e % nb;
                if (k > i) continue;
                const double2 ci = cj[i], ck = cj[k];
                double2& t = band[(size_t)(j + k) * LDB + (i - k)];
                cfms(t, cmulb(ci, dinv), ck);
            }
            __syncthreads();
            for (int i = 1 + tid; i <= nb; i += nt) cj[i] = cmulb(cj[i], dinv);
            if (tid == 0) cj[0] = dinv;
            __syncthreads();
        }
    }
}

// ------------------------------------------------------------------ sweep
// One warp per subdomain. The factor stream is what bounds it (375 KB per
// subdomain at p = 4, the band read twice): every load is issued ahead of its
// use -- the next cell's condensation coefficients under the current cell, the
// band columns D = 4 columns ahead of the substitution (registers, NV entries
// per lane with bw <= 32 NV) -- so a warp keeps several DRAM requests in flight
// instead of one latency per column.
template <int NV>
__device__ __forceinline__ void band_col(double2 (&v)[NV], const double2* band, int col, int ns, int LDB, int bw,
                                         int lane) {
#pragma unroll
    for (int t = 0; t < NV; ++t) {
        const int i = 1 + lane + 32 * t;
        v[t] = (col < ns && i <= bw) ? band[(size_t)col * LDB + i] : make_double2(0.0, 0.0);
    }
}

#ifndef HTG_BAND_D
#define HTG_BAND_D 12
#endif
#ifndef HTG_BAND_THREADS
#define HTG_BAND_THREADS 384
#endif
constexpr int kBandD = HTG_BAND_D, kBandThreads = HTG_BAND_THREADS;

// INV: the same solve with a unit right-hand side e_{U_u} per item, every cell's
// bubbles back-substituted, writing row u of B_c = A^-1[U, :] (A_s is complex
// symmetric, so A^-1 e_{U_u} is that row) for the dense-path classes
template <int P, int NV, bool INV = false>
__global__ void __launch_bounds__(kBandThreads) k_band_solve(FineGeom g, BandLaunch L, const double2* __restrict__ r,
                                                    double2* __restrict__ ystage, int nu_max) {
    constexpr int NB = 4 * P, NI = (P - 1) * (P - 1), NO = NI + NB, NR = (NO + 31) / 32;
    constexpr int D = NV <= 2 ? kBandD : 4;  // band columns in flight per lane
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double2* vec = reinterpret_cast<double2*>(smem_raw) + (size_t)warp * L.warp_elems;
    auto bub = [](int base, int NXn, int j) { return base + (1 + j / (P - 1)) * NXn + 1 + j % (P - 1); };
    const int nitems = INV ? L.ninv : L.nsub;
    for (int bs = blockIdx.x * nw + warp; bs < nitems; bs += gridDim.x * nw) {
        const int4 sd = INV ? L.inv_rows[bs] : L.subs[bs];  // INV: (factor unit, geometry, U row, kpad)
        const BandGeomDev G = L.geoms[sd.y];
        const int ox = sd.z & 0xffff, oy = sd.z >> 16;
        const double2* F = L.pool + (INV ? L.ffoff[sd.x] : L.foff[bs]);
        const double2* band = F + (size_t)G.ncell * G.cellstride;
        const int ns = G.ns, bw = G.bw, LDB = bw + 1, nn = G.NXn * G.NYn, NXn = G.NXn;
        double2* xs = vec + nn;  // skeleton vector
        // condensation coefficients of the next cell in registers (p <= 4: 9 per
        // lane at p = 4); larger cells read them in the loop
        constexpr bool PRE = NR * NI <= 16;
        double2 cf[PRE ? NR : 1][PRE ? NI : 1];
        auto load_cell = [&](int cell) {
            if constexpr (PRE) {
                const double2* Fc = F + (size_t)cell * G.cellstride;
#pragma unroll
                for (int t = 0; t < NR; ++t)
#pragma unroll
                    for (int j = 0; j < NI; ++j) {
                        const int o = lane + 32 * t;
                        cf[t][j] = o < NO ? Fc[j * NO + o] : make_double2(0.0, 0.0);
                    }
            }
        };
        load_cell(0);
        // gather g = r on Omega (lattice node order); INV: the unit vector of U row sd.z
        if constexpr (INV) {
            const int hot = G.uout[2 * sd.z];
            for (int n = lane; n < nn; n += 32) vec[n] = make_double2(n == hot ? 1.0 : 0.0, 0.0);
        } else {
            for (int n = lane; n < nn; n += 32) {
                const int gx = n % NXn, gy = n / NXn;
                vec[n] = r[dof_index(g.nx, g.ny, P, ox * P + gx, oy * P + gy)];
            }
        }
        __syncwarp();
        for (int s = lane; s < ns; s += 32) xs[s] = vec[G.skel_node[s]];
        __syncwarp();
        // condensation: y_I = A_II^-1 g_I (into the bubble nodes), g_B -= W^T g_I
        for (int cell = 0; cell < G.ncell; ++cell) {
            const int cx = cell % G.onx, cy = cell / G.onx;
            const int base = cy * P * NXn + cx * P;
            const int* cb = G.cell_bnd + (size_t)cell * NB;
            const double2* Fc = F + (size_t)cell * G.cellstride;
            double2 out[NR];
#pragma unroll
            for (int t = 0; t < NR; ++t) {
                const int o = lane + 32 * t;
                double2 s = make_double2(0.0, 0.0);
                if (o >= NI && o < NO) s = xs[cb[o - NI]];
#pragma unroll 7
                for (int j = 0; j < NI; ++j) {
                    const double2 gj = vec[bub(base, NXn, j)];
                    double2 c;
                    if constexpr (PRE) c = cf[PRE ? t : 0][PRE ? j : 0];
                    else c = o < NO ? Fc[j * NO + o] : make_double2(0.0, 0.0);
                    if (o < NI) cfma(s, c, gj);
                    else cfms(s, c, gj);
                }
                out[t] = s;
            }
            if (cell + 1 < G.ncell) load_cell(cell + 1);
            __syncwarp();
#pragma unroll
            for (int t = 0; t < NR; ++t) {
                const int o = lane + 32 * t;
                if (o < NI) vec[bub(base, NXn, o)] = out[t];
                else if (o < NO) xs[cb[o - NI]] = out[t];
            }
            __syncwarp();
        }
        // skeleton: L z = g (unit lower, by columns), z /= d, L^T x = z (dots); band
        // columns D ahead in registers
        double2 bv[D][NV];
#pragma unroll
        for (int t = 0; t < D; ++t) band_col<NV>(bv[t], band, t, ns, LDB, bw, lane);
        for (int j0 = 0; j0 < ns; j0 += D) {
#pragma unroll
            for (int t = 0; t < D; ++t) {
                const int j = j0 + t;
                if (j < ns) {
                    const double2 yj = xs[j];
#pragma unroll
                    for (int q = 0; q < NV; ++q) {
                        const int i = 1 + lane + 32 * q;
                        if (i <= bw && j + i < ns) cfms(xs[j + i], bv[t][q], yj);
                    }
                }
                band_col<NV>(bv[t], band, j + D, ns, LDB, bw, lane);
                __syncwarp();
            }
        }
        for (int j = lane; j < ns; j += 32) xs[j] = cmulb(xs[j], band[(size_t)j * LDB]);
        __syncwarp();
#pragma unroll
        for (int t = 0; t < D; ++t) band_col<NV>(bv[t], band, ns - 1 - t, ns, LDB, bw, lane);
        for (int j0 = ns - 1; j0 >= 0; j0 -= D) {
#pragma unroll
            for (int t = 0; t < D; ++t) {
                const int j = j0 - t;
                if (j >= 0) {
                    double2 s = make_double2(0.0, 0.0);
#pragma unroll
                    for (int q = 0; q < NV; ++q) {
                        const int i = 1 + lane + 32 * q;
                        if (i <= bw && j + i < ns) cfma(s, bv[t][q], xs[j + i]);
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
                        s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
                    }
                    if (lane == 0) xs[j] = make_double2(xs[j].x - s.x, xs[j].y - s.y);
                }
                if (j - D >= 0) band_col<NV>(bv[t], band, j - D, ns, LDB, bw, lane);
                __syncwarp();
            }
        }
        for (int s = lane; s < ns; s += 32) vec[G.skel_node[s]] = xs[s];
        __syncwarp();
        // bubbles of the U cells (INV: of every cell): x_I = y_I - W x_B (W row o of the
        // cell block: entries o * NO + NI + k)
        for (int uc = 0; uc < (INV ? G.ncell : G.nucell); ++uc) {
            const int cell = INV ? uc : G.ucells[uc];
            const int cx = cell % G.onx, cy = cell / G.onx;
            const int base = cy * P * NXn + cx * P;
            const double2* Fc = F + (size_t)cell * G.cellstride;
            const int* cb = G.cell_bnd + (size_t)cell * NB;
            for (int o = lane; o < NI; o += 32) {
                const int no = bub(base, NXn, o);
                double2 s = vec[no];
                for (int k = 0; k < NB; ++k) cfms(s, Fc[o * NO + NI + k], xs[cb[k]]);
                vec[no] = s;
            }
        }
        __syncwarp();
        if constexpr (INV) {
            double2* brow = L.Bmat + L.inv_off[bs];
            for (int l = lane; l < G.nloc; l += 32) brow[l] = vec[G.lnode[l]];
        } else {
            double2* yrow = ystage + (size_t)sd.x * nu_max;
            for (int e = lane; e < G.nu; e += 32) yrow[G.uout[2 * e + 1]] = vec[G.uout[2 * e]];
        }
        __syncwarp();
    }
}

}  // namespace

// ------------------------------------------------------------------ host
// Geometry of an Omega type: skeleton order (lattice rows; vertex-line rows
// carry every node, the other rows the vertical-edge nodes), half bandwidth,
// per-cell boundary-node -> skeleton maps, U outputs (node, U row) with the
// U-row order of the class (local reference dof order, as the combine table).
struct BandGeomHost {
    int onx, ony, ns = 0, bw = 0, nu = 0;
    std::vector<int> node_code, skel_node, cell_bnd, uout, ucells, lnode;
};

static BandGeomHost make_band_geom(int p, int onx, int ony, const std::vector<int>& umem) {
    BandGeomHost G;
    G.onx = onx;
    G.ony = ony;
    const int NXn = onx * p + 1, NYn = ony * p + 1, NB = 4 * p;
    G.node_code.assign(size_t(NXn) * NYn, -1);
    for (int gy = 0; gy < NYn; ++gy)
        for (int gx = 0; gx < NXn; ++gx)
            if (gx % p == 0 || gy % p == 0) {
                G.node_code[size_t(gy) * NXn + gx] = G.ns++;
                G.skel_node.push_back(gy * NXn + gx);
            }
    // per cell: skeleton index of each boundary slot (same slot order as bnd_node<P>)
    for (int cy = 0; cy < ony; ++cy)
        for (int cx = 0; cx < onx; ++cx) {
            std::vector<int> sl;
            for (int k = 0; k < NB; ++k) {
                int a, b;
                const int NE1 = p + 1;
                if (k < NE1) a = k, b = 0;
                else if (k >= 4 * p - NE1) a = k - (4 * p - NE1), b = p;
                else {
                    const int r = k - NE1;
                    b = 1 + r / 2;
                    a = (r & 1) ? p : 0;
                }
                const int s = G.node_code[size_t(cy * p + b) * NXn + cx * p + a];
                sl.push_back(s);
            }
            int lo = *std::min_element(sl.begin(), sl.end()), hi = *std::max_element(sl.begin(), sl.end());
            G.bw = std::max(G.bw, hi - lo);
            G.cell_bnd.insert(G.cell_bnd.end(), sl.begin(), sl.end());
        }
    // U outputs: local reference dof l = dof_index(onx, ony, p, gx, gy) -> lattice node
    std::vector<int> node_of(size_t(NXn) * NYn);
    for (int gy = 0; gy < NYn; ++gy)
        for (int gx = 0; gx < NXn; ++gx) node_of[size_t(dof_index(onx, ony, p, gx, gy))] = gy * NXn + gx;
    std::vector<char> ucell(size_t(onx) * ony, 0);
    for (int rI = 0; rI < int(umem.size()); ++rI) {
        const int node = node_of[size_t(umem[rI])];
        G.uout.push_back(node);
        G.uout.push_back(rI);
        const int gx = node % NXn, gy = node / NXn;
        if (gx % p && gy % p) ucell[size_t(gy / p) * onx + gx / p] = 1;  // a bubble of this cell is a U member
    }
    G.nu = int(umem.size());
    G.lnode = node_of;
    for (int c = 0; c < onx * ony; ++c)
        if (ucell[c]) G.ucells.push_back(c);
    return G;
}

BandLaunch band_setup(const FineGeom& g, const std::vector<BandSubdomain>& subs, const std::vector<BandInvJob>& jobs,
                      double2* Bmat, const Basis1D& basis, const std::vector<double>& khtab,
                      std::vector<void*>& allocs, size_t& bytes, cudaStream_t st) {
    BandLaunch L{};
    if (subs.empty() && jobs.empty()) return L;
    const int p = g.p;
    const int NI = (p - 1) * (p - 1), NB = 4 * p;
    std::map<std::vector<int>, int> gid;
    std::vector<BandGeomHost> geoms;
    std::vector<int4> sd, fsd;
    std::vector<long long> foff, ffoff;
    std::map<int, long long> cls_off;  // class -> its factor
    long long pool = 0;
    for (const BandSubdomain& s : subs) {
        std::vector<int> key{s.onx, s.ony};
        key.insert(key.end(), s.umem->begin(), s.umem->end());
        auto it = gid.find(key);
        if (it == gid.end()) {
            it = gid.emplace(key, int(geoms.size())).first;
            geoms.push_back(make_band_geom(p, s.onx, s.ony, *s.umem));
        }
        const BandGeomHost& G = geoms[it->second];
        const int4 e = make_int4(s.sid, it->second, s.ox | (s.oy << 16), 0);
        auto ct = cls_off.find(s.cls);
        if (ct == cls_off.end()) {  // first member: the class's factor unit
            ct = cls_off.emplace(s.cls, pool).first;
            fsd.push_back(e);
            ffoff.push_back(pool);
            pool += (long long)G.onx * G.ony * (NI * NI + NI * NB) + (long long)G.ns * (G.bw + 1);
        }
        sd.push_back(e);
        foff.push_back(ct->second);
    }
    // dense-path classes: their factor unit (the first member) and one item per U row
    std::vector<int4> inv_rows;
    std::vector<long long> inv_off;
    for (const BandInvJob& j : jobs) {
        std::vector<int> key{j.onx, j.ony};
        key.insert(key.end(), j.umem->begin(), j.umem->end());
        auto it = gid.find(key);
        if (it == gid.end()) {
            it = gid.emplace(key, int(geoms.size())).first;
            geoms.push_back(make_band_geom(p, j.onx, j.ony, *j.umem));
        }
        const BandGeomHost& G = geoms[it->second];
        const int unit = int(fsd.size());
        fsd.push_back(make_int4(j.sid, it->second, j.ox | (j.oy << 16), 0));
        ffoff.push_back(pool);
        pool += (long long)G.onx * G.ony * (NI * NI + NI * NB) + (long long)G.ns * (G.bw + 1);
        for (int u = 0; u < G.nu; ++u) {
            inv_rows.push_back(make_int4(unit, it->second, u, j.kpad));
            inv_off.push_back(j.boff + (long long)u * j.kpad);
        }
    }
    auto up = [&](const auto& v) {
        using T = typename std::decay_t<decltype(v)>::value_type;
        void* ptr = nullptr;
        HTG_CUDA(cudaMalloc(&ptr, std::max<size_t>(1, v.size()) * sizeof(T)));
        allocs.push_back(ptr);
        bytes += v.size() * sizeof(T);
        if (!v.empty()) HTG_CUDA(cudaMemcpyAsync(ptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
        return static_cast<const T*>(ptr);
    };
    std::vector<BandGeomDev> gd;
    size_t max_warp = 0;
    for (const BandGeomHost& G : geoms) {
        BandGeomDev d{};
        d.onx = G.onx;
        d.ony = G.ony;
        d.NXn = G.onx * p + 1;
        d.NYn = G.ony * p + 1;
        d.ns = G.ns;
        d.bw = G.bw;
        d.ncell = G.onx * G.ony;
        d.cellstride = NI * NI + NI * NB;
        d.nu = G.nu;
        d.nucell = int(G.ucells.size());
        d.node_code = up(G.node_code);
        d.skel_node = up(G.skel_node);
        d.cell_bnd = up(G.cell_bnd);
        d.uout = up(G.uout);
        d.ucells = up(G.ucells);
        d.lnode = up(G.lnode);
        d.nloc = int(G.lnode.size());
        gd.push_back(d);
        max_warp = std::max(max_warp, size_t(d.NXn) * d.NYn + size_t(d.ns));
    }
    L.geoms = up(gd);
    L.subs = up(sd);
    L.foff = up(foff);
    L.fsubs = up(fsd);
    L.ffoff = up(ffoff);
    L.nfac = int(fsd.size());
    L.inv_rows = up(inv_rows);
    L.inv_off = up(inv_off);
    L.ninv = int(inv_rows.size());
    L.Bmat = Bmat;
    L.khtab = up(khtab);
    std::vector<double> bt(2 * size_t(p + 1) * (p + 1));
    for (int a = 0; a <= p; ++a)
        for (int b = 0; b <= p; ++b) {
            bt[size_t(a) * (p + 1) + b] = basis.M[a][b];
            bt[size_t(p + 1) * (p + 1) + size_t(a) * (p + 1) + b] = basis.S[a][b];
        }
    L.basis = up(bt);
    void* pp = nullptr;
    HTG_CUDA(cudaMalloc(&pp, size_t(std::max<long long>(pool, 1)) * sizeof(double2)));
    allocs.push_back(pp);
    bytes += size_t(pool) * sizeof(double2);
    L.pool = static_cast<double2*>(pp);
    L.pool_elems = pool;
    L.nsub = int(subs.size());
    L.warp_elems = int((max_warp + 1) / 2 * 2);
    // sweep launch: as many warps per CTA as the per-warp vectors allow (<= 16)
    constexpr int kSmem = 232448;
    L.warps = int(std::min<size_t>(kBandThreads / 32, kSmem / (size_t(L.warp_elems) * sizeof(double2))));
    if (L.warps < 1) throw RuntimeError("band subdomain solver: Omega too large for shared memory");
    L.solve_smem = size_t(L.warps) * L.warp_elems * sizeof(double2);
    // setup: assemble, condense and factor every band subdomain on the device
    const int NE = (p + 1) * (p + 1);
    int ns_max = 0;
    for (const BandGeomDev& d : gd) ns_max = std::max(ns_max, d.ns), L.bw_max = std::max(L.bw_max, d.bw);
    const size_t fsm = (size_t(NE) * NE + size_t(NI) * NI + size_t(NI) * NB + NI) * sizeof(double2) + size_t(ns_max) * 4;
    if (fsm > size_t(kSmem) - 4096) throw RuntimeError("band subdomain solver: element too large for shared memory");
    const int nsm = current_sm_count();
    const int fgrid = std::min(L.nfac, nsm * std::max(1, std::min(8, int((kSmem - 4096) / fsm))));
    auto go = [&](auto kern) {
        // (the kernel also holds ~1.6 KB of static shared memory)
        HTG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem - 4096));
        kern<<<fgrid, 256, fsm, st>>>(g, L);
    };
    switch (p) {
        case 2: go(k_band_factor<2>); break;
        case 4: go(k_band_factor<4>); break;
        case 6: go(k_band_factor<6>); break;
        default: go(k_band_factor<8>); break;
    }
    HTG_CUDA(cudaGetLastError());
    count_launch();
    if (L.ninv > 0) {  // explicit restricted inverses of the dense-path classes
        const int nv = L.bw_max <= 64 ? 2 : (L.bw_max <= 128 ? 4 : 8);
        const int grid = (L.ninv + L.warps - 1) / L.warps;
        auto gi = [&](auto kern) {
            HTG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
            kern<<<grid, L.warps * 32, L.solve_smem, st>>>(g, L, nullptr, nullptr, 0);
        };
        switch (p * 10 + nv) {
            case 22: gi(k_band_solve<2, 2, true>); break;
            case 24: gi(k_band_solve<2, 4, true>); break;
            case 28: gi(k_band_solve<2, 8, true>); break;
            case 42: gi(k_band_solve<4, 2, true>); break;
            case 44: gi(k_band_solve<4, 4, true>); break;
            case 48: gi(k_band_solve<4, 8, true>); break;
            case 62: gi(k_band_solve<6, 2, true>); break;
            case 64: gi(k_band_solve<6, 4, true>); break;
            case 68: gi(k_band_solve<6, 8, true>); break;
            case 82: gi(k_band_solve<8, 2, true>); break;
            case 84: gi(k_band_solve<8, 4, true>); break;
            default: gi(k_band_solve<8, 8, true>); break;
        }
        HTG_CUDA(cudaGetLastError());
        count_launch();
    }
    HTG_CUDA(cudaStreamSynchronize(st));
    return L;
}

void band_solve_launch(const FineGeom& g, const BandLaunch& L, const double2* r, double2* ystage, int nu_max,
                       cudaStream_t st) {
    if (L.nsub == 0) return;
    static bool attr[12] = {};
    const int nsm = current_sm_count();
    const int grid = std::min((L.nsub + L.warps - 1) / L.warps, nsm * std::max(1, 16 / L.warps));
    auto go = [&](auto kern, int slot) {
        if (!attr[slot]) {
            HTG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
            attr[slot] = true;
        }
        kern<<<grid, L.warps * 32, L.solve_smem, st>>>(g, L, r, ystage, nu_max);
    };
    // band entries per lane: bw <= 32 NV
    const int nv = L.bw_max <= 64 ? 2 : (L.bw_max <= 128 ? 4 : 8);
    if (L.bw_max > 256) throw RuntimeError("band subdomain solver: half bandwidth above 256");
    switch (g.p * 10 + nv) {
        case 22: go(k_band_solve<2, 2>, 0); break;
        case 24: go(k_band_solve<2, 4>, 1); break;
        case 28: go(k_band_solve<2, 8>, 2); break;
        case 42: go(k_band_solve<4, 2>, 3); break;
        case 44: go(k_band_solve<4, 4>, 4); break;
        case 48: go(k_band_solve<4, 8>, 5); break;
        case 62: go(k_band_solve<6, 2>, 6); break;
        case 64: go(k_band_solve<6, 4>, 7); break;
        case 68: go(k_band_solve<6, 8>, 8); break;
        case 82: go(k_band_solve<8, 2>, 9); break;
        case 84: go(k_band_solve<8, 4>, 10); break;
        default: go(k_band_solve<8, 8>, 11); break;
    }
    HTG_CUDA(cudaGetLastError());
    count_launch();
}

}  // namespace htg
