// k_dd.cu -- K2: the CSDD smoother's subdomain solves as one batched
// complex-fp64 GEMM on the FP64 tensor cores, plus the partition-of-unity combine.
//
// Reference: dd_step (proj/core/src/twogrid.cpp:92-112) gathers g on every
// Omega_i, runs one SparseLU solve per subdomain and averages the U-parts
// with 1/L_j. Subdomains with identical local operators share one factor; the
// host precomputes per class B_c = (A_s^(i))^-1[Dofs(U_i), :], so a sweep is
//   Y_c (|U| x N_c) = B_c (|U| x |Omega|) * G_c (|Omega| x N_c)
// where column s of G_c is the gathered residual of subdomain s. Each CTA
// computes a 64 x 64 tile of Y with mma.sync.m8n8k4.f64 (DMMA), the complex
// product as 4 real products; the gather is fused into the cp.async producer.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "common.hpp"
#include "kernels.hpp"
#include "setup.hpp"

namespace htg {

namespace {

constexpr int kTM = 64, kTN = 64, kKC = 8, kLD = kKC + 4, kStages = 4, kThreads = 256;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int sz = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

struct GemmSmem {
    double2 A[kStages][kTM][kLD];
    double2 B[kStages][kTN][kLD];
};

// 8 warps, warp tile 32 (rows) x 16 (subdomains): 4 x 2 DMMA accumulator tiles
template <int P>
__global__ void __launch_bounds__(kThreads, 2) k_dd_gemm(FineGeom g, DDDevice d, const double2* __restrict__ r,
                                                         double2* __restrict__ ystage) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    GemmSmem& sm = *reinterpret_cast<GemmSmem*>(smem_raw);
    const int4 tile = d.tiles[blockIdx.x];
    const int c = tile.x, m0 = tile.y, n0 = tile.z;
    const int* ci = d.cls_info + 8 * c;
    const int nu = ci[3], kpad = ci[4], loff = ci[6], ncol = ci[7];
    const int sub0 = tile.w;  // offset of this class's subdomain list
    const double2* Bc = d.Bmat + d.cls_boff[c];
    const int* locg = d.loc_g + loff;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 2, wn = warp & 3;

    // producer assignment: row/col tid/4, 2 k values each
    const int prow = tid >> 2, pk = (tid & 3) * 2;
    const double2* arow = Bc + (size_t)(m0 + prow) * kpad;
    const int col = n0 + prow;
    const bool colok = col < ncol;
    int ox = 0, oy = 0;
    if (colok) {
        const int so = d.sub_o[d.class_subs[sub0 + col]];
        ox = (so & 0xffff) * P;
        oy = (so >> 16) * P;
    }
    const int nkc = kpad / kKC;
    // m8 tiles of this warp that hold real U rows (the last M-tile is partial)
    const int mt_valid = max(0, min(4, (nu - (m0 + wm * 32) + 7) / 8));
    const bool nt_any = n0 + wn * 16 < ncol;

    auto load_stage = [&](int stage, int kc) {
        const int k0 = kc * kKC + pk;
#pragma unroll
        for (int i = 0; i < 2; ++i) cp_async16(&sm.A[stage][prow][pk + i], arow + k0 + i, true);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int lg = locg[k0 + i];
            const bool ok = colok && lg >= 0;
            const double2* src = r;
            if (ok) src = r + dof_index(g.nx, g.ny, P, ox + (lg & 0xffff), oy + (lg >> 16));
            cp_async16(&sm.B[stage][prow][pk + i], src, ok);
        }
    };

    double cr[4][2][2], cim[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            cr[a][b][0] = cr[a][b][1] = 0.0;
            cim[a][b][0] = cim[a][b][1] = 0.0;
        }

#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < nkc) load_stage(s, s);
        cp_commit();
    }
    for (int kc = 0; kc < nkc; ++kc) {
        cp_wait<kStages - 2>();
        __syncthreads();
        const int stage = kc % kStages;
        const int nxt = kc + kStages - 1;
        if (nxt < nkc) load_stage(nxt % kStages, nxt);
        cp_commit();
        if (nt_any) {
#pragma unroll
            for (int ks = 0; ks < kKC / 4; ++ks) {
                const int kk = ks * 4 + (lane & 3);
                double2 af[4], bf[2];
#pragma unroll
                for (int t = 0; t < 4; ++t) af[t] = sm.A[stage][wm * 32 + t * 8 + (lane >> 2)][kk];
#pragma unroll
                for (int t = 0; t < 2; ++t) bf[t] = sm.B[stage][wn * 16 + t * 8 + (lane >> 2)][kk];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) {
                    if (mt >= mt_valid) break;
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt) {
                        dmma(cr[mt][nt][0], cr[mt][nt][1], af[mt].x, bf[nt].x);
                        dmma(cim[mt][nt][0], cim[mt][nt][1], af[mt].x, bf[nt].y);
                    }
                }
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) {
                    if (mt >= mt_valid) break;
                    const double nai = -af[mt].y;
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt) {
                        dmma(cr[mt][nt][0], cr[mt][nt][1], nai, bf[nt].y);
                        dmma(cim[mt][nt][0], cim[mt][nt][1], af[mt].y, bf[nt].x);
                    }
                }
            }
        }
    }
    cp_wait<0>();
    // epilogue: C[row][col], row = lane/4, col = 2 (lane%4) + i
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
        const int row = m0 + wm * 32 + mt * 8 + (lane >> 2);
        if (row >= nu) continue;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int cc = n0 + wn * 16 + nt * 8 + 2 * (lane & 3) + i;
                if (cc >= ncol) continue;
                const int s = d.class_subs[sub0 + cc];
                ystage[(size_t)s * d.nu_max + row] = make_double2(cr[mt][nt][i], cim[mt][nt][i]);
            }
    }
}

// out = u + (sum over U-memberships of Y) / L, summed in subdomain order; one
// thread per fine dof in storage order (coalesced u / out / table), the staged
// values are gathered (they were just written and sit in L2)
__global__ void k_dd_combine(long long ndof, DDDevice d, const double2* __restrict__ ystage, const double2* u,
                             double2* out) {
    const long long di = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (di >= ndof) return;
    const int src = d.srcmap[di];
    double2 acc;
    double inv = 1.0;
    if (src >= 0) {
        acc = ystage[src];
    } else {
        const int k = -1 - src, b0 = d.bptr[k], b1 = d.bptr[k + 1];
        acc = make_double2(0.0, 0.0);
        for (int b = b0; b < b1; ++b) {
            const double2 yv = ystage[d.bsrc[b]];
            acc.x += yv.x;
            acc.y += yv.y;
        }
        inv = 1.0 / double(b1 - b0);
    }
    const double2 base = u ? u[di] : make_double2(0.0, 0.0);
    out[di] = make_double2(base.x + acc.x * inv, base.y + acc.y * inv);
}

}  // namespace

void dd_gemm_launch(const FineGeom& g, const DDDevice& d, const double2* r, double2* ystage, cudaStream_t st) {
    if (d.ntiles == 0) return;
    const size_t smem = sizeof(GemmSmem);
    static bool attr[9] = {};
    auto go = [&](auto kern, int p) {
        if (!attr[p]) {
            HTG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            attr[p] = true;
        }
        kern<<<d.ntiles, kThreads, smem, st>>>(g, d, r, ystage);
    };
    switch (g.p) {
        case 2: go(k_dd_gemm<2>, 2); break;
        case 4: go(k_dd_gemm<4>, 4); break;
        case 6: go(k_dd_gemm<6>, 6); break;
        default: go(k_dd_gemm<8>, 8); break;
    }
    HTG_CUDA(cudaGetLastError());
    count_launch();
}

void dd_combine_launch(const FineGeom& g, const DDDevice& d, const double2* ystage, const double2* u, double2* out,
                       cudaStream_t st) {
    k_dd_combine<<<unsigned((g.ndof + 255) / 256), 256, 0, st>>>(g.ndof, d, ystage, u, out);
    HTG_CUDA(cudaGetLastError());
    count_launch();
}

// Host: lay the classes out for the kernels (padded B_c, local gather tables,
// U-row maps, tile list) and upload.
DDDevice upload_dd_impl(const DDSetup& dd, const HostProblem& hp, std::vector<void*>& allocs, size_t& bytes,
                        cudaStream_t st, double2*& ystage, std::vector<FdmClassDev>& fdm,
                        std::vector<BandSubdomain>& band, std::vector<BandInvJob>& jobs) {
    DDDevice d;
    const int nc = int(dd.classes.size());
    d.nclass = nc;
    d.nbx = dd.nbx;
    d.nby = dd.nby;
    d.nsub = dd.nbx * dd.nby;
    d.l_dd = dd.l_dd;
    const int p = hp.p;
    std::vector<int> info(8 * nc), locg, rowmap, class_subs;
    std::vector<long long> boff(nc);
    std::vector<double2> Bm;
    std::vector<int4> tiles;
    std::vector<std::vector<int>> subs(nc);
    for (int s = 0; s < d.nsub; ++s) subs[dd.sub_class[s]].push_back(s);
    int nu_max = 0;
    for (int ci = 0; ci < nc; ++ci) {
        const DDClass& c = dd.classes[ci];
        const int kpad = (c.nloc + kKC - 1) / kKC * kKC;
        const int rpad = (c.nu + kTM - 1) / kTM * kTM;
        nu_max = std::max(nu_max, c.nu);
        int* in = &info[8 * ci];
        in[0] = c.onx;
        in[1] = c.ony;
        in[2] = c.nloc;
        in[3] = c.nu;
        in[4] = kpad;
        in[5] = 0;
        boff[ci] = (long long)Bm.size();
        in[6] = int(locg.size());
        in[7] = int(subs[ci].size());
        const size_t b0 = Bm.size();
        const bool fdm_cls = c.fdm && fdm_supported(p, c.fdm_nx, c.fdm_ny);  // no dense B (setup.cpp)
        if (!c.band && !fdm_cls) Bm.resize(b0 + size_t(rpad) * kpad, make_double2(0.0, 0.0));
        if (c.devB && !subs[ci].empty()) {  // B_c filled on the device (k_band.cu) from a band factor
            const int s0 = subs[ci][0];
            jobs.push_back({s0, dd.sub_ox[s0], dd.sub_oy[s0], c.onx, c.ony, &c.umem, ci, (long long)b0, kpad});
        }
        for (int rI = 0; rI < (c.band || c.devB || fdm_cls ? 0 : c.nu); ++rI)
            for (int l = 0; l < c.nloc; ++l) {
                const cplx v = c.B[size_t(rI) * c.nloc + l];
                Bm[b0 + size_t(rI) * kpad + l] = make_double2(v.real(), v.imag());
            }
        // local dof -> (lgx, lgy), and local dof -> U row
        std::vector<int> lg(kpad, -1), rm(kpad, -1);
        for (int gy = 0; gy <= c.ony * p; ++gy)
            for (int gx = 0; gx <= c.onx * p; ++gx) lg[dof_index(c.onx, c.ony, p, gx, gy)] = gx | (gy << 16);
        for (int rI = 0; rI < c.nu; ++rI) rm[c.umem[rI]] = rI;
        locg.insert(locg.end(), lg.begin(), lg.end());
        rowmap.insert(rowmap.end(), rm.begin(), rm.end());
        const int off = int(class_subs.size());
        class_subs.insert(class_subs.end(), subs[ci].begin(), subs[ci].end());
        if (c.band) {  // per-member device factors (k_band.cu)
            for (int sI : subs[ci]) band.push_back({sI, dd.sub_ox[sI], dd.sub_oy[sI], c.onx, c.ony, &c.umem, ci});
            continue;
        }
        if (c.fdm && fdm_supported(p, c.fdm_nx, c.fdm_ny)) {
            FdmClassDev f{};
            f.nx = c.fdm_nx;
            f.ny = c.fdm_ny;
            f.nux = c.fdm_nux;
            f.nuy = c.fdm_nuy;
            f.ux0 = c.fdm_ux0;
            f.uy0 = c.fdm_uy0;
            f.onx = c.onx;
            f.ony = c.ony;
            f.nsub = int(subs[ci].size());
            f.rowmap = reinterpret_cast<const int*>(size_t(in[6]));  // offsets, patched below
            f.subs = reinterpret_cast<const int*>(size_t(off));
            std::vector<double2> vx(c.Vx.size()), vy(c.Vy.size()), dv(c.Dinv.size());
            for (size_t i = 0; i < vx.size(); ++i) vx[i] = make_double2(c.Vx[i].real(), c.Vx[i].imag());
            for (size_t i = 0; i < vy.size(); ++i) vy[i] = make_double2(c.Vy[i].real(), c.Vy[i].imag());
            for (size_t i = 0; i < dv.size(); ++i) dv[i] = make_double2(c.Dinv[i].real(), c.Dinv[i].imag());
            auto put = [&](const std::vector<double2>& v) {
                void* ptr = nullptr;
                HTG_CUDA(cudaMalloc(&ptr, v.size() * sizeof(double2)));
                allocs.push_back(ptr);
                bytes += v.size() * sizeof(double2);
                HTG_CUDA(cudaMemcpyAsync(ptr, v.data(), v.size() * sizeof(double2), cudaMemcpyHostToDevice, st));
                HTG_CUDA(cudaStreamSynchronize(st));
                return static_cast<const double2*>(ptr);
            };
            f.Vx = put(vx);
            f.Vy = put(vy);
            f.Dinv = put(dv);
            if (c.fdm_sym) {
                auto putc = [&](const std::vector<cplx>& v) {
                    std::vector<double2> w(v.size());
                    for (size_t i = 0; i < v.size(); ++i) w[i] = make_double2(v[i].real(), v[i].imag());
                    return put(w);
                };
                f.sym = 1;
                f.Vxe = putc(c.Vxe);
                f.Vxo = putc(c.Vxo);
                f.Vye = putc(c.Vye);
                f.Vyo = putc(c.Vyo);
                std::vector<int> mr(c.mirror.size());
                for (size_t i = 0; i < mr.size(); ++i) mr[i] = c.mirror[i] | ((c.msign[i] > 0 ? 1 : 0) << 16);
                void* ptr = nullptr;
                HTG_CUDA(cudaMalloc(&ptr, mr.size() * sizeof(int)));
                allocs.push_back(ptr);
                bytes += mr.size() * sizeof(int);
                HTG_CUDA(cudaMemcpy(ptr, mr.data(), mr.size() * sizeof(int), cudaMemcpyHostToDevice));
                f.mir = static_cast<const int*>(ptr);
            }
            {  // relative gather offsets, shared by every member of the class (checked)
                const int nx = f.nx, ny = f.ny;
                std::vector<int> go(size_t(nx) * ny);
                bool same = true;
                for (size_t m = 0; m < subs[ci].size() && same; ++m) {
                    const int sI = subs[ci][m];
                    const int gx0 = dd.sub_ox[sI] * p, gy0 = dd.sub_oy[sI] * p;
                    const long long base = dof_index(hp.nx, hp.ny, p, gx0, gy0);
                    for (int iy = 0; iy < ny && same; ++iy)
                        for (int ix = 0; ix < nx; ++ix) {
                            const int o = int(dof_index(hp.nx, hp.ny, p, gx0 + ix, gy0 + iy) - base);
                            if (m == 0) go[size_t(iy) * nx + ix] = o;
                            else if (go[size_t(iy) * nx + ix] != o) { same = false; break; }
                        }
                }
                if (same) {
                    void* ptr = nullptr;
                    HTG_CUDA(cudaMalloc(&ptr, go.size() * sizeof(int)));
                    allocs.push_back(ptr);
                    bytes += go.size() * sizeof(int);
                    HTG_CUDA(cudaMemcpy(ptr, go.data(), go.size() * sizeof(int), cudaMemcpyHostToDevice));
                    f.goff = static_cast<const int*>(ptr);
                    // memory order of the gather: consecutive lanes copy consecutive 16-byte dofs
                    std::vector<int> ord(go.size());
                    for (size_t i = 0; i < ord.size(); ++i) ord[i] = int(i);
                    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return go[a] < go[b]; });
                    void* po = nullptr;
                    HTG_CUDA(cudaMalloc(&po, ord.size() * sizeof(int)));
                    allocs.push_back(po);
                    bytes += ord.size() * sizeof(int);
                    HTG_CUDA(cudaMemcpy(po, ord.data(), ord.size() * sizeof(int), cudaMemcpyHostToDevice));
                    f.gord = static_cast<const int*>(po);
                }
            }
            fdm.push_back(f);
            continue;
        }
        for (int m0 = 0; m0 < c.nu; m0 += kTM)
            for (int n0 = 0; n0 < int(subs[ci].size()); n0 += kTN) tiles.push_back(make_int4(ci, m0, n0, off));
    }
    // partition-of-unity combine table: every fine dof's staged values in subdomain order
    std::vector<int> srcmap(size_t(hp.ndof()), 0), bptr{0}, bsrc;
    {
        // counting sort of the (subdomain, U row) pairs by fine dof, subdomain order kept
        const size_t nd = size_t(hp.ndof());
        std::vector<int> start(nd + 1, 0);
        std::vector<long long> pair_dof;
        pair_dof.reserve(size_t(d.nsub) * nu_max);
        for (int s = 0; s < d.nsub; ++s) {
            const int ci = dd.sub_class[s];
            const DDClass& c = dd.classes[ci];
            const int lo = info[8 * ci + 6];
            for (int rI = 0; rI < c.nu; ++rI) {
                const int lxy = locg[lo + c.umem[rI]];
                const int gx = dd.sub_ox[s] * p + (lxy & 0xffff), gy = dd.sub_oy[s] * p + (lxy >> 16);
                const long long di = dof_index(hp.nx, hp.ny, p, gx, gy);
                pair_dof.push_back(di);
                ++start[size_t(di) + 1];
            }
        }
        for (size_t di = 0; di < nd; ++di) start[di + 1] += start[di];
        std::vector<int> flat(pair_dof.size()), fill(start.begin(), start.end() - 1);
        {
            size_t k = 0;
            for (int s = 0; s < d.nsub; ++s) {
                const int nu = dd.classes[dd.sub_class[s]].nu;
                for (int rI = 0; rI < nu; ++rI) flat[size_t(fill[size_t(pair_dof[k++])]++)] = s * nu_max + rI;
            }
        }
        for (size_t di = 0; di < nd; ++di) {
            const int b0 = start[di], n = start[di + 1] - b0;
            if (n == 0) throw RuntimeError("dd setup: fine dof outside every subdomain U");
            if (n == 1) {
                srcmap[di] = flat[size_t(b0)];
            } else {
                srcmap[di] = -int(bptr.size());
                bsrc.insert(bsrc.end(), flat.begin() + b0, flat.begin() + b0 + n);
                bptr.push_back(int(bsrc.size()));
            }
        }
    }
    // big classes first
    std::stable_sort(tiles.begin(), tiles.end(), [&](const int4& a, const int4& b) {
        return info[8 * a.x + 4] * 1.0 > info[8 * b.x + 4] * 1.0;
    });
    std::vector<int> sub_o(d.nsub);
    for (int s = 0; s < d.nsub; ++s) sub_o[s] = dd.sub_ox[s] | (dd.sub_oy[s] << 16);
    auto up = [&](const auto& v) {
        using T = typename std::decay_t<decltype(v)>::value_type;
        void* ptr = nullptr;
        HTG_CUDA(cudaMalloc(&ptr, std::max<size_t>(1, v.size()) * sizeof(T)));
        allocs.push_back(ptr);
        bytes += v.size() * sizeof(T);
        if (!v.empty()) HTG_CUDA(cudaMemcpyAsync(ptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
        return static_cast<const T*>(ptr);
    };
    d.cls_info = up(info);
    d.cls_boff = up(boff);
    d.Bmat = up(Bm);
    d.loc_g = up(locg);
    d.rowmap = up(rowmap);
    d.sub_class = up(dd.sub_class);
    d.sub_o = up(sub_o);
    d.tiles = up(tiles);
    d.class_subs = up(class_subs);
    d.ntiles = int(tiles.size());
    d.nu_max = nu_max;
    d.srcmap = up(srcmap);
    d.bptr = up(bptr);
    d.bsrc = up(bsrc);
    for (FdmClassDev& f : fdm) {  // patch offsets into device pointers
        f.rowmap = d.rowmap + size_t(f.rowmap);
        f.subs = d.class_subs + size_t(f.subs);
        f.sub_o = d.sub_o;
    }
    void* ys = nullptr;
    const size_t ysz = size_t(d.nsub) * nu_max * sizeof(double2);
    HTG_CUDA(cudaMalloc(&ys, std::max<size_t>(ysz, 16)));
    allocs.push_back(ys);
    bytes += ysz;
    ystage = static_cast<double2*>(ys);
    return d;
}

}  // namespace htg

// ------------------------------------------------------------------ FP64 tensor peak
namespace htg {
namespace {
__global__ void k_dmma_peak(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[8][2];
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0.0;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int t = 0; t < 8; ++t) dmma(c[t][0], c[t][1], a, b);
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
}  // namespace
}  // namespace htg

extern "C" int htg_measure_fp64_tensor_peak(double* tflops) {
    using namespace htg;
    try {
        int sms = 0;
        sms = current_sm_count();
        const int blocks = sms * 2, threads = 512, iters = 4096;
        double* out = nullptr;
        HTG_CUDA(cudaMalloc(&out, sizeof(double) * blocks * threads));
        cudaEvent_t e0, e1;
        HTG_CUDA(cudaEventCreate(&e0));
        HTG_CUDA(cudaEventCreate(&e1));
        k_dmma_peak<<<blocks, threads>>>(out, 64);
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            HTG_CUDA(cudaEventRecord(e0));
            k_dmma_peak<<<blocks, threads>>>(out, iters);
            HTG_CUDA(cudaEventRecord(e1));
            HTG_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            HTG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            best = std::min(best, ms);
        }
        count_launch(4);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(out);
        const double flops = double(blocks) * (threads / 32) * iters * 8 * 512.0;
        *tflops = flops / (best * 1e-3) / 1e12;
        return 0;
    } catch (const std::exception& e) {
        return 1;
    }
}
