// common.hpp -- shared host/device types of the helmtg_b200 library.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace htg {

// Errors: thrown on the host, mapped to status codes at the C-ABI boundary.
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct RuntimeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define HTG_CUDA(call)                                                                          \
    do {                                                                                        \
        cudaError_t e_ = (call);                                                                \
        if (e_ != cudaSuccess)                                                                  \
            throw ::htg::RuntimeError(std::string("CUDA error ") + cudaGetErrorString(e_) +     \
                                      " at " __FILE__ ":" + std::to_string(__LINE__));          \
    } while (0)

// SM count of the calling thread's current device (handles may live on any device)
inline int current_sm_count() {
    int dev = 0, n = 0;
    HTG_CUDA(cudaGetDevice(&dev));
    HTG_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    return n;
}

constexpr int kMaxP = 8;
constexpr int8_t kDirichlet = 0, kNeumann = 1, kAbsorbing = 2;

// Geometry + coefficients of the fine level as the kernels see them. The dof
// numbering is the reference's (proj/core/src/fespace.cpp:37-54): lattice point
// (x, y) owns vertex, h-edge (p-1), v-edge (p-1), interior (p-1)^2, with
// offset(x, y) = y (nx p^2 + p) + (y < ny ? x p^2 : x p).
// In tensor form a dof is a pair (gx, gy) of 1-D hierarchical indices,
// g = x p + j, j = 0 the vertex function, j >= 1 the bubble of degree j + 1.
struct FineGeom {
    int nx, ny, p;
    long long ndof;
    // per-cell coefficient class (nullptr: one class for every cell)
    const uint32_t* cls;
    // complex mass weight m = (k^2 (1 + i alpha) + i eps) h^2 per class, for
    // alpha = 0 (mtab0) and alpha = alpha_s (mtabS)
    const double2* mtab0;
    const double2* mtabS;
    // Robin k h per boundary edge (0 when the edge is not absorbing) and tags
    const double *kh_b, *kh_t, *kh_l, *kh_r;
    const int8_t *tg_b, *tg_t, *tg_l, *tg_r;
    int has_dirichlet;
};

// Coarse (QSFEM, p = 1) lattice: (nx m + 1) x (ny m + 1) vertices, m = p/2.
struct CoarseGeom {
    int cnx, cny, m;
    long long ndof;
    // per fine cell coefficient class -> stencil weights (q0, q1, q2) and the
    // i eps hc^2 mass weight; Robin k hc per coarse boundary edge (by fine edge)
    const double4* qtab;  // q0, q1, q2, eps*hc^2
    double hc;
};

inline __host__ __device__ long long dof_index(int nx, int ny, int p, int gx, int gy) {
    const int x = gx / p, jx = gx - x * p;
    const int y = gy / p, jy = gy - y * p;
    const long long row = (long long)nx * p * p + p;
    const long long base = (long long)y * row + (y < ny ? (long long)x * p * p : (long long)x * p);
    if (jx == 0 && jy == 0) return base;
    if (jy == 0) return base + jx;
    if (jx == 0) return base + (x < nx ? p : 1) + (jy - 1);
    return base + 2 * p - 1 + (long long)(jx - 1) * (p - 1) + (jy - 1);
}

}  // namespace htg

// The mirror-symmetric (parity) path of the FDM subdomain kernel (k_fdm.cu) and its
// host factors (fdm.cpp, HTG_FDM_SYM=1) are compiled only on request: the path halves
// the DMMA work but was never faster (0.212 vs 0.216 ms at cfg4), and its code slows
// the default path through the instruction cache (187.5 vs 196.5 us without / with it).
#ifndef HTG_FDM_SYM_CODE
#define HTG_FDM_SYM_CODE 0
#endif
