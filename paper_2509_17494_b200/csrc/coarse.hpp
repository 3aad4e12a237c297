// coarse.hpp -- QSFEM coarse operator and its direct solver (factored once).
#pragma once

#include <cuda_runtime.h>

#include <memory>

#include "common.hpp"
#include "setup.hpp"

namespace htg {

// proj/core/src/qsfem.cpp:8-39: per-cell weights q0 = N P0/4, q1 = N P1/2,
// q2 = N P2 of the dispersion-minimising 9-point stencil at eta = k h_c.
struct QsfemWeights {
    double eta, P0, P1, P2, N, q0, q1, q2;
};
QsfemWeights qsfem_weights(double eta);

// Direct solve with the QSFEM coarse matrix (the reference factors it once with
// Eigen SparseLU, proj/core/src/twogrid.cpp:244, and solves at :273).
// Implementation: geometric nested dissection of the coarse vertex lattice,
// multifrontal LU with partial pivoting inside each front, factored on the host
// at setup; the per-level triangular solves run on the GPU as batched dense
// complex matvecs with explicit (L^-1 P), U^-1 blocks.
class CoarseSolver {
  public:
    virtual ~CoarseSolver() = default;
    virtual void solve(const double2* rc, double2* uc, cudaStream_t st) = 0;
    virtual size_t device_bytes() const = 0;
    virtual int levels() const = 0;
};
std::unique_ptr<CoarseSolver> make_coarse_solver(const HostProblem& hp, cudaStream_t st);

// 9-point coarse matrix rows: A9[v*9 + (dy+1)*3 + (dx+1)] = A_c[v][v + (dx, dy)]
// in the coarse p=1 vertex numbering (Y*(CX+1) + X), Dirichlet eliminated.
std::vector<cplx> coarse_stencil(const HostProblem& hp);

}  // namespace htg
