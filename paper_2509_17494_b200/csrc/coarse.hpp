// coarse.hpp -- QSFEM coarse operator and its direct solver (factored once).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <vector>

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

// ------------------------------------------------------------------ nested dissection
// Geometric nested dissection of the coarse vertex lattice. Each front is
// factored by LU with threshold partial pivoting inside its pivot block;
// columns without an acceptable pivot are delayed to the parent (coarse_nd.cpp).
// The factors are stored as explicit L11^-1, L21, U11^-1 and Z = U11^-1 U12
// blocks (row-major) for the GPU level kernels.
struct NDNode {
    int x0 = 0, x1 = 0, y0 = 0, y1 = 0;  // box of the subtree (inclusive vertex coordinates)
    int depth = 0;
    int parent = -1;
    bool leaf = false;
    std::vector<int> vars, ring, children;  // own separator vertices, boundary ring, child nodes
    // after factoring: front row / column labels in pivot order, F = sN + ring,
    // ke eliminated here, rows/cols [ke, F) form the contribution block
    int sN = 0, F = 0, ke = 0;
    std::vector<int> rows, cols;
    std::vector<int> rc;  // per front row: coarse vertex whose rhs entry is injected here, or -1
    std::vector<cplx> Finv, L21, Uinv, Z, S;  // factor blocks (host, freed after upload)
};
struct NDTree {
    int CX = 0, CY = 0;
    std::vector<NDNode> nodes;  // postorder: children before parents, root last
    int max_depth = 0;
    long long delayed = 0;  // pivots delayed to an ancestor (summed over nodes)
    int max_front = 0;
};
// Build and factor the tree. leaf_max: vertices per leaf box; pivtol: the
// threshold-pivoting tolerance in (0, 1] (0 = plain partial pivoting inside the block).
void nd_factor(const HostProblem& hp, NDTree& t, int leaf_max, double pivtol);

}  // namespace htg
