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
    // algorithmic bytes one solve reads: the nonzero halves of the triangular
    // pivot-block inverses plus the off-diagonal factor blocks, 16 B per entry
    virtual size_t solve_read_bytes() const = 0;
};
std::unique_ptr<CoarseSolver> make_coarse_solver(const HostProblem& hp, cudaStream_t st);

// 9-point coarse matrix rows: A9[v*9 + (dy+1)*3 + (dx+1)] = A_c[v][v + (dx, dy)]
// in the coarse p=1 vertex numbering (Y*(CX+1) + X), Dirichlet eliminated.
std::vector<cplx> coarse_stencil(const HostProblem& hp);

// ------------------------------------------------------------------ lattice matrices
// A sparse matrix with one unknown per node of a W x H lattice. The nested
// dissection cuts along lattice lines X % q == 0 (Y % q == 0): q = 1 for the
// 9-point QSFEM lattice; for an order-q FE space on the fine mesh a line of
// element-boundary nodes (vertices and edge functions of one mesh line)
// separates the cells on its two sides.
struct LatticeMatrix {
    int W = 0, H = 0, q = 1;
    std::vector<int> id;      // node Y * W + X -> unknown (row) index
    std::vector<int> rp, ci;  // CSR over unknowns, columns sorted
    std::vector<cplx> v;
    cplx at(int i, int j) const;
};
// the QSFEM coarse matrix on the (n m + 1)^2 vertex lattice (lexicographic unknowns)
LatticeMatrix qsfem_lattice(const HostProblem& hp);
// the order-q Helmholtz matrix A = sum_cells [K_e - (k^2 (1 + i alpha) + i eps) h^2 M_e]
// - sum_{absorbing edges} i k h m_e on the fine mesh, unknowns in the reference
// dof numbering of the order-q space, Dirichlet rows / columns replaced by the
// identity (proj/core/src/fespace.cpp:181-210,246-258). The order-q hierarchical
// functions are the first q + 1 of the order-p family, so the element factors
// are the leading blocks of the 1-D M, S.
LatticeMatrix fe_lattice(const HostProblem& hp, const Basis1D& b, int q, double alpha);
// per node (Y W + X) of the order-q lattice: on the closure of a Dirichlet edge
// (proj/core/src/fespace.cpp:146-153)
std::vector<char> fe_dirichlet(const HostProblem& hp, int q);

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
    // Fronts of one depth whose assembled matrices are bit-identical (the boxes of a
    // uniform medium away from the boundary) are factored once: rep >= 0 names the node
    // holding the blocks (this node's are empty; its rows / cols / rc are its own, in the
    // representative's pivot order). perm_r / perm_c: initial position of each final front
    // row / column (kept by representatives for their sharers).
    int rep = -1;
    std::vector<int> perm_r, perm_c;
};
// the node holding n's factor blocks
inline const NDNode& nd_blocks(const std::vector<NDNode>& nodes, const NDNode& n) {
    return n.rep < 0 ? n : nodes[size_t(n.rep)];
}
struct NDTree {
    int W = 0, H = 0, q = 1, nv = 0;
    std::vector<NDNode> nodes;  // postorder: children before parents, root last
    int max_depth = 0;
    long long delayed = 0;  // pivots delayed to an ancestor (summed over nodes)
    long long shared = 0;   // fronts that share another front's factor blocks
    int max_front = 0;
};
// Build and factor the tree. leaf_max: nodes per leaf box; pivtol: the
// threshold-pivoting tolerance in (0, 1] (0 = plain partial pivoting inside the block).
void nd_factor(const LatticeMatrix& A, NDTree& t, int leaf_max, double pivtol);
// the GPU direct solver of a lattice matrix (coarse.cu); make_coarse_solver is
// make_nd_solver(qsfem_lattice(hp))
std::unique_ptr<CoarseSolver> make_nd_solver(const LatticeMatrix& A, cudaStream_t st);

}  // namespace htg
