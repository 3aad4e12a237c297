// nd_check.cpp -- TEST INFRASTRUCTURE (not part of the product library).
// Runs the coarse nested-dissection factorization of csrc/coarse_nd.cpp on the
// host and applies its explicit factors in the same order as the GPU level
// kernels (coarse.cu), so the factorization's accuracy (node amalgamation of
// near-resonant boxes) can be checked in the CPU test suite without a GPU.
#include <complex>
#include <cstring>
#include <exception>
#include <vector>

#include "coarse.hpp"

using htg::cplx;

namespace {
void matvec_sub(const std::vector<cplx>& M, int rows, int cols, const cplx* x, cplx* y, bool add) {
    for (int i = 0; i < rows; ++i) {
        cplx acc = 0.0;
        for (int j = 0; j < cols; ++j) acc += M[size_t(i) * cols + j] * x[j];
        y[i] = add ? y[i] + acc : acc;
    }
}
}  // namespace

extern "C" {

// The product's triangle element (csrc/tri.cpp): K, M (n x n), E (n x npts) and
// the lattice placement (4 ints per dof).
int nd_tri_element(int p, int sub, double* K, double* M, double* E, int* place, int* n, int* npts) {
    try {
        const htg::TriElement& T = htg::tri_element(p, sub);
        *n = T.n;
        *npts = T.npts;
        std::memcpy(K, T.K.data(), T.K.size() * sizeof(double));
        std::memcpy(M, T.M.data(), T.M.size() * sizeof(double));
        std::memcpy(E, T.E.data(), T.E.size() * sizeof(double));
        for (int i = 0; i < T.n; ++i)
            for (int c = 0; c < 4; ++c) place[4 * i + c] = T.place[i][c];
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// A9 stencil rows of the coarse matrix (nv * 9 complex = 18 doubles per vertex).
int nd_stencil(const htg_problem* prob, double* a9, long long cap) {
    try {
        const htg::HostProblem hp = htg::make_problem(*prob);
        const std::vector<cplx> A9 = htg::coarse_stencil(hp);
        if ((long long)A9.size() > cap) return 2;
        std::memcpy(a9, A9.data(), A9.size() * sizeof(cplx));
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// Factor and solve A_c x = rc for nrhs right-hand sides (interleaved complex),
// applying the explicit blocks exactly as the GPU level kernels do.
// stats: [delayed pivots, max front, live nodes, fronts sharing another front's factors]
static int nd_run(const htg::LatticeMatrix& A, int leaf, double pivtol, const double* rc, double* x, int nrhs,
                  double* stats) {
    try {
        htg::NDTree t;
        htg::nd_factor(A, t, leaf, pivtol);
        const int nv = t.nv;
        stats[0] = double(t.delayed);
        stats[1] = t.max_front;
        stats[2] = double(t.nodes.size());
        stats[3] = double(t.shared);
        const cplx* R = reinterpret_cast<const cplx*>(rc);
        cplx* X = reinterpret_cast<cplx*>(x);
        const int nn = int(t.nodes.size());
        std::vector<int> rpos(nv, -1);
        for (int r = 0; r < nrhs; ++r) {
            std::vector<std::vector<cplx>> contrib(nn);
            std::vector<cplx> Y(nv);
            const cplx* b = R + size_t(r) * nv;
            cplx* xo = X + size_t(r) * nv;
            for (int i = 0; i < nn; ++i) {  // postorder = children first
                const auto& n = t.nodes[i];
                const int s = n.ke, u = n.F - n.ke;
                std::vector<cplx> v(n.F, cplx(0.0));
                for (int k = 0; k < n.F; ++k) {
                    if (n.rc[k] >= 0) v[k] = b[n.rc[k]];
                    rpos[n.rows[k]] = k;
                }
                for (int c : n.children) {
                    const auto& ch = t.nodes[c];
                    for (int k = 0; k < ch.F - ch.ke; ++k) v[rpos[ch.rows[ch.ke + k]]] += contrib[c][k];
                }
                for (int k = 0; k < n.F; ++k) rpos[n.rows[k]] = -1;
                std::vector<cplx> y(s);
                matvec_sub(htg::nd_blocks(t.nodes, n).Finv, s, s, v.data(), y.data(), false);
                for (int k = 0; k < s; ++k) Y[n.cols[k]] = y[k];
                contrib[i].assign(v.begin() + s, v.end());
                std::vector<cplx> ly(u);
                matvec_sub(htg::nd_blocks(t.nodes, n).L21, u, s, y.data(), ly.data(), false);
                for (int k = 0; k < u; ++k) contrib[i][k] -= ly[k];
            }
            for (int i = nn - 1; i >= 0; --i) {
                const auto& n = t.nodes[i];
                const int s = n.ke, u = n.F - n.ke;
                std::vector<cplx> y1(s), x2(u), x1(s), z(s);
                for (int k = 0; k < s; ++k) y1[k] = Y[n.cols[k]];
                for (int k = 0; k < u; ++k) x2[k] = xo[n.cols[s + k]];
                matvec_sub(htg::nd_blocks(t.nodes, n).Uinv, s, s, y1.data(), x1.data(), false);
                if (u) matvec_sub(htg::nd_blocks(t.nodes, n).Z, s, u, x2.data(), z.data(), false);
                for (int k = 0; k < s; ++k) xo[n.cols[k]] = x1[k] - (u ? z[k] : cplx(0.0));
            }
        }
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

int nd_check(const htg_problem* prob, int leaf, double pivtol, const double* rc, double* x, int nrhs,
             double* stats) {
    try {
        const htg::HostProblem hp = htg::make_problem(*prob);
        return nd_run(htg::qsfem_lattice(hp), leaf, pivtol, rc, x, nrhs, stats);
    } catch (const std::exception&) {
        return 1;
    }
}

// the order-q FE lattice matrix of the product (GalerkinP coarse operator for
// q = p/2, the shifted fine operator of the ExactShifted smoother for q = p)
int nd_fe_apply(const htg_problem* prob, int q, double alpha, const double* xin, double* yout) {
    try {
        const htg::HostProblem hp = htg::make_problem(*prob);
        const htg::Basis1D b = htg::make_basis(hp.p);
        const htg::LatticeMatrix A = htg::fe_lattice(hp, b, q, alpha);
        const cplx* X = reinterpret_cast<const cplx*>(xin);
        cplx* Y = reinterpret_cast<cplx*>(yout);
        const int n = A.W * A.H;
        for (int i = 0; i < n; ++i) {
            cplx acc = 0.0;
            for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) acc += A.v[k] * X[A.ci[k]];
            Y[i] = acc;
        }
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

int nd_check_fe(const htg_problem* prob, int q, double alpha, int leaf, double pivtol, const double* rc, double* x,
                int nrhs, double* stats) {
    try {
        const htg::HostProblem hp = htg::make_problem(*prob);
        const htg::Basis1D b = htg::make_basis(hp.p);
        return nd_run(htg::fe_lattice(hp, b, q, alpha), leaf, pivtol, rc, x, nrhs, stats);
    } catch (const std::exception&) {
        return 1;
    }
}
}
