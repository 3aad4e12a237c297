// Eigen::SparseLU stand-in for the reference build (oracle/_ref). TEST
// INFRASTRUCTURE ONLY.
//
// Eigen's SparseLU (supernodal, COLAMD column ordering, partial pivoting with
// diagonal threshold 1.0) is restated as:
//  * analyzePattern: a nested-dissection column ordering of the symmetric
//    pattern A + A^T (BFS level-structure separators from a pseudo-peripheral
//    node, thinned; leaves <= 32 nodes kept in natural order);
//  * factorize: left-looking sparse LU (Gilbert-Peierls: sparse triangular
//    solve per column over the depth-first reach in the graph of L) with
//    partial pivoting; the diagonal row is taken when it is the largest
//    candidate (threshold 1.0, as Eigen's default);
//  * solve: P A Q = L U, forward/back substitution.
// Results agree with Eigen's at round-off (both are backward-stable LU).
#pragma once

#include <string>

#include "sparse.hpp"

namespace Eigen {

template <class T> struct COLAMDOrdering {};

template <class SparseMatrixType, class Ordering = COLAMDOrdering<int>>
class SparseLU {
  public:
    using S = typename SparseMatrixType::Scalar;

    SparseLU() = default;
    explicit SparseLU(const SparseMatrixType& a) { compute(a); }
    void compute(const SparseMatrixType& a) {
        analyzePattern(a);
        factorize(a);
    }
    void setPivotThreshold(double t) { thresh_ = t; }

    void analyzePattern(const SparseMatrixType& a) {
        n_ = a.rows();
        if (a.cols() != n_) throw std::invalid_argument("SparseLU: square matrix required");
        q_ = nested_dissection(a);
    }

    void factorize(const SparseMatrixType& a) {
        info_ = Success;
        msg_.clear();
        const Index n = n_;
        const auto* Ap = a.outerIndexPtr();
        const auto* Ai = a.innerIndexPtr();
        const S* Ax = a.valuePtr();
        Lp_.assign(std::size_t(n + 1), 0);
        Up_.assign(std::size_t(n + 1), 0);
        Li_.clear(); Lx_.clear(); Ui_.clear(); Ux_.clear();
        Li_.reserve(std::size_t(a.nonZeros()) * 4);
        Lx_.reserve(std::size_t(a.nonZeros()) * 4);
        Ui_.reserve(std::size_t(a.nonZeros()) * 4);
        Ux_.reserve(std::size_t(a.nonZeros()) * 4);
        Ud_.assign(std::size_t(n), S(0));
        pinv_.assign(std::size_t(n), -1);
        std::vector<S> x(std::size_t(n), S(0));
        std::vector<Index> xi(static_cast<std::size_t>(n)), stack(static_cast<std::size_t>(n)), pstack(static_cast<std::size_t>(n));
        std::vector<Index> mark(std::size_t(n), -1);
        for (Index k = 0; k < n; ++k) {
            const Index col = q_[std::size_t(k)];
            // depth-first reach of A(:, col) in the graph of L (original row ids)
            Index top = n;
            for (auto p = Ap[col]; p < Ap[col + 1]; ++p) {
                const Index i0 = Ai[p];
                if (mark[std::size_t(i0)] == k) continue;
                Index head = 0;
                stack[0] = i0;
                while (head >= 0) {
                    const Index j = stack[std::size_t(head)];
                    const Index jc = pinv_[std::size_t(j)];
                    if (mark[std::size_t(j)] != k) {
                        mark[std::size_t(j)] = k;
                        pstack[std::size_t(head)] = jc < 0 ? 0 : Lp_[std::size_t(jc)];
                    }
                    bool done = true;
                    const Index pend = jc < 0 ? 0 : Lp_[std::size_t(jc + 1)];
                    for (Index q = pstack[std::size_t(head)]; q < pend; ++q) {
                        const Index i = Li_[std::size_t(q)];
                        if (mark[std::size_t(i)] == k) continue;
                        pstack[std::size_t(head)] = q + 1;
                        stack[std::size_t(++head)] = i;
                        done = false;
                        break;
                    }
                    if (done) {
                        --head;
                        xi[std::size_t(--top)] = j;
                    }
                }
            }
            for (auto p = Ap[col]; p < Ap[col + 1]; ++p) x[std::size_t(Ai[p])] = Ax[p];
            for (Index t = top; t < n; ++t) {
                const Index i = xi[std::size_t(t)];
                const Index jc = pinv_[std::size_t(i)];
                if (jc < 0) continue;
                const S xj = x[std::size_t(i)];
                if (xj == S(0)) continue;
                for (Index q = Lp_[std::size_t(jc)]; q < Lp_[std::size_t(jc + 1)]; ++q)
                    x[std::size_t(Li_[std::size_t(q)])] -= Lx_[std::size_t(q)] * xj;
            }
            // pivot among the non-pivotal rows of the reach
            Index piv = -1;
            double best = -1;
            for (Index t = top; t < n; ++t) {
                const Index i = xi[std::size_t(t)];
                if (pinv_[std::size_t(i)] >= 0) {
                    Ui_.push_back(int(pinv_[std::size_t(i)]));
                    Ux_.push_back(x[std::size_t(i)]);
                    continue;
                }
                const double v = std::abs(x[std::size_t(i)]);
                if (v > best) { best = v; piv = i; }
            }
            if (piv < 0 || best <= 0.0) {
                info_ = NumericalIssue;
                msg_ = "THE MATRIX IS STRUCTURALLY OR NUMERICALLY SINGULAR at column " + std::to_string(k);
                return;
            }
            if (pinv_[std::size_t(col)] < 0 && mark[std::size_t(col)] == k &&
                std::abs(x[std::size_t(col)]) >= thresh_ * best)
                piv = col;
            const S pv = x[std::size_t(piv)];
            Ud_[std::size_t(k)] = pv;
            pinv_[std::size_t(piv)] = k;
            for (Index t = top; t < n; ++t) {
                const Index i = xi[std::size_t(t)];
                if (pinv_[std::size_t(i)] < 0) {
                    Li_.push_back(int(i));
                    Lx_.push_back(x[std::size_t(i)] / pv);
                }
                x[std::size_t(i)] = S(0);
            }
            Lp_[std::size_t(k + 1)] = Index(Li_.size());
            Up_[std::size_t(k + 1)] = Index(Ui_.size());
        }
        for (auto& i : Li_) i = int(pinv_[std::size_t(i)]);
        Li_.shrink_to_fit(); Lx_.shrink_to_fit(); Ui_.shrink_to_fit(); Ux_.shrink_to_fit();
        prow_.assign(std::size_t(n), 0);
        for (Index i = 0; i < n; ++i) prow_[std::size_t(pinv_[std::size_t(i)])] = i;
    }

    ComputationInfo info() const { return info_; }
    std::string lastErrorMessage() const { return msg_; }
    Index rows() const { return n_; }
    Index cols() const { return n_; }
    Index nnzL() const { return Index(Li_.size()); }
    Index nnzU() const { return Index(Ui_.size()) + n_; }

    template <class M> Matrix<S, Dynamic, 1> solve(const M& b_) const {
        const auto& b = shim::ev(b_);
        const Index n = n_;
        std::vector<S> c(static_cast<std::size_t>(n));
        for (Index k = 0; k < n; ++k) c[std::size_t(k)] = b(prow_[std::size_t(k)]);
        for (Index k = 0; k < n; ++k) {
            const S ck = c[std::size_t(k)];
            if (ck == S(0)) continue;
            for (Index q = Lp_[std::size_t(k)]; q < Lp_[std::size_t(k + 1)]; ++q)
                c[std::size_t(Li_[std::size_t(q)])] -= Lx_[std::size_t(q)] * ck;
        }
        for (Index k = n - 1; k >= 0; --k) {
            c[std::size_t(k)] /= Ud_[std::size_t(k)];
            const S ck = c[std::size_t(k)];
            if (ck == S(0)) continue;
            for (Index q = Up_[std::size_t(k)]; q < Up_[std::size_t(k + 1)]; ++q)
                c[std::size_t(Ui_[std::size_t(q)])] -= Ux_[std::size_t(q)] * ck;
        }
        Matrix<S, Dynamic, 1> x(n);
        for (Index k = 0; k < n; ++k) x(q_[std::size_t(k)]) = c[std::size_t(k)];
        return x;
    }

  private:
    static std::vector<Index> nested_dissection(const SparseMatrixType& a) {
        const Index n = a.rows();
        // symmetric adjacency of A + A^T without the diagonal
        std::vector<std::vector<Index>> adj(static_cast<std::size_t>(n));
        const auto* Ap = a.outerIndexPtr();
        const auto* Ai = a.innerIndexPtr();
        for (Index j = 0; j < n; ++j)
            for (auto p = Ap[j]; p < Ap[j + 1]; ++p) {
                const Index i = Ai[p];
                if (i == j) continue;
                adj[std::size_t(i)].push_back(j);
                adj[std::size_t(j)].push_back(i);
            }
        std::vector<Index> xadj(std::size_t(n + 1), 0), nbr;
        for (Index i = 0; i < n; ++i) {
            auto& v = adj[std::size_t(i)];
            std::sort(v.begin(), v.end());
            v.erase(std::unique(v.begin(), v.end()), v.end());
            xadj[std::size_t(i + 1)] = xadj[std::size_t(i)] + Index(v.size());
        }
        nbr.reserve(std::size_t(xadj[std::size_t(n)]));
        for (auto& v : adj) nbr.insert(nbr.end(), v.begin(), v.end());
        adj.clear();
        adj.shrink_to_fit();

        std::vector<Index> order;
        order.reserve(static_cast<std::size_t>(n));
        std::vector<Index> part(std::size_t(n), 0), level(std::size_t(n), -1);
        Index next_part = 1;
        std::vector<Index> all(static_cast<std::size_t>(n));
        std::iota(all.begin(), all.end(), 0);
        // explicit work stack: (node list, part id); separators are emitted after both halves
        struct Item { std::vector<Index> nodes; Index id; bool emit; };
        std::vector<Item> work;
        work.push_back({std::move(all), 0, false});
        std::vector<Index> queue;
        auto bfs = [&](Index root, Index id, std::vector<Index>& out) {
            out.clear();
            out.push_back(root);
            level[std::size_t(root)] = 0;
            for (std::size_t h = 0; h < out.size(); ++h) {
                const Index u = out[h];
                for (Index p = xadj[std::size_t(u)]; p < xadj[std::size_t(u + 1)]; ++p) {
                    const Index v = nbr[std::size_t(p)];
                    if (part[std::size_t(v)] != id || level[std::size_t(v)] >= 0) continue;
                    level[std::size_t(v)] = level[std::size_t(u)] + 1;
                    out.push_back(v);
                }
            }
        };
        auto reset = [&](const std::vector<Index>& nodes) {
            for (Index v : nodes) level[std::size_t(v)] = -1;
        };
        while (!work.empty()) {
            Item it = std::move(work.back());
            work.pop_back();
            if (it.emit || it.nodes.size() <= 32) {
                std::vector<Index> s = std::move(it.nodes);
                std::sort(s.begin(), s.end());
                order.insert(order.end(), s.begin(), s.end());
                continue;
            }
            const Index id = it.id;
            // pseudo-peripheral root
            Index root = *std::min_element(it.nodes.begin(), it.nodes.end());
            Index ecc = -1;
            for (int sweep = 0; sweep < 4; ++sweep) {
                bfs(root, id, queue);
                const Index far = queue.back();
                const Index e = level[std::size_t(far)];
                reset(queue);
                if (e <= ecc) break;
                ecc = e;
                root = far;
            }
            bfs(root, id, queue);
            if (queue.size() < it.nodes.size()) {  // disconnected: split off this component
                std::vector<Index> comp = queue, rest;
                reset(queue);
                const Index ida = next_part++, idb = next_part++;
                for (Index v : comp) part[std::size_t(v)] = ida;
                for (Index v : it.nodes)
                    if (part[std::size_t(v)] == id) { part[std::size_t(v)] = idb; rest.push_back(v); }
                work.push_back({std::move(rest), idb, false});
                work.push_back({std::move(comp), ida, false});
                continue;
            }
            const Index nlev = level[std::size_t(queue.back())] + 1;
            if (nlev < 3) {
                reset(queue);
                work.push_back({std::move(it.nodes), id, true});
                continue;
            }
            std::vector<Index> cnt(std::size_t(nlev), 0);
            for (Index v : queue) cnt[std::size_t(level[std::size_t(v)])]++;
            Index m = 1, cum = cnt[0];
            while (m < nlev - 2 && 2 * (cum + cnt[std::size_t(m)]) < Index(queue.size())) cum += cnt[std::size_t(m++)];
            std::vector<Index> A, B, Sep;
            for (Index v : queue) {
                const Index l = level[std::size_t(v)];
                if (l < m) A.push_back(v);
                else if (l > m) B.push_back(v);
                else {
                    bool touches_b = false;
                    for (Index p = xadj[std::size_t(v)]; p < xadj[std::size_t(v + 1)] && !touches_b; ++p) {
                        const Index w = nbr[std::size_t(p)];
                        touches_b = part[std::size_t(w)] == id && level[std::size_t(w)] == m + 1;
                    }
                    (touches_b ? Sep : A).push_back(v);
                }
            }
            reset(queue);
            if (Sep.empty() || B.empty()) {  // no usable separator: order this set as a leaf
                work.push_back({std::move(it.nodes), id, true});
                continue;
            }
            const Index ida = next_part++, idb = next_part++, ids = next_part++;
            for (Index v : A) part[std::size_t(v)] = ida;
            for (Index v : B) part[std::size_t(v)] = idb;
            for (Index v : Sep) part[std::size_t(v)] = ids;
            work.push_back({std::move(Sep), ids, true});
            work.push_back({std::move(B), idb, false});
            work.push_back({std::move(A), ida, false});
        }
        return order;
    }

    Index n_ = 0;
    double thresh_ = 1.0;
    ComputationInfo info_ = InvalidInput;
    std::string msg_;
    std::vector<Index> q_, pinv_, prow_;
    std::vector<Index> Lp_, Up_;
    std::vector<int> Li_, Ui_;  // 32-bit row ids keep the factors of large problems compact
    std::vector<S> Lx_, Ux_, Ud_;
};

}  // namespace Eigen
