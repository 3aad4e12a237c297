// Minimal SparseMatrix subset of the Eigen 3.3+ API (compressed column storage),
// enough for the reference sources named in dense.hpp. TEST INFRASTRUCTURE ONLY.
//
// Semantics restated from Eigen's documentation:
//  * setFromTriplets sums duplicate entries in the order the triplets are given;
//  * prune(keep) drops the stored entries for which keep(row, col, value) is false;
//  * InnerIterator walks one column in increasing row order;
//  * coeffRef(i, j) inserts a zero entry when (i, j) is not stored;
//  * A * x is a column-oriented product (y += x_j A(:, j) in column order);
//  * A.adjoint() * x is the conjugate-transpose product.
#pragma once

#include <algorithm>
#include <numeric>

#include "dense.hpp"

namespace Eigen {

enum { ColMajor = 0, RowMajor = 0x1 };

template <class S, class SI = int>
class Triplet {
  public:
    Triplet() = default;
    Triplet(Index r, Index c, const S& v) : r_(SI(r)), c_(SI(c)), v_(v) {}
    SI row() const { return r_; }
    SI col() const { return c_; }
    const S& value() const { return v_; }

  private:
    SI r_ = 0, c_ = 0;
    S v_{};
};

template <class SM> class SparseAdjoint;

template <class S, int Options = ColMajor, class SI = int>
class SparseMatrix {
  public:
    using Scalar = S;
    using StorageIndex = SI;

    SparseMatrix() = default;
    SparseMatrix(Index rows, Index cols) { resize(rows, cols); }

    void resize(Index rows, Index cols) {
        rows_ = rows;
        cols_ = cols;
        outer_.assign(std::size_t(cols + 1), 0);
        inner_.clear();
        val_.clear();
    }
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index outerSize() const { return cols_; }
    Index innerSize() const { return rows_; }
    Index nonZeros() const { return Index(val_.size()); }
    void makeCompressed() {}
    bool isCompressed() const { return true; }

    const SI* outerIndexPtr() const { return outer_.data(); }
    const SI* innerIndexPtr() const { return inner_.data(); }
    const S* valuePtr() const { return val_.data(); }

    template <class It> void setFromTriplets(It begin, It end) {
        const std::size_t nt = std::size_t(std::distance(begin, end));
        std::vector<std::size_t> order(nt);
        std::vector<SI> tr(nt), tc(nt);
        std::vector<S> tv(nt);
        std::size_t t = 0;
        for (It it = begin; it != end; ++it, ++t) {
            tr[t] = SI(it->row());
            tc[t] = SI(it->col());
            tv[t] = S(it->value());
            if (tr[t] < 0 || tr[t] >= rows_ || tc[t] < 0 || tc[t] >= cols_)
                throw std::out_of_range("SparseMatrix::setFromTriplets: index out of range");
        }
        std::iota(order.begin(), order.end(), 0);
        // stable: duplicates keep their input order and are summed in that order
        std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) {
            return tc[a] != tc[b] ? tc[a] < tc[b] : tr[a] < tr[b];
        });
        outer_.assign(std::size_t(cols_ + 1), 0);
        inner_.clear();
        val_.clear();
        for (std::size_t q = 0; q < nt; ++q) {
            const std::size_t k = order[q];
            if (!inner_.empty() && q > 0 && tc[order[q - 1]] == tc[k] && inner_.back() == tr[k]) {
                val_.back() += tv[k];
                continue;
            }
            inner_.push_back(tr[k]);
            val_.push_back(tv[k]);
            outer_[std::size_t(tc[k]) + 1]++;
        }
        for (Index j = 0; j < cols_; ++j) outer_[std::size_t(j + 1)] += outer_[std::size_t(j)];
    }

    template <class Keep> void prune(Keep keep) {
        std::size_t w = 0;
        std::vector<SI> no(std::size_t(cols_ + 1), 0);
        for (Index j = 0; j < cols_; ++j) {
            for (SI p = outer_[std::size_t(j)]; p < outer_[std::size_t(j + 1)]; ++p) {
                if (keep(Index(inner_[std::size_t(p)]), j, val_[std::size_t(p)])) {
                    inner_[w] = inner_[std::size_t(p)];
                    val_[w] = val_[std::size_t(p)];
                    ++w;
                }
            }
            no[std::size_t(j + 1)] = SI(w);
        }
        inner_.resize(w);
        val_.resize(w);
        outer_ = std::move(no);
    }

    S coeff(Index i, Index j) const {
        const SI* b = inner_.data() + outer_[std::size_t(j)];
        const SI* e = inner_.data() + outer_[std::size_t(j + 1)];
        const SI* p = std::lower_bound(b, e, SI(i));
        return (p != e && *p == i) ? val_[std::size_t(p - inner_.data())] : S(0);
    }
    S& coeffRef(Index i, Index j) {
        const SI* b = inner_.data() + outer_[std::size_t(j)];
        const SI* e = inner_.data() + outer_[std::size_t(j + 1)];
        const SI* p = std::lower_bound(b, e, SI(i));
        std::size_t pos = std::size_t(p - inner_.data());
        if (p != e && *p == i) return val_[pos];
        inner_.insert(inner_.begin() + std::ptrdiff_t(pos), SI(i));
        val_.insert(val_.begin() + std::ptrdiff_t(pos), S(0));
        for (Index c = j + 1; c <= cols_; ++c) outer_[std::size_t(c)]++;
        return val_[pos];
    }

    class InnerIterator {
      public:
        InnerIterator(const SparseMatrix& m, Index outer)
            : m_(const_cast<SparseMatrix*>(&m)), j_(outer), p_(m.outer_[std::size_t(outer)]),
              end_(m.outer_[std::size_t(outer + 1)]) {}
        explicit operator bool() const { return p_ < end_; }
        InnerIterator& operator++() { ++p_; return *this; }
        Index row() const { return Index(m_->inner_[std::size_t(p_)]); }
        Index col() const { return j_; }
        Index index() const { return row(); }
        Index outer() const { return j_; }
        const S& value() const { return m_->val_[std::size_t(p_)]; }
        S& valueRef() { return m_->val_[std::size_t(p_)]; }

      private:
        SparseMatrix* m_;
        Index j_;
        SI p_, end_;
    };

    SparseMatrix& operator+=(const SparseMatrix& o) { return *this = combine(o, S(1)); }
    SparseMatrix& operator-=(const SparseMatrix& o) { return *this = combine(o, S(-1)); }

    SparseAdjoint<SparseMatrix> adjoint() const { return SparseAdjoint<SparseMatrix>(*this); }

    template <class S2, int R2, int C2> auto operator*(const Matrix<S2, R2, C2>& x) const {
        using T = shim::prod_t<S, S2>;
        if (x.rows() != cols_) throw std::invalid_argument("sparse * dense: size mismatch");
        Matrix<T, Dynamic, C2> y(rows_, x.cols());
        for (Index c = 0; c < x.cols(); ++c)
            for (Index j = 0; j < cols_; ++j) {
                const S2 xj = x(j, c);
                for (SI p = outer_[std::size_t(j)]; p < outer_[std::size_t(j + 1)]; ++p)
                    y(inner_[std::size_t(p)], c) += val_[std::size_t(p)] * xj;
            }
        return y;
    }
    template <class M> auto operator*(const Block<M>& x) const { return (*this) * x.eval(); }

  private:
    SparseMatrix combine(const SparseMatrix& o, S sign) const {
        if (o.rows_ != rows_ || o.cols_ != cols_) throw std::invalid_argument("sparse +/-: size mismatch");
        SparseMatrix r(rows_, cols_);
        r.inner_.reserve(inner_.size() + o.inner_.size());
        r.val_.reserve(inner_.size() + o.inner_.size());
        for (Index j = 0; j < cols_; ++j) {
            SI a = outer_[std::size_t(j)], ae = outer_[std::size_t(j + 1)];
            SI b = o.outer_[std::size_t(j)], be = o.outer_[std::size_t(j + 1)];
            while (a < ae || b < be) {
                const SI ra = a < ae ? inner_[std::size_t(a)] : SI(rows_);
                const SI rb = b < be ? o.inner_[std::size_t(b)] : SI(rows_);
                if (ra == rb) {
                    r.inner_.push_back(ra);
                    r.val_.push_back(val_[std::size_t(a++)] + sign * o.val_[std::size_t(b++)]);
                } else if (ra < rb) {
                    r.inner_.push_back(ra);
                    r.val_.push_back(val_[std::size_t(a++)]);
                } else {
                    r.inner_.push_back(rb);
                    r.val_.push_back(sign * o.val_[std::size_t(b++)]);
                }
            }
            r.outer_[std::size_t(j + 1)] = SI(r.inner_.size());
        }
        return r;
    }

    Index rows_ = 0, cols_ = 0;
    std::vector<SI> outer_{0};
    std::vector<SI> inner_;
    std::vector<S> val_;
};

/// Conjugate-transpose view; only its product with a dense vector is used.
template <class SM>
class SparseAdjoint {
  public:
    explicit SparseAdjoint(const SM& m) : m_(&m) {}
    template <class S2, int R2, int C2> auto operator*(const Matrix<S2, R2, C2>& x) const {
        using S = typename SM::Scalar;
        using T = shim::prod_t<S, S2>;
        if (x.rows() != m_->rows()) throw std::invalid_argument("adjoint * dense: size mismatch");
        Matrix<T, Dynamic, C2> y(m_->cols(), x.cols());
        const auto* op = m_->outerIndexPtr();
        const auto* ip = m_->innerIndexPtr();
        const auto* vp = m_->valuePtr();
        for (Index c = 0; c < x.cols(); ++c)
            for (Index j = 0; j < m_->cols(); ++j) {
                T s(0);
                for (auto p = op[j]; p < op[j + 1]; ++p) s += shim::conj_(vp[p]) * x(ip[p], c);
                y(j, c) = s;
            }
        return y;
    }

  private:
    const SM* m_;
};

}  // namespace Eigen
