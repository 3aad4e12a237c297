// Minimal dense-matrix subset of the Eigen 3.3+ API, written for this repo so
// that the UNMODIFIED reference hot-path sources
//   /root/reference/proj/core/src/{basis,fespace,mesh,qsfem,twogrid,linalg,parallel}.cpp
// compile here (Eigen itself is absent: proj/core/CMakeLists.txt:1 requires it).
//
// TEST INFRASTRUCTURE ONLY (oracle/_ref). This is not Eigen's source: it is an
// eager (no expression templates), column-major restatement of the documented
// semantics of the calls those files make. Only what they use is provided.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <concepts>
#include <cstddef>
#include <initializer_list>
#include <limits>
#include <stdexcept>
#include <type_traits>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };
enum DecompositionOptions { EigenvaluesOnly = 0x40, ComputeEigenvectors = 0x80 };

namespace shim {
template <class T> struct is_complex : std::false_type {};
template <class T> struct is_complex<std::complex<T>> : std::true_type {};
template <class T> inline T conj_(const T& v) {
    if constexpr (is_complex<T>::value) return std::conj(v); else return v;
}
template <class T> inline double abs_(const T& v) { return std::abs(v); }
template <class T> inline double abs2_(const T& v) {
    if constexpr (is_complex<T>::value) return std::norm(v); else return v * v;
}
template <class T> concept ScalarT = std::is_arithmetic_v<T> || is_complex<T>::value;
template <class A, class B> using prod_t = decltype(std::declval<A>() * std::declval<B>());
}  // namespace shim

template <class S, int R = Dynamic, int C = Dynamic> class Matrix;
template <class M> class Block;
template <class M> class ArrayRef;
template <class M> class PartialPivLU;
template <class M> class ColPivHouseholderQR;

template <class T> struct is_dense : std::false_type {};
template <class S, int R, int C> struct is_dense<Matrix<S, R, C>> : std::true_type {};
template <class M> struct is_dense<Block<M>> : std::true_type {};
template <class T> concept DenseT = is_dense<std::remove_cvref_t<T>>::value;

namespace shim {
// operand access without copies for matrices (a block is materialised)
template <class S, int R, int C> const Matrix<S, R, C>& ev(const Matrix<S, R, C>& m);
template <class M> Matrix<typename M::Scalar> ev(const Block<M>& b);
}  // namespace shim

template <class S, int R, int C>
class Matrix {
  public:
    using Scalar = S;
    using RealScalar = double;
    static constexpr int RowsAtCompileTime = R, ColsAtCompileTime = C;

    Matrix() : r_(R == Dynamic ? 0 : R), c_(C == Dynamic ? 0 : C), d_(std::size_t(r_ * c_)) {}
    explicit Matrix(Index n) { resize(n); }
    Matrix(Index r, Index c) { resize(r, c); }
    Matrix(const Matrix&) = default;
    Matrix(Matrix&&) noexcept = default;
    Matrix& operator=(const Matrix&) = default;
    Matrix& operator=(Matrix&&) noexcept = default;

    template <class S2, int R2, int C2>
        requires std::convertible_to<S2, S>
    Matrix(const Matrix<S2, R2, C2>& o) : r_(o.rows()), c_(o.cols()), d_(o.size()) {
        for (Index i = 0; i < size(); ++i) d_[i] = S(o.data()[i]);
    }
    template <class M> Matrix(const Block<M>& b) : Matrix(b.eval()) {}
    template <class S2, int R2, int C2>
        requires std::convertible_to<S2, S>
    Matrix& operator=(const Matrix<S2, R2, C2>& o) { return *this = Matrix(o); }
    template <class M> Matrix& operator=(const Block<M>& b) { return *this = Matrix(b.eval()); }

    static Matrix Zero() { return Matrix(); }
    static Matrix Zero(Index n) { return Matrix(n); }
    static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
    static Matrix Identity(Index r, Index c) {
        Matrix m(r, c);
        for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = S(1);
        return m;
    }
    static Matrix Identity() { return Identity(R, C); }

    void resize(Index n) {
        if constexpr (R == 1) resize(1, n); else resize(n, 1);
    }
    void resize(Index r, Index c) {
        r_ = r;
        c_ = c;
        d_.assign(std::size_t(r * c), S(0));
    }
    void setZero() { std::fill(d_.begin(), d_.end(), S(0)); }
    void setZero(Index r, Index c) { resize(r, c); }

    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    S* data() { return d_.data(); }
    const S* data() const { return d_.data(); }

    S& operator()(Index i) { return d_[std::size_t(i)]; }
    const S& operator()(Index i) const { return d_[std::size_t(i)]; }
    S& operator()(Index i, Index j) { return d_[std::size_t(i + j * r_)]; }
    const S& operator()(Index i, Index j) const { return d_[std::size_t(i + j * r_)]; }
    S& operator[](Index i) { return d_[std::size_t(i)]; }
    const S& operator[](Index i) const { return d_[std::size_t(i)]; }

    Block<Matrix> row(Index i) { return Block<Matrix>(*this, i, 0, 1, c_); }
    Block<Matrix> col(Index j) { return Block<Matrix>(*this, 0, j, r_, 1); }
    Matrix<S, 1, Dynamic> row(Index i) const { return block_copy<1, Dynamic>(i, 0, 1, c_); }
    Matrix<S, Dynamic, 1> col(Index j) const { return block_copy<Dynamic, 1>(0, j, r_, 1); }
    Block<Matrix> block(Index i, Index j, Index r, Index c) { return Block<Matrix>(*this, i, j, r, c); }
    Matrix<S> block(Index i, Index j, Index r, Index c) const { return block_copy<Dynamic, Dynamic>(i, j, r, c); }
    Matrix<S> topLeftCorner(Index r, Index c) const { return block_copy<Dynamic, Dynamic>(0, 0, r, c); }

    Matrix<S, C, R> transpose() const {
        Matrix<S, C, R> t(c_, r_);
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) t(j, i) = (*this)(i, j);
        return t;
    }
    Matrix<S, C, R> adjoint() const {
        Matrix<S, C, R> t(c_, r_);
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) t(j, i) = shim::conj_((*this)(i, j));
        return t;
    }
    Matrix conjugate() const {
        Matrix t(*this);
        for (auto& v : t.d_) v = shim::conj_(v);
        return t;
    }
    Matrix eval() const { return *this; }
    template <class T> Matrix<T, R, C> cast() const {
        Matrix<T, R, C> t(r_, c_);
        for (Index i = 0; i < size(); ++i) t.data()[i] = T(d_[std::size_t(i)]);
        return t;
    }
    Matrix<double, R, C> cwiseAbs() const {
        Matrix<double, R, C> t(r_, c_);
        for (Index i = 0; i < size(); ++i) t.data()[i] = std::abs(d_[std::size_t(i)]);
        return t;
    }

    double squaredNorm() const {
        double s = 0;
        for (const auto& v : d_) s += shim::abs2_(v);
        return s;
    }
    double norm() const { return std::sqrt(squaredNorm()); }
    S sum() const {
        S s(0);
        for (const auto& v : d_) s += v;
        return s;
    }
    /// conjugate-linear in the first argument (Eigen's dot)
    template <class S2, int R2, int C2> auto dot(const Matrix<S2, R2, C2>& o) const {
        shim::prod_t<S, S2> s(0);
        for (Index i = 0; i < size(); ++i) s += shim::conj_(d_[std::size_t(i)]) * o.data()[i];
        return s;
    }
    S minCoeff() const { return *std::min_element(d_.begin(), d_.end()); }
    S maxCoeff() const { return *std::max_element(d_.begin(), d_.end()); }

    Matrix inverse() const;  // defined with PartialPivLU below
    PartialPivLU<Matrix<S>> partialPivLu() const;
    ColPivHouseholderQR<Matrix<S>> colPivHouseholderQr() const;

    ArrayRef<Matrix> array() { return ArrayRef<Matrix>(*this); }
    ArrayRef<const Matrix> array() const { return ArrayRef<const Matrix>(*this); }

    template <DenseT O> Matrix& operator+=(const O& o) {
        const auto& e = shim::ev(o);
        check_same(e);
        for (Index i = 0; i < size(); ++i) d_[std::size_t(i)] += e.data()[i];
        return *this;
    }
    template <DenseT O> Matrix& operator-=(const O& o) {
        const auto& e = shim::ev(o);
        check_same(e);
        for (Index i = 0; i < size(); ++i) d_[std::size_t(i)] -= e.data()[i];
        return *this;
    }
    template <shim::ScalarT T> Matrix& operator*=(const T& s) {
        for (auto& v : d_) v *= s;
        return *this;
    }
    template <shim::ScalarT T> Matrix& operator/=(const T& s) {
        for (auto& v : d_) v /= s;
        return *this;
    }

    class CommaInit;
    CommaInit operator<<(const S& v) { return CommaInit(this, v); }

  private:
    template <int R2, int C2> Matrix<S, R2, C2> block_copy(Index i0, Index j0, Index r, Index c) const {
        Matrix<S, R2, C2> b(r, c);
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) b(i, j) = (*this)(i0 + i, j0 + j);
        return b;
    }
    template <class E> void check_same(const E& e) const {
        if (e.rows() != r_ || e.cols() != c_) throw std::invalid_argument("eigen shim: size mismatch");
    }
    Index r_ = 0, c_ = 0;
    std::vector<S> d_;
    template <class S2, int R2, int C2> friend class Matrix;
};

/// Comma initializer: fills row-major, as Eigen does.
template <class S, int R, int C>
class Matrix<S, R, C>::CommaInit {
  public:
    CommaInit(Matrix* m, const S& v) : m_(m) { put(v); }
    CommaInit& operator,(const S& v) { put(v); return *this; }
  private:
    void put(const S& v) {
        const Index i = k_ / m_->cols(), j = k_ % m_->cols();
        (*m_)(i, j) = v;
        ++k_;
    }
    Matrix* m_;
    Index k_ = 0;
};

/// Writable rectangular view of a matrix (row(), col(), block() of a non-const matrix).
template <class M>
class Block {
  public:
    using Scalar = typename M::Scalar;
    Block(M& m, Index i0, Index j0, Index r, Index c) : m_(&m), i0_(i0), j0_(j0), r_(r), c_(c) {}
    Block(const Block&) = default;
    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    Scalar& operator()(Index i, Index j) { return (*m_)(i0_ + i, j0_ + j); }
    const Scalar& operator()(Index i, Index j) const { return (*m_)(i0_ + i, j0_ + j); }
    Scalar& operator()(Index k) { return r_ == 1 ? (*this)(0, k) : (*this)(k, 0); }
    const Scalar& operator()(Index k) const { return r_ == 1 ? (*this)(0, k) : (*this)(k, 0); }

    Matrix<Scalar> eval() const {
        Matrix<Scalar> out(r_, c_);
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) out(i, j) = (*this)(i, j);
        return out;
    }
    Block& operator=(const Block& o) { return assign(o.eval()); }
    template <DenseT O> Block& operator=(const O& o) { return assign(o.eval()); }
    template <DenseT O> Block& operator+=(const O& o) { return assign(eval() + o.eval()); }
    template <DenseT O> Block& operator-=(const O& o) { return assign(eval() - o.eval()); }
    auto transpose() const { return eval().transpose(); }
    double norm() const { return eval().norm(); }
    auto cwiseAbs() const { return eval().cwiseAbs(); }
    Scalar maxCoeff() const { return eval().maxCoeff(); }

    class CommaInit {
      public:
        CommaInit(Block* b, const Scalar& v) : b_(b) { put(v); }
        CommaInit& operator,(const Scalar& v) { put(v); return *this; }
      private:
        void put(const Scalar& v) {
            (*b_)(k_ / b_->cols(), k_ % b_->cols()) = v;
            ++k_;
        }
        Block* b_;
        Index k_ = 0;
    };
    CommaInit operator<<(const Scalar& v) { return CommaInit(this, v); }

  private:
    template <class E> Block& assign(const E& e) {
        if (e.rows() * e.cols() != r_ * c_) throw std::invalid_argument("eigen shim: block size mismatch");
        // vectors may be assigned across orientation (row <- column of equal length)
        const bool same = e.rows() == r_;
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) (*this)(i, j) = same ? e(i, j) : e.data()[i + j * r_];
        return *this;
    }
    M* m_;
    Index i0_, j0_, r_, c_;
};

/// Coefficient-wise view (array()); only the compound division the reference uses.
template <class M>
class ArrayRef {
  public:
    explicit ArrayRef(M& m) : m_(&m) {}
    M& matrix() const { return *m_; }
    template <class M2> ArrayRef& operator/=(const ArrayRef<M2>& o) {
        for (Index i = 0; i < m_->size(); ++i) m_->data()[i] /= o.matrix().data()[i];
        return *this;
    }
    template <class M2> ArrayRef& operator*=(const ArrayRef<M2>& o) {
        for (Index i = 0; i < m_->size(); ++i) m_->data()[i] *= o.matrix().data()[i];
        return *this;
    }
  private:
    M* m_;
};

namespace shim {
template <class S, int R, int C> inline const Matrix<S, R, C>& ev(const Matrix<S, R, C>& m) { return m; }
template <class M> inline Matrix<typename M::Scalar> ev(const Block<M>& b) { return b.eval(); }
template <class E> struct eval_type { using type = std::remove_cvref_t<decltype(std::declval<const E&>().eval())>; };
template <class E> using ev_t = typename eval_type<std::remove_cvref_t<E>>::type;
}  // namespace shim

// ---- arithmetic (eager) ----
template <DenseT A, DenseT B> auto operator+(const A& a_, const B& b_) {
    const auto& a = shim::ev(a_);
    const auto& b = shim::ev(b_);
    using S = decltype(a.data()[0] + b.data()[0]);
    using EA = shim::ev_t<A>;
    Matrix<S, EA::RowsAtCompileTime, EA::ColsAtCompileTime> out(a.rows(), a.cols());
    if (a.size() != b.size()) throw std::invalid_argument("eigen shim: + size mismatch");
    for (Index i = 0; i < a.size(); ++i) out.data()[i] = a.data()[i] + b.data()[i];
    return out;
}
template <DenseT A, DenseT B> auto operator-(const A& a_, const B& b_) {
    const auto& a = shim::ev(a_);
    const auto& b = shim::ev(b_);
    using S = decltype(a.data()[0] - b.data()[0]);
    using EA = shim::ev_t<A>;
    Matrix<S, EA::RowsAtCompileTime, EA::ColsAtCompileTime> out(a.rows(), a.cols());
    if (a.size() != b.size()) throw std::invalid_argument("eigen shim: - size mismatch");
    for (Index i = 0; i < a.size(); ++i) out.data()[i] = a.data()[i] - b.data()[i];
    return out;
}
template <DenseT A> auto operator-(const A& a_) {
    auto out = shim::ev(a_).eval();
    for (Index i = 0; i < out.size(); ++i) out.data()[i] = -out.data()[i];
    return out;
}
template <DenseT A, shim::ScalarT T> auto operator*(const A& a_, const T& s) {
    const auto& a = shim::ev(a_);
    using S = shim::prod_t<typename shim::ev_t<A>::Scalar, T>;
    using EA = shim::ev_t<A>;
    Matrix<S, EA::RowsAtCompileTime, EA::ColsAtCompileTime> out(a.rows(), a.cols());
    for (Index i = 0; i < a.size(); ++i) out.data()[i] = a.data()[i] * s;
    return out;
}
template <shim::ScalarT T, DenseT A> auto operator*(const T& s, const A& a_) {
    const auto& a = shim::ev(a_);
    using S = shim::prod_t<T, typename shim::ev_t<A>::Scalar>;
    using EA = shim::ev_t<A>;
    Matrix<S, EA::RowsAtCompileTime, EA::ColsAtCompileTime> out(a.rows(), a.cols());
    for (Index i = 0; i < a.size(); ++i) out.data()[i] = s * a.data()[i];
    return out;
}
template <DenseT A, shim::ScalarT T> auto operator/(const A& a_, const T& s) {
    const auto& a = shim::ev(a_);
    using S = decltype(std::declval<typename shim::ev_t<A>::Scalar>() / s);
    using EA = shim::ev_t<A>;
    Matrix<S, EA::RowsAtCompileTime, EA::ColsAtCompileTime> out(a.rows(), a.cols());
    for (Index i = 0; i < a.size(); ++i) out.data()[i] = a.data()[i] / s;
    return out;
}
template <DenseT A, DenseT B> auto operator*(const A& a_, const B& b_) {
    const auto& a = shim::ev(a_);
    const auto& b = shim::ev(b_);
    using SA = typename shim::ev_t<A>::Scalar;
    using SB = typename shim::ev_t<B>::Scalar;
    using S = shim::prod_t<SA, SB>;
    if (a.cols() != b.rows()) throw std::invalid_argument("eigen shim: product size mismatch");
    Matrix<S, shim::ev_t<A>::RowsAtCompileTime, shim::ev_t<B>::ColsAtCompileTime> out(a.rows(), b.cols());
    for (Index j = 0; j < b.cols(); ++j)
        for (Index k = 0; k < a.cols(); ++k) {
            const SB bkj = b(k, j);
            for (Index i = 0; i < a.rows(); ++i) out(i, j) += a(i, k) * bkj;
        }
    return out;
}

// ---- dense decompositions ----

/// LU with partial (row) pivoting, P A = L U.
template <class MatrixType>
class PartialPivLU {
  public:
    using S = typename MatrixType::Scalar;
    PartialPivLU() = default;
    template <class M> explicit PartialPivLU(const M& a) { compute(a.eval()); }
    template <class M> PartialPivLU& compute(const M& a_) {
        lu_ = Matrix<S>(a_.eval());
        const Index n = lu_.rows();
        if (lu_.cols() != n) throw std::invalid_argument("PartialPivLU: square matrix required");
        perm_.resize(std::size_t(n));
        for (Index i = 0; i < n; ++i) perm_[std::size_t(i)] = i;
        norm1_ = 0;
        for (Index j = 0; j < n; ++j) {
            double s = 0;
            for (Index i = 0; i < n; ++i) s += std::abs(lu_(i, j));
            norm1_ = std::max(norm1_, s);
        }
        for (Index k = 0; k < n; ++k) {
            Index piv = k;
            double best = std::abs(lu_(k, k));
            for (Index i = k + 1; i < n; ++i)
                if (std::abs(lu_(i, k)) > best) { best = std::abs(lu_(i, k)); piv = i; }
            if (piv != k) {
                for (Index j = 0; j < n; ++j) std::swap(lu_(k, j), lu_(piv, j));
                std::swap(perm_[std::size_t(k)], perm_[std::size_t(piv)]);
            }
            if (lu_(k, k) == S(0)) continue;
            for (Index i = k + 1; i < n; ++i) {
                lu_(i, k) /= lu_(k, k);
                const S l = lu_(i, k);
                if (l == S(0)) continue;
                for (Index j = k + 1; j < n; ++j) lu_(i, j) -= l * lu_(k, j);
            }
        }
        return *this;
    }
    template <class M> auto solve(const M& b_) const {
        const auto& b = shim::ev(b_);
        using SB = typename shim::ev_t<M>::Scalar;
        using SR = decltype(std::declval<SB>() / std::declval<S>());
        const Index n = lu_.rows();
        Matrix<SR, Dynamic, shim::ev_t<M>::ColsAtCompileTime> x(n, b.cols());
        for (Index c = 0; c < b.cols(); ++c) {
            for (Index i = 0; i < n; ++i) x(i, c) = b(perm_[std::size_t(i)], c);
            for (Index i = 0; i < n; ++i)
                for (Index k = 0; k < i; ++k) x(i, c) -= lu_(i, k) * x(k, c);
            for (Index i = n - 1; i >= 0; --i) {
                for (Index k = i + 1; k < n; ++k) x(i, c) -= lu_(i, k) * x(k, c);
                x(i, c) /= lu_(i, i);
            }
        }
        return x;
    }
    Matrix<S> inverse() const { return solve(Matrix<S>::Identity(lu_.rows(), lu_.rows())); }
    /// Reciprocal 1-norm condition number (computed exactly from the inverse;
    /// Eigen estimates it — only ever compared against a singularity threshold).
    double rcond() const {
        const Index n = lu_.rows();
        for (Index i = 0; i < n; ++i)
            if (lu_(i, i) == S(0)) return 0.0;
        const Matrix<S> inv = inverse();
        double ninv = 0;
        for (Index j = 0; j < n; ++j) {
            double s = 0;
            for (Index i = 0; i < n; ++i) s += std::abs(inv(i, j));
            ninv = std::max(ninv, s);
        }
        return (norm1_ == 0 || ninv == 0) ? 0.0 : 1.0 / (norm1_ * ninv);
    }
    const Matrix<S>& matrixLU() const { return lu_; }

  private:
    Matrix<S> lu_;
    std::vector<Index> perm_;
    double norm1_ = 0;
};

template <class S, int R, int C>
Matrix<S, R, C> Matrix<S, R, C>::inverse() const {
    return Matrix<S, R, C>(PartialPivLU<Matrix<S>>(*this).inverse());
}

/// Householder QR with column pivoting; solve() returns the basic least-squares
/// solution on the numerical rank (threshold eps * min(m, n) * |R_00|, Eigen's default).
template <class MatrixType>
class ColPivHouseholderQR {
  public:
    using S = typename MatrixType::Scalar;
    template <class M> explicit ColPivHouseholderQR(const M& a_) {
        qr_ = Matrix<S>(a_.eval());
        const Index m = qr_.rows(), n = qr_.cols(), kmax = std::min(m, n);
        perm_.resize(std::size_t(n));
        for (Index j = 0; j < n; ++j) perm_[std::size_t(j)] = j;
        tau_.assign(std::size_t(kmax), S(0));
        double maxpiv = 0;
        rank_ = 0;
        for (Index k = 0; k < kmax; ++k) {
            // pivot: the remaining column of largest norm (recomputed exactly)
            Index best = k;
            double bn = -1;
            for (Index j = k; j < n; ++j) {
                double s = 0;
                for (Index i = k; i < m; ++i) s += shim::abs2_(qr_(i, j));
                if (s > bn) { bn = s; best = j; }
            }
            if (best != k) {
                for (Index i = 0; i < m; ++i) std::swap(qr_(i, k), qr_(i, best));
                std::swap(perm_[std::size_t(k)], perm_[std::size_t(best)]);
            }
            // Householder reflector H = I - tau v v^H with v(0) = 1 mapping x to beta e1
            double xnorm2 = 0;
            for (Index i = k + 1; i < m; ++i) xnorm2 += shim::abs2_(qr_(i, k));
            const S alpha = qr_(k, k);
            if (xnorm2 == 0 && std::imag(std::complex<double>(alpha)) == 0) {
                tau_[std::size_t(k)] = S(0);
            } else {
                const double anorm = std::sqrt(shim::abs2_(alpha) + xnorm2);
                const double beta = std::real(std::complex<double>(alpha)) >= 0 ? -anorm : anorm;
                tau_[std::size_t(k)] = (S(beta) - alpha) / S(beta);
                const S scale = S(1) / (alpha - S(beta));
                for (Index i = k + 1; i < m; ++i) qr_(i, k) *= scale;
                qr_(k, k) = S(beta);
                // apply H^H to the trailing columns
                for (Index j = k + 1; j < n; ++j) {
                    S w = qr_(k, j);
                    for (Index i = k + 1; i < m; ++i) w += shim::conj_(qr_(i, k)) * qr_(i, j);
                    w *= shim::conj_(tau_[std::size_t(k)]);
                    qr_(k, j) -= w;
                    for (Index i = k + 1; i < m; ++i) qr_(i, j) -= qr_(i, k) * w;
                }
            }
            const double piv = std::abs(qr_(k, k));
            if (k == 0) maxpiv = piv;
            if (piv > std::numeric_limits<double>::epsilon() * double(kmax) * maxpiv) ++rank_;
        }
    }
    template <class M> Matrix<S, Dynamic, 1> solve(const M& b_) const {
        Matrix<S, Dynamic, 1> c(b_.eval());
        const Index m = qr_.rows(), n = qr_.cols(), kmax = std::min(m, n);
        for (Index k = 0; k < kmax; ++k) {  // c <- Q^H c
            S w = c(k);
            for (Index i = k + 1; i < m; ++i) w += shim::conj_(qr_(i, k)) * c(i);
            w *= shim::conj_(tau_[std::size_t(k)]);
            c(k) -= w;
            for (Index i = k + 1; i < m; ++i) c(i) -= qr_(i, k) * w;
        }
        Matrix<S, Dynamic, 1> z(n), x(n);
        for (Index i = rank_ - 1; i >= 0; --i) {
            S s = c(i);
            for (Index j = i + 1; j < rank_; ++j) s -= qr_(i, j) * z(j);
            z(i) = s / qr_(i, i);
        }
        for (Index j = 0; j < n; ++j) x(perm_[std::size_t(j)]) = z(j);
        return x;
    }
    Index rank() const { return rank_; }

  private:
    Matrix<S> qr_;
    std::vector<S> tau_;
    std::vector<Index> perm_;
    Index rank_ = 0;
};

template <class S, int R, int C>
PartialPivLU<Matrix<S>> Matrix<S, R, C>::partialPivLu() const { return PartialPivLU<Matrix<S>>(*this); }
template <class S, int R, int C>
ColPivHouseholderQR<Matrix<S>> Matrix<S, R, C>::colPivHouseholderQr() const {
    return ColPivHouseholderQR<Matrix<S>>(*this);
}

// ---- typedefs used by the reference ----
using MatrixXd = Matrix<double>;
using MatrixXcd = Matrix<std::complex<double>>;
using VectorXd = Matrix<double, Dynamic, 1>;
using VectorXcd = Matrix<std::complex<double>, Dynamic, 1>;
using RowVectorXd = Matrix<double, 1, Dynamic>;
using MatrixX2d = Matrix<double, Dynamic, 2>;
using Matrix2cd = Matrix<std::complex<double>, 2, 2>;
using Matrix3d = Matrix<double, 3, 3>;
using Vector3d = Matrix<double, 3, 1>;
using Vector2d = Matrix<double, 2, 1>;
using RowVector2d = Matrix<double, 1, 2>;
template <class S, int N> using Vector = Matrix<S, N, 1>;
template <class S, int N> using RowVector = Matrix<S, 1, N>;
template <class S> using MatrixX = Matrix<S>;

}  // namespace Eigen
