// Eigenvalue solvers appear in the reference only in linalg.cpp's
// dense_eigenvalues (LFA / dispersion analysis, out of scope for the hot path).
// They are declared so that linalg.cpp compiles unmodified; a call reports
// failure (info() != Success), which dense_eigenvalues turns into an exception.
// TEST INFRASTRUCTURE ONLY.
#pragma once

#include "dense.hpp"

namespace Eigen {

template <class MatrixType>
class ComplexEigenSolver {
  public:
    template <class M> ComplexEigenSolver(const M&, bool = true) {}
    ComputationInfo info() const { return InvalidInput; }
    const Matrix<std::complex<double>, Dynamic, 1>& eigenvalues() const { return ev_; }

  private:
    Matrix<std::complex<double>, Dynamic, 1> ev_;
};

template <class MatrixType>
class SelfAdjointEigenSolver {
  public:
    template <class M> SelfAdjointEigenSolver(const M&, int = ComputeEigenvectors) {}
    ComputationInfo info() const { return InvalidInput; }
    const Matrix<double, Dynamic, 1>& eigenvalues() const { return ev_; }

  private:
    Matrix<double, Dynamic, 1> ev_;
};

}  // namespace Eigen
