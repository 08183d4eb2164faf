// matrix.hpp — the dense matrix type of the drop-in API.
//
// The reference uses Eigen::MatrixXd (proj/include/lora_fleet/fused_lora.hpp:20). When
// Eigen is available it is used as-is; otherwise (this image has no Eigen) a small
// column-major double matrix provides exactly the Eigen surface the reference's hot-path
// callers use: rows/cols, operator(), row(i) (assign, +=, * matrix), cwiseAbs, maxCoeff,
// Zero, comma initialiser <<, +, -, scalar *, *=, matrix *.
// Host-side value type only: no arithmetic of the fused layer runs here.
#pragma once

#if __has_include(<Eigen/Dense>) && !defined(LORA_FLEET_NO_EIGEN)
#include <Eigen/Dense>
namespace lora_fleet {
using Matrix = Eigen::MatrixXd;
using Index = Eigen::Index;
}  // namespace lora_fleet
#else
#include <algorithm>
#include <cmath>
#include <cstddef>
#include <stdexcept>
#include <vector>

namespace lora_fleet {

using Index = std::ptrdiff_t;

class Matrix {
 public:
  class Row {
   public:
    Row(Matrix& m, Index r) : m_(&m), r_(r) {}
    Row& operator=(const Row& o) {
      for (Index c = 0; c < m_->cols(); ++c) (*m_)(r_, c) = (*o.m_)(o.r_, c);
      return *this;
    }
    Row& operator=(const Matrix& o) {  // o is 1 x cols
      if (o.rows() != 1 || o.cols() != m_->cols()) throw std::logic_error("row shape mismatch");
      for (Index c = 0; c < m_->cols(); ++c) (*m_)(r_, c) = o(0, c);
      return *this;
    }
    Row& operator+=(const Row& o) {
      for (Index c = 0; c < m_->cols(); ++c) (*m_)(r_, c) += (*o.m_)(o.r_, c);
      return *this;
    }
    double operator()(Index c) const { return (*m_)(r_, c); }
    Index cols() const { return m_->cols(); }
    friend Matrix operator*(const Row& r, const Matrix& b) {
      if (r.cols() != b.rows()) throw std::logic_error("inner dimension mismatch");
      Matrix o(1, b.cols());
      for (Index j = 0; j < b.cols(); ++j) {
        double acc = 0.0;
        for (Index p = 0; p < b.rows(); ++p) acc += r(p) * b(p, j);
        o(0, j) = acc;
      }
      return o;
    }

   private:
    Matrix* m_;
    Index r_;
  };

  Matrix() = default;
  Matrix(Index r, Index c) : r_(r), c_(c), v_(static_cast<size_t>(r * c), 0.0) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  double& operator()(Index i, Index j) { return v_[static_cast<size_t>(j * r_ + i)]; }
  double operator()(Index i, Index j) const { return v_[static_cast<size_t>(j * r_ + i)]; }
  Row row(Index i) { return Row(*this, i); }
  Row row(Index i) const { return Row(const_cast<Matrix&>(*this), i); }
  static Matrix Zero(Index r, Index c) { return Matrix(r, c); }

  Matrix cwiseAbs() const {
    Matrix o(r_, c_);
    for (size_t i = 0; i < v_.size(); ++i) o.v_[i] = std::fabs(v_[i]);
    return o;
  }
  double maxCoeff() const {
    if (v_.empty()) throw std::logic_error("maxCoeff of empty matrix");
    return *std::max_element(v_.begin(), v_.end());
  }
  Matrix& operator*=(double s) {
    for (auto& x : v_) x *= s;
    return *this;
  }
  friend Matrix operator*(double s, Matrix m) { return m *= s; }
  friend Matrix operator*(Matrix m, double s) { return m *= s; }
  friend Matrix operator+(Matrix a, const Matrix& b) {
    if (a.r_ != b.r_ || a.c_ != b.c_) throw std::logic_error("shape mismatch");
    for (size_t i = 0; i < a.v_.size(); ++i) a.v_[i] += b.v_[i];
    return a;
  }
  friend Matrix operator-(Matrix a, const Matrix& b) {
    if (a.r_ != b.r_ || a.c_ != b.c_) throw std::logic_error("shape mismatch");
    for (size_t i = 0; i < a.v_.size(); ++i) a.v_[i] -= b.v_[i];
    return a;
  }
  friend Matrix operator*(const Matrix& a, const Matrix& b) {
    if (a.c_ != b.r_) throw std::logic_error("inner dimension mismatch");
    Matrix o(a.r_, b.c_);
    for (Index j = 0; j < b.c_; ++j)
      for (Index p = 0; p < a.c_; ++p) {
        const double bv = b(p, j);
        for (Index i = 0; i < a.r_; ++i) o(i, j) += a(i, p) * bv;
      }
    return o;
  }

  class CommaInit {
   public:
    CommaInit(Matrix& m, double first) : m_(m) { put(first); }
    CommaInit& operator,(double x) {
      put(x);
      return *this;
    }

   private:
    void put(double x) {
      if (i_ >= m_.r_ * m_.c_) throw std::logic_error("too many coefficients");
      m_(i_ / m_.c_, i_ % m_.c_) = x;  // row-major fill order, as Eigen
      ++i_;
    }
    Matrix& m_;
    Index i_ = 0;
  };
  CommaInit operator<<(double x) { return CommaInit(*this, x); }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> v_;
};

}  // namespace lora_fleet
#endif
