// l1solve/types.hpp -- drop-in for proj/core/include/l1solve/types.hpp (B200 build).
//
// The reference aliases Eigen::VectorXd / MatrixXd (types.hpp:8-10); Eigen is not part of
// this build, so Vector and Matrix are small dense containers with the subset of the Eigen
// interface the solver API and its callers use.  Reductions follow the library's canonical
// order and run on the GPU through libl1g (l1g_reduce), like every other computation here.
#pragma once
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <vector>

namespace l1solve {

using Index = std::ptrdiff_t;
constexpr int Infinity = -1;  // for lpNorm<Infinity>()

class Vector {
 public:
  Vector() = default;
  explicit Vector(Index n) : v_(static_cast<std::size_t>(n), 0.0) {}
  Vector(std::initializer_list<double> il) : v_(il) {}
  static Vector Zero(Index n) { return Vector(n); }
  static Vector Ones(Index n) { return Constant(n, 1.0); }
  static Vector Constant(Index n, double c) {
    Vector r(n);
    for (auto& x : r.v_) x = c;
    return r;
  }
  Index size() const { return static_cast<Index>(v_.size()); }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator[](Index i) { return v_[static_cast<std::size_t>(i)]; }
  double operator[](Index i) const { return v_[static_cast<std::size_t>(i)]; }
  double& operator()(Index i) { return v_[static_cast<std::size_t>(i)]; }
  double operator()(Index i) const { return v_[static_cast<std::size_t>(i)]; }

  double dot(const Vector& o) const;
  double squaredNorm() const;
  double norm() const;
  template <int P>
  double lpNorm() const;

  Vector& operator+=(const Vector& o);
  Vector& operator-=(const Vector& o);
  Vector& operator*=(double c);
  Vector& operator/=(double c);

 private:
  std::vector<double> v_;
};

template <>
double Vector::lpNorm<1>() const;
template <>
double Vector::lpNorm<Infinity>() const;

Vector operator+(Vector a, const Vector& b);
Vector operator-(Vector a, const Vector& b);
Vector operator-(Vector a);
Vector operator*(double c, Vector a);
Vector operator*(Vector a, double c);
Vector operator/(Vector a, double c);

// Column-major dense matrix (Eigen's default storage order).
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index rows, Index cols)
      : r_(rows), c_(cols), d_(static_cast<std::size_t>(rows * cols), 0.0) {}
  static Matrix Zero(Index rows, Index cols) { return Matrix(rows, cols); }
  static Matrix Identity(Index rows, Index cols) {
    Matrix m(rows, cols);
    for (Index i = 0; i < (rows < cols ? rows : cols); ++i) m(i, i) = 1.0;
    return m;
  }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double& operator()(Index i, Index j) { return d_[static_cast<std::size_t>(j * r_ + i)]; }
  double operator()(Index i, Index j) const { return d_[static_cast<std::size_t>(j * r_ + i)]; }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> d_;
};

/// Counts applications of K and K^T (types.hpp:15-17).
struct MatvecCounter {
  std::int64_t count = 0;
};

}  // namespace l1solve

// source compatibility with callers written against Eigen (x.lpNorm<Eigen::Infinity>())
namespace Eigen {
using l1solve::Infinity;
}
