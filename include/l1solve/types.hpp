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

  /// Eigen's comma initializer: v << a, b, c;
  struct CommaInit {
    Vector* v;
    Index i;
    CommaInit& operator,(double x) {
      (*v)[i++] = x;
      return *this;
    }
  };
  CommaInit operator<<(double x) {
    (*this)[0] = x;
    return CommaInit{this, 1};
  }
  /// coefficient-wise view for (a.array() == b.array()).all()
  struct Array {
    const std::vector<double>* v;
    struct Mask {
      bool ok;
      bool all() const { return ok; }
    };
    Mask operator==(const Array& o) const {
      if (v->size() != o.v->size()) return {false};
      for (std::size_t i = 0; i < v->size(); ++i)
        if (!((*v)[i] == (*o.v)[i])) return {false};
      return {true};
    }
  };
  Array array() const { return Array{&v_}; }

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

  // host-side helpers for callers written against Eigen (tests, generators); the solver's
  // products run on the GPU through DenseOperator
  Matrix transpose() const {
    Matrix t(c_, r_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  Matrix& operator+=(const Matrix& o) {
    for (std::size_t k = 0; k < d_.size(); ++k) d_[k] = d_[k] + o.d_[k];
    return *this;
  }
  Matrix& operator/=(double c) {
    for (auto& x : d_) x = x / c;
    return *this;
  }
  Matrix& operator*=(double c) {
    for (auto& x : d_) x = x * c;
    return *this;
  }
  /// Eigen's comma initializer, row by row: m << a, b, c, d;
  struct CommaInit {
    Matrix* m;
    Index k;
    CommaInit& operator,(double x) {
      (*m)(k / m->c_, k % m->c_) = x;
      ++k;
      return *this;
    }
  };
  CommaInit operator<<(double x) {
    (*this)(0, 0) = x;
    return CommaInit{this, 1};
  }
  struct Array {
    const Matrix* m;
    Vector::Array::Mask operator==(const Array& o) const {
      return {m->r_ == o.m->r_ && m->c_ == o.m->c_ && m->d_ == o.m->d_};
    }
  };
  Array array() const { return Array{this}; }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> d_;
};

inline Matrix operator*(double c, Matrix m) { return m *= c; }
inline Matrix operator+(Matrix a, const Matrix& b) { return a += b; }
/// host product (column-major accumulation, Eigen's plain GEMV order)
inline Vector operator*(const Matrix& m, const Vector& x) {
  Vector out(m.rows());
  for (Index j = 0; j < m.cols(); ++j)
    for (Index i = 0; i < m.rows(); ++i) out[i] = out[i] + m(i, j) * x[j];
  return out;
}

/// Counts applications of K and K^T (types.hpp:15-17).
struct MatvecCounter {
  std::int64_t count = 0;
};

}  // namespace l1solve

// source compatibility with callers written against Eigen (x.lpNorm<Eigen::Infinity>())
namespace Eigen {
using l1solve::Infinity;
}
