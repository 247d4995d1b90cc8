// eigen_shim -- TEST INFRASTRUCTURE ONLY.
//
// A minimal, eagerly evaluated stand-in for the subset of the Eigen 3 API that the
// reference's headers (/root/reference/proj/include/tpmg/{types,geometry,profiles,
// discretization,relaxation,multigrid}.hpp) use, so that those headers can be compiled
// unmodified into oracle/_ref/ (Eigen itself is not installed in this image).  Written from
// the public Eigen API semantics, not from Eigen's sources.
//
// Semantics that matter for bitwise comparisons:
//  * column-major storage;
//  * element-wise expressions are evaluated left to right, one IEEE operation per Eigen
//    operation (what Eigen's lazy evaluation computes too, absent FMA contraction; build
//    with -ffp-contract=off);
//  * col()/row()/leftCols() are views (reference semantics, assignment copies values);
//  * reductions (sum, squaredNorm, norm, mean, dot) are sequential left-to-right sums.
//    Eigen's vectorised reduction order is NOT reproduced (the reference's tests never pin
//    it).
#pragma once

#include <algorithm>
#include <cassert>
#include <cmath>
#include <cstddef>
#include <initializer_list>
#include <map>
#include <stdexcept>
#include <type_traits>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;

template <typename Derived>
struct MatrixBase {
  const Derived& derived() const { return static_cast<const Derived&>(*this); }
  bool allFinite() const { return derived().allFinite(); }
};

template <typename T, int R = Dynamic, int C = Dynamic>
class Matrix;

// ---- strided 1-D views (a column, a row, a column block) ----------------------------------
template <typename T>
class VecView {
 public:
  VecView(T* p, Index n, Index stride) : p_(p), n_(n), s_(stride) {}
  VecView(const VecView&) = default;  // binds to the same storage (Eigen Block semantics)
  Index size() const { return n_; }
  Index rows() const { return n_; }
  Index cols() const { return 1; }
  T& operator[](Index i) const { return p_[i * s_]; }
  T& operator()(Index i) const { return p_[i * s_]; }
  template <typename Src>
  VecView& operator=(const Src& src) {  // value copy
    const Matrix<std::remove_const_t<T>> tmp = Matrix<std::remove_const_t<T>>::from(src);
    check(tmp.size());
    for (Index i = 0; i < n_; ++i) (*this)[i] = tmp.data()[i];
    return *this;
  }
  VecView& operator=(const VecView& src) {
    const Matrix<std::remove_const_t<T>> tmp = Matrix<std::remove_const_t<T>>::from(src);
    check(tmp.size());
    for (Index i = 0; i < n_; ++i) (*this)[i] = tmp.data()[i];
    return *this;
  }
  template <typename Src>
  VecView& operator+=(const Src& src) {
    const auto tmp = Matrix<std::remove_const_t<T>>::from(src);
    check(tmp.size());
    for (Index i = 0; i < n_; ++i) (*this)[i] = (*this)[i] + tmp.data()[i];
    return *this;
  }
  template <typename Src>
  VecView& operator-=(const Src& src) {
    const auto tmp = Matrix<std::remove_const_t<T>>::from(src);
    check(tmp.size());
    for (Index i = 0; i < n_; ++i) (*this)[i] = (*this)[i] - tmp.data()[i];
    return *this;
  }
  VecView& operator/=(std::remove_const_t<T> s) {
    for (Index i = 0; i < n_; ++i) (*this)[i] = (*this)[i] / s;
    return *this;
  }
  VecView& operator*=(std::remove_const_t<T> s) {
    for (Index i = 0; i < n_; ++i) (*this)[i] = (*this)[i] * s;
    return *this;
  }
  void setZero() const {
    for (Index i = 0; i < n_; ++i) (*this)[i] = T(0);
  }
  std::remove_const_t<T> sum() const {
    std::remove_const_t<T> s = (*this)[0];
    for (Index i = 1; i < n_; ++i) s = s + (*this)[i];
    return s;
  }
  template <typename O>
  auto cwiseProduct(const O& o) const;
  template <typename O>
  std::remove_const_t<T> dot(const O& o) const;
  std::remove_const_t<T> squaredNorm() const { return dot(*this); }
  std::remove_const_t<T> norm() const { return std::sqrt(squaredNorm()); }

 private:
  void check(Index n) const {
    if (n != n_) throw std::runtime_error("eigen_shim: size mismatch in view assignment");
  }
  T* p_;
  Index n_, s_;
};

// ---- the one dense type (fixed sizes are checked at run time) -----------------------------
template <typename T, int R, int C>
class Matrix : public MatrixBase<Matrix<T, R, C>> {
 public:
  using Scalar = T;
  Matrix() : r_(R > 0 ? R : 0), c_(C > 0 ? C : (R > 0 && C == Dynamic ? 0 : 0)) {
    if (R > 0 && C > 0) d_.assign(R * C, T(0));
    if (R > 0 && C == 1) { r_ = R; c_ = 1; d_.assign(R, T(0)); }
    if (R == Dynamic && C == 1) { r_ = 0; c_ = 1; }
  }
  Matrix(Index r, Index c) { resize(r, c); }
  explicit Matrix(Index n) {  // vectors
    if (C == 1) resize(n, 1);
    else resize(n, 1);
  }
  Matrix(T x, T y, T z) {
    resize(3, 1);
    d_[0] = x; d_[1] = y; d_[2] = z;
  }
  template <int R2, int C2>
  Matrix(const Matrix<T, R2, C2>& o) : r_(o.rows()), c_(o.cols()), d_(o.data(), o.data() + o.size()) {}
  template <typename V>
  Matrix(const VecView<V>& v) {
    resize(v.size(), 1);
    for (Index i = 0; i < v.size(); ++i) d_[i] = v[i];
  }
  template <typename Src>
  static Matrix from(const Src& s) {
    return Matrix(s);
  }
  static Matrix from(T) = delete;

  static Matrix Zero(Index r, Index c) { Matrix m(r, c); return m; }
  static Matrix Zero(Index n) { Matrix m; m.resize(n, 1); return m; }
  static Matrix Ones(Index n) { Matrix m; m.resize(n, 1); m.setConstant(T(1)); return m; }
  static Matrix Ones(Index r, Index c) { Matrix m(r, c); m.setConstant(T(1)); return m; }
  static Matrix Constant(Index r, Index c, T v) { Matrix m(r, c); m.setConstant(v); return m; }
  static Matrix Constant(Index n, T v) { Matrix m; m.resize(n, 1); m.setConstant(v); return m; }

  void resize(Index r, Index c) {
    r_ = r;
    c_ = c;
    d_.assign(static_cast<size_t>(r * c), T(0));
  }
  void resize(Index n) { resize(n, 1); }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  T* data() { return d_.data(); }
  const T* data() const { return d_.data(); }

  T& operator()(Index i, Index j) { return d_[static_cast<size_t>(j * r_ + i)]; }
  const T& operator()(Index i, Index j) const { return d_[static_cast<size_t>(j * r_ + i)]; }
  T& operator()(Index i) { return d_[static_cast<size_t>(i)]; }
  const T& operator()(Index i) const { return d_[static_cast<size_t>(i)]; }
  T& operator[](Index i) { return d_[static_cast<size_t>(i)]; }
  const T& operator[](Index i) const { return d_[static_cast<size_t>(i)]; }

  VecView<T> col(Index j) { return VecView<T>(d_.data() + j * r_, r_, 1); }
  VecView<const T> col(Index j) const { return VecView<const T>(d_.data() + j * r_, r_, 1); }
  VecView<T> row(Index i) { return VecView<T>(d_.data() + i, c_, r_); }
  VecView<const T> row(Index i) const { return VecView<const T>(d_.data() + i, c_, r_); }

  struct ColBlock {  // leftCols(n) = other
    Matrix* m;
    Index n;
    template <typename Src>
    ColBlock& operator=(const Src& src) {
      if (src.rows() != m->rows() || src.cols() != n)
        throw std::runtime_error("eigen_shim: leftCols size mismatch");
      for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < m->rows(); ++i) (*m)(i, j) = src(i, j);
      return *this;
    }
  };
  ColBlock leftCols(Index n) { return ColBlock{this, n}; }

  void setZero() { std::fill(d_.begin(), d_.end(), T(0)); }
  void setOnes() { std::fill(d_.begin(), d_.end(), T(1)); }
  void setConstant(T v) { std::fill(d_.begin(), d_.end(), v); }
  void setConstant(Index r, Index c, T v) { resize(r, c); setConstant(v); }

  bool allFinite() const {
    for (const T& v : d_)
      if (!std::isfinite(static_cast<double>(v))) return false;
    return true;
  }
  T sum() const {
    T s = d_.empty() ? T(0) : d_[0];
    for (size_t i = 1; i < d_.size(); ++i) s = s + d_[i];
    return s;
  }
  T mean() const { return sum() / T(size()); }
  template <typename O>
  T dot(const O& o) const {
    const Matrix b = from(o);
    T s = T(0);
    for (Index i = 0; i < size(); ++i) s = s + d_[i] * b.d_[i];
    return s;
  }
  T squaredNorm() const { return dot(*this); }
  T norm() const { return std::sqrt(squaredNorm()); }
  Matrix normalized() const {
    Matrix m(*this);
    const T n = norm();
    for (T& v : m.d_) v = v / n;
    return m;
  }
  template <typename O>
  Matrix cross(const O& o) const {
    const Matrix b = from(o);
    const Matrix& a = *this;
    return Matrix(a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]);
  }
  template <typename O>
  Matrix cwiseProduct(const O& o) const {
    const Matrix b = from(o);
    Matrix m(r_, c_);
    for (Index i = 0; i < size(); ++i) m.d_[i] = d_[i] * b.d_[i];
    return m;
  }
  Matrix cwiseAbs() const {
    Matrix m(*this);
    for (T& v : m.d_) v = std::abs(v);
    return m;
  }
  T maxCoeff() const { return *std::max_element(d_.begin(), d_.end()); }
  Matrix<T, Dynamic, Dynamic> transpose() const {
    Matrix<T, Dynamic, Dynamic> t(c_, r_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  template <typename Src>
  Matrix& operator+=(const Src& s) {
    const Matrix b = from(s);
    for (Index i = 0; i < size(); ++i) d_[i] = d_[i] + b.d_[i];
    return *this;
  }
  template <typename Src>
  Matrix& operator-=(const Src& s) {
    const Matrix b = from(s);
    for (Index i = 0; i < size(); ++i) d_[i] = d_[i] - b.d_[i];
    return *this;
  }
  Matrix& operator*=(T s) {
    for (T& v : d_) v = v * s;
    return *this;
  }
  Matrix& operator/=(T s) {
    for (T& v : d_) v = v / s;
    return *this;
  }
  Matrix operator-() const {
    Matrix m(*this);
    for (T& v : m.d_) v = -v;
    return m;
  }

 private:
  template <typename, int, int>
  friend class Matrix;
  Index r_ = 0, c_ = 0;
  std::vector<T> d_;
};

template <typename T>
using Vector3 = Matrix<T, 3, 1>;
using VectorXd = Matrix<double, Dynamic, 1>;
using MatrixXd = Matrix<double, Dynamic, Dynamic>;

// ---- free arithmetic: everything evaluates to a dense Matrix -----------------------------
template <typename X>
struct is_eig : std::false_type {};
template <typename T, int R, int C>
struct is_eig<Matrix<T, R, C>> : std::true_type {};
template <typename T>
struct is_eig<VecView<T>> : std::true_type {};

template <typename X>
struct scalar_of;
template <typename T, int R, int C>
struct scalar_of<Matrix<T, R, C>> { using type = T; };
template <typename T>
struct scalar_of<VecView<T>> { using type = std::remove_const_t<T>; };

template <typename X>
auto ev(const X& x) {
  using T = typename scalar_of<X>::type;
  return Matrix<T, Dynamic, Dynamic>(x);
}

template <typename A, typename B, typename F>
auto zipw(const A& a, const B& b, F f) {
  auto x = ev(a);
  const auto y = ev(b);
  if (x.rows() != y.rows() || x.cols() != y.cols())
    throw std::runtime_error("eigen_shim: size mismatch");
  for (Index i = 0; i < x.size(); ++i) x.data()[i] = f(x.data()[i], y.data()[i]);
  return x;
}

template <typename A, typename B, typename = std::enable_if_t<is_eig<A>::value && is_eig<B>::value>>
auto operator+(const A& a, const B& b) {
  return zipw(a, b, [](auto p, auto q) { return p + q; });
}
template <typename A, typename B, typename = std::enable_if_t<is_eig<A>::value && is_eig<B>::value>>
auto operator-(const A& a, const B& b) {
  return zipw(a, b, [](auto p, auto q) { return p - q; });
}
template <typename A, typename = std::enable_if_t<is_eig<A>::value>>
auto operator*(typename scalar_of<A>::type s, const A& a) {
  auto x = ev(a);
  for (Index i = 0; i < x.size(); ++i) x.data()[i] = s * x.data()[i];
  return x;
}
template <typename A, typename = std::enable_if_t<is_eig<A>::value>>
auto operator*(const A& a, typename scalar_of<A>::type s) {
  auto x = ev(a);
  for (Index i = 0; i < x.size(); ++i) x.data()[i] = x.data()[i] * s;
  return x;
}
template <typename A, typename = std::enable_if_t<is_eig<A>::value>>
auto operator/(const A& a, typename scalar_of<A>::type s) {
  auto x = ev(a);
  for (Index i = 0; i < x.size(); ++i) x.data()[i] = x.data()[i] / s;
  return x;
}
template <typename T>
auto operator-(const VecView<T>& a) {
  return -ev(a);
}
// matrix product (used for outer products vert * horiz^T)
template <typename T, int R1, int C1, int R2, int C2>
Matrix<T, Dynamic, Dynamic> operator*(const Matrix<T, R1, C1>& a, const Matrix<T, R2, C2>& b) {
  if (a.cols() != b.rows()) throw std::runtime_error("eigen_shim: product size mismatch");
  Matrix<T, Dynamic, Dynamic> m(a.rows(), b.cols());
  for (Index j = 0; j < b.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) {
      T s = T(0);
      for (Index k = 0; k < a.cols(); ++k) s = s + a(i, k) * b(k, j);
      m(i, j) = s;
    }
  return m;
}

template <typename T>
template <typename O>
auto VecView<T>::cwiseProduct(const O& o) const {
  return ev(*this).cwiseProduct(o);
}
template <typename T>
template <typename O>
std::remove_const_t<T> VecView<T>::dot(const O& o) const {
  return ev(*this).dot(o);
}

// ---- Sparse subset (dense_assemble / dump_coordinate_format) -------------------------------
template <typename T>
class Triplet {
 public:
  Triplet(Index r, Index c, T v) : r_(r), c_(c), v_(v) {}
  Index row() const { return r_; }
  Index col() const { return c_; }
  T value() const { return v_; }

 private:
  Index r_, c_;
  T v_;
};

template <typename T>
class SparseMatrix {
 public:
  SparseMatrix(Index r, Index c) : r_(r), c_(c), cols_(static_cast<size_t>(c)) {}
  template <typename It>
  void setFromTriplets(It b, It e) {
    for (; b != e; ++b) {
      auto& cm = cols_[static_cast<size_t>(b->col())];
      auto it = cm.find(b->row());
      if (it == cm.end()) cm.emplace(b->row(), b->value());
      else it->second = it->second + b->value();
    }
  }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index outerSize() const { return c_; }
  class InnerIterator {
   public:
    InnerIterator(const SparseMatrix& m, Index outer)
        : it_(m.cols_[static_cast<size_t>(outer)].begin()),
          end_(m.cols_[static_cast<size_t>(outer)].end()), col_(outer) {}
    explicit operator bool() const { return it_ != end_; }
    InnerIterator& operator++() {
      ++it_;
      return *this;
    }
    Index row() const { return it_->first; }
    Index col() const { return col_; }
    T value() const { return it_->second; }

   private:
    typename std::map<Index, T>::const_iterator it_, end_;
    Index col_;
  };

 private:
  Index r_, c_;
  std::vector<std::map<Index, T>> cols_;
};

}  // namespace Eigen
