// Eigen-subset shim — TEST INFRASTRUCTURE ONLY (oracle build).
//
// The reference (voxrf, /root/reference/proj) is written against Eigen 3
// (find_package(Eigen3 3.3), proj/CMakeLists.txt:12), which is not installed
// in this image. This header implements exactly the part of the Eigen API the
// reference's hot-path translation units and unit tests use, so that those
// sources compile *unchanged* from where they lie (see oracle/Makefile).
//
// Arithmetic order follows Eigen 3.3/3.4 on x86-64 with SSE2 and no FMA:
//  * element-wise ops evaluate per coefficient, left to right;
//  * redux (sum / squaredNorm / dot) over 3-vectors is (e0+e1)+e2, over
//    4-vectors the SSE2 packet order (e0+e2)+(e1+e3);
//  * normalized() = v / sqrt(squaredNorm());
//  * Quaternion * vector uses Eigen's _transformVector:
//      uv = vec x v; uv += uv; return v + w*uv + vec x uv;
//  * cross product is the generic cross3_impl.
// Bit-level agreement with a real Eigen build is NOT pinned (no Eigen here);
// the reference's own tests (test_renderer.cpp:30-57) pin this layer to
// <= 1e-12 / 1e-15 and pass against this shim.
#pragma once

#include <algorithm>
#include <cassert>
#include <cmath>
#include <cstddef>
#include <initializer_list>
#include <limits>
#include <stdexcept>
#include <type_traits>

namespace Eigen {

using Index = std::ptrdiff_t;

template <typename T, int R, int C>
class Matrix;

namespace internal {
template <typename T, int N>
inline T redux_sum(const T* v) {
  if constexpr (N == 4) {
    return (v[0] + v[2]) + (v[1] + v[3]);  // SSE2 Packet2d order
  } else {
    T s = v[0];
    for (int i = 1; i < N; ++i) s = s + v[i];
    return s;
  }
}
}  // namespace internal

// Comma initializer: fills coefficients (row-major walk) from scalars or
// column vectors (blocks).
template <typename M>
class CommaInitializer {
 public:
  using Scalar = typename M::Scalar;
  CommaInitializer(M& m, const Scalar& s) : m_(m), pos_(0) { put(s); }
  template <int R2, int C2>
  CommaInitializer(M& m, const Matrix<Scalar, R2, C2>& b) : m_(m), pos_(0) { put(b); }
  template <typename S, typename = std::enable_if_t<std::is_arithmetic_v<S>>>
  CommaInitializer& operator,(const S& s) {
    put(Scalar(s));
    return *this;
  }
  template <int R2, int C2>
  CommaInitializer& operator,(const Matrix<Scalar, R2, C2>& b) {
    put(b);
    return *this;
  }

 private:
  void put(const Scalar& s) {
    const int r = pos_ / M::kCols, c = pos_ % M::kCols;
    m_(r, c) = s;
    ++pos_;
  }
  template <int R2, int C2>
  void put(const Matrix<Scalar, R2, C2>& b) {
    static_assert(C2 == 1, "shim: only column blocks in comma init");
    static_assert(M::kCols == 1, "shim: block comma init only for vectors");
    for (int i = 0; i < R2; ++i) m_(pos_ + i, 0) = b(i, 0);
    pos_ += R2;
  }
  M& m_;
  int pos_;
};

// Row / column proxies for assignment (A.row(k) << ..., rot.col(0) = v).
template <typename M>
class RowRef {
 public:
  using Scalar = typename M::Scalar;
  RowRef(M& m, int r) : m_(m), r_(r) {}
  struct Filler {
    M& m;
    int r;
    int c;
    template <typename S>
    Filler& operator,(const S& s) {
      m(r, c++) = Scalar(s);
      return *this;
    }
  };
  template <typename S>
  Filler operator<<(const S& s) {
    m_(r_, 0) = Scalar(s);
    return Filler{m_, r_, 1};
  }

 private:
  M& m_;
  int r_;
};

template <typename M>
class ColRef {
 public:
  using Scalar = typename M::Scalar;
  ColRef(M& m, int c) : m_(m), c_(c) {}
  ColRef& operator=(const Matrix<Scalar, M::kRows, 1>& v) {
    for (int i = 0; i < M::kRows; ++i) m_(i, c_) = v(i, 0);
    return *this;
  }

 private:
  M& m_;
  int c_;
};

template <typename M>
class ColPivHouseholderQR;

template <typename T, int R, int C>
class Matrix {
 public:
  using Scalar = T;
  static constexpr int kRows = R;
  static constexpr int kCols = C;
  static constexpr int kSize = R * C;
  enum { RowsAtCompileTime = R, ColsAtCompileTime = C, SizeAtCompileTime = R * C };

  Matrix() {
    for (int i = 0; i < kSize; ++i) d_[i] = T(0);
  }
  template <typename A, typename B, typename D,
            typename = std::enable_if_t<kSize == 3 && std::is_arithmetic_v<A> &&
                                        std::is_arithmetic_v<B> && std::is_arithmetic_v<D>>>
  Matrix(const A& x, const B& y, const D& z) {
    d_[0] = T(x);
    d_[1] = T(y);
    d_[2] = T(z);
  }
  template <typename A, typename B, typename D, typename E,
            typename = std::enable_if_t<kSize == 4 && std::is_arithmetic_v<A>>>
  Matrix(const A& x, const B& y, const D& z, const E& w) {
    d_[0] = T(x);
    d_[1] = T(y);
    d_[2] = T(z);
    d_[3] = T(w);
  }

  static Matrix Zero() { return Constant(T(0)); }
  static Matrix Ones() { return Constant(T(1)); }
  static Matrix Constant(const T& v) {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.d_[i] = v;
    return m;
  }
  static Matrix Identity() {
    Matrix m;
    for (int i = 0; i < R && i < C; ++i) m(i, i) = T(1);
    return m;
  }

  // Column-major storage, like Eigen's default.
  T& operator()(Index r, Index c) { return d_[c * R + r]; }
  const T& operator()(Index r, Index c) const { return d_[c * R + r]; }
  T& operator()(Index i) { return d_[i]; }
  const T& operator()(Index i) const { return d_[i]; }
  T& operator[](Index i) { return d_[i]; }
  const T& operator[](Index i) const { return d_[i]; }
  T coeff(Index r, Index c) const { return (*this)(r, c); }
  T coeff(Index i) const { return d_[i]; }
  T& coeffRef(Index i) { return d_[i]; }

  T& x() { return d_[0]; }
  T& y() { return d_[1]; }
  T& z() { return d_[2]; }
  T& w() { return d_[3]; }
  const T& x() const { return d_[0]; }
  const T& y() const { return d_[1]; }
  const T& z() const { return d_[2]; }
  const T& w() const { return d_[3]; }

  T* data() { return d_; }
  const T* data() const { return d_; }
  static constexpr Index size() { return kSize; }
  static constexpr Index rows() { return R; }
  static constexpr Index cols() { return C; }

  void setZero() {
    for (int i = 0; i < kSize; ++i) d_[i] = T(0);
  }
  Matrix& setConstant(const T& v) {
    for (int i = 0; i < kSize; ++i) d_[i] = v;
    return *this;
  }

  template <typename U>
  Matrix<U, R, C> cast() const {
    Matrix<U, R, C> m;
    for (int i = 0; i < kSize; ++i) m[i] = U(d_[i]);
    return m;
  }

  // ---- element-wise arithmetic
  Matrix operator+(const Matrix& o) const {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.d_[i] = d_[i] + o.d_[i];
    return m;
  }
  Matrix operator-(const Matrix& o) const {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.d_[i] = d_[i] - o.d_[i];
    return m;
  }
  Matrix operator-() const {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.d_[i] = -d_[i];
    return m;
  }
  Matrix operator*(const T& s) const {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.d_[i] = d_[i] * s;
    return m;
  }
  Matrix operator/(const T& s) const {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.d_[i] = d_[i] / s;
    return m;
  }
  Matrix& operator+=(const Matrix& o) {
    for (int i = 0; i < kSize; ++i) d_[i] = d_[i] + o.d_[i];
    return *this;
  }
  Matrix& operator-=(const Matrix& o) {
    for (int i = 0; i < kSize; ++i) d_[i] = d_[i] - o.d_[i];
    return *this;
  }
  Matrix& operator*=(const T& s) {
    for (int i = 0; i < kSize; ++i) d_[i] = d_[i] * s;
    return *this;
  }
  Matrix& operator/=(const T& s) {
    for (int i = 0; i < kSize; ++i) d_[i] = d_[i] / s;
    return *this;
  }
  Matrix cwiseProduct(const Matrix& o) const {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.d_[i] = d_[i] * o.d_[i];
    return m;
  }
  Matrix cwiseMin(const Matrix& o) const {
    Matrix m;
    // Eigen's scalar_min_op: numext::mini(a, b) = (b < a) ? b : a
    for (int i = 0; i < kSize; ++i) m.d_[i] = (o.d_[i] < d_[i]) ? o.d_[i] : d_[i];
    return m;
  }
  Matrix cwiseMax(const Matrix& o) const {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.d_[i] = (d_[i] < o.d_[i]) ? o.d_[i] : d_[i];
    return m;
  }
  Matrix cwiseAbs() const {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.d_[i] = std::abs(d_[i]);
    return m;
  }

  bool operator==(const Matrix& o) const {
    for (int i = 0; i < kSize; ++i)
      if (!(d_[i] == o.d_[i])) return false;
    return true;
  }
  bool operator!=(const Matrix& o) const { return !(*this == o); }

  // ---- reductions
  T sum() const { return internal::redux_sum<T, kSize>(d_); }
  T squaredNorm() const {
    T sq[kSize];
    for (int i = 0; i < kSize; ++i) sq[i] = d_[i] * d_[i];
    return internal::redux_sum<T, kSize>(sq);
  }
  T norm() const { return std::sqrt(squaredNorm()); }
  Matrix normalized() const {
    const T z = squaredNorm();
    if (z > T(0)) return *this / std::sqrt(z);
    return *this;
  }
  void normalize() {
    const T z = squaredNorm();
    if (z > T(0)) *this /= std::sqrt(z);
  }
  T dot(const Matrix& o) const {
    T pr[kSize];
    for (int i = 0; i < kSize; ++i) pr[i] = d_[i] * o.d_[i];
    return internal::redux_sum<T, kSize>(pr);
  }
  Matrix cross(const Matrix& r) const {
    static_assert(kSize == 3, "cross needs 3-vectors");
    return Matrix(d_[1] * r.d_[2] - d_[2] * r.d_[1], d_[2] * r.d_[0] - d_[0] * r.d_[2],
                  d_[0] * r.d_[1] - d_[1] * r.d_[0]);
  }
  T minCoeff() const {
    T m = d_[0];
    for (int i = 1; i < kSize; ++i) m = (d_[i] < m) ? d_[i] : m;
    return m;
  }
  T maxCoeff() const {
    T m = d_[0];
    for (int i = 1; i < kSize; ++i) m = (m < d_[i]) ? d_[i] : m;
    return m;
  }
  bool allFinite() const {
    for (int i = 0; i < kSize; ++i)
      if (!std::isfinite(double(d_[i]))) return false;
    return true;
  }

  // ---- matrix algebra (small, test/eval use only)
  template <int C2>
  Matrix<T, R, C2> operator*(const Matrix<T, C, C2>& o) const {
    Matrix<T, R, C2> m;
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < C2; ++j) {
        T s = T(0);
        for (int k = 0; k < C; ++k) s = s + (*this)(i, k) * o(k, j);
        m(i, j) = s;
      }
    return m;
  }
  Matrix<T, C, R> transpose() const {
    Matrix<T, C, R> m;
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < C; ++j) m(j, i) = (*this)(i, j);
    return m;
  }
  T trace() const {
    T s = T(0);
    for (int i = 0; i < R && i < C; ++i) s = s + (*this)(i, i);
    return s;
  }
  // Eigen determinant_impl<3>: sum of bruteforce_det3_helper(m, a, b, c) =
  // m(0,a) * (m(1,b) m(2,c) - m(1,c) m(2,b)) over the first column's cofactors
  T determinant() const {
    static_assert(R == 3 && C == 3, "shim: 3x3 determinant only");
    const Matrix& m = *this;
    auto h = [&m](int a, int b, int c) { return m(0, a) * (m(1, b) * m(2, c) - m(1, c) * m(2, b)); };
    return h(0, 1, 2) - h(1, 0, 2) + h(2, 0, 1);
  }

  CommaInitializer<Matrix> operator<<(const T& s) { return CommaInitializer<Matrix>(*this, s); }
  template <typename S, typename = std::enable_if_t<std::is_arithmetic_v<S> && !std::is_same_v<S, T>>>
  CommaInitializer<Matrix> operator<<(const S& s) {
    return CommaInitializer<Matrix>(*this, T(s));
  }
  template <int R2, int C2>
  CommaInitializer<Matrix> operator<<(const Matrix<T, R2, C2>& b) {
    return CommaInitializer<Matrix>(*this, b);
  }

  RowRef<Matrix> row(int r) { return RowRef<Matrix>(*this, r); }
  ColRef<Matrix> col(int c) { return ColRef<Matrix>(*this, c); }
  Matrix<T, R, 1> col(int c) const {
    Matrix<T, R, 1> v;
    for (int i = 0; i < R; ++i) v[i] = (*this)(i, c);
    return v;
  }

  ColPivHouseholderQR<Matrix> colPivHouseholderQr() const { return ColPivHouseholderQR<Matrix>(*this); }

 private:
  T d_[kSize];
};

template <typename T, int R, int C>
inline Matrix<T, R, C> operator*(const T& s, const Matrix<T, R, C>& m) {
  Matrix<T, R, C> out;
  for (int i = 0; i < R * C; ++i) out[i] = s * m[i];
  return out;
}
// int * Vector3i and the like where the scalar literal type differs.
template <typename S, typename T, int R, int C,
          typename = std::enable_if_t<std::is_arithmetic_v<S> && !std::is_same_v<S, T>>>
inline Matrix<T, R, C> operator*(const S& s, const Matrix<T, R, C>& m) {
  return T(s) * m;
}

// Dense solve for the reference's 8x8 interpolation test
// (test_voxel_grid.cpp:67); Gaussian elimination with partial pivoting.
template <typename M>
class ColPivHouseholderQR {
 public:
  using T = typename M::Scalar;
  explicit ColPivHouseholderQR(const M& a) : a_(a) {}
  Matrix<T, M::kRows, 1> solve(const Matrix<T, M::kRows, 1>& b) const {
    constexpr int n = M::kRows;
    M a = a_;
    Matrix<T, n, 1> x = b;
    for (int col = 0; col < n; ++col) {
      int piv = col;
      for (int r = col + 1; r < n; ++r)
        if (std::abs(a(r, col)) > std::abs(a(piv, col))) piv = r;
      if (piv != col) {
        for (int c = 0; c < n; ++c) std::swap(a(col, c), a(piv, c));
        std::swap(x[col], x[piv]);
      }
      for (int r = col + 1; r < n; ++r) {
        const T f = a(r, col) / a(col, col);
        for (int c = col; c < n; ++c) a(r, c) -= f * a(col, c);
        x[r] -= f * x[col];
      }
    }
    for (int r = n - 1; r >= 0; --r) {
      T s = x[r];
      for (int c = r + 1; c < n; ++c) s -= a(r, c) * x[c];
      x[r] = s / a(r, r);
    }
    return x;
  }

 private:
  M a_;
};

using Vector3d = Matrix<double, 3, 1>;
using Vector3i = Matrix<int, 3, 1>;
using Vector4d = Matrix<double, 4, 1>;
using Matrix3d = Matrix<double, 3, 3>;

template <typename T>
class Quaternion;

template <typename T>
class AngleAxis {
 public:
  AngleAxis() = default;
  AngleAxis(const T& angle, const Matrix<T, 3, 1>& axis) : angle_(angle), axis_(axis) {}
  // Eigen AngleAxis::operator=(const QuaternionBase&)
  explicit AngleAxis(const Quaternion<T>& q);
  T angle() const { return angle_; }
  const Matrix<T, 3, 1>& axis() const { return axis_; }

 private:
  T angle_ = T(0);
  Matrix<T, 3, 1> axis_;
};

template <typename T>
class Quaternion {
 public:
  using Scalar = T;
  Quaternion() = default;
  // Eigen ctor order is (w, x, y, z); storage is (x, y, z, w).
  Quaternion(const T& w, const T& x, const T& y, const T& z) : c_(x, y, z, w) {}
  explicit Quaternion(const AngleAxis<T>& aa) {
    const T ha = T(0.5) * aa.angle();
    c_[3] = std::cos(ha);
    const Matrix<T, 3, 1> v = std::sin(ha) * aa.axis();
    c_[0] = v[0];
    c_[1] = v[1];
    c_[2] = v[2];
  }
  explicit Quaternion(const Matrix<T, 3, 3>& mat) {
    // Eigen quaternionbase_assign_impl<Other,3,3>::run
    T t = mat.trace();
    if (t > T(0)) {
      t = std::sqrt(t + T(1.0));
      c_[3] = T(0.5) * t;
      t = T(0.5) / t;
      c_[0] = (mat.coeff(2, 1) - mat.coeff(1, 2)) * t;
      c_[1] = (mat.coeff(0, 2) - mat.coeff(2, 0)) * t;
      c_[2] = (mat.coeff(1, 0) - mat.coeff(0, 1)) * t;
    } else {
      int i = 0;
      if (mat.coeff(1, 1) > mat.coeff(0, 0)) i = 1;
      if (mat.coeff(2, 2) > mat.coeff(i, i)) i = 2;
      const int j = (i + 1) % 3;
      const int k = (j + 1) % 3;
      t = std::sqrt(mat.coeff(i, i) - mat.coeff(j, j) - mat.coeff(k, k) + T(1.0));
      c_[i] = T(0.5) * t;
      t = T(0.5) / t;
      c_[3] = (mat.coeff(k, j) - mat.coeff(j, k)) * t;
      c_[j] = (mat.coeff(j, i) + mat.coeff(i, j)) * t;
      c_[k] = (mat.coeff(k, i) + mat.coeff(i, k)) * t;
    }
  }

  T& w() { return c_[3]; }
  T& x() { return c_[0]; }
  T& y() { return c_[1]; }
  T& z() { return c_[2]; }
  const T& w() const { return c_[3]; }
  const T& x() const { return c_[0]; }
  const T& y() const { return c_[1]; }
  const T& z() const { return c_[2]; }
  Matrix<T, 4, 1>& coeffs() { return c_; }
  const Matrix<T, 4, 1>& coeffs() const { return c_; }
  Matrix<T, 3, 1> vec() const { return Matrix<T, 3, 1>(c_[0], c_[1], c_[2]); }

  T squaredNorm() const { return c_.squaredNorm(); }
  T norm() const { return c_.norm(); }
  void normalize() { c_.normalize(); }
  Quaternion normalized() const {
    Quaternion q;
    q.c_ = c_.normalized();
    return q;
  }
  Quaternion conjugate() const { return Quaternion(c_[3], -c_[0], -c_[1], -c_[2]); }
  Quaternion inverse() const {
    const T n2 = squaredNorm();
    if (n2 > T(0)) {
      Quaternion q = conjugate();
      q.c_ /= n2;
      return q;
    }
    Quaternion q;
    q.c_.setZero();
    return q;
  }

  // Generic quat_product.
  Quaternion operator*(const Quaternion& b) const {
    const Quaternion& a = *this;
    return Quaternion(a.w() * b.w() - a.x() * b.x() - a.y() * b.y() - a.z() * b.z(),
                      a.w() * b.x() + a.x() * b.w() + a.y() * b.z() - a.z() * b.y(),
                      a.w() * b.y() + a.y() * b.w() + a.z() * b.x() - a.x() * b.z(),
                      a.w() * b.z() + a.z() * b.w() + a.x() * b.y() - a.y() * b.x());
  }
  // QuaternionBase::_transformVector.
  Matrix<T, 3, 1> operator*(const Matrix<T, 3, 1>& v) const {
    const Matrix<T, 3, 1> qv = vec();
    Matrix<T, 3, 1> uv = qv.cross(v);
    uv += uv;
    return v + w() * uv + qv.cross(uv);
  }

  Matrix<T, 3, 3> toRotationMatrix() const {
    // Eigen toRotationMatrix
    Matrix<T, 3, 3> res;
    const T tx = T(2) * x(), ty = T(2) * y(), tz = T(2) * z();
    const T twx = tx * w(), twy = ty * w(), twz = tz * w();
    const T txx = tx * x(), txy = ty * x(), txz = tz * x();
    const T tyy = ty * y(), tyz = tz * y(), tzz = tz * z();
    res(0, 0) = T(1) - (tyy + tzz);
    res(0, 1) = txy - twz;
    res(0, 2) = txz + twy;
    res(1, 0) = txy + twz;
    res(1, 1) = T(1) - (txx + tzz);
    res(1, 2) = tyz - twx;
    res(2, 0) = txz - twy;
    res(2, 1) = tyz + twx;
    res(2, 2) = T(1) - (txx + tyy);
    return res;
  }

 private:
  Matrix<T, 4, 1> c_{T(0), T(0), T(0), T(1)};
};

template <typename T>
AngleAxis<T>::AngleAxis(const Quaternion<T>& q) {
  T n = q.vec().norm();
  if (n != T(0)) {
    angle_ = T(2) * std::atan2(n, std::abs(q.w()));
    if (q.w() < T(0)) n = -n;
    axis_ = q.vec() / n;
  } else {
    angle_ = T(0);
    axis_ = Matrix<T, 3, 1>(T(1), T(0), T(0));
  }
}

using Quaterniond = Quaternion<double>;
using AngleAxisd = AngleAxis<double>;

}  // namespace Eigen

#include "EigenEval.h"
