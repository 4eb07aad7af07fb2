// Eigen-subset shim, evaluation part — TEST INFRASTRUCTURE ONLY (oracle build).
//
// What eval.cpp's ATE alignment (eval.cpp:140-172) uses beyond the hot-path
// subset: a 3 x N dynamic matrix (columns, rowwise().mean(), colwise() - v,
// A * B.transpose()) and JacobiSVD<Matrix3d> with full U / V. The SVD follows
// Eigen 3's two-sided Jacobi algorithm for square matrices (JacobiSVD.h:
// scale by the max |coefficient|, sweep the (p, q) pairs with
// real_2x2_jacobi_svd until every off-diagonal entry is below the threshold,
// make the singular values positive, sort them descending). The rotation the
// ATE alignment builds from U V^T is unique for a non-degenerate covariance, so
// agreement with a real Eigen build is at rounding level (not bit-pinned).
#pragma once

#include <vector>

namespace Eigen {

constexpr int Dynamic = -1;

template <typename M>
struct RowwiseMean;
template <typename M>
struct ColwiseMinus;
template <typename M>
struct Transposed3X;

// Matrix<T, 3, Dynamic>: column storage of 3-vectors.
template <typename T>
class Matrix<T, 3, Dynamic> {
 public:
  using Scalar = T;
  using Col = Matrix<T, 3, 1>;
  Matrix() = default;
  Matrix(Index rows, Index cols) : c_((size_t)cols) {
    if (rows != 3) throw std::invalid_argument("shim: Matrix3X needs 3 rows");
  }
  Index rows() const { return 3; }
  Index cols() const { return (Index)c_.size(); }
  Col& col(Index k) { return c_[(size_t)k]; }
  const Col& col(Index k) const { return c_[(size_t)k]; }
  T& operator()(Index r, Index c) { return c_[(size_t)c][r]; }
  const T& operator()(Index r, Index c) const { return c_[(size_t)c][r]; }
  RowwiseMean<Matrix> rowwise() const { return RowwiseMean<Matrix>{*this}; }
  ColwiseMinus<Matrix> colwise() const { return ColwiseMinus<Matrix>{*this}; }
  Transposed3X<Matrix> transpose() const { return Transposed3X<Matrix>{*this}; }
  // (3 x N) * (N x 3): sequential sums over the columns
  Matrix<T, 3, 3> operator*(const Transposed3X<Matrix>& bt) const {
    Matrix<T, 3, 3> out;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        T s = T(0);
        for (Index k = 0; k < cols(); ++k) s = s + (*this)(i, k) * bt.m(j, k);
        out(i, j) = s;
      }
    return out;
  }

 private:
  std::vector<Col> c_;
};

template <typename M>
struct RowwiseMean {
  const M& m;
  // Eigen: rowwise().mean() = rowwise().sum() / cols
  Matrix<typename M::Scalar, 3, 1> mean() const {
    Matrix<typename M::Scalar, 3, 1> s;
    for (Index k = 0; k < m.cols(); ++k) s += m.col(k);
    return s / typename M::Scalar(m.cols());
  }
};

template <typename M>
struct ColwiseMinus {
  const M& m;
  M operator-(const Matrix<typename M::Scalar, 3, 1>& v) const {
    M out(3, m.cols());
    for (Index k = 0; k < m.cols(); ++k) out.col(k) = m.col(k) - v;
    return out;
  }
};

template <typename M>
struct Transposed3X {
  const M& m;
};

using Matrix3Xd = Matrix<double, 3, Dynamic>;

enum DecompositionOptions { ComputeFullU = 0x04, ComputeThinU = 0x08, ComputeFullV = 0x10,
                            ComputeThinV = 0x20 };

namespace internal {
// JacobiRotation (Jacobi.h) for real scalars
template <typename T>
struct JacobiRotation {
  T c = T(1), s = T(0);
  JacobiRotation transpose() const { return {c, -s}; }
  JacobiRotation operator*(const JacobiRotation& o) const {
    return {c * o.c - s * o.s, c * o.s + s * o.c};
  }
  // makeJacobi(x, y, z): the rotation diagonalising [[x, y], [y, z]]
  void make(T x, T y, T z) {
    const T deno = T(2) * std::abs(y);
    if (deno < std::numeric_limits<T>::min()) {
      c = T(1);
      s = T(0);
    } else {
      const T tau = (x - z) / deno;
      const T w = std::sqrt(tau * tau + T(1));
      const T t = tau > T(0) ? T(1) / (tau + w) : T(1) / (tau - w);
      const T sign_t = t > T(0) ? T(1) : T(-1);
      const T n = T(1) / std::sqrt(t * t + T(1));
      s = -sign_t * (y / std::abs(y)) * std::abs(t) * n;
      c = n;
    }
  }
};
// apply_rotation_in_the_plane: x' = c x + s y, y' = -s x + c y
template <typename T>
inline void rot_rows(Matrix<T, 3, 3>& m, int p, int q, const JacobiRotation<T>& j) {
  for (int i = 0; i < 3; ++i) {
    const T xi = m(p, i), yi = m(q, i);
    m(p, i) = j.c * xi + j.s * yi;
    m(q, i) = -j.s * xi + j.c * yi;
  }
}
template <typename T>
inline void rot_cols(Matrix<T, 3, 3>& m, int p, int q, const JacobiRotation<T>& jr) {
  const JacobiRotation<T> j = jr.transpose();  // applyOnTheRight uses j.transpose()
  for (int i = 0; i < 3; ++i) {
    const T xi = m(i, p), yi = m(i, q);
    m(i, p) = j.c * xi + j.s * yi;
    m(i, q) = -j.s * xi + j.c * yi;
  }
}
}  // namespace internal

template <typename M>
class JacobiSVD {
 public:
  using T = typename M::Scalar;
  JacobiSVD(const M& a, unsigned int /*options*/) {
    static_assert(M::kRows == 3 && M::kCols == 3, "shim: 3x3 JacobiSVD only");
    using internal::JacobiRotation;
    T scale = a.cwiseAbs().maxCoeff();
    if (!(scale > T(0)) || !std::isfinite(scale)) scale = T(1);
    M w = a / scale;
    u_ = M::Identity();
    v_ = M::Identity();
    const T consider_zero = std::numeric_limits<T>::min();
    const T precision = T(2) * std::numeric_limits<T>::epsilon();
    T max_diag = std::max(std::abs(w(0, 0)), std::max(std::abs(w(1, 1)), std::abs(w(2, 2))));
    bool finished = false;
    while (!finished) {
      finished = true;
      for (int p = 1; p < 3; ++p)
        for (int q = 0; q < p; ++q) {
          const T threshold = std::max(consider_zero, precision * max_diag);
          if (std::max(std::abs(w(p, q)), std::abs(w(q, p))) > threshold) {
            finished = false;
            // real_2x2_jacobi_svd (RealSvd2x2.h)
            T m00 = w(p, p), m01 = w(p, q), m10 = w(q, p), m11 = w(q, q);
            JacobiRotation<T> rot1;
            const T t = m00 + m11, d = m10 - m01;
            if (std::abs(d) < std::numeric_limits<T>::min()) {
              rot1.s = T(0);
              rot1.c = T(1);
            } else {
              const T uu = t / d, tmp = std::sqrt(T(1) + uu * uu);
              rot1.s = T(1) / tmp;
              rot1.c = uu / tmp;
            }
            // m.applyOnTheLeft(0, 1, rot1)
            const T n00 = rot1.c * m00 + rot1.s * m10, n01 = rot1.c * m01 + rot1.s * m11;
            const T n11 = -rot1.s * m01 + rot1.c * m11;
            JacobiRotation<T> jr;
            jr.make(n00, n01, n11);
            const JacobiRotation<T> jl = rot1 * jr.transpose();
            internal::rot_rows(w, p, q, jl);
            internal::rot_cols(u_, p, q, jl.transpose());
            internal::rot_cols(w, p, q, jr);
            internal::rot_cols(v_, p, q, jr);
            max_diag = std::max(max_diag, std::max(std::abs(w(p, p)), std::abs(w(q, q))));
          }
        }
    }
    for (int i = 0; i < 3; ++i) {
      const T a_ii = w(i, i);
      sv_[i] = std::abs(a_ii) * scale;
      if (a_ii < T(0))
        for (int r = 0; r < 3; ++r) u_(r, i) = -u_(r, i);
    }
    // descending order (selection of the largest remaining, swapping columns)
    for (int i = 0; i < 3; ++i) {
      int pos = i;
      for (int k = i + 1; k < 3; ++k)
        if (sv_[k] > sv_[pos]) pos = k;
      if (pos != i) {
        std::swap(sv_[i], sv_[pos]);
        for (int r = 0; r < 3; ++r) {
          std::swap(u_(r, i), u_(r, pos));
          std::swap(v_(r, i), v_(r, pos));
        }
      }
    }
  }
  const M& matrixU() const { return u_; }
  const M& matrixV() const { return v_; }
  Matrix<T, 3, 1> singularValues() const { return sv_; }

 private:
  M u_, v_;
  Matrix<T, 3, 1> sv_;
};

}  // namespace Eigen
