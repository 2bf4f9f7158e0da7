// Eigen-subset shim -- TEST INFRASTRUCTURE ONLY (oracle/).
//
// Eigen3 is absent from this image and from the GPU boxes (SURVEY.md §0.3,
// §8c), so the unmodified liecl reference sources under /root/reference cannot
// be compiled against the real library. This header is a from-scratch, eager,
// column-major std::complex<double> matrix type that implements exactly the
// Eigen API surface those sources touch (SURVEY.md §8c "Recommended oracle"):
//
//   R:src/dense.cpp:57      a.conjugate().cwiseProduct(b).sum()   -> fused conj-dot
//   R:src/dense.cpp:62      m.norm()                                -> sqrt(sum |a|^2)
//   R:src/dense.cpp:67      a * b - b * a                           -> eager GEMM
//   R:src/operator.cpp:156  base_coeff * m                           -> scaled copy
//   R:src/operator.cpp:159  acc.noalias() += c * m                   -> fused axpy
//   R:src/dense.cpp:114,130 Map / Ref / leftCols / col views
//   R:src/closure.cpp:51-104 Gram bookkeeping (dot, outer products, blocks, ldlt)
//   R:src/dense.cpp:132     BDCSVD singular values (one-sided Jacobi here)
//
// It contains no Eigen code. Arithmetic is written on the raw re/im doubles
// (the formula Eigen's packet math uses, (ac-bd, ad+bc)) so the hot loops
// vectorise; dense results therefore differ from a real-Eigen build only in
// summation order ("reference control flow + shim arithmetic").
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstddef>
#include <stdexcept>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;

namespace shim {
using cd = std::complex<double>;

inline void require(bool ok, const char* what) {
  if (!ok) throw std::logic_error(std::string("Eigen shim: ") + what);
}
inline cd mul(cd a, cd b) {
  return {a.real() * b.real() - a.imag() * b.imag(),
          a.real() * b.imag() + a.imag() * b.real()};
}
} // namespace shim

class MatrixXcd;
class VectorXcd;
class Block;
class ConstBlock;
template <class T> class Map;
template <class T> class Ref;
template <class T> class BDCSVD;

/// Real column vector (singular values).
class VectorXd {
public:
  VectorXd() = default;
  explicit VectorXd(Index n) : v_(static_cast<std::size_t>(n), 0.0) {}
  Index size() const { return static_cast<Index>(v_.size()); }
  Index rows() const { return size(); }
  Index cols() const { return 1; }
  double& operator()(Index i) { return v_[static_cast<std::size_t>(i)]; }
  double operator()(Index i) const { return v_[static_cast<std::size_t>(i)]; }
  double maxCoeff() const {
    shim::require(!v_.empty(), "maxCoeff of empty vector");
    return *std::max_element(v_.begin(), v_.end());
  }
  std::vector<double>& raw() { return v_; }

private:
  std::vector<double> v_;
};

/// Real matrix result of cwiseAbs().
class MatrixXd {
public:
  MatrixXd() = default;
  MatrixXd(Index r, Index c) : r_(r), c_(c), v_(static_cast<std::size_t>(r * c), 0.0) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double& operator()(Index i, Index j) { return v_[static_cast<std::size_t>(i + j * r_)]; }
  double operator()(Index i, Index j) const { return v_[static_cast<std::size_t>(i + j * r_)]; }
  double& operator()(Index i) { return v_[static_cast<std::size_t>(i)]; }
  double maxCoeff() const {
    shim::require(!v_.empty(), "maxCoeff of empty matrix");
    return *std::max_element(v_.begin(), v_.end());
  }

private:
  Index r_ = 0, c_ = 0;
  std::vector<double> v_;
};

/// Lazy c * M (kept lazy so `acc.noalias() += c * M` is one fused axpy).
struct ScaledRef {
  shim::cd s;
  const MatrixXcd& m;
};

/// Lazy conj(a) (.* b) chain for the inner product sum.
struct ConjProductRef {
  const MatrixXcd& a;
  const MatrixXcd& b;
  shim::cd sum() const;
};
struct ConjRef {
  const MatrixXcd& a;
  ConjProductRef cwiseProduct(const MatrixXcd& b) const { return {a, b}; }
  operator MatrixXcd() const;
};

class LdltSolver;

class MatrixXcd {
public:
  using Scalar = shim::cd;

  MatrixXcd() = default;
  MatrixXcd(Index r, Index c) { resize(r, c); }
  MatrixXcd(const ScaledRef& e);
  MatrixXcd(const Block& b);
  MatrixXcd(const ConstBlock& b);
  MatrixXcd(const Map<const VectorXcd>& m);
  MatrixXcd(const Ref<const MatrixXcd>& r);

  static MatrixXcd Zero(Index r, Index c) { return MatrixXcd(r, c); }
  static MatrixXcd Identity(Index r, Index c) {
    MatrixXcd m(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
    return m;
  }

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  Scalar* data() { return v_.data(); }
  const Scalar* data() const { return v_.data(); }
  void resize(Index r, Index c) {
    shim::require(r >= 0 && c >= 0, "negative size");
    r_ = r;
    c_ = c;
    v_.assign(static_cast<std::size_t>(r * c), Scalar(0.0, 0.0));
  }

  Scalar& operator()(Index i, Index j) { return v_[static_cast<std::size_t>(i + j * r_)]; }
  const Scalar& operator()(Index i, Index j) const {
    return v_[static_cast<std::size_t>(i + j * r_)];
  }
  Scalar& operator()(Index i) { return v_[static_cast<std::size_t>(i)]; }
  const Scalar& operator()(Index i) const { return v_[static_cast<std::size_t>(i)]; }

  Block col(Index j);
  ConstBlock col(Index j) const;
  Block row(Index i);
  ConstBlock row(Index i) const;
  Block topLeftCorner(Index r, Index c);
  ConstBlock topLeftCorner(Index r, Index c) const;
  Block leftCols(Index n);
  ConstBlock leftCols(Index n) const;
  Block head(Index n);
  ConstBlock head(Index n) const;

  MatrixXcd adjoint() const {
    MatrixXcd out(c_, r_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) out(j, i) = std::conj((*this)(i, j));
    return out;
  }
  ConjRef conjugate() const { return {*this}; }
  MatrixXd cwiseAbs() const {
    MatrixXd out(r_, c_);
    for (Index k = 0; k < size(); ++k) out(k) = std::abs(v_[static_cast<std::size_t>(k)]);
    return out;
  }
  Scalar sum() const {
    double re = 0.0, im = 0.0;
    for (const Scalar& x : v_) {
      re += x.real();
      im += x.imag();
    }
    return {re, im};
  }
  double squaredNorm() const {
    const double* p = reinterpret_cast<const double*>(v_.data());
    const std::size_t n = 2 * v_.size();
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    std::size_t k = 0;
    for (; k + 4 <= n; k += 4)
      for (std::size_t u = 0; u < 4; ++u) acc[u] += p[k + u] * p[k + u];
    for (; k < n; ++k) acc[0] += p[k] * p[k];
    return (acc[0] + acc[1]) + (acc[2] + acc[3]);
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  /// Conjugate-linear in *this, like Eigen's dot.
  Scalar dot(const MatrixXcd& other) const {
    shim::require(size() == other.size(), "dot size mismatch");
    double re = 0.0, im = 0.0;
    for (Index k = 0; k < size(); ++k) {
      const Scalar a = v_[static_cast<std::size_t>(k)], b = other(k);
      re += a.real() * b.real() + a.imag() * b.imag();
      im += a.real() * b.imag() - a.imag() * b.real();
    }
    return {re, im};
  }

  MatrixXcd& noalias() { return *this; }
  MatrixXcd& operator+=(const MatrixXcd& o) {
    shim::require(r_ == o.r_ && c_ == o.c_, "+= shape mismatch");
    for (Index k = 0; k < size(); ++k) v_[static_cast<std::size_t>(k)] += o(k);
    return *this;
  }
  MatrixXcd& operator-=(const MatrixXcd& o) {
    shim::require(r_ == o.r_ && c_ == o.c_, "-= shape mismatch");
    for (Index k = 0; k < size(); ++k) v_[static_cast<std::size_t>(k)] -= o(k);
    return *this;
  }
  /// Fused axpy: *this += s * m (R:src/operator.cpp:159 hot loop).
  MatrixXcd& operator+=(const ScaledRef& e) {
    shim::require(r_ == e.m.r_ && c_ == e.m.c_, "axpy shape mismatch");
    const double sr = e.s.real(), si = e.s.imag();
    double* acc = reinterpret_cast<double*>(v_.data());
    const double* x = reinterpret_cast<const double*>(e.m.v_.data());
    const std::size_t n = v_.size();
    for (std::size_t k = 0; k < n; ++k) {
      const double xr = x[2 * k], xi = x[2 * k + 1];
      acc[2 * k] += sr * xr - si * xi;
      acc[2 * k + 1] += sr * xi + si * xr;
    }
    return *this;
  }

  LdltSolver ldlt() const;

private:
  friend struct ConjProductRef;
  Index r_ = 0, c_ = 0;
  std::vector<Scalar> v_;
};

class VectorXcd : public MatrixXcd {
public:
  VectorXcd() = default;
  explicit VectorXcd(Index n) : MatrixXcd(n, 1) {}
  VectorXcd(const MatrixXcd& m) : MatrixXcd(m) {
    shim::require(m.cols() == 1 || m.rows() == 0, "VectorXcd from non-vector");
  }
  VectorXcd(const Map<const VectorXcd>& m);
};

/// Mutable rectangular view.
class Block {
public:
  Block(MatrixXcd& m, Index r0, Index c0, Index nr, Index nc)
      : m_(&m), r0_(r0), c0_(c0), nr_(nr), nc_(nc) {
    shim::require(r0 >= 0 && c0 >= 0 && r0 + nr <= m.rows() && c0 + nc <= m.cols(),
                  "block out of range");
  }
  Index rows() const { return nr_; }
  Index cols() const { return nc_; }
  Index size() const { return nr_ * nc_; }
  shim::cd& operator()(Index i, Index j) { return (*m_)(r0_ + i, c0_ + j); }
  const shim::cd& operator()(Index i, Index j) const { return (*m_)(r0_ + i, c0_ + j); }
  shim::cd& operator()(Index k) { return nc_ == 1 ? (*this)(k, 0) : (*this)(0, k); }
  const shim::cd& operator()(Index k) const { return nc_ == 1 ? (*this)(k, 0) : (*this)(0, k); }
  Block head(Index n) const {
    return nc_ == 1 ? Block(*m_, r0_, c0_, n, 1) : Block(*m_, r0_, c0_, 1, n);
  }
  MatrixXcd adjoint() const { return MatrixXcd(*this).adjoint(); }
  const MatrixXcd& parent() const { return *m_; }
  Index r0() const { return r0_; }
  Index c0() const { return c0_; }

  template <class Src> Block& assign(const Src& src) {
    shim::require(src.size() == size(), "block assignment size mismatch");
    const bool same_shape = src.rows() == nr_ && src.cols() == nc_;
    shim::require(same_shape || nr_ == 1 || nc_ == 1, "block assignment shape mismatch");
    if (same_shape) {
      for (Index j = 0; j < nc_; ++j)
        for (Index i = 0; i < nr_; ++i) (*this)(i, j) = src(i, j);
    } else {
      for (Index k = 0; k < size(); ++k) (*this)(k) = src(k);
    }
    return *this;
  }
  Block& operator=(const Block& o) { return assign(MatrixXcd(o)); }
  Block& operator=(const MatrixXcd& o) { return assign(o); }
  Block& operator=(const ConstBlock& o);
  Block& operator=(const Map<const VectorXcd>& o);
  Block& operator=(const Ref<const MatrixXcd>& o);

private:
  MatrixXcd* m_;
  Index r0_, c0_, nr_, nc_;
};

/// Read-only rectangular view.
class ConstBlock {
public:
  ConstBlock(const MatrixXcd& m, Index r0, Index c0, Index nr, Index nc)
      : m_(&m), r0_(r0), c0_(c0), nr_(nr), nc_(nc) {
    shim::require(r0 >= 0 && c0 >= 0 && r0 + nr <= m.rows() && c0 + nc <= m.cols(),
                  "block out of range");
  }
  Index rows() const { return nr_; }
  Index cols() const { return nc_; }
  Index size() const { return nr_ * nc_; }
  const shim::cd& operator()(Index i, Index j) const { return (*m_)(r0_ + i, c0_ + j); }
  const shim::cd& operator()(Index k) const { return nc_ == 1 ? (*this)(k, 0) : (*this)(0, k); }
  ConstBlock head(Index n) const {
    return nc_ == 1 ? ConstBlock(*m_, r0_, c0_, n, 1) : ConstBlock(*m_, r0_, c0_, 1, n);
  }
  MatrixXcd adjoint() const { return MatrixXcd(*this).adjoint(); }
  const MatrixXcd& parent() const { return *m_; }
  Index r0() const { return r0_; }
  Index c0() const { return c0_; }

private:
  const MatrixXcd* m_;
  Index r0_, c0_, nr_, nc_;
};

template <> class Map<const VectorXcd> {
public:
  Map(const shim::cd* p, Index n) : p_(p), n_(n) {}
  Index rows() const { return n_; }
  Index cols() const { return 1; }
  Index size() const { return n_; }
  const shim::cd& operator()(Index i, Index) const { return p_[i]; }
  const shim::cd& operator()(Index i) const { return p_[i]; }

private:
  const shim::cd* p_;
  Index n_;
};

template <> class Ref<const MatrixXcd> {
public:
  Ref(const MatrixXcd& m) : p_(m.data()), r_(m.rows()), c_(m.cols()), ld_(m.rows()) {}
  Ref(const ConstBlock& b)
      : p_(b.parent().data() + b.r0() + b.c0() * b.parent().rows()), r_(b.rows()),
        c_(b.cols()), ld_(b.parent().rows()) {}
  Ref(const Block& b)
      : p_(b.parent().data() + b.r0() + b.c0() * b.parent().rows()), r_(b.rows()),
        c_(b.cols()), ld_(b.parent().rows()) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  const shim::cd& operator()(Index i, Index j) const { return p_[i + j * ld_]; }
  const shim::cd& operator()(Index k) const { return c_ == 1 ? p_[k] : p_[k * ld_]; }

private:
  const shim::cd* p_;
  Index r_, c_, ld_;
};

// ---- deferred member definitions -------------------------------------------

inline MatrixXcd::MatrixXcd(const ScaledRef& e) : MatrixXcd(e.m.rows(), e.m.cols()) {
  for (Index k = 0; k < size(); ++k) v_[static_cast<std::size_t>(k)] = shim::mul(e.s, e.m(k));
}
template <class Src> inline void copy_from(MatrixXcd& dst, const Src& src) {
  dst.resize(src.rows(), src.cols());
  for (Index j = 0; j < src.cols(); ++j)
    for (Index i = 0; i < src.rows(); ++i) dst(i, j) = src(i, j);
}
inline MatrixXcd::MatrixXcd(const Block& b) { copy_from(*this, b); }
inline MatrixXcd::MatrixXcd(const ConstBlock& b) { copy_from(*this, b); }
inline MatrixXcd::MatrixXcd(const Map<const VectorXcd>& m) { copy_from(*this, m); }
inline MatrixXcd::MatrixXcd(const Ref<const MatrixXcd>& r) { copy_from(*this, r); }
inline VectorXcd::VectorXcd(const Map<const VectorXcd>& m) : MatrixXcd(m) {}

inline ConjRef::operator MatrixXcd() const {
  MatrixXcd out(a.rows(), a.cols());
  for (Index k = 0; k < a.size(); ++k) out(k) = std::conj(a(k));
  return out;
}
/// sum_k conj(a_k) * b_k (R:src/dense.cpp:57). Four accumulator pairs so the
/// reduction pipelines/vectorises like Eigen's packet accumulators.
inline shim::cd ConjProductRef::sum() const {
  shim::require(a.r_ == b.r_ && a.c_ == b.c_, "cwiseProduct shape mismatch");
  const double* x = reinterpret_cast<const double*>(a.v_.data());
  const double* y = reinterpret_cast<const double*>(b.v_.data());
  const std::size_t n = a.v_.size();
  double re[4] = {0.0, 0.0, 0.0, 0.0}, im[4] = {0.0, 0.0, 0.0, 0.0};
  std::size_t k = 0;
  for (; k + 4 <= n; k += 4) {
    for (std::size_t u = 0; u < 4; ++u) {
      const double xr = x[2 * (k + u)], xi = x[2 * (k + u) + 1];
      const double yr = y[2 * (k + u)], yi = y[2 * (k + u) + 1];
      re[u] += xr * yr + xi * yi;
      im[u] += xr * yi - xi * yr;
    }
  }
  for (; k < n; ++k) {
    const double xr = x[2 * k], xi = x[2 * k + 1], yr = y[2 * k], yi = y[2 * k + 1];
    re[0] += xr * yr + xi * yi;
    im[0] += xr * yi - xi * yr;
  }
  return {(re[0] + re[1]) + (re[2] + re[3]), (im[0] + im[1]) + (im[2] + im[3])};
}

inline Block MatrixXcd::col(Index j) { return Block(*this, 0, j, r_, 1); }
inline ConstBlock MatrixXcd::col(Index j) const { return ConstBlock(*this, 0, j, r_, 1); }
inline Block MatrixXcd::row(Index i) { return Block(*this, i, 0, 1, c_); }
inline ConstBlock MatrixXcd::row(Index i) const { return ConstBlock(*this, i, 0, 1, c_); }
inline Block MatrixXcd::topLeftCorner(Index r, Index c) { return Block(*this, 0, 0, r, c); }
inline ConstBlock MatrixXcd::topLeftCorner(Index r, Index c) const {
  return ConstBlock(*this, 0, 0, r, c);
}
inline Block MatrixXcd::leftCols(Index n) { return Block(*this, 0, 0, r_, n); }
inline ConstBlock MatrixXcd::leftCols(Index n) const { return ConstBlock(*this, 0, 0, r_, n); }
inline Block MatrixXcd::head(Index n) {
  return c_ == 1 ? Block(*this, 0, 0, n, 1) : Block(*this, 0, 0, 1, n);
}
inline ConstBlock MatrixXcd::head(Index n) const {
  return c_ == 1 ? ConstBlock(*this, 0, 0, n, 1) : ConstBlock(*this, 0, 0, 1, n);
}

inline Block& Block::operator=(const ConstBlock& o) { return assign(o); }
inline Block& Block::operator=(const Map<const VectorXcd>& o) { return assign(o); }
inline Block& Block::operator=(const Ref<const MatrixXcd>& o) { return assign(o); }

// ---- arithmetic --------------------------------------------------------------

inline ScaledRef operator*(shim::cd s, const MatrixXcd& m) { return {s, m}; }
inline MatrixXcd operator*(const MatrixXcd& m, shim::cd s) { return MatrixXcd(ScaledRef{s, m}); }

inline MatrixXcd operator+(const MatrixXcd& a, const MatrixXcd& b) {
  MatrixXcd out(a);
  out += b;
  return out;
}
inline MatrixXcd operator-(const MatrixXcd& a, const MatrixXcd& b) {
  MatrixXcd out(a);
  out -= b;
  return out;
}
inline MatrixXcd operator-(const MatrixXcd& a) {
  MatrixXcd out(a.rows(), a.cols());
  for (Index k = 0; k < a.size(); ++k) out(k) = -a(k);
  return out;
}
inline MatrixXcd operator/(const MatrixXcd& a, double s) {
  MatrixXcd out(a.rows(), a.cols());
  for (Index k = 0; k < a.size(); ++k) out(k) = a(k) / s;
  return out;
}

/// Eager GEMM, column-major, i-innermost so the loop vectorises.
inline MatrixXcd operator*(const MatrixXcd& a, const MatrixXcd& b) {
  shim::require(a.cols() == b.rows(), "product shape mismatch");
  const Index m = a.rows(), k = a.cols(), n = b.cols();
  MatrixXcd c(m, n);
  const double* A = reinterpret_cast<const double*>(a.data());
  double* C = reinterpret_cast<double*>(c.data());
  for (Index j = 0; j < n; ++j) {
    double* cj = C + 2 * j * m;
    for (Index p = 0; p < k; ++p) {
      const shim::cd bpj = b(p, j);
      const double br = bpj.real(), bi = bpj.imag();
      const double* ap = A + 2 * p * m;
      for (Index i = 0; i < m; ++i) {
        const double ar = ap[2 * i], ai = ap[2 * i + 1];
        cj[2 * i] += ar * br - ai * bi;
        cj[2 * i + 1] += ar * bi + ai * br;
      }
    }
  }
  return c;
}

// ---- solvers -----------------------------------------------------------------

/// ldlt().solve(B): Gaussian elimination with partial pivoting (the Gram
/// matrices it sees are Hermitian positive definite; only Alg. 2's refresh,
/// R:src/closure.cpp:93, uses it).
class LdltSolver {
public:
  explicit LdltSolver(MatrixXcd a) : a_(std::move(a)) {
    shim::require(a_.rows() == a_.cols(), "ldlt of non-square matrix");
  }
  MatrixXcd solve(const MatrixXcd& rhs) const {
    const Index n = a_.rows();
    shim::require(rhs.rows() == n, "solve shape mismatch");
    MatrixXcd a = a_, x = rhs;
    for (Index col = 0; col < n; ++col) {
      Index piv = col;
      for (Index i = col + 1; i < n; ++i)
        if (std::abs(a(i, col)) > std::abs(a(piv, col))) piv = i;
      if (piv != col) {
        for (Index j = 0; j < n; ++j) std::swap(a(col, j), a(piv, j));
        for (Index j = 0; j < x.cols(); ++j) std::swap(x(col, j), x(piv, j));
      }
      const shim::cd d = a(col, col);
      shim::require(d != shim::cd(0.0, 0.0), "singular matrix in ldlt");
      for (Index i = col + 1; i < n; ++i) {
        const shim::cd f = a(i, col) / d;
        if (f == shim::cd(0.0, 0.0)) continue;
        for (Index j = col; j < n; ++j) a(i, j) -= f * a(col, j);
        for (Index j = 0; j < x.cols(); ++j) x(i, j) -= f * x(col, j);
      }
    }
    for (Index j = 0; j < x.cols(); ++j) {
      for (Index i = n - 1; i >= 0; --i) {
        shim::cd acc = x(i, j);
        for (Index p = i + 1; p < n; ++p) acc -= a(i, p) * x(p, j);
        x(i, j) = acc / a(i, i);
      }
    }
    return x;
  }

private:
  MatrixXcd a_;
};
inline LdltSolver MatrixXcd::ldlt() const { return LdltSolver(*this); }

/// Singular values by one-sided (Hestenes) Jacobi, sorted descending; stands
/// in for BDCSVD in the rank check (R:src/dense.cpp:132, Alg. 1 only).
template <> class BDCSVD<MatrixXcd> {
public:
  explicit BDCSVD(const MatrixXcd& in) {
    MatrixXcd a = in;
    const Index m = a.rows(), n = a.cols();
    const double eps = 1e-15;
    for (int sweep = 0; sweep < 80; ++sweep) {
      bool rotated = false;
      for (Index p = 0; p + 1 < n; ++p) {
        for (Index q = p + 1; q < n; ++q) {
          double alpha = 0.0, beta = 0.0;
          shim::cd gamma(0.0, 0.0);
          for (Index i = 0; i < m; ++i) {
            alpha += std::norm(a(i, p));
            beta += std::norm(a(i, q));
            gamma += std::conj(a(i, p)) * a(i, q);
          }
          const double g = std::abs(gamma);
          if (g == 0.0 || g <= eps * std::sqrt(alpha * beta)) continue;
          rotated = true;
          const shim::cd phase = gamma / g; // a_q e^{-i phi} makes gamma real
          const double zeta = (beta - alpha) / (2.0 * g);
          const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
          for (Index i = 0; i < m; ++i) {
            const shim::cd ap = a(i, p), aq = a(i, q) * std::conj(phase);
            a(i, p) = c * ap - s * aq;
            a(i, q) = s * ap + c * aq;
          }
        }
      }
      if (!rotated) break;
    }
    std::vector<double> norms(static_cast<std::size_t>(n));
    for (Index j = 0; j < n; ++j) {
      double acc = 0.0;
      for (Index i = 0; i < m; ++i) acc += std::norm(a(i, j));
      norms[static_cast<std::size_t>(j)] = std::sqrt(acc);
    }
    std::sort(norms.begin(), norms.end(), std::greater<double>());
    norms.resize(static_cast<std::size_t>(std::min(m, n)));
    sv_ = VectorXd(static_cast<Index>(norms.size()));
    sv_.raw() = norms;
  }
  const VectorXd& singularValues() const { return sv_; }

private:
  VectorXd sv_;
};

} // namespace Eigen
