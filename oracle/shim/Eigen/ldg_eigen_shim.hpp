// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// A minimal, eager (no expression templates) subset of the Eigen 3 API,
// exactly the surface that the reference headers (/root/reference/proj/
// include/ldg/{fields,assembly,system,convergence,vtkout}.hpp) and their unit
// tests use, so that the UNMODIFIED reference can be compiled here as the
// parity oracle.  Eigen itself is not installed in this image.
//
// Semantics that matter for parity are reproduced deliberately:
//  * SparseMatrix<double> is column-major CSC with int indices;
//  * setFromTriplets sums duplicates in triplet order (Eigen's
//    set_from_triplets: bucket per inner vector in insertion order, then
//    collapseDuplicates left-to-right), and keeps explicit zeros;
//  * sparse * dense walks columns (y += A(:,j) x_j), as Eigen does for CSC.
// SparseLU is a stand-in: a registered external solver hook (SciPy SuperLU,
// installed from Python via ldgref_set_sparse_solver) or, without a hook, a
// dense partial-pivoting LU.  It is labelled "Eigen-shim" wherever timed.
#ifndef LDG_EIGEN_SHIM_HPP
#define LDG_EIGEN_SHIM_HPP

#include <algorithm>
#include <cassert>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };

inline void setNbThreads(int) {}

class VectorXd;
class MatrixXd;
template <typename Scalar, int Options = 0, typename StorageIndex = int>
class SparseMatrix;

// ---------------------------------------------------------------- comma init
template <typename Target>
class CommaInit {
 public:
  CommaInit(Target& t, double v) : t_(t), i_(0) { t_.comma_set(i_++, v); }
  CommaInit& operator,(double v) {
    t_.comma_set(i_++, v);
    return *this;
  }

 private:
  Target& t_;
  Index i_;
};

// ---------------------------------------------------------------- RowVector
// Result of VectorXd::transpose(); only used as the right-hand side of
// MatrixXd::row(k) = ....
struct RowVectorXd {
  std::vector<double> v;
};

// ---------------------------------------------------------------- VectorXd
class VectorXd {
 public:
  VectorXd() = default;
  explicit VectorXd(Index n) : v_(static_cast<size_t>(n), 0.0) {}

  static VectorXd Zero(Index n) { return VectorXd(n); }
  static VectorXd Constant(Index n, double c) {
    VectorXd r(n);
    std::fill(r.v_.begin(), r.v_.end(), c);
    return r;
  }

  Index size() const { return static_cast<Index>(v_.size()); }
  Index rows() const { return size(); }
  Index cols() const { return 1; }
  void resize(Index n) { v_.assign(static_cast<size_t>(n), 0.0); }
  void setZero() { std::fill(v_.begin(), v_.end(), 0.0); }
  VectorXd& setConstant(double c) {
    std::fill(v_.begin(), v_.end(), c);
    return *this;
  }

  double& operator[](Index i) { return v_[static_cast<size_t>(i)]; }
  double operator[](Index i) const { return v_[static_cast<size_t>(i)]; }
  double& operator()(Index i) { return v_[static_cast<size_t>(i)]; }
  double operator()(Index i) const { return v_[static_cast<size_t>(i)]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }

  // Segment proxy: assignable view into the vector.
  class Segment {
   public:
    Segment(VectorXd& v, Index s, Index n) : v_(v), s_(s), n_(n) {}
    Segment& operator=(const VectorXd& x) {
      if (x.size() != n_) throw std::invalid_argument("segment size mismatch");
      for (Index i = 0; i < n_; ++i) v_[s_ + i] = x[i];
      return *this;
    }
    Segment& operator=(const Segment& x) { return *this = VectorXd(x); }
    operator VectorXd() const {
      VectorXd r(n_);
      for (Index i = 0; i < n_; ++i) r[i] = v_[s_ + i];
      return r;
    }
    Index size() const { return n_; }
    double norm() const { return VectorXd(*this).norm(); }
    VectorXd cwiseAbs() const { return VectorXd(*this).cwiseAbs(); }

   private:
    VectorXd& v_;
    Index s_, n_;
  };

  Segment segment(Index s, Index n) { return Segment(*this, s, n); }
  VectorXd segment(Index s, Index n) const { return slice(s, n); }
  Segment head(Index n) { return Segment(*this, 0, n); }
  VectorXd head(Index n) const { return slice(0, n); }
  Segment tail(Index n) { return Segment(*this, size() - n, n); }
  VectorXd tail(Index n) const { return slice(size() - n, n); }

  double squaredNorm() const {
    double s = 0.0;
    for (double x : v_) s += x * x;
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  double dot(const VectorXd& o) const {
    if (o.size() != size()) throw std::invalid_argument("dot size mismatch");
    double s = 0.0;
    for (size_t i = 0; i < v_.size(); ++i) s += v_[i] * o.v_[i];
    return s;
  }
  bool allFinite() const {
    for (double x : v_)
      if (!std::isfinite(x)) return false;
    return true;
  }
  VectorXd cwiseAbs() const {
    VectorXd r(size());
    for (size_t i = 0; i < v_.size(); ++i) r.v_[i] = std::abs(v_[i]);
    return r;
  }
  double maxCoeff() const {
    if (v_.empty()) throw std::invalid_argument("maxCoeff of empty vector");
    return *std::max_element(v_.begin(), v_.end());
  }
  double minCoeff() const {
    if (v_.empty()) throw std::invalid_argument("minCoeff of empty vector");
    return *std::min_element(v_.begin(), v_.end());
  }
  double sum() const {
    double s = 0.0;
    for (double x : v_) s += x;
    return s;
  }
  RowVectorXd transpose() const { return RowVectorXd{v_}; }
  VectorXd eval() const { return *this; }

  VectorXd& operator+=(const VectorXd& o) {
    check(o);
    for (size_t i = 0; i < v_.size(); ++i) v_[i] += o.v_[i];
    return *this;
  }
  VectorXd& operator-=(const VectorXd& o) {
    check(o);
    for (size_t i = 0; i < v_.size(); ++i) v_[i] -= o.v_[i];
    return *this;
  }
  VectorXd& operator*=(double s) {
    for (double& x : v_) x *= s;
    return *this;
  }

  CommaInit<VectorXd> operator<<(double v) { return CommaInit<VectorXd>(*this, v); }
  void comma_set(Index i, double v) { v_.at(static_cast<size_t>(i)) = v; }

  void check(const VectorXd& o) const {
    if (o.size() != size()) throw std::invalid_argument("vector size mismatch");
  }

 private:
  VectorXd slice(Index s, Index n) const {
    VectorXd r(n);
    for (Index i = 0; i < n; ++i) r[i] = v_[static_cast<size_t>(s + i)];
    return r;
  }
  std::vector<double> v_;
};

inline VectorXd operator+(VectorXd a, const VectorXd& b) { return a += b; }
inline VectorXd operator-(VectorXd a, const VectorXd& b) { return a -= b; }
inline VectorXd operator-(VectorXd a) {
  for (Index i = 0; i < a.size(); ++i) a[i] = -a[i];
  return a;
}
inline VectorXd operator*(double s, VectorXd a) { return a *= s; }
inline VectorXd operator*(VectorXd a, double s) { return a *= s; }

// ---------------------------------------------------------------- MatrixXd
// Column-major dense matrix, like Eigen's default.
class MatrixXd {
 public:
  MatrixXd() = default;
  MatrixXd(Index r, Index c) : r_(r), c_(c), a_(static_cast<size_t>(r * c), 0.0) {}
  template <typename S, int O, typename I>
  explicit MatrixXd(const SparseMatrix<S, O, I>& sp);

  static MatrixXd Zero(Index r, Index c) { return MatrixXd(r, c); }
  static MatrixXd Constant(Index r, Index c, double v) {
    MatrixXd m(r, c);
    std::fill(m.a_.begin(), m.a_.end(), v);
    return m;
  }
  static MatrixXd Identity(Index r, Index c) {
    MatrixXd m(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
    return m;
  }

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double& operator()(Index i, Index j) { return a_[static_cast<size_t>(j * r_ + i)]; }
  double operator()(Index i, Index j) const { return a_[static_cast<size_t>(j * r_ + i)]; }
  void setZero() { std::fill(a_.begin(), a_.end(), 0.0); }
  void resize(Index r, Index c) {
    r_ = r;
    c_ = c;
    a_.assign(static_cast<size_t>(r * c), 0.0);
  }
  MatrixXd eval() const { return *this; }

  class Row {
   public:
    Row(MatrixXd& m, Index k) : m_(m), k_(k) {}
    Row& operator=(const RowVectorXd& v) {
      if (static_cast<Index>(v.v.size()) != m_.cols())
        throw std::invalid_argument("row size mismatch");
      for (Index j = 0; j < m_.cols(); ++j) m_(k_, j) = v.v[static_cast<size_t>(j)];
      return *this;
    }

   private:
    MatrixXd& m_;
    Index k_;
  };
  class Col {
   public:
    Col(MatrixXd& m, Index j) : m_(m), j_(j) {}
    Col& setConstant(double v) {
      for (Index i = 0; i < m_.rows(); ++i) m_(i, j_) = v;
      return *this;
    }
    Col& setZero() { return setConstant(0.0); }
    operator VectorXd() const {
      VectorXd r(m_.rows());
      for (Index i = 0; i < m_.rows(); ++i) r[i] = m_(i, j_);
      return r;
    }

   private:
    MatrixXd& m_;
    Index j_;
  };
  class Diagonal {
   public:
    explicit Diagonal(MatrixXd& m) : m_(m) {}
    CommaInit<Diagonal> operator<<(double v) { return CommaInit<Diagonal>(*this, v); }
    void comma_set(Index i, double v) {
      if (i >= std::min(m_.rows(), m_.cols())) throw std::out_of_range("diagonal init");
      m_(i, i) = v;
    }

   private:
    MatrixXd& m_;
  };

  Row row(Index k) { return Row(*this, k); }
  Col col(Index j) { return Col(*this, j); }
  VectorXd col(Index j) const {
    VectorXd r(r_);
    for (Index i = 0; i < r_; ++i) r[i] = (*this)(i, j);
    return r;
  }
  Diagonal diagonal() { return Diagonal(*this); }
  MatrixXd block(Index i0, Index j0, Index nr, Index nc) const {
    MatrixXd b(nr, nc);
    for (Index j = 0; j < nc; ++j)
      for (Index i = 0; i < nr; ++i) b(i, j) = (*this)(i0 + i, j0 + j);
    return b;
  }
  MatrixXd topRows(Index n) const { return block(0, 0, n, c_); }
  MatrixXd bottomRows(Index n) const { return block(r_ - n, 0, n, c_); }

  MatrixXd cwiseAbs() const {
    MatrixXd m(*this);
    for (double& x : m.a_) x = std::abs(x);
    return m;
  }
  double maxCoeff() const {
    if (a_.empty()) throw std::invalid_argument("maxCoeff of empty matrix");
    return *std::max_element(a_.begin(), a_.end());
  }
  double minCoeff() const {
    if (a_.empty()) throw std::invalid_argument("minCoeff of empty matrix");
    return *std::min_element(a_.begin(), a_.end());
  }

  MatrixXd& operator+=(const MatrixXd& o) {
    check(o);
    for (size_t i = 0; i < a_.size(); ++i) a_[i] += o.a_[i];
    return *this;
  }
  MatrixXd& operator-=(const MatrixXd& o) {
    check(o);
    for (size_t i = 0; i < a_.size(); ++i) a_[i] -= o.a_[i];
    return *this;
  }
  MatrixXd& operator*=(double s) {
    for (double& x : a_) x *= s;
    return *this;
  }

  // Row-major fill order, as Eigen's comma initializer.
  CommaInit<MatrixXd> operator<<(double v) { return CommaInit<MatrixXd>(*this, v); }
  void comma_set(Index idx, double v) {
    if (idx >= size()) throw std::out_of_range("too many coefficients in comma initializer");
    (*this)(idx / c_, idx % c_) = v;
  }

  class ColPivHouseholderQR;
  ColPivHouseholderQR colPivHouseholderQr() const;

  void check(const MatrixXd& o) const {
    if (o.r_ != r_ || o.c_ != c_) throw std::invalid_argument("matrix size mismatch");
  }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> a_;
};

inline MatrixXd operator+(MatrixXd a, const MatrixXd& b) { return a += b; }
inline MatrixXd operator-(MatrixXd a, const MatrixXd& b) { return a -= b; }
inline MatrixXd operator*(double s, MatrixXd a) { return a *= s; }
inline MatrixXd operator*(MatrixXd a, double s) { return a *= s; }
inline VectorXd operator*(const MatrixXd& a, const VectorXd& x) {
  if (a.cols() != x.size()) throw std::invalid_argument("matvec size mismatch");
  VectorXd y(a.rows());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) y[i] += a(i, j) * x[j];
  return y;
}

// Least-squares solve by Householder QR with column pivoting (tests only).
class MatrixXd::ColPivHouseholderQR {
 public:
  explicit ColPivHouseholderQR(const MatrixXd& a) : a_(a) {}
  VectorXd solve(const VectorXd& b) const {
    const Index m = a_.rows(), n = a_.cols();
    MatrixXd r = a_;
    VectorXd y = b;
    std::vector<Index> perm(static_cast<size_t>(n));
    std::iota(perm.begin(), perm.end(), 0);
    const Index steps = std::min(m, n);
    Index rank = 0;
    double max_first = 0.0;
    for (Index k = 0; k < steps; ++k) {
      // pivot: column of largest remaining norm
      Index best = k;
      double bestn = -1.0;
      for (Index j = k; j < n; ++j) {
        double s = 0.0;
        for (Index i = k; i < m; ++i) s += r(i, j) * r(i, j);
        if (s > bestn) {
          bestn = s;
          best = j;
        }
      }
      if (k == 0) max_first = std::sqrt(bestn);
      if (std::sqrt(bestn) <= 1e-13 * std::max(max_first, 1e-300)) break;
      if (best != k) {
        for (Index i = 0; i < m; ++i) std::swap(r(i, k), r(i, best));
        std::swap(perm[static_cast<size_t>(k)], perm[static_cast<size_t>(best)]);
      }
      double alpha = 0.0;
      for (Index i = k; i < m; ++i) alpha += r(i, k) * r(i, k);
      alpha = std::sqrt(alpha);
      if (r(k, k) > 0) alpha = -alpha;
      std::vector<double> v(static_cast<size_t>(m - k));
      for (Index i = k; i < m; ++i) v[static_cast<size_t>(i - k)] = r(i, k);
      v[0] -= alpha;
      double vn = 0.0;
      for (double x : v) vn += x * x;
      if (vn > 0.0) {
        for (Index j = k; j < n; ++j) {
          double s = 0.0;
          for (Index i = k; i < m; ++i) s += v[static_cast<size_t>(i - k)] * r(i, j);
          s = 2.0 * s / vn;
          for (Index i = k; i < m; ++i) r(i, j) -= s * v[static_cast<size_t>(i - k)];
        }
        double s = 0.0;
        for (Index i = k; i < m; ++i) s += v[static_cast<size_t>(i - k)] * y[i];
        s = 2.0 * s / vn;
        for (Index i = k; i < m; ++i) y[i] -= s * v[static_cast<size_t>(i - k)];
      }
      ++rank;
    }
    VectorXd z(n);
    for (Index k = rank - 1; k >= 0; --k) {
      double s = y[k];
      for (Index j = k + 1; j < rank; ++j) s -= r(k, j) * z[j];
      z[k] = s / r(k, k);
    }
    VectorXd x(n);
    for (Index k = 0; k < n; ++k) x[perm[static_cast<size_t>(k)]] = z[k];
    return x;
  }

 private:
  MatrixXd a_;
};
inline MatrixXd::ColPivHouseholderQR MatrixXd::colPivHouseholderQr() const {
  return ColPivHouseholderQR(*this);
}

// ---------------------------------------------------------------- FullPivLU
template <typename MatrixType>
class FullPivLU {
 public:
  explicit FullPivLU(const MatrixXd& a) : lu_(a), n_(a.rows()) {
    if (a.rows() != a.cols()) throw std::invalid_argument("FullPivLU needs a square matrix");
    rp_.resize(static_cast<size_t>(n_));
    cp_.resize(static_cast<size_t>(n_));
    std::iota(rp_.begin(), rp_.end(), 0);
    std::iota(cp_.begin(), cp_.end(), 0);
    double maxpivot = 0.0;
    rank_ = n_;
    for (Index k = 0; k < n_; ++k) {
      Index bi = k, bj = k;
      double best = -1.0;
      for (Index j = k; j < n_; ++j)
        for (Index i = k; i < n_; ++i)
          if (std::abs(lu_(i, j)) > best) {
            best = std::abs(lu_(i, j));
            bi = i;
            bj = j;
          }
      if (k == 0) maxpivot = best;
      if (best <= std::numeric_limits<double>::epsilon() * n_ * maxpivot || best == 0.0) {
        rank_ = k;
        break;
      }
      if (bi != k) {
        for (Index j = 0; j < n_; ++j) std::swap(lu_(k, j), lu_(bi, j));
        std::swap(rp_[static_cast<size_t>(k)], rp_[static_cast<size_t>(bi)]);
      }
      if (bj != k) {
        for (Index i = 0; i < n_; ++i) std::swap(lu_(i, k), lu_(i, bj));
        std::swap(cp_[static_cast<size_t>(k)], cp_[static_cast<size_t>(bj)]);
      }
      for (Index i = k + 1; i < n_; ++i) {
        lu_(i, k) /= lu_(k, k);
        for (Index j = k + 1; j < n_; ++j) lu_(i, j) -= lu_(i, k) * lu_(k, j);
      }
    }
  }
  bool isInvertible() const { return rank_ == n_; }
  VectorXd solve(const VectorXd& b) const {
    VectorXd y(n_);
    for (Index i = 0; i < n_; ++i) y[i] = b[rp_[static_cast<size_t>(i)]];
    for (Index i = 0; i < n_; ++i)
      for (Index j = 0; j < i; ++j) y[i] -= lu_(i, j) * y[j];
    for (Index i = n_ - 1; i >= 0; --i) {
      for (Index j = i + 1; j < n_; ++j) y[i] -= lu_(i, j) * y[j];
      y[i] /= lu_(i, i);
    }
    VectorXd x(n_);
    for (Index i = 0; i < n_; ++i) x[cp_[static_cast<size_t>(i)]] = y[i];
    return x;
  }

 private:
  MatrixXd lu_;
  Index n_, rank_;
  std::vector<Index> rp_, cp_;
};

// ---------------------------------------------------------------- Triplet
template <typename Scalar = double, typename StorageIndex = int>
class Triplet {
 public:
  Triplet() = default;
  Triplet(StorageIndex r, StorageIndex c, Scalar v) : r_(r), c_(c), v_(v) {}
  StorageIndex row() const { return r_; }
  StorageIndex col() const { return c_; }
  Scalar value() const { return v_; }

 private:
  StorageIndex r_ = 0, c_ = 0;
  Scalar v_ = 0;
};

// ---------------------------------------------------------------- SparseMatrix
template <typename Scalar, int Options, typename StorageIndex>
class SparseMatrix {
 public:
  SparseMatrix() : outer_(1, 0) {}
  SparseMatrix(Index r, Index c) { resize(r, c); }

  void resize(Index r, Index c) {
    r_ = r;
    c_ = c;
    outer_.assign(static_cast<size_t>(c + 1), 0);
    inner_.clear();
    val_.clear();
  }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index outerSize() const { return c_; }
  Index nonZeros() const { return static_cast<Index>(val_.size()); }
  void makeCompressed() {}

  // Eigen set_from_triplets semantics (see file header).
  template <typename It>
  void setFromTriplets(It begin, It end) {
    std::vector<StorageIndex> count(static_cast<size_t>(c_) + 1, 0);
    size_t n = 0;
    for (It it = begin; it != end; ++it, ++n) {
      if (it->row() < 0 || it->row() >= r_ || it->col() < 0 || it->col() >= c_)
        throw std::out_of_range("triplet index out of range");
      ++count[static_cast<size_t>(it->col()) + 1];
    }
    for (Index j = 0; j < c_; ++j) count[static_cast<size_t>(j + 1)] += count[static_cast<size_t>(j)];
    std::vector<StorageIndex> rows(n);
    std::vector<Scalar> vals(n);
    std::vector<StorageIndex> fill(count.begin(), count.end() - 1);
    for (It it = begin; it != end; ++it) {
      const size_t p = static_cast<size_t>(fill[static_cast<size_t>(it->col())]++);
      rows[p] = it->row();
      vals[p] = it->value();
    }
    outer_.assign(static_cast<size_t>(c_) + 1, 0);
    inner_.clear();
    val_.clear();
    inner_.reserve(n);
    val_.reserve(n);
    std::vector<size_t> order;
    for (Index j = 0; j < c_; ++j) {
      const size_t b = static_cast<size_t>(count[static_cast<size_t>(j)]);
      const size_t e = static_cast<size_t>(count[static_cast<size_t>(j + 1)]);
      order.resize(e - b);
      std::iota(order.begin(), order.end(), b);
      std::stable_sort(order.begin(), order.end(),
                       [&](size_t x, size_t y) { return rows[x] < rows[y]; });
      for (size_t q = 0; q < order.size(); ++q) {
        const size_t p = order[q];
        if (q > 0 && rows[order[q - 1]] == rows[p])
          val_.back() = val_.back() + vals[p];
        else {
          inner_.push_back(rows[p]);
          val_.push_back(vals[p]);
        }
      }
      outer_[static_cast<size_t>(j + 1)] = static_cast<StorageIndex>(val_.size());
    }
  }

  class InnerIterator {
   public:
    InnerIterator(const SparseMatrix& m, Index col)
        : m_(m), p_(m.outer_[static_cast<size_t>(col)]),
          e_(m.outer_[static_cast<size_t>(col + 1)]), col_(col) {}
    explicit operator bool() const { return p_ < e_; }
    InnerIterator& operator++() {
      ++p_;
      return *this;
    }
    Index row() const { return m_.inner_[static_cast<size_t>(p_)]; }
    Index col() const { return col_; }
    Index index() const { return row(); }
    Scalar value() const { return m_.val_[static_cast<size_t>(p_)]; }

   private:
    const SparseMatrix& m_;
    StorageIndex p_, e_;
    Index col_;
  };

  SparseMatrix& operator*=(Scalar s) {
    for (auto& v : val_) v *= s;
    return *this;
  }
  // Union-pattern addition (explicit zeros kept).
  SparseMatrix& operator+=(const SparseMatrix& o) {
    if (o.r_ != r_ || o.c_ != c_) throw std::invalid_argument("sparse size mismatch");
    std::vector<StorageIndex> outer(static_cast<size_t>(c_) + 1, 0);
    std::vector<StorageIndex> inner;
    std::vector<Scalar> val;
    inner.reserve(inner_.size() + o.inner_.size());
    val.reserve(inner_.size() + o.inner_.size());
    for (Index j = 0; j < c_; ++j) {
      StorageIndex a = outer_[static_cast<size_t>(j)], ae = outer_[static_cast<size_t>(j + 1)];
      StorageIndex b = o.outer_[static_cast<size_t>(j)], be = o.outer_[static_cast<size_t>(j + 1)];
      while (a < ae || b < be) {
        if (b >= be || (a < ae && inner_[static_cast<size_t>(a)] < o.inner_[static_cast<size_t>(b)])) {
          inner.push_back(inner_[static_cast<size_t>(a)]);
          val.push_back(val_[static_cast<size_t>(a++)]);
        } else if (a >= ae || o.inner_[static_cast<size_t>(b)] < inner_[static_cast<size_t>(a)]) {
          inner.push_back(o.inner_[static_cast<size_t>(b)]);
          val.push_back(o.val_[static_cast<size_t>(b++)]);
        } else {
          inner.push_back(inner_[static_cast<size_t>(a)]);
          val.push_back(val_[static_cast<size_t>(a++)] + o.val_[static_cast<size_t>(b++)]);
        }
      }
      outer[static_cast<size_t>(j + 1)] = static_cast<StorageIndex>(val.size());
    }
    outer_.swap(outer);
    inner_.swap(inner);
    val_.swap(val);
    return *this;
  }

  const std::vector<StorageIndex>& outer_index() const { return outer_; }
  const std::vector<StorageIndex>& inner_index() const { return inner_; }
  const std::vector<Scalar>& values() const { return val_; }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<StorageIndex> outer_, inner_;
  std::vector<Scalar> val_;
};

template <typename S, int O, typename I>
SparseMatrix<S, O, I> operator*(SparseMatrix<S, O, I> a, double s) {
  return a *= s;
}
template <typename S, int O, typename I>
SparseMatrix<S, O, I> operator*(double s, SparseMatrix<S, O, I> a) {
  return a *= s;
}
template <typename S, int O, typename I>
VectorXd operator*(const SparseMatrix<S, O, I>& a, const VectorXd& x) {
  if (a.cols() != x.size()) throw std::invalid_argument("sparse matvec size mismatch");
  VectorXd y(a.rows());
  for (Index j = 0; j < a.outerSize(); ++j) {
    const double xj = x[j];
    for (typename SparseMatrix<S, O, I>::InnerIterator it(a, j); it; ++it) y[it.row()] += it.value() * xj;
  }
  return y;
}

template <typename S, int O, typename I>
MatrixXd::MatrixXd(const SparseMatrix<S, O, I>& sp) : MatrixXd(sp.rows(), sp.cols()) {
  for (Index j = 0; j < sp.outerSize(); ++j)
    for (typename SparseMatrix<S, O, I>::InnerIterator it(sp, j); it; ++it) (*this)(it.row(), j) = it.value();
}

// ---------------------------------------------------------------- SparseLU
// External solver hook: solves A x = b for the CSC matrix (n x n, colptr,
// rowind, values).  Returns 0 on success.
using SparseSolverHook = int (*)(int n, int nnz, const int* colptr, const int* rowind,
                                 const double* values, const double* rhs, double* x);
inline SparseSolverHook& sparse_solver_hook() {
  static SparseSolverHook hook = nullptr;
  return hook;
}

template <typename MatrixType>
class SparseLU {
 public:
  void compute(const MatrixType& a) {
    a_ = a;
    info_ = (a.rows() == a.cols()) ? Success : InvalidInput;
    factored_ = false;
    if (info_ != Success) return;
    if (sparse_solver_hook() == nullptr) factor_dense();
  }
  ComputationInfo info() const { return info_; }
  VectorXd solve(const VectorXd& b) {
    const Index n = a_.rows();
    VectorXd x(n);
    if (SparseSolverHook hook = sparse_solver_hook()) {
      const int rc = hook(static_cast<int>(n), static_cast<int>(a_.nonZeros()), a_.outer_index().data(),
                          a_.inner_index().data(), a_.values().data(), b.data(), x.data());
      if (rc != 0) {
        info_ = NumericalIssue;
        for (Index i = 0; i < n; ++i) x[i] = std::numeric_limits<double>::quiet_NaN();
      }
      return x;
    }
    if (!factored_) factor_dense();
    for (Index i = 0; i < n; ++i) x[i] = b[piv_[static_cast<size_t>(i)]];
    for (Index i = 0; i < n; ++i) {
      double s = x[i];
      const double* row = &lu_[static_cast<size_t>(i * n)];
      for (Index j = 0; j < i; ++j) s -= row[j] * x[j];
      x[i] = s;
    }
    for (Index i = n - 1; i >= 0; --i) {
      double s = x[i];
      const double* row = &lu_[static_cast<size_t>(i * n)];
      for (Index j = i + 1; j < n; ++j) s -= row[j] * x[j];
      x[i] = s / row[i];
    }
    return x;
  }

 private:
  // Row-major dense LU with partial pivoting (fallback for small systems).
  void factor_dense() {
    const Index n = a_.rows();
    if (n > 20000) throw std::runtime_error("Eigen-shim SparseLU: no solver hook for n > 20000");
    lu_.assign(static_cast<size_t>(n * n), 0.0);
    for (Index j = 0; j < n; ++j)
      for (typename MatrixType::InnerIterator it(a_, j); it; ++it)
        lu_[static_cast<size_t>(it.row() * n + j)] += it.value();
    piv_.resize(static_cast<size_t>(n));
    std::iota(piv_.begin(), piv_.end(), 0);
    for (Index k = 0; k < n; ++k) {
      Index p = k;
      double best = std::abs(lu_[static_cast<size_t>(k * n + k)]);
      for (Index i = k + 1; i < n; ++i)
        if (std::abs(lu_[static_cast<size_t>(i * n + k)]) > best) {
          best = std::abs(lu_[static_cast<size_t>(i * n + k)]);
          p = i;
        }
      if (best == 0.0) {
        info_ = NumericalIssue;
        return;
      }
      if (p != k) {
        std::swap_ranges(lu_.begin() + k * n, lu_.begin() + (k + 1) * n, lu_.begin() + p * n);
        std::swap(piv_[static_cast<size_t>(k)], piv_[static_cast<size_t>(p)]);
      }
      const double* rk = &lu_[static_cast<size_t>(k * n)];
      for (Index i = k + 1; i < n; ++i) {
        double* ri = &lu_[static_cast<size_t>(i * n)];
        if (ri[k] == 0.0) continue;
        ri[k] /= rk[k];
        const double f = ri[k];
        for (Index j = k + 1; j < n; ++j) ri[j] -= f * rk[j];
      }
    }
    factored_ = true;
  }

  MatrixType a_;
  ComputationInfo info_ = Success;
  bool factored_ = false;
  std::vector<double> lu_;
  std::vector<Index> piv_;
};

}  // namespace Eigen

#endif  // LDG_EIGEN_SHIM_HPP
