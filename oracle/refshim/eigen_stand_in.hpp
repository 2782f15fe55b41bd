// eigen_stand_in.hpp — TEST INFRASTRUCTURE.  A small, self-written stand-in for the subset of
// the Eigen API that the reference's hot-path sources (kernels/grid/interp/solvers/gp .cpp)
// use, so those sources compile unmodified in an image without Eigen (oracle/refshim/README.md).
// Eager evaluation, no expression templates; reductions are plain left-to-right sums.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
enum StorageOrder { ColMajor = 0, RowMajor = 1 };
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };

class MatrixXd;
template <typename Scalar, int Options, typename StorageIndex>
class SparseMatrixBase;

// ------------------------------------------------------------------ dense vector
class VectorXd {
 public:
  VectorXd() = default;
  explicit VectorXd(Index n) : v_(static_cast<std::size_t>(n), 0.0) {}
  VectorXd(std::vector<double> v) : v_(std::move(v)) {}  // NOLINT (implicit on purpose)

  static VectorXd Zero(Index n) { return VectorXd(n); }
  static VectorXd Ones(Index n) { return Constant(n, 1.0); }
  static VectorXd Constant(Index n, double c) {
    VectorXd o(n);
    std::fill(o.v_.begin(), o.v_.end(), c);
    return o;
  }

  Index size() const { return static_cast<Index>(v_.size()); }
  Index rows() const { return size(); }
  Index cols() const { return 1; }
  void resize(Index n) { v_.assign(static_cast<std::size_t>(n), 0.0); }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator[](Index i) { return v_[static_cast<std::size_t>(i)]; }
  double operator[](Index i) const { return v_[static_cast<std::size_t>(i)]; }
  double& operator()(Index i) { return v_[static_cast<std::size_t>(i)]; }
  double operator()(Index i) const { return v_[static_cast<std::size_t>(i)]; }
  void setZero() { std::fill(v_.begin(), v_.end(), 0.0); }

  double dot(const VectorXd& o) const {
    check(o);
    double s = 0.0;
    for (std::size_t i = 0; i < v_.size(); ++i) s += v_[i] * o.v_[i];
    return s;
  }
  double squaredNorm() const { return dot(*this); }
  double norm() const { return std::sqrt(squaredNorm()); }
  double sum() const {
    double s = 0.0;
    for (double x : v_) s += x;
    return s;
  }
  double maxCoeff() const { return *std::max_element(v_.begin(), v_.end()); }
  double minCoeff() const { return *std::min_element(v_.begin(), v_.end()); }
  VectorXd cwiseAbs() const {
    VectorXd o(size());
    for (std::size_t i = 0; i < v_.size(); ++i) o.v_[i] = std::abs(v_[i]);
    return o;
  }
  VectorXd head(Index n) const { return VectorXd(std::vector<double>(v_.begin(), v_.begin() + n)); }
  VectorXd tail(Index n) const { return VectorXd(std::vector<double>(v_.end() - n, v_.end())); }
  VectorXd segment(Index s, Index n) const {
    return VectorXd(std::vector<double>(v_.begin() + s, v_.begin() + s + n));
  }
  // column vector ↔ row vector carry the same storage here
  const VectorXd& transpose() const { return *this; }
  const VectorXd& eval() const { return *this; }

  VectorXd& operator+=(const VectorXd& o) {
    check(o);
    for (std::size_t i = 0; i < v_.size(); ++i) v_[i] += o.v_[i];
    return *this;
  }
  VectorXd& operator-=(const VectorXd& o) {
    check(o);
    for (std::size_t i = 0; i < v_.size(); ++i) v_[i] -= o.v_[i];
    return *this;
  }
  VectorXd& operator*=(double c) {
    for (double& x : v_) x *= c;
    return *this;
  }
  VectorXd& operator/=(double c) {
    for (double& x : v_) x /= c;
    return *this;
  }
  VectorXd operator-() const {
    VectorXd o(size());
    for (std::size_t i = 0; i < v_.size(); ++i) o.v_[i] = -v_[i];
    return o;
  }

 private:
  void check(const VectorXd& o) const {
    if (o.v_.size() != v_.size()) throw std::logic_error("eigen_stand_in: vector size mismatch");
  }
  std::vector<double> v_;
};

inline VectorXd operator+(VectorXd a, const VectorXd& b) { return a += b; }
inline VectorXd operator-(VectorXd a, const VectorXd& b) { return a -= b; }
inline VectorXd operator*(VectorXd a, double c) { return a *= c; }
inline VectorXd operator*(double c, VectorXd a) { return a *= c; }
inline VectorXd operator/(VectorXd a, double c) { return a /= c; }

template <typename T>
class Map;
template <>
class Map<VectorXd> {
 public:
  Map(double* p, Index n) : p_(p), n_(n) {}
  Map(double* p, std::size_t n) : p_(p), n_(static_cast<Index>(n)) {}
  operator VectorXd() const { return VectorXd(std::vector<double>(p_, p_ + n_)); }  // NOLINT

 private:
  double* p_;
  Index n_;
};

// ------------------------------------------------------------------ dense matrix (column-major)
class MatrixXd {
 public:
  MatrixXd() = default;
  MatrixXd(Index r, Index c) : r_(r), c_(c), v_(static_cast<std::size_t>(r * c), 0.0) {}
  template <typename S, int O, typename I>
  explicit MatrixXd(const SparseMatrixBase<S, O, I>& s);

  static MatrixXd Zero(Index r, Index c) { return MatrixXd(r, c); }
  static MatrixXd Identity(Index r, Index c) {
    MatrixXd m(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
    return m;
  }

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  void resize(Index r, Index c) {
    r_ = r;
    c_ = c;
    v_.assign(static_cast<std::size_t>(r * c), 0.0);
  }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator()(Index i, Index j) { return v_[static_cast<std::size_t>(j * r_ + i)]; }
  double operator()(Index i, Index j) const { return v_[static_cast<std::size_t>(j * r_ + i)]; }

  // writable column view; reads convert to VectorXd
  class ColXpr {
   public:
    ColXpr(MatrixXd& m, Index j) : m_(m), j_(j) {}
    ColXpr& operator=(const VectorXd& v) {
      if (v.size() != m_.r_) throw std::logic_error("eigen_stand_in: column size mismatch");
      for (Index i = 0; i < m_.r_; ++i) m_(i, j_) = v[i];
      return *this;
    }
    ColXpr& operator=(const ColXpr& o) { return *this = static_cast<VectorXd>(o); }
    operator VectorXd() const {  // NOLINT
      VectorXd v(m_.r_);
      for (Index i = 0; i < m_.r_; ++i) v[i] = m_(i, j_);
      return v;
    }
    double dot(const VectorXd& o) const { return static_cast<VectorXd>(*this).dot(o); }
    double norm() const { return static_cast<VectorXd>(*this).norm(); }
    double squaredNorm() const { return static_cast<VectorXd>(*this).squaredNorm(); }
    Index size() const { return m_.r_; }
    double operator[](Index i) const { return m_(i, j_); }
    double& operator[](Index i) { return m_(i, j_); }

   private:
    MatrixXd& m_;
    Index j_;
  };
  ColXpr col(Index j) { return ColXpr(*this, j); }
  VectorXd col(Index j) const {
    VectorXd v(r_);
    for (Index i = 0; i < r_; ++i) v[i] = (*this)(i, j);
    return v;
  }
  VectorXd row(Index i) const {
    VectorXd v(c_);
    for (Index j = 0; j < c_; ++j) v[j] = (*this)(i, j);
    return v;
  }
  MatrixXd leftCols(Index k) const {
    MatrixXd o(r_, k);
    std::copy(v_.begin(), v_.begin() + r_ * k, o.v_.begin());
    return o;
  }
  MatrixXd transpose() const {
    MatrixXd o(c_, r_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) o(j, i) = (*this)(i, j);
    return o;
  }
  const MatrixXd& eval() const { return *this; }
  MatrixXd cwiseAbs() const {
    MatrixXd o(r_, c_);
    for (std::size_t i = 0; i < v_.size(); ++i) o.v_[i] = std::abs(v_[i]);
    return o;
  }
  double maxCoeff() const { return *std::max_element(v_.begin(), v_.end()); }
  double minCoeff() const { return *std::min_element(v_.begin(), v_.end()); }

  // m.diagonal().array() += c
  class DiagXpr {
   public:
    explicit DiagXpr(MatrixXd& m) : m_(m) {}
    DiagXpr& array() { return *this; }
    DiagXpr& operator+=(double c) {
      for (Index i = 0; i < std::min(m_.r_, m_.c_); ++i) m_(i, i) += c;
      return *this;
    }
    double operator[](Index i) const { return m_(i, i); }

   private:
    MatrixXd& m_;
  };
  DiagXpr diagonal() { return DiagXpr(*this); }

  MatrixXd& operator+=(const MatrixXd& o) {
    check(o);
    for (std::size_t i = 0; i < v_.size(); ++i) v_[i] += o.v_[i];
    return *this;
  }
  MatrixXd& operator-=(const MatrixXd& o) {
    check(o);
    for (std::size_t i = 0; i < v_.size(); ++i) v_[i] -= o.v_[i];
    return *this;
  }
  MatrixXd& operator*=(double c) {
    for (double& x : v_) x *= c;
    return *this;
  }

 private:
  void check(const MatrixXd& o) const {
    if (o.r_ != r_ || o.c_ != c_) throw std::logic_error("eigen_stand_in: matrix size mismatch");
  }
  Index r_ = 0, c_ = 0;
  std::vector<double> v_;
};

inline MatrixXd operator+(MatrixXd a, const MatrixXd& b) { return a += b; }
inline MatrixXd operator-(MatrixXd a, const MatrixXd& b) { return a -= b; }
inline MatrixXd operator*(MatrixXd a, double c) { return a *= c; }
inline MatrixXd operator*(double c, MatrixXd a) { return a *= c; }
inline VectorXd operator*(const MatrixXd& a, const VectorXd& x) {
  if (a.cols() != x.size()) throw std::logic_error("eigen_stand_in: A x size mismatch");
  VectorXd y(a.rows());
  for (Index i = 0; i < a.rows(); ++i) {
    double s = 0.0;
    for (Index j = 0; j < a.cols(); ++j) s += a(i, j) * x[j];
    y[i] = s;
  }
  return y;
}
inline MatrixXd operator*(const MatrixXd& a, const MatrixXd& b) {
  if (a.cols() != b.rows()) throw std::logic_error("eigen_stand_in: A B size mismatch");
  MatrixXd c(a.rows(), b.cols());
  for (Index j = 0; j < b.cols(); ++j)
    for (Index k = 0; k < a.cols(); ++k) {
      const double bkj = b(k, j);
      for (Index i = 0; i < a.rows(); ++i) c(i, j) += a(i, k) * bkj;
    }
  return c;
}

// ------------------------------------------------------------------ sparse
template <typename Scalar, typename StorageIndex = int>
class Triplet {
 public:
  Triplet() = default;
  Triplet(StorageIndex i, StorageIndex j, Scalar v) : i_(i), j_(j), v_(v) {}
  StorageIndex row() const { return i_; }
  StorageIndex col() const { return j_; }
  Scalar value() const { return v_; }

 private:
  StorageIndex i_ = 0, j_ = 0;
  Scalar v_ = Scalar();
};

// compressed storage: outer = rows (RowMajor) or columns (ColMajor); inner indices sorted
template <typename Scalar, int Options, typename StorageIndex>
class SparseMatrixBase {
 public:
  SparseMatrixBase() : outer_(1, 0) {}
  SparseMatrixBase(Index r, Index c) : r_(r), c_(c), outer_(static_cast<std::size_t>(outer_dim(r, c)) + 1, 0) {}

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index outerSize() const { return Options == RowMajor ? r_ : c_; }
  Index innerSize() const { return Options == RowMajor ? c_ : r_; }
  Index nonZeros() const { return static_cast<Index>(inner_.size()); }
  const StorageIndex* outerIndexPtr() const { return outer_.data(); }
  const StorageIndex* innerIndexPtr() const { return inner_.data(); }
  const Scalar* valuePtr() const { return val_.data(); }
  void makeCompressed() {}

  // duplicates are summed in input order; explicit zeros are kept.  Linear time like the real
  // library: a counting pass over the outer index, then a stable sort of each outer vector.
  template <typename It>
  void setFromTriplets(It first, It last) {
    const Index no = outerSize(), ni = innerSize();
    std::vector<std::size_t> start(static_cast<std::size_t>(no) + 1, 0);
    std::size_t total = 0;
    for (It t = first; t != last; ++t, ++total) {
      const Index o = Options == RowMajor ? t->row() : t->col();
      const Index i = Options == RowMajor ? t->col() : t->row();
      if (o < 0 || o >= no || i < 0 || i >= ni) throw std::logic_error("eigen_stand_in: triplet out of range");
      ++start[static_cast<std::size_t>(o) + 1];
    }
    for (Index o = 0; o < no; ++o) start[o + 1] += start[o];
    std::vector<std::pair<StorageIndex, Scalar>> e(total);
    {
      std::vector<std::size_t> cur(start.begin(), start.end() - 1);
      for (It t = first; t != last; ++t) {
        const Index o = Options == RowMajor ? t->row() : t->col();
        const StorageIndex i = Options == RowMajor ? t->col() : t->row();
        e[cur[static_cast<std::size_t>(o)]++] = {i, t->value()};
      }
    }
    outer_.assign(static_cast<std::size_t>(no) + 1, 0);
    inner_.clear();
    val_.clear();
    inner_.reserve(total);
    val_.reserve(total);
    for (Index o = 0; o < no; ++o) {
      auto b = e.begin() + static_cast<std::ptrdiff_t>(start[o]), en = e.begin() + static_cast<std::ptrdiff_t>(start[o + 1]);
      std::stable_sort(b, en, [](const auto& x, const auto& y) { return x.first < y.first; });
      for (auto it = b; it != en; ++it) {
        if (it != b && it->first == (it - 1)->first) {
          val_.back() += it->second;
        } else {
          inner_.push_back(it->first);
          val_.push_back(it->second);
        }
      }
      outer_[static_cast<std::size_t>(o) + 1] = static_cast<StorageIndex>(inner_.size());
    }
  }

  // drops entries with |v| <= ref (Eigen's prune(ref) with the default epsilon keeps |v| > 0 for ref = 0)
  void prune(Scalar ref) {
    std::vector<StorageIndex> no(outer_.size(), 0), ni;
    std::vector<Scalar> nv;
    for (Index o = 0; o < outerSize(); ++o) {
      for (StorageIndex k = outer_[o]; k < outer_[o + 1]; ++k) {
        if (std::abs(val_[k]) > std::abs(ref)) {
          ni.push_back(inner_[k]);
          nv.push_back(val_[k]);
        }
      }
      no[static_cast<std::size_t>(o) + 1] = static_cast<StorageIndex>(ni.size());
    }
    outer_ = std::move(no);
    inner_ = std::move(ni);
    val_ = std::move(nv);
  }

  VectorXd operator*(const VectorXd& x) const {
    if (x.size() != c_) throw std::logic_error("eigen_stand_in: sparse A x size mismatch");
    VectorXd y(r_);
    for (Index o = 0; o < outerSize(); ++o) {
      if (Options == RowMajor) {
        double s = 0.0;
        for (StorageIndex k = outer_[o]; k < outer_[o + 1]; ++k) s += val_[k] * x[inner_[k]];
        y[o] = s;
      } else {
        const double xo = x[o];
        for (StorageIndex k = outer_[o]; k < outer_[o + 1]; ++k) y[inner_[k]] += val_[k] * xo;
      }
    }
    return y;
  }

  class InnerIterator {
   public:
    InnerIterator(const SparseMatrixBase& m, Index outer)
        : m_(m), o_(outer), k_(m.outer_[outer]), e_(m.outer_[outer + 1]) {}
    explicit operator bool() const { return k_ < e_; }
    InnerIterator& operator++() {
      ++k_;
      return *this;
    }
    Scalar value() const { return m_.val_[k_]; }
    Index index() const { return m_.inner_[k_]; }
    Index row() const { return Options == RowMajor ? o_ : index(); }
    Index col() const { return Options == RowMajor ? index() : o_; }

   private:
    const SparseMatrixBase& m_;
    Index o_;
    StorageIndex k_, e_;
  };

  // raw access for conversions between the two storage orders
  std::vector<StorageIndex>& outer_raw() { return outer_; }
  std::vector<StorageIndex>& inner_raw() { return inner_; }
  std::vector<Scalar>& val_raw() { return val_; }
  const std::vector<StorageIndex>& outer_raw() const { return outer_; }
  const std::vector<StorageIndex>& inner_raw() const { return inner_; }
  const std::vector<Scalar>& val_raw() const { return val_; }

 protected:
  static Index outer_dim(Index r, Index c) { return Options == RowMajor ? r : c; }
  Index r_ = 0, c_ = 0;
  std::vector<StorageIndex> outer_, inner_;
  std::vector<Scalar> val_;
};

template <typename Scalar, int Options = ColMajor, typename StorageIndex = int>
class SparseMatrix : public SparseMatrixBase<Scalar, Options, StorageIndex> {
  using Base = SparseMatrixBase<Scalar, Options, StorageIndex>;

 public:
  SparseMatrix() = default;
  SparseMatrix(Index r, Index c) : Base(r, c) {}
  // conversion from the other storage order (re-sorted by the new outer index)
  template <int O2>
  SparseMatrix(const SparseMatrix<Scalar, O2, StorageIndex>& o) : Base(o.rows(), o.cols()) {  // NOLINT
    if (O2 == Options) {
      this->outer_ = o.outer_raw();
      this->inner_ = o.inner_raw();
      this->val_ = o.val_raw();
      return;
    }
    std::vector<Triplet<Scalar, StorageIndex>> t;
    for (Index oo = 0; oo < o.outerSize(); ++oo)
      for (typename SparseMatrix<Scalar, O2, StorageIndex>::InnerIterator it(o, oo); it; ++it)
        t.emplace_back(static_cast<StorageIndex>(it.row()), static_cast<StorageIndex>(it.col()), it.value());
    this->setFromTriplets(t.begin(), t.end());
  }

  // the transpose of a compressed matrix is the same arrays read in the other storage order
  SparseMatrix<Scalar, Options == RowMajor ? ColMajor : RowMajor, StorageIndex> transpose() const {
    SparseMatrix<Scalar, Options == RowMajor ? ColMajor : RowMajor, StorageIndex> t(this->c_, this->r_);
    t.outer_raw() = this->outer_;
    t.inner_raw() = this->inner_;
    t.val_raw() = this->val_;
    return t;
  }
};

// sparse × sparse (result column-major; structural zeros from cancellation are kept)
template <typename S, int O1, int O2, typename I>
SparseMatrix<S, ColMajor, I> operator*(const SparseMatrix<S, O1, I>& a, const SparseMatrix<S, O2, I>& b) {
  if (a.cols() != b.rows()) throw std::logic_error("eigen_stand_in: sparse A B size mismatch");
  const SparseMatrix<S, ColMajor, I> ac(a), bc(b);
  std::vector<Triplet<S, I>> t;
  std::vector<S> acc(static_cast<std::size_t>(a.rows()), S());
  std::vector<char> hit(static_cast<std::size_t>(a.rows()), 0);
  std::vector<I> rows;
  for (Index j = 0; j < bc.cols(); ++j) {
    rows.clear();
    for (typename SparseMatrix<S, ColMajor, I>::InnerIterator ib(bc, j); ib; ++ib) {
      for (typename SparseMatrix<S, ColMajor, I>::InnerIterator ia(ac, ib.index()); ia; ++ia) {
        const std::size_t r = static_cast<std::size_t>(ia.index());
        if (!hit[r]) {
          hit[r] = 1;
          rows.push_back(static_cast<I>(r));
        }
        acc[r] += ia.value() * ib.value();
      }
    }
    for (I r : rows) {
      t.emplace_back(r, static_cast<I>(j), acc[static_cast<std::size_t>(r)]);
      acc[static_cast<std::size_t>(r)] = S();
      hit[static_cast<std::size_t>(r)] = 0;
    }
  }
  SparseMatrix<S, ColMajor, I> c(a.rows(), b.cols());
  c.setFromTriplets(t.begin(), t.end());
  return c;
}

template <typename S, int O, typename I>
MatrixXd::MatrixXd(const SparseMatrixBase<S, O, I>& s) : MatrixXd(s.rows(), s.cols()) {
  for (Index o = 0; o < s.outerSize(); ++o)
    for (typename SparseMatrixBase<S, O, I>::InnerIterator it(s, o); it; ++it) (*this)(it.row(), it.col()) += it.value();
}

// ------------------------------------------------------------------ dense factorizations
template <typename M>
class LLT {
 public:
  LLT() = default;
  explicit LLT(const M& a) { compute(a); }
  LLT& compute(const M& a) {
    const Index n = a.rows();
    l_ = a;
    info_ = Success;
    for (Index j = 0; j < n; ++j) {
      double d = l_(j, j);
      for (Index k = 0; k < j; ++k) d -= l_(j, k) * l_(j, k);
      if (!(d > 0.0)) {
        info_ = NumericalIssue;
        return *this;
      }
      const double ljj = std::sqrt(d);
      l_(j, j) = ljj;
      for (Index i = j + 1; i < n; ++i) {
        double s = l_(i, j);
        for (Index k = 0; k < j; ++k) s -= l_(i, k) * l_(j, k);
        l_(i, j) = s / ljj;
      }
    }
    return *this;
  }
  ComputationInfo info() const { return info_; }
  const M& matrixLLT() const { return l_; }
  VectorXd solve(const VectorXd& b) const {
    const Index n = l_.rows();
    VectorXd x = b;
    for (Index i = 0; i < n; ++i) {
      double s = x[i];
      for (Index k = 0; k < i; ++k) s -= l_(i, k) * x[k];
      x[i] = s / l_(i, i);
    }
    for (Index i = n - 1; i >= 0; --i) {
      double s = x[i];
      for (Index k = i + 1; k < n; ++k) s -= l_(k, i) * x[k];
      x[i] = s / l_(i, i);
    }
    return x;
  }
  M solve(const M& b) const {
    M x(b.rows(), b.cols());
    for (Index j = 0; j < b.cols(); ++j) x.col(j) = solve(b.col(j));
    return x;
  }

 private:
  M l_;
  ComputationInfo info_ = InvalidInput;
};

// symmetric indefinite LDLᵀ with diagonal pivoting (largest remaining |d|)
template <typename M>
class LDLT {
 public:
  LDLT() = default;
  explicit LDLT(const M& a) { compute(a); }
  LDLT& compute(const M& a) {
    const Index n = a.rows();
    M w = a;
    perm_.resize(static_cast<std::size_t>(n));
    std::iota(perm_.begin(), perm_.end(), Index{0});
    l_ = M::Identity(n, n);
    d_.assign(static_cast<std::size_t>(n), 0.0);
    info_ = Success;
    for (Index j = 0; j < n; ++j) {
      Index p = j;
      for (Index i = j + 1; i < n; ++i)
        if (std::abs(w(i, i)) > std::abs(w(p, p))) p = i;
      if (p != j) {  // symmetric swap of rows/columns j and p, and of the finished part of L
        for (Index k = 0; k < n; ++k) std::swap(w(j, k), w(p, k));
        for (Index k = 0; k < n; ++k) std::swap(w(k, j), w(k, p));
        for (Index k = 0; k < j; ++k) std::swap(l_(j, k), l_(p, k));
        std::swap(perm_[static_cast<std::size_t>(j)], perm_[static_cast<std::size_t>(p)]);
      }
      const double d = w(j, j);
      d_[static_cast<std::size_t>(j)] = d;
      if (d == 0.0) continue;
      for (Index i = j + 1; i < n; ++i) l_(i, j) = w(i, j) / d;
      for (Index c = j + 1; c < n; ++c)
        for (Index r = j + 1; r < n; ++r) w(r, c) -= l_(r, j) * d * l_(c, j);
    }
    return *this;
  }
  ComputationInfo info() const { return info_; }
  VectorXd solve(const VectorXd& b) const {
    const Index n = static_cast<Index>(d_.size());
    VectorXd x(n);
    for (Index i = 0; i < n; ++i) x[i] = b[perm_[static_cast<std::size_t>(i)]];
    for (Index i = 0; i < n; ++i)
      for (Index k = 0; k < i; ++k) x[i] -= l_(i, k) * x[k];
    for (Index i = 0; i < n; ++i) {
      const double d = d_[static_cast<std::size_t>(i)];
      x[i] = d != 0.0 ? x[i] / d : 0.0;
    }
    for (Index i = n - 1; i >= 0; --i)
      for (Index k = i + 1; k < n; ++k) x[i] -= l_(k, i) * x[k];
    VectorXd out(n);
    for (Index i = 0; i < n; ++i) out[perm_[static_cast<std::size_t>(i)]] = x[i];
    return out;
  }
  M solve(const M& b) const {
    M x(b.rows(), b.cols());
    for (Index j = 0; j < b.cols(); ++j) x.col(j) = solve(b.col(j));
    return x;
  }

 private:
  M l_;
  std::vector<double> d_;
  std::vector<Index> perm_;
  ComputationInfo info_ = InvalidInput;
};

template <typename M>
class PartialPivLU {
 public:
  PartialPivLU() = default;
  explicit PartialPivLU(const M& a) { compute(a); }
  PartialPivLU& compute(const M& a) {
    const Index n = a.rows();
    lu_ = a;
    for (Index j = 0; j < n; ++j) {
      Index p = j;
      for (Index i = j + 1; i < n; ++i)
        if (std::abs(lu_(i, j)) > std::abs(lu_(p, j))) p = i;
      if (p != j)
        for (Index k = 0; k < n; ++k) std::swap(lu_(j, k), lu_(p, k));
      const double d = lu_(j, j);
      if (d == 0.0) continue;
      for (Index i = j + 1; i < n; ++i) lu_(i, j) /= d;
      for (Index c = j + 1; c < n; ++c) {
        const double u = lu_(j, c);
        for (Index i = j + 1; i < n; ++i) lu_(i, c) -= lu_(i, j) * u;
      }
    }
    return *this;
  }
  const M& matrixLU() const { return lu_; }

 private:
  M lu_;
};

// symmetric tridiagonal eigen-decomposition (implicit QL with Wilkinson shifts), eigenvalues
// ascending, eigenvectors in the columns
template <typename M>
class SelfAdjointEigenSolver {
 public:
  SelfAdjointEigenSolver() = default;
  SelfAdjointEigenSolver& computeFromTridiagonal(const VectorXd& diag, const VectorXd& sub) {
    const Index n = diag.size();
    std::vector<double> d(diag.data(), diag.data() + n), e(static_cast<std::size_t>(n), 0.0);
    for (Index i = 0; i + 1 < n; ++i) e[static_cast<std::size_t>(i)] = sub[i];
    M z = M::Identity(n, n);
    info_ = Success;
    for (Index l = 0; l < n; ++l) {
      int iter = 0;
      Index m;
      do {
        for (m = l; m + 1 < n; ++m) {
          const double dd = std::abs(d[m]) + std::abs(d[m + 1]);
          if (std::abs(e[m]) <= 2.220446049250313e-16 * dd) break;
        }
        if (m != l) {
          if (++iter > 200) {
            info_ = NoConvergence;
            break;
          }
          double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
          double r = std::hypot(g, 1.0);
          g = d[m] - d[l] + e[l] / (g + (g >= 0.0 ? std::abs(r) : -std::abs(r)));
          double s = 1.0, c = 1.0, p = 0.0;
          Index i;
          for (i = m - 1; i >= l; --i) {
            double f = s * e[i];
            const double b = c * e[i];
            r = std::hypot(f, g);
            e[i + 1] = r;
            if (r == 0.0) {
              d[i + 1] -= p;
              e[m] = 0.0;
              break;
            }
            s = f / r;
            c = g / r;
            g = d[i + 1] - p;
            r = (d[i] - g) * s + 2.0 * c * b;
            p = s * r;
            d[i + 1] = g + p;
            g = c * r - b;
            for (Index k = 0; k < n; ++k) {
              f = z(k, i + 1);
              z(k, i + 1) = s * z(k, i) + c * f;
              z(k, i) = c * z(k, i) - s * f;
            }
          }
          if (r == 0.0 && i >= l) continue;
          d[l] -= p;
          e[l] = g;
          e[m] = 0.0;
        }
      } while (m != l);
    }
    std::vector<Index> order(static_cast<std::size_t>(n));
    std::iota(order.begin(), order.end(), Index{0});
    std::stable_sort(order.begin(), order.end(), [&](Index a, Index b) { return d[a] < d[b]; });
    vals_ = VectorXd(n);
    vecs_ = M(n, n);
    for (Index j = 0; j < n; ++j) {
      vals_[j] = d[order[static_cast<std::size_t>(j)]];
      for (Index k = 0; k < n; ++k) vecs_(k, j) = z(k, order[static_cast<std::size_t>(j)]);
    }
    return *this;
  }
  const VectorXd& eigenvalues() const { return vals_; }
  const M& eigenvectors() const { return vecs_; }
  ComputationInfo info() const { return info_; }

 private:
  VectorXd vals_;
  M vecs_;
  ComputationInfo info_ = InvalidInput;
};

}  // namespace Eigen
