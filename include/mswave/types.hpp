// mswave/types.hpp -- B200 drop-in mirror of proj/include/mswave/types.hpp.
//
// With -DMSWAVE_USE_EIGEN every alias is the reference's own (Vec, Mat, CVec,
// CMat, SpMat, CSpMat, Triplet, Cpx), so the structs of the other headers are
// layout-identical to the reference's and objects pass freely between the
// reference's off-line sources and this library.
//
// The reference aliases Vec/Mat to Eigen (types.hpp:14-21).  Eigen is not a
// dependency of the B200 library: without MSWAVE_USE_EIGEN the aliases bind
// to the minimal column-major containers below, which expose the subset of
// the Eigen interface the on-line API uses (size/rows/cols/data, (i)/(i,j),
// [], Zero/Constant/Identity, segment reads).  With -DMSWAVE_USE_EIGEN the
// reference's own aliases are used and the same sources compile unchanged
// (the implementation only touches data()/size()/rows()/cols()).
#ifndef MSWAVE_TYPES_HPP
#define MSWAVE_TYPES_HPP

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef MSWAVE_USE_EIGEN
#include <Eigen/Dense>
#include <Eigen/Sparse>
#endif

namespace mswave {

using Cpx = std::complex<double>;

#ifdef MSWAVE_USE_EIGEN
// exactly the reference's aliases (types.hpp:14-21)
using Vec = Eigen::VectorXd;
using Mat = Eigen::MatrixXd;
using CVec = Eigen::VectorXcd;
using CMat = Eigen::MatrixXcd;
using SpMat = Eigen::SparseMatrix<double>;
using CSpMat = Eigen::SparseMatrix<std::complex<double>>;
using Triplet = Eigen::Triplet<double>;
#else
class Vec {
 public:
  Vec() = default;
  explicit Vec(long n) : d_(static_cast<size_t>(n), 0.0) {}
  static Vec Zero(long n) { return Vec(n); }
  static Vec Ones(long n) { return Constant(n, 1.0); }
  static Vec Constant(long n, double v) {
    Vec x(n);
    std::fill(x.d_.begin(), x.d_.end(), v);
    return x;
  }
  long size() const { return static_cast<long>(d_.size()); }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double& operator[](long i) { return d_[static_cast<size_t>(i)]; }
  double operator[](long i) const { return d_[static_cast<size_t>(i)]; }
  double& operator()(long i) { return d_[static_cast<size_t>(i)]; }
  double operator()(long i) const { return d_[static_cast<size_t>(i)]; }
  void setZero() { std::fill(d_.begin(), d_.end(), 0.0); }
  void resize(long n) { d_.resize(static_cast<size_t>(n)); }
  Vec segment(long off, long n) const {
    Vec s(n);
    std::copy(d_.begin() + off, d_.begin() + off + n, s.d_.begin());
    return s;
  }
  double maxAbs() const {
    double m = 0.0;
    for (double v : d_) m = std::max(m, std::abs(v));
    return m;
  }
  double dot(const Vec& o) const {
    double s = 0.0;
    for (size_t i = 0; i < d_.size(); ++i) s += d_[i] * o.d_[i];
    return s;
  }

 private:
  std::vector<double> d_;
};

class Mat {  // column-major, like Eigen::MatrixXd
 public:
  Mat() = default;
  Mat(long r, long c) : r_(r), c_(c), d_(static_cast<size_t>(r * c), 0.0) {}
  static Mat Zero(long r, long c) { return Mat(r, c); }
  static Mat Constant(long r, long c, double v) {
    Mat m(r, c);
    std::fill(m.d_.begin(), m.d_.end(), v);
    return m;
  }
  static Mat Identity(long r, long c) {
    Mat m(r, c);
    for (long i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
    return m;
  }
  long rows() const { return r_; }
  long cols() const { return c_; }
  long size() const { return r_ * c_; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double& operator()(long i, long j) { return d_[static_cast<size_t>(i + j * r_)]; }
  double operator()(long i, long j) const { return d_[static_cast<size_t>(i + j * r_)]; }

 private:
  long r_ = 0, c_ = 0;
  std::vector<double> d_;
};

// (row, col, value) entry for SpMat::setFromTriplets (Eigen::Triplet<double>).
class Triplet {
 public:
  Triplet() = default;
  Triplet(int r, int c, double v) : r_(r), c_(c), v_(v) {}
  int row() const { return r_; }
  int col() const { return c_; }
  double value() const { return v_; }

 private:
  int r_ = 0, c_ = 0;
  double v_ = 0.0;
};

// Compressed sparse column matrix with Eigen::SparseMatrix<double>'s storage
// (32-bit indices, outer = column pointers, inner = sorted row indices) and
// the subset of its interface the fine-grid path uses.
class SpMat {
 public:
  using StorageIndex = int;
  SpMat() = default;
  SpMat(long r, long c) { resize(r, c); }
  void resize(long r, long c) {
    r_ = r;
    c_ = c;
    outer_.assign(static_cast<size_t>(c) + 1, 0);
    inner_.clear();
    val_.clear();
  }
  long rows() const { return r_; }
  long cols() const { return c_; }
  long outerSize() const { return c_; }
  long innerSize() const { return r_; }
  long nonZeros() const { return static_cast<long>(val_.size()); }
  bool isCompressed() const { return true; }
  void makeCompressed() {}
  const int* outerIndexPtr() const { return outer_.data(); }
  const int* innerIndexPtr() const { return inner_.data(); }
  const double* valuePtr() const { return val_.data(); }
  int* outerIndexPtr() { return outer_.data(); }
  int* innerIndexPtr() { return inner_.data(); }
  double* valuePtr() { return val_.data(); }
  // duplicates are summed in input order, rows sorted within each column
  template <typename It>
  void setFromTriplets(It begin, It end) {
    std::vector<long> cnt(static_cast<size_t>(c_) + 1, 0);
    for (It it = begin; it != end; ++it) ++cnt[static_cast<size_t>(it->col()) + 1];
    for (long j = 0; j < c_; ++j) cnt[j + 1] += cnt[j];
    std::vector<int> rows(static_cast<size_t>(cnt[c_]));
    std::vector<double> vals(rows.size());
    std::vector<long> fill(cnt.begin(), cnt.end() - 1);
    for (It it = begin; it != end; ++it) {
      const long q = fill[it->col()]++;
      rows[q] = it->row();
      vals[q] = it->value();
    }
    outer_.assign(static_cast<size_t>(c_) + 1, 0);
    inner_.clear();
    val_.clear();
    for (long j = 0; j < c_; ++j) {
      std::vector<std::pair<int, long>> col;
      for (long q = cnt[j]; q < cnt[j + 1]; ++q) col.push_back({rows[q], q});
      std::stable_sort(col.begin(), col.end(),
                       [](const std::pair<int, long>& a, const std::pair<int, long>& b) { return a.first < b.first; });
      for (size_t k = 0; k < col.size(); ++k) {
        if (k > 0 && col[k].first == col[k - 1].first) {
          val_.back() += vals[col[k].second];
        } else {
          inner_.push_back(col[k].first);
          val_.push_back(vals[col[k].second]);
        }
      }
      outer_[j + 1] = static_cast<int>(inner_.size());
    }
  }
  double coeff(long i, long j) const {
    for (int q = outer_[j]; q < outer_[j + 1]; ++q)
      if (inner_[q] == i) return val_[q];
    return 0.0;
  }
  class InnerIterator {
   public:
    InnerIterator(const SpMat& m, long outer) : m_(m), j_(outer), q_(m.outer_[outer]), e_(m.outer_[outer + 1]) {}
    explicit operator bool() const { return q_ < e_; }
    InnerIterator& operator++() {
      ++q_;
      return *this;
    }
    double value() const { return m_.val_[q_]; }
    long row() const { return m_.inner_[q_]; }
    long col() const { return j_; }
    long index() const { return m_.inner_[q_]; }

   private:
    const SpMat& m_;
    long j_;
    int q_, e_;
  };

 private:
  long r_ = 0, c_ = 0;
  std::vector<int> outer_{0};
  std::vector<int> inner_;
  std::vector<double> val_;
};
#endif

// Thrown when a numerical contract is violated (instability, breakdown,
// non-SPD ladder).  The CLI maps it to exit code 3 (types.hpp:23-29).
class NumericalError : public std::runtime_error {
 public:
  explicit NumericalError(const std::string& what) : std::runtime_error(what) {}
};

// Thrown on invalid configuration or malformed artifacts.  Exit code 2.
class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& what) : std::runtime_error(what) {}
};

// Device/runtime failure of the B200 backend (no reference analogue).
class DeviceError : public std::runtime_error {
 public:
  explicit DeviceError(const std::string& what) : std::runtime_error(what) {}
};

inline double rel_diff(double a, double b) {
  const double d = std::abs(a - b);
  const double s = std::max(std::abs(a), std::abs(b));
  return s > 0.0 ? d / s : d;
}

}  // namespace mswave

#endif  // MSWAVE_TYPES_HPP
