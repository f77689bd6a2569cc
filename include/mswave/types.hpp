// mswave/types.hpp -- B200 drop-in mirror of proj/include/mswave/types.hpp.
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
#include <stdexcept>
#include <string>
#include <vector>

#ifdef MSWAVE_USE_EIGEN
#include <Eigen/Dense>
#endif

namespace mswave {

#ifdef MSWAVE_USE_EIGEN
using Vec = Eigen::VectorXd;
using Mat = Eigen::MatrixXd;
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
