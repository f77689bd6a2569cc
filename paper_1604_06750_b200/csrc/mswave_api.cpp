// C++ drop-in mirror of the reference's on-line API (namespace mswave,
// include/mswave/*.hpp) implemented on top of the C ABI (mswave_b200.h).
// Every compute call runs on the B200 kernels; this file only marshals
// host data, mirroring the reference's signatures and error behaviour.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <map>
#include <list>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/mswave/msolver.hpp"
#include "../../include/mswave/reference.hpp"
#include "../../include/mswave/trace_io.hpp"
#include "../../include/mswave_b200.h"

namespace mswave {

namespace {

void check(int rc) {
  if (rc == MSW_OK) return;
  const std::string msg = msw_last_error();
  if (rc == MSW_CONFIG_ERROR) throw ConfigError(msg);
  if (rc == MSW_NUMERICAL_ERROR) throw NumericalError(msg);
  throw DeviceError(msg);
}

// Cholesky inverse (Eigen llt().solve(I), msolver.cpp:71-73).
std::vector<double> spd_inverse(const std::vector<double>& A, int n) {
  std::vector<double> L(static_cast<size_t>(n) * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double d = A[j + j * n];
    for (int k = 0; k < j; ++k) d -= L[j + k * n] * L[j + k * n];
    if (!(d > 0.0)) throw NumericalError("assemble_system: interface mass block is not SPD");
    const double ljj = std::sqrt(d);
    L[j + j * n] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double s = A[i + j * n];
      for (int k = 0; k < j; ++k) s -= L[i + k * n] * L[j + k * n];
      L[i + j * n] = s / ljj;
    }
  }
  std::vector<double> X(static_cast<size_t>(n) * n, 0.0), y(n);
  for (int c = 0; c < n; ++c) {
    for (int i = 0; i < n; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) s -= L[i + k * n] * y[k];
      y[i] = s / L[i + i * n];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < n; ++k) s -= L[k + i * n] * X[k + c * n];
      X[i + c * n] = s / L[i + i * n];
    }
  }
  return X;
}

void symmetrize(std::vector<double>& M, int n) {
  const std::vector<double> T(M);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) M[i + j * n] = 0.5 * (T[i + j * n] + T[j + i * n]);
}

std::vector<double> to_vec(const Mat& m) {
  return std::vector<double>(m.data(), m.data() + m.rows() * m.cols());
}

Mat from_vec(const std::vector<double>& v, int r, int c) {
  Mat m = Mat::Zero(r, c);
  std::copy(v.begin(), v.end(), m.data());
  return m;
}

}  // namespace

// ============================== wavelet ====================================

double Wavelet::operator()(double t) const {  // wavelet.cpp:9-19 (+ Ricker)
  const double x = (t - delay()) / tau();
  switch (kind) {
    case Kind::GaussianDerivative: return -x * std::exp(0.5 - 0.5 * x * x);
    case Kind::Gaussian: return std::exp(-0.5 * x * x);
    case Kind::Ricker: return (1.0 - x * x) * std::exp(-0.5 * x * x);
  }
  return 0.0;
}

Wavelet::Kind Wavelet::kind_from_string(const std::string& s) {
  if (s == "gaussian_derivative") return Kind::GaussianDerivative;
  if (s == "gaussian") return Kind::Gaussian;
  if (s == "ricker") return Kind::Ricker;
  throw ConfigError("unknown wavelet kind: " + s);
}

std::string Wavelet::to_string(Kind k) {
  switch (k) {
    case Kind::GaussianDerivative: return "gaussian_derivative";
    case Kind::Gaussian: return "gaussian";
    case Kind::Ricker: return "ricker";
  }
  return "?";
}

// ============================== fine grid ==================================

long GridMedium::node_count() const {
  long n = 1;
  for (int d : dims) n *= d;
  return n;
}

long GridMedium::node_id(const std::array<int, 3>& c) const {
  long id = 0;
  for (int a = 0; a < ndim(); ++a) id = id * dims[a] + c[a];
  return id;
}

GridMedium make_uniform_medium(std::vector<int> dims, double h, double sigma_value,
                               double rho_value) {
  GridMedium m;
  m.dims = std::move(dims);
  m.h = h;
  m.sigma = Vec::Constant(m.node_count(), sigma_value);
  m.rho = Vec::Constant(m.node_count(), rho_value);
  return m;
}

long SparsePencil::node_of(const std::array<int, 3>& c) const {
  long id = 0;
  for (int a = 0; a < ndim; ++a) {
    if (c[a] < 1 || c[a] > dims[a] - 2) return -1;
    id = id * (dims[a] - 2) + (c[a] - 1);
  }
  return id;
}

namespace {
void validate_medium(const GridMedium& medium) {  // fine_grid.cpp:40-53
  if (medium.ndim() < 1 || medium.ndim() > 3) throw ConfigError("medium must have 1-3 axes");
  if (medium.h <= 0.0) throw ConfigError("grid step h must be positive");
  for (int d : medium.dims)
    if (d < 3) throw ConfigError("every axis needs at least 3 nodes (no interior otherwise)");
  if (medium.sigma.size() != medium.node_count() || medium.rho.size() != medium.node_count())
    throw ConfigError("sigma/rho length does not match dims");
  for (long i = 0; i < medium.node_count(); ++i) {
    if (medium.sigma[i] < 0.0) throw ConfigError("sigma must be nonnegative");
    if (medium.rho[i] <= 0.0) throw ConfigError("rho must be strictly positive");
  }
}
}  // namespace

// fine_grid.cpp:58-112: the 3/5/7-point conservative pencil, edge stiffness
// 0.5 (sigma_i + sigma_j) / h^2, Dirichlet neighbours on the diagonal only,
// B = rho; the same per-row arithmetic and triplet order (this file is built
// without FMA contraction, like the reference's flag-less build).
SparsePencil assemble_nd(const GridMedium& medium) {
  validate_medium(medium);
  const int nd = medium.ndim();
  const double inv_h2 = 1.0 / (medium.h * medium.h);
  SparsePencil p;
  p.ndim = nd;
  p.dims = medium.dims;
  std::array<int, 3> idims = {1, 1, 1};
  long n = 1;
  for (int a = 0; a < nd; ++a) {
    idims[a] = medium.dims[a] - 2;
    n *= idims[a];
  }
  p.coords.resize(n);
  p.B = Vec::Zero(n);
  std::vector<Triplet> trips;
  trips.reserve(static_cast<size_t>(n) * (2 * nd + 1));
  std::array<int, 3> c = {0, 0, 0};
  for (long row = 0; row < n; ++row) {
    long r = row;
    for (int a = nd - 1; a >= 0; --a) {
      c[a] = 1 + static_cast<int>(r % idims[a]);
      r /= idims[a];
    }
    p.coords[row] = c;
    const long gid = medium.node_id(c);
    p.B[row] = medium.rho[gid];
    double diag = 0.0;
    for (int a = 0; a < nd; ++a)
      for (int dir = -1; dir <= 1; dir += 2) {
        std::array<int, 3> nb = c;
        nb[a] += dir;
        const double edge = 0.5 * (medium.sigma[gid] + medium.sigma[medium.node_id(nb)]);
        diag -= edge * inv_h2;
        if (nb[a] >= 1 && nb[a] <= medium.dims[a] - 2) {
          long col = 0;
          for (int b = 0; b < nd; ++b) col = col * idims[b] + (nb[b] - 1);
          trips.emplace_back(static_cast<int>(row), static_cast<int>(col), edge * inv_h2);
        }
      }
    trips.emplace_back(static_cast<int>(row), static_cast<int>(row), diag);
  }
  p.A.resize(n, n);
  p.A.setFromTriplets(trips.begin(), trips.end());
  p.A.makeCompressed();
  return p;
}

SparsePencil assemble_1d(const GridMedium& medium) {
  if (medium.ndim() != 1) throw ConfigError("assemble_1d expects one axis");
  return assemble_nd(medium);
}

SourceReceiver make_source(const SparsePencil& pencil, const std::array<int, 3>& location,
                           SourceKind kind, int taper_axis, double taper_halfwidth) {
  SourceReceiver sr;  // fine_grid.cpp:119-165
  sr.g = Vec::Zero(pencil.n());
  sr.q = Vec::Zero(pencil.n());
  const long k = pencil.node_of(location);
  if (k < 0) throw ConfigError("source location outside the interior grid");
  switch (kind) {
    case SourceKind::Point:
      sr.g[k] = 1.0;
      sr.g_support = {k};
      break;
    case SourceKind::UnitImpulse:
      sr.g[k] = 1.0 / pencil.B[k];
      sr.g_support = {k};
      break;
    case SourceKind::Taper: {
      if (taper_axis < 0 || taper_axis >= pencil.ndim) throw ConfigError("taper axis out of range");
      const double hw = taper_halfwidth;
      const int reach = static_cast<int>(std::ceil(3.0 * hw));
      double total = 0.0;
      for (long row = 0; row < pencil.n(); ++row) {
        if (pencil.coords[row][taper_axis] != location[taper_axis]) continue;
        double d2 = 0.0;
        bool close = true;
        for (int a = 0; a < pencil.ndim; ++a) {
          if (a == taper_axis) continue;
          const int d = pencil.coords[row][a] - location[a];
          if (std::abs(d) > reach) {
            close = false;
            break;
          }
          d2 += static_cast<double>(d) * d;
        }
        if (!close) continue;
        const double w = std::exp(-0.5 * d2 / (hw * hw));
        sr.g[row] = w;
        sr.g_support.push_back(row);
        total += w;
      }
      if (total <= 0.0) throw ConfigError("taper source has empty support");
      for (long row : sr.g_support) sr.g[row] /= total;
      break;
    }
  }
  return sr;
}

void set_receiver(SourceReceiver& sr, const SparsePencil& pencil, const std::array<int, 3>& location) {
  const long k = pencil.node_of(location);
  if (k < 0) throw ConfigError("receiver location outside the interior grid");
  if (sr.q.size() != pencil.n()) sr.q = Vec::Zero(pencil.n());
  sr.q[k] = 1.0;
  sr.q_support = {k};
}

namespace {

using FineGuard = std::unique_ptr<msw_fine, void (*)(msw_fine_handle)>;

FineGuard pencil_handle(const SparsePencil& pencil) {
  if (pencil.A.rows() != pencil.A.cols() || pencil.B.size() != pencil.A.rows())
    throw ConfigError("fine pencil: A must be square and match B");
  msw_fine_handle fh = nullptr;
  if (pencil.A.isCompressed()) {
    check(msw_fine_create_csc(pencil.A.rows(), pencil.A.outerIndexPtr(), pencil.A.innerIndexPtr(),
                              pencil.A.valuePtr(), pencil.B.data(), 0, &fh));
  } else {
    SpMat a = pencil.A;
    a.makeCompressed();
    check(msw_fine_create_csc(a.rows(), a.outerIndexPtr(), a.innerIndexPtr(), a.valuePtr(), pencil.B.data(), 0,
                              &fh));
  }
  return FineGuard(fh, msw_fine_destroy);
}

FineGuard medium_handle(const GridMedium& medium) {
  validate_medium(medium);
  std::vector<int32_t> dims(medium.dims.begin(), medium.dims.end());
  msw_fine_handle fh = nullptr;
  check(msw_fine_create(medium.ndim(), dims.data(), medium.h, medium.sigma.data(), medium.rho.data(), 0, &fh));
  return FineGuard(fh, msw_fine_destroy);
}

// reference.cpp:49-80 for S sources x R receivers on a device handle
std::vector<std::vector<Trace>> leapfrog_on(msw_fine_handle fh, long n, const std::vector<Vec>& g,
                                            const std::vector<Vec>& q, const Wavelet& wavelet, double t_final,
                                            double dt) {
  if (dt <= 0.0) throw ConfigError("fine_leapfrog: dt must be positive");
  for (const Vec& v : g)
    if (v.size() != n) throw ConfigError("fine_leapfrog: vector size mismatch");
  for (const Vec& v : q)
    if (v.size() != n) throw ConfigError("fine_leapfrog: vector size mismatch");
  const long steps = static_cast<long>(std::ceil(t_final / dt - 1e-12));
  const int S = static_cast<int>(g.size()), R = static_cast<int>(q.size());
  auto sparse = [&](const std::vector<Vec>& vs, std::vector<int32_t>& ptr, std::vector<int64_t>& rows,
                    std::vector<double>& vals) {
    ptr.assign(1, 0);
    for (const Vec& v : vs) {
      for (long i = 0; i < n; ++i)
        if (v[i] != 0.0) {
          rows.push_back(i);
          vals.push_back(v[i]);
        }
      ptr.push_back(static_cast<int32_t>(rows.size()));
    }
  };
  std::vector<int32_t> sp, rp;
  std::vector<int64_t> sr, rr;
  std::vector<double> sv, rv;
  sparse(g, sp, sr, sv);
  sparse(q, rp, rr, rv);
  std::vector<double> w(static_cast<size_t>(std::max<long>(steps, 1)));
  for (long s = 0; s < steps; ++s) w[s] = wavelet(static_cast<double>(s) * dt);  // reference.cpp:67
  std::vector<double> traces(static_cast<size_t>(steps + 1) * R * S);
  int64_t bad = 0;
  check(msw_fine_leapfrog(fh, S, sp.data(), sr.data(), sv.data(), R, rp.data(), rr.data(), rv.data(), dt, steps,
                          w.data(), 1, traces.data(), &bad));
  std::vector<std::vector<Trace>> out(S, std::vector<Trace>(R));
  for (int s = 0; s < S; ++s)
    for (int r = 0; r < R; ++r) {
      Trace& tr = out[s][r];
      tr.dt = dt;
      for (long k = 0; k <= steps; ++k) {
        tr.times.push_back(static_cast<double>(k) * dt);
        tr.values.push_back(traces[(static_cast<size_t>(k) * R + r) * S + s]);
      }
    }
  return out;
}

}  // namespace

std::vector<std::vector<Trace>> fine_leapfrog_batched(const SparsePencil& pencil, const std::vector<Vec>& g,
                                                      const std::vector<Vec>& q, const Wavelet& wavelet,
                                                      double t_final, double dt) {
  if (dt <= 0.0) throw ConfigError("fine_leapfrog: dt must be positive");
  FineGuard fh = pencil_handle(pencil);
  return leapfrog_on(fh.get(), pencil.n(), g, q, wavelet, t_final, dt);
}

std::vector<std::vector<Trace>> fine_leapfrog_batched(const GridMedium& medium, const std::vector<Vec>& g,
                                                      const std::vector<Vec>& q, const Wavelet& wavelet,
                                                      double t_final, double dt) {
  if (dt <= 0.0) throw ConfigError("fine_leapfrog: dt must be positive");
  FineGuard fh = medium_handle(medium);
  long n = 1;
  for (int d : medium.dims) n *= d - 2;
  return leapfrog_on(fh.get(), n, g, q, wavelet, t_final, dt);
}

Trace fine_leapfrog(const SparsePencil& pencil, const Vec& g, const Vec& q, const Wavelet& wavelet,
                    double t_final, double dt) {
  return fine_leapfrog_batched(pencil, {g}, {q}, wavelet, t_final, dt)[0][0];
}

double fine_cfl(const SparsePencil& pencil) {  // reference.cpp:24-47 on the device
  FineGuard fh = pencil_handle(pencil);
  double dt = 0.0;
  check(msw_fine_cfl(fh.get(), &dt));
  return dt;
}

double fine_cfl(const GridMedium& medium) {
  FineGuard fh = medium_handle(medium);
  double dt = 0.0;
  check(msw_fine_cfl(fh.get(), &dt));
  return dt;
}

// ============================== trace I/O ==================================

void write_trace_csv(const Trace& trace, const std::string& path) {  // trace_io.cpp:9-16
  std::FILE* f = std::fopen(path.c_str(), "w");
  if (!f) throw ConfigError("cannot open trace file for writing: " + path);
  std::fputs("t,value\n", f);
  for (size_t i = 0; i < trace.times.size(); ++i)
    std::fprintf(f, "%.17g,%.17g\n", trace.times[i], trace.values[i]);
  std::fclose(f);
}

Trace read_trace_csv(const std::string& path) {  // trace_io.cpp:18-34
  std::ifstream in(path);
  if (!in) throw ConfigError("cannot open trace file: " + path);
  std::string line;
  if (!std::getline(in, line) || line.rfind("t,value", 0) != 0)
    throw ConfigError("trace file missing 't,value' header: " + path);
  Trace t;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    const auto comma = line.find(',');
    if (comma == std::string::npos) throw ConfigError("malformed trace row: " + line);
    t.times.push_back(std::stod(line.substr(0, comma)));
    t.values.push_back(std::stod(line.substr(comma + 1)));
  }
  if (t.times.size() >= 2) t.dt = t.times[1] - t.times[0];
  return t;
}

ComparisonReport compare_traces(const Trace& a, const Trace& b) {  // trace_io.cpp:36-67
  if (a.times.empty() || b.times.empty()) throw ConfigError("cannot compare empty traces");
  ComparisonReport rep;
  rep.steps_a = static_cast<long>(a.times.size()) - 1;
  rep.steps_b = static_cast<long>(b.times.size()) - 1;
  rep.dt_a = a.dt;
  rep.dt_b = b.dt;
  auto sample_b = [&](double t) {
    const auto& ts = b.times;
    if (t <= ts.front()) return b.values.front();
    if (t >= ts.back()) return b.values.back();
    const auto it = std::upper_bound(ts.begin(), ts.end(), t);
    const size_t hi = it - ts.begin();
    const size_t lo = hi - 1;
    const double w = (t - ts[lo]) / (ts[hi] - ts[lo]);
    return (1.0 - w) * b.values[lo] + w * b.values[hi];
  };
  double num2 = 0.0, den2 = 0.0;
  const double t_end = std::min(a.times.back(), b.times.back());
  for (size_t i = 0; i < a.times.size(); ++i) {
    if (a.times[i] > t_end + 1e-12) break;
    const double bv = sample_b(a.times[i]);
    const double d = a.values[i] - bv;
    rep.max_abs_error = std::max(rep.max_abs_error, std::abs(d));
    num2 += d * d;
    den2 += bv * bv;
  }
  rep.rel_l2_error = den2 > 0.0 ? std::sqrt(num2 / den2) : std::sqrt(num2);
  return rep;
}

// ============================== on-line ROM ================================

int MultiscaleSystem::total_reduced_io() const {
  int k = 0;
  for (const auto& f : ifaces) k += f.size;
  return k;
}

long MultiscaleSystem::reduced_dof() const {
  long k = 0;
  for (const auto& r : roms) k += static_cast<long>(r.m) * r.ktilde;
  return k;
}

long MultiscaleSystem::flops_per_step() const {
  long flops = 0;
  for (const auto& r : roms) {
    const long kt = r.ktilde;
    flops += 2 * kt * kt + static_cast<long>(r.m - 1) * 3 * 2 * kt * kt;
  }
  for (const auto& f : ifaces) flops += 2L * f.size * f.size;
  return flops;
}

MultiscaleSystem assemble_system(const Partition& partition, const BoundaryBasis& basis,
                                 std::vector<SubdomainROM> roms, const Vec& B_diag) {
  MultiscaleSystem sys;  // msolver.cpp:31-106
  sys.roms = std::move(roms);
  for (int f = 0; f < static_cast<int>(partition.interfaces.size()); ++f) {
    const Interface& pf = partition.interfaces[f];
    CoupledInterface cf;
    cf.part_iface = f;
    cf.ci = pf.ci;
    cf.cj = pf.cj;
    cf.S = basis.S[f];
    cf.size = static_cast<int>(cf.S.cols());
    auto find_local = [&](int cell) {
      const auto& ids = sys.roms[cell].iface_ids;
      const auto it = std::find(ids.begin(), ids.end(), f);
      if (it == ids.end())
        throw ConfigError("cell " + std::to_string(cell) + " is missing interface " + std::to_string(f));
      return static_cast<int>(it - ids.begin());
    };
    cf.li = find_local(pf.ci);
    cf.lj = find_local(pf.cj);
    const SubdomainROM& ri = sys.roms[pf.ci];
    const SubdomainROM& rj = sys.roms[pf.cj];
    if (ri.block_size(cf.li) != cf.size || rj.block_size(cf.lj) != cf.size)
      throw ConfigError("mismatched interface bases between cells " + std::to_string(pf.ci) + " and " +
                        std::to_string(pf.cj));
    for (int i = 0; i < cf.size; ++i)
      if (ri.g_proj[cf.li][i] != rj.g_proj[cf.lj][i] || ri.q_proj[cf.li][i] != rj.q_proj[cf.lj][i])
        throw ConfigError("projected I/O disagrees between the two sides of interface " + std::to_string(f));
    const int M = cf.size;
    auto block = [&](const SubdomainROM& r, int li) {
      std::vector<double> B(static_cast<size_t>(M) * M);
      const int o = r.block_offset(li);
      for (int j = 0; j < M; ++j)
        for (int i = 0; i < M; ++i) B[i + j * M] = r.ladder_hat[0](o + i, o + j);
      return B;
    };
    std::vector<double> form = spd_inverse(block(ri, cf.li), M);
    const std::vector<double> inv_j = spd_inverse(block(rj, cf.lj), M);
    for (size_t k = 0; k < form.size(); ++k) form[k] += inv_j[k];
    symmetrize(form, M);
    std::vector<double> mass = spd_inverse(form, M);
    symmetrize(mass, M);
    cf.mass_form = from_vec(form, M, M);
    cf.mass = from_vec(mass, M, M);
    cf.g_proj = ri.g_proj[cf.li];
    cf.q_proj = ri.q_proj[cf.li];
    sys.ifaces.push_back(std::move(cf));
  }
  std::map<long, CornerGroup> groups;  // msolver.cpp:81-104
  for (const HangingNode& hn : partition.hanging) {
    int f = -1;
    for (int i = 0; i < static_cast<int>(partition.interfaces.size()); ++i) {
      if (partition.interfaces[i].ci == hn.ci && partition.interfaces[i].cj == hn.cj &&
          std::binary_search(partition.interfaces[i].nodes.begin(), partition.interfaces[i].nodes.end(),
                             hn.id)) {
        f = i;
        break;
      }
    }
    if (f < 0) throw ConfigError("hanging node without a matching interface");
    const auto& nodes = partition.interfaces[f].nodes;
    CornerGroup::Copy copy;
    copy.iface = f;
    copy.row = static_cast<int>(std::lower_bound(nodes.begin(), nodes.end(), hn.id) - nodes.begin());
    copy.mass = B_diag[hn.id];
    auto& grp = groups[hn.parent];
    grp.parent = hn.parent;
    grp.copies.push_back(copy);
  }
  for (auto& kv : groups) sys.corners.push_back(std::move(kv.second));
  return sys;
}

namespace detail {

// Device-resident copy of a MultiscaleSystem: the msw_handle plus the host
// layout needed to translate WaveState <-> the ABI's flat state arrays.
struct DeviceSystem {
  msw_handle h = nullptr;
  int S = 1, R = 0;
  std::vector<long> cell_u_off;
  std::vector<long> iface_off;
  long total_u = 0, total_io = 0;
  bool has_state = false;
  double dt = 0.0;
  ~DeviceSystem() {
    if (h) msw_destroy(h);
  }
};

// Device copies live in a small registry instead of a MultiscaleSystem member,
// so MultiscaleSystem keeps the reference's exact layout (msolver.hpp:38-46).
// An entry is found by a fingerprint of the system: its address, the heap
// buffers of its vectors (distinct for distinct live systems) and a sample of
// its values (ladder corners, masses, the full projected source / receiver),
// so a later system that happens to reuse a dead one's storage is not
// mistaken for it unless it is the same system.  At most kRegistry systems
// stay resident (least recently used evicted first).
constexpr size_t kRegistry = 4;

uint64_t fingerprint(const MultiscaleSystem& sys) {
  uint64_t h = 1469598103934665603ull;
  auto mix_bytes = [&](const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) {
      h ^= b[i];
      h *= 1099511628211ull;
    }
  };
  auto mix = [&](auto v) { mix_bytes(&v, sizeof(v)); };
  auto mix_mat = [&](const Mat& m) {
    mix(static_cast<const void*>(m.data()));
    mix(static_cast<long>(m.rows()));
    mix(static_cast<long>(m.cols()));
    if (m.size() > 0) {
      mix(m.data()[0]);
      mix(m.data()[m.size() / 2]);
      mix(m.data()[m.size() - 1]);
    }
  };
  auto mix_vec = [&](const Vec& v) {
    mix(static_cast<long>(v.size()));
    if (v.size() > 0) mix_bytes(v.data(), sizeof(double) * static_cast<size_t>(v.size()));
  };
  mix(static_cast<const void*>(&sys));
  mix(static_cast<const void*>(sys.roms.data()));
  mix(static_cast<const void*>(sys.ifaces.data()));
  mix(sys.roms.size());
  mix(sys.ifaces.size());
  mix(sys.corners.size());
  for (const SubdomainROM& r : sys.roms) {
    mix(r.m);
    mix(r.ktilde);
    for (const Mat& L : r.ladder) mix_mat(L);
    for (const Mat& L : r.ladder_hat) mix_mat(L);
  }
  for (const CoupledInterface& cf : sys.ifaces) {
    mix(cf.ci);
    mix(cf.cj);
    mix(cf.li);
    mix(cf.lj);
    mix(cf.size);
    mix_mat(cf.mass);
    mix_vec(cf.g_proj);
    mix_vec(cf.q_proj);
  }
  for (const CornerGroup& g : sys.corners) {
    mix(g.parent);
    for (const auto& cp : g.copies) {
      mix(cp.iface);
      mix(cp.row);
      mix(cp.mass);
    }
  }
  return h;
}

std::mutex g_reg_mu;
std::list<std::pair<uint64_t, std::shared_ptr<DeviceSystem>>> g_registry;  // most recent first

std::shared_ptr<DeviceSystem> build_device(const MultiscaleSystem& sys);

std::shared_ptr<DeviceSystem> bind(const MultiscaleSystem& sys) {
  const uint64_t key = fingerprint(sys);
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    for (auto it = g_registry.begin(); it != g_registry.end(); ++it)
      if (it->first == key) {
        g_registry.splice(g_registry.begin(), g_registry, it);
        return g_registry.front().second;
      }
  }
  auto dev = build_device(sys);
  std::lock_guard<std::mutex> lk(g_reg_mu);
  g_registry.emplace_front(key, dev);
  while (g_registry.size() > kRegistry) g_registry.pop_back();
  return dev;
}

void unbind(const MultiscaleSystem& sys) {
  const uint64_t key = fingerprint(sys);
  std::lock_guard<std::mutex> lk(g_reg_mu);
  g_registry.remove_if([&](const std::pair<uint64_t, std::shared_ptr<DeviceSystem>>& e) { return e.first == key; });
}

std::shared_ptr<DeviceSystem> build_device(const MultiscaleSystem& sys) {
  auto dev = std::make_shared<DeviceSystem>();
  const int nc = static_cast<int>(sys.roms.size()), nf = static_cast<int>(sys.ifaces.size());
  std::vector<int32_t> cm(nc), ckt(nc), cptr(1, 0), cids, coff, ci(nf), cj(nf), li(nf), lj(nf), sz(nf);
  std::vector<int64_t> loff(nc);
  std::vector<double> lad, mass;
  dev->cell_u_off.assign(nc + 1, 0);
  for (int c = 0; c < nc; ++c) {
    const SubdomainROM& r = sys.roms[c];
    cm[c] = r.m;
    ckt[c] = r.ktilde;
    for (size_t l = 0; l < r.iface_ids.size(); ++l) {
      cids.push_back(r.iface_ids[l]);
      coff.push_back(r.iface_offsets[l]);
    }
    cptr.push_back(static_cast<int32_t>(cids.size()));
    loff[c] = static_cast<int64_t>(lad.size());
    if (static_cast<int>(r.ladder.size()) != r.m || static_cast<int>(r.ladder_hat.size()) != r.m)
      throw ConfigError("cell " + std::to_string(c) + ": ladder count != m");
    for (const Mat& L : r.ladder) {
      const std::vector<double> v = to_vec(L);
      lad.insert(lad.end(), v.begin(), v.end());
    }
    for (const Mat& L : r.ladder_hat) {
      const std::vector<double> v = to_vec(L);
      lad.insert(lad.end(), v.begin(), v.end());
    }
    dev->cell_u_off[c + 1] = dev->cell_u_off[c] + static_cast<long>(r.m) * r.ktilde;
  }
  dev->iface_off.assign(nf + 1, 0);
  for (int f = 0; f < nf; ++f) {
    const CoupledInterface& cf = sys.ifaces[f];
    ci[f] = cf.ci;
    cj[f] = cf.cj;
    li[f] = cf.li;
    lj[f] = cf.cj >= 0 ? cf.lj : -1;
    sz[f] = cf.size;
    if (cf.mass.rows() != cf.size || cf.mass.cols() != cf.size)
      throw ConfigError("interface " + std::to_string(f) + " has no shared mass (use assemble_system)");
    const std::vector<double> v = to_vec(cf.mass);
    mass.insert(mass.end(), v.begin(), v.end());
    dev->iface_off[f + 1] = dev->iface_off[f] + cf.size;
  }
  dev->total_u = dev->cell_u_off[nc];
  dev->total_io = dev->iface_off[nf];
  msw_system_desc d{};
  d.n_cells = nc;
  d.n_ifaces = nf;
  d.cell_m = cm.data();
  d.cell_ktilde = ckt.data();
  d.cell_iface_ptr = cptr.data();
  d.cell_iface_ids = cids.data();
  d.cell_iface_offsets = coff.data();
  d.cell_ladder_off = loff.data();
  d.ladders = lad.data();
  d.iface_ci = ci.data();
  d.iface_cj = cj.data();
  d.iface_li = li.data();
  d.iface_lj = lj.data();
  d.iface_size = sz.data();
  d.iface_mass = mass.data();
  check(msw_create(&d, 0, &dev->h));
  // the system's own single source / receiver (CoupledInterface g/q_proj)
  std::vector<double> g(dev->total_io, 0.0);
  std::vector<int32_t> rptr{0}, rif;
  std::vector<double> rq;
  for (int f = 0; f < nf; ++f) {
    const CoupledInterface& cf = sys.ifaces[f];
    bool nz = false;
    for (int i = 0; i < cf.size; ++i) {
      if (cf.g_proj.size() == cf.size) g[dev->iface_off[f] + i] = cf.g_proj[i];
      if (cf.q_proj.size() == cf.size && cf.q_proj[i] != 0.0) nz = true;
    }
    if (nz) {
      rif.push_back(f);
      for (int i = 0; i < cf.size; ++i) rq.push_back(cf.q_proj[i]);
    }
  }
  rptr.push_back(static_cast<int32_t>(rif.size()));
  check(msw_set_sources(dev->h, 1, g.data()));
  check(msw_set_receivers(dev->h, 1, rptr.data(), rif.data(), rq.data()));
  dev->R = 1;
  if (!sys.corners.empty()) {
    std::vector<int32_t> gp{0}, cif, crow, K(nf);
    std::vector<double> cmass, basis;
    for (const CornerGroup& grp : sys.corners) {
      for (const auto& cp : grp.copies) {
        cif.push_back(cp.iface);
        crow.push_back(cp.row);
        cmass.push_back(cp.mass);
      }
      gp.push_back(static_cast<int32_t>(cif.size()));
    }
    for (int f = 0; f < nf; ++f) {
      K[f] = static_cast<int32_t>(sys.ifaces[f].S.rows());
      const std::vector<double> v = to_vec(sys.ifaces[f].S);
      basis.insert(basis.end(), v.begin(), v.end());
    }
    check(msw_set_corners(dev->h, static_cast<int32_t>(sys.corners.size()), gp.data(), cif.data(),
                          crow.data(), cmass.data(), K.data(), basis.data()));
  }
  return dev;
}

void upload(DeviceSystem& dev, const MultiscaleSystem& sys, const WaveState& st) {
  if (!dev.has_state || dev.dt != st.dt) {
    check(msw_make_state(dev.h, st.dt));
    dev.has_state = true;
    dev.dt = st.dt;
  }
  std::vector<double> uc(dev.total_u), up(dev.total_u), bc(dev.total_io), bp(dev.total_io);
  for (size_t c = 0; c < sys.roms.size(); ++c) {
    std::copy(st.u_cur[c].data(), st.u_cur[c].data() + st.u_cur[c].size(), uc.begin() + dev.cell_u_off[c]);
    std::copy(st.u_prev[c].data(), st.u_prev[c].data() + st.u_prev[c].size(), up.begin() + dev.cell_u_off[c]);
  }
  for (size_t f = 0; f < sys.ifaces.size(); ++f) {
    std::copy(st.ubar_cur[f].data(), st.ubar_cur[f].data() + st.ubar_cur[f].size(), bc.begin() + dev.iface_off[f]);
    std::copy(st.ubar_prev[f].data(), st.ubar_prev[f].data() + st.ubar_prev[f].size(),
              bp.begin() + dev.iface_off[f]);
  }
  check(msw_set_state(dev.h, uc.data(), up.data(), bc.data(), bp.data(), st.t, st.step_index));
}

void download(DeviceSystem& dev, const MultiscaleSystem& sys, WaveState& st) {
  std::vector<double> uc(dev.total_u), up(dev.total_u), bc(dev.total_io), bp(dev.total_io);
  double t = 0.0;
  int64_t si = 0;
  check(msw_get_state(dev.h, uc.data(), up.data(), bc.data(), bp.data(), &t, &si));
  for (size_t c = 0; c < sys.roms.size(); ++c) {
    std::copy(uc.begin() + dev.cell_u_off[c], uc.begin() + dev.cell_u_off[c + 1], st.u_cur[c].data());
    std::copy(up.begin() + dev.cell_u_off[c], up.begin() + dev.cell_u_off[c + 1], st.u_prev[c].data());
  }
  for (size_t f = 0; f < sys.ifaces.size(); ++f) {
    std::copy(bc.begin() + dev.iface_off[f], bc.begin() + dev.iface_off[f + 1], st.ubar_cur[f].data());
    std::copy(bp.begin() + dev.iface_off[f], bp.begin() + dev.iface_off[f + 1], st.ubar_prev[f].data());
  }
  st.t = t;
  st.step_index = si;
}

}  // namespace detail

void invalidate_device(const MultiscaleSystem& system) { detail::unbind(system); }

WaveState make_state(const MultiscaleSystem& system, double dt) {  // msolver.cpp:108-121
  if (dt <= 0.0) throw ConfigError("dt must be positive");
  WaveState st;
  st.dt = dt;
  for (const auto& r : system.roms) {
    st.u_cur.push_back(Vec::Zero(static_cast<long>(r.m) * r.ktilde));
    st.u_prev.push_back(Vec::Zero(static_cast<long>(r.m) * r.ktilde));
  }
  for (const auto& f : system.ifaces) {
    st.ubar_cur.push_back(Vec::Zero(f.size));
    st.ubar_prev.push_back(Vec::Zero(f.size));
  }
  return st;
}

void step(const MultiscaleSystem& system, WaveState& state, double source_value) {
  auto dev = detail::bind(system);
  detail::upload(*dev, system, state);
  const int rc = msw_step(dev->h, &source_value, 1);
  const std::string msg = rc == MSW_OK ? std::string() : std::string(msw_last_error());
  detail::download(*dev, system, state);  // reference mutates the state before throwing
  if (rc == MSW_NUMERICAL_ERROR) throw NumericalError(msg);
  if (rc == MSW_CONFIG_ERROR) throw ConfigError(msg);
  if (rc != MSW_OK) throw DeviceError(msg);
}

void corner_correct(const MultiscaleSystem& system, WaveState& state) {
  if (system.corners.empty()) return;
  auto dev = detail::bind(system);
  detail::upload(*dev, system, state);
  check(msw_corner_correct(dev->h));
  detail::download(*dev, system, state);
}

double estimate_dt(const MultiscaleSystem& system, double safety) {
  auto dev = detail::bind(system);
  double dt = 0.0;
  check(msw_estimate_dt(dev->h, safety, &dt));
  return dt;
}

double energy(const MultiscaleSystem& system, const WaveState& state) {
  auto dev = detail::bind(system);
  detail::upload(*dev, system, state);
  std::vector<double> e(static_cast<size_t>(std::max<long>(dev->S, 1)));
  check(msw_energy(dev->h, e.data()));
  return e[0];
}

RunResult run_simulation(const MultiscaleSystem& system, const Wavelet& wavelet, double t_final,
                         double dt, bool corner_correction, long energy_stride) {
  auto dev = detail::bind(system);
  if (dt <= 0.0) throw ConfigError("dt must be positive");
  check(msw_make_state(dev->h, dt));
  dev->has_state = true;
  dev->dt = dt;
  RunResult res;  // msolver.cpp:397-424
  const long steps = static_cast<long>(std::ceil(t_final / dt - 1e-12));
  res.steps = steps;
  res.trace.dt = dt;
  std::vector<double> w(static_cast<size_t>(std::max<long>(steps, 1)));
  double t = 0.0;
  for (long s = 0; s < steps; ++s) {
    w[s] = wavelet(t);  // wavelet at the accumulated time (msolver.cpp:191,415)
    t += dt;
  }
  res.trace.times.resize(steps + 1);
  res.trace.values.resize(steps + 1);
  int64_t bad = 0;
  if (energy_stride <= 0) {
    check(msw_run(dev->h, steps, w.data(), 1, corner_correction ? 1 : 0, res.trace.values.data(),
                  res.trace.times.data(), &bad));
    return res;
  }
  // energy every energy_stride steps (msolver.cpp:415-420): run in chunks;
  // each chunk's trace row 0 repeats the previous chunk's last sample
  std::vector<double> e(static_cast<size_t>(std::max<long>(dev->S, 1)));
  std::vector<double> tv, tt;
  long done = 0;
  while (done < steps) {
    const long chunk = std::min(energy_stride, steps - done);
    tv.assign(static_cast<size_t>(chunk + 1), 0.0);
    tt.assign(static_cast<size_t>(chunk + 1), 0.0);
    check(msw_run(dev->h, chunk, w.data() + done, 1, corner_correction ? 1 : 0, tv.data(), tt.data(), &bad));
    for (long i = (done == 0 ? 0 : 1); i <= chunk; ++i) {
      res.trace.values[done + i] = tv[i];
      res.trace.times[done + i] = tt[i];
    }
    done += chunk;
    if (chunk == energy_stride) {
      check(msw_energy(dev->h, e.data()));
      res.energy_times.push_back(tt[chunk]);
      res.energy_values.push_back(e[0]);
    }
  }
  return res;
}

std::vector<std::vector<Trace>> run_simulation_batched(
    const MultiscaleSystem& system, const std::vector<std::vector<Vec>>& g_proj_per_source,
    const std::vector<std::vector<Vec>>& q_proj_per_receiver, const Wavelet& wavelet, double t_final,
    double dt, bool corner_correction) {
  auto dev = detail::bind(system);
  const int S = static_cast<int>(g_proj_per_source.size());
  const int R = static_cast<int>(q_proj_per_receiver.size());
  const int nf = static_cast<int>(system.ifaces.size());
  std::vector<double> g(static_cast<size_t>(dev->total_io) * S, 0.0);
  for (int s = 0; s < S; ++s)
    for (int f = 0; f < nf; ++f)
      for (int i = 0; i < system.ifaces[f].size; ++i)
        g[(dev->iface_off[f] + i) * S + s] = g_proj_per_source[s][f][i];
  std::vector<int32_t> rptr{0}, rif;
  std::vector<double> rq;
  for (int r = 0; r < R; ++r) {
    for (int f = 0; f < nf; ++f) {
      const Vec& q = q_proj_per_receiver[r][f];
      bool nz = false;
      for (int i = 0; i < q.size(); ++i) nz |= q[i] != 0.0;
      if (!nz) continue;
      rif.push_back(f);
      for (int i = 0; i < q.size(); ++i) rq.push_back(q[i]);
    }
    rptr.push_back(static_cast<int32_t>(rif.size()));
  }
  check(msw_set_sources(dev->h, S, g.data()));
  check(msw_set_receivers(dev->h, R, rptr.data(), rif.data(), rq.data()));
  check(msw_make_state(dev->h, dt));
  const long steps = static_cast<long>(std::ceil(t_final / dt - 1e-12));
  std::vector<double> w(static_cast<size_t>(std::max<long>(steps, 1)));
  double t = 0.0;
  for (long s = 0; s < steps; ++s) {
    w[s] = wavelet(t);
    t += dt;
  }
  std::vector<double> traces(static_cast<size_t>(steps + 1) * R * S), times(steps + 1);
  int64_t bad = 0;
  const int rc = msw_run(dev->h, steps, w.data(), 1, corner_correction ? 1 : 0, traces.data(),
                         times.data(), &bad);
  // restore the system's own single source/receiver binding for later calls
  detail::unbind(system);
  check(rc);
  std::vector<std::vector<Trace>> out(R, std::vector<Trace>(S));
  for (int r = 0; r < R; ++r)
    for (int s = 0; s < S; ++s) {
      Trace& tr = out[r][s];
      tr.dt = dt;
      tr.times = times;
      tr.values.resize(steps + 1);
      for (long k = 0; k <= steps; ++k) tr.values[k] = traces[(static_cast<size_t>(k) * R + r) * S + s];
    }
  return out;
}

}  // namespace mswave
