// ===========================================================================
// TEST INFRASTRUCTURE ONLY -- CPU oracle for the on-line ROM stepper and the
// fine-grid leapfrog of arXiv 1604.06750 (reference: /root/reference/proj).
//
// This file is a faithful, Eigen-free, single-threaded C++ restatement of the
// reference's algorithm.  It is the CHECKER: only tests/, __graft_entry__
// .smoke() and bench.py's cpu_baseline / --impl reference leg may load it.
// The product library (paper_1604_06750_b200/libmswave_b200.so) never links
// or calls it.
//
// Why a restatement: the reference cannot be compiled here -- Eigen3 is not
// installed anywhere and there is no network (proj/CMakeLists.txt:13), so
// `oracle/_ref` cannot be built.  Parity of this
// restatement is pinned by the reference's own known-answer tests
// (proj/tests/test_msolver.cpp, test_reference.cpp), re-run in
// tests/test_oracle_kat.py.
//
// Arithmetic conventions (to stay as close as possible to the reference
// build, which has no -march flags and therefore no FMA contraction):
//   * compiled with -ffp-contract=off;
//   * dense mat-vec y = A x accumulates y_i over columns j in ascending order
//     (Eigen col-major GEMV order is unspecified; bitwise parity with the
//     reference is therefore unpinned and checked at 1e-10);
//   * sparse mat-vec follows Eigen's col-major SparseMatrix * dense product:
//     for each column j ascending, y_i += a_ij x_j (reference.cpp:68).
// ===========================================================================

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "../include/mswave_b200.h"

namespace {

thread_local std::string g_err;

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

using Vec = std::vector<double>;

// y = A x, A n x n column-major, ascending-column accumulation.
inline void gemv(const double* A, int n, const double* x, double* y) {
  for (int i = 0; i < n; ++i) y[i] = 0.0;
  for (int j = 0; j < n; ++j) {
    const double xj = x[j];
    const double* col = A + static_cast<size_t>(j) * n;
    for (int i = 0; i < n; ++i) y[i] += col[i] * xj;
  }
}

// Cholesky A = L L^T (lower, column-major, n x n); throws if not SPD.
void cholesky(const double* A, int n, std::vector<double>& L) {
  L.assign(static_cast<size_t>(n) * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double d = A[j + j * n];
    for (int k = 0; k < j; ++k) d -= L[j + k * n] * L[j + k * n];
    if (!(d > 0.0)) throw NumericalError("oracle: LLT of a non-SPD block");
    const double ljj = std::sqrt(d);
    L[j + j * n] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double s = A[i + j * n];
      for (int k = 0; k < j; ++k) s -= L[i + k * n] * L[j + k * n];
      L[i + j * n] = s / ljj;
    }
  }
}

// X = A^{-1} via LLT solve against the identity (Eigen llt().solve(I)).
std::vector<double> spd_inverse(const double* A, int n) {
  std::vector<double> L;
  cholesky(A, n, L);
  std::vector<double> X(static_cast<size_t>(n) * n, 0.0);
  std::vector<double> y(n);
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

// x = A^{-1} b for SPD A (llt().solve(b), used by FlatOps::mass_apply).
void spd_solve(const double* A, int n, const double* b, double* x) {
  std::vector<double> L;
  cholesky(A, n, L);
  std::vector<double> y(n);
  for (int i = 0; i < n; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= L[i + k * n] * y[k];
    y[i] = s / L[i + i * n];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = y[i];
    for (int k = i + 1; k < n; ++k) s -= L[k + i * n] * x[k];
    x[i] = s / L[i + i * n];
  }
}

void symmetrize(std::vector<double>& M, int n) {  // 0.5 (M + M^T)
  std::vector<double> T(M);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) M[i + j * n] = 0.5 * (T[i + j * n] + T[j + i * n]);
}

struct Cell {
  int m = 0, kt = 0;
  std::vector<int> iface_ids, iface_off;
  const double* lad = nullptr;  // ladder[0..m-1], ladder_hat[0..m-1]
  const double* L(int k) const { return lad + static_cast<size_t>(k) * kt * kt; }
  const double* Lhat(int k) const { return lad + static_cast<size_t>(m + k) * kt * kt; }
};

struct Iface {
  int ci = -1, cj = -1, li = -1, lj = -1, M = 0;
  std::vector<double> mass, mass_form;
};

struct CornerCopy {
  int iface, row;
  double mass;
};

struct State {  // WaveState, msolver.hpp:53-59 (one per source)
  std::vector<Vec> u_cur, u_prev, ubar_cur, ubar_prev;
};

struct System {
  std::vector<Cell> cells;
  std::vector<Iface> ifaces;
  std::vector<double> ladders;  // owned copy
  std::vector<int> iface_row_off;
  int total_io = 0;
  // io
  int S = 1;
  std::vector<double> gproj;  // [total_io][S]
  int R = 0;
  std::vector<int> rcv_ptr, term_iface;
  std::vector<long> term_qoff;
  std::vector<double> term_q;
  // corners
  std::vector<std::vector<CornerCopy>> corners;
  std::vector<int> iface_K;
  std::vector<long> basis_off;
  std::vector<double> basis;
  // state
  std::vector<State> st;
  double t = 0.0, dt = 0.0;
  long step_index = 0;
  bool has_state = false;

  int off(int c, int li) const { return cells[c].iface_off[li]; }
};

// assemble_system (msolver.cpp:31-79): shared mass per interface.
void assemble(System& sys, const msw_system_desc* d) {
  const int nc = d->n_cells, nf = d->n_ifaces;
  if (nc < 0 || nf < 0) throw ConfigError("negative sizes");
  size_t lad_total = 0;
  for (int c = 0; c < nc; ++c) {
    const size_t kt = d->cell_ktilde[c];
    lad_total = std::max(lad_total, static_cast<size_t>(d->cell_ladder_off[c]) +
                                        2 * static_cast<size_t>(d->cell_m[c]) * kt * kt);
  }
  sys.ladders.assign(d->ladders, d->ladders + lad_total);
  sys.cells.resize(nc);
  for (int c = 0; c < nc; ++c) {
    Cell& cl = sys.cells[c];
    cl.m = d->cell_m[c];
    cl.kt = d->cell_ktilde[c];
    if (cl.m < 1) throw ConfigError("cell with m < 1");
    for (int p = d->cell_iface_ptr[c]; p < d->cell_iface_ptr[c + 1]; ++p) {
      cl.iface_ids.push_back(d->cell_iface_ids[p]);
      cl.iface_off.push_back(d->cell_iface_offsets[p]);
    }
    cl.iface_off.push_back(cl.kt);
    cl.lad = sys.ladders.data() + d->cell_ladder_off[c];
  }
  sys.ifaces.resize(nf);
  sys.iface_row_off.assign(nf + 1, 0);
  long mass_off = 0;
  for (int f = 0; f < nf; ++f) {
    Iface& cf = sys.ifaces[f];
    cf.ci = d->iface_ci[f];
    cf.cj = d->iface_cj[f];
    cf.li = d->iface_li[f];
    cf.lj = d->iface_lj[f];
    cf.M = d->iface_size[f];
    sys.iface_row_off[f + 1] = sys.iface_row_off[f] + cf.M;
    auto check_side = [&](int c, int li) {
      if (c < 0 || c >= nc) throw ConfigError("interface cell out of range");
      const Cell& cl = sys.cells[c];
      if (li < 0 || li >= static_cast<int>(cl.iface_ids.size()) || cl.iface_ids[li] != f)
        throw ConfigError("cell " + std::to_string(c) + " is missing interface " +
                          std::to_string(f));
      if (cl.iface_off[li + 1] - cl.iface_off[li] != cf.M)
        throw ConfigError("mismatched interface bases between cells");
    };
    check_side(cf.ci, cf.li);
    if (cf.cj >= 0) check_side(cf.cj, cf.lj);
    const int M = cf.M;
    if (d->iface_mass) {
      cf.mass.assign(d->iface_mass + mass_off, d->iface_mass + mass_off + M * M);
      cf.mass_form = spd_inverse(cf.mass.data(), M);
    } else {
      auto block = [&](int c, int li) {
        const Cell& cl = sys.cells[c];
        std::vector<double> B(static_cast<size_t>(M) * M);
        const int o = cl.iface_off[li];
        const double* H = cl.Lhat(0);
        for (int j = 0; j < M; ++j)
          for (int i = 0; i < M; ++i) B[i + j * M] = H[(o + i) + static_cast<size_t>(o + j) * cl.kt];
        return B;
      };
      std::vector<double> Mi = block(cf.ci, cf.li);
      cf.mass_form = spd_inverse(Mi.data(), M);
      if (cf.cj >= 0) {
        std::vector<double> Mj = block(cf.cj, cf.lj);
        std::vector<double> inv_j = spd_inverse(Mj.data(), M);
        for (size_t k = 0; k < inv_j.size(); ++k) cf.mass_form[k] += inv_j[k];
      }
      symmetrize(cf.mass_form, M);
      cf.mass = spd_inverse(cf.mass_form.data(), M);
      symmetrize(cf.mass, M);
    }
    mass_off += static_cast<long>(M) * M;
  }
  sys.total_io = sys.iface_row_off[nf];
  sys.S = 1;
  sys.gproj.assign(sys.total_io, 0.0);
}

void make_state(System& sys, double dt) {  // msolver.cpp:108-121
  if (dt <= 0.0) throw ConfigError("dt must be positive");
  sys.dt = dt;
  sys.t = 0.0;
  sys.step_index = 0;
  sys.st.assign(sys.S, State());
  for (State& s : sys.st) {
    for (const Cell& c : sys.cells) {
      s.u_cur.emplace_back(static_cast<size_t>(c.m) * c.kt, 0.0);
      s.u_prev.emplace_back(static_cast<size_t>(c.m) * c.kt, 0.0);
    }
    for (const Iface& f : sys.ifaces) {
      s.ubar_cur.emplace_back(f.M, 0.0);
      s.ubar_prev.emplace_back(f.M, 0.0);
    }
  }
  sys.has_state = true;
}

// first_layer_flux (msolver.cpp:126-130)
Vec first_layer_flux(const Cell& r, const Vec& u) {
  const int kt = r.kt;
  Vec d(kt), out(kt);
  if (r.m == 1)
    for (int i = 0; i < kt; ++i) d[i] = -u[i];
  else
    for (int i = 0; i < kt; ++i) d[i] = u[kt + i] - u[i];
  gemv(r.L(0), kt, d.data(), out.data());
  return out;
}

// interior_accelerations (msolver.cpp:133-145), three GEMVs per layer as in
// the reference.
Vec interior_accelerations(const Cell& r, const Vec& u) {
  const int kt = r.kt;
  Vec acc(u.size(), 0.0), d(kt), t1(kt), t2(kt), flux(kt);
  for (int k = 2; k <= r.m; ++k) {
    const double* uk = u.data() + static_cast<size_t>(k - 1) * kt;
    const double* ukm = u.data() + static_cast<size_t>(k - 2) * kt;
    for (int i = 0; i < kt; ++i) d[i] = uk[i] - ukm[i];
    gemv(r.L(k - 2), kt, d.data(), t1.data());
    for (int i = 0; i < kt; ++i) flux[i] = -t1[i];
    if (k < r.m) {
      const double* ukp = u.data() + static_cast<size_t>(k) * kt;
      for (int i = 0; i < kt; ++i) d[i] = ukp[i] - uk[i];
    } else {
      for (int i = 0; i < kt; ++i) d[i] = -uk[i];
    }
    gemv(r.L(k - 1), kt, d.data(), t2.data());
    for (int i = 0; i < kt; ++i) flux[i] += t2[i];
    gemv(r.Lhat(k - 1), kt, flux.data(), acc.data() + static_cast<size_t>(k - 1) * kt);
  }
  return acc;
}

// step (msolver.cpp:154-194) for one source.  Returns amp = max|u_cur|.
double step_one(const System& sys, State& st, const double* g_col, int g_stride,
                double source_value, double dt) {
  const int nc = static_cast<int>(sys.cells.size());
  const int nf = static_cast<int>(sys.ifaces.size());
  const double dt2 = dt * dt;
  std::vector<Vec> flux(nc);
  for (int c = 0; c < nc; ++c) flux[c] = first_layer_flux(sys.cells[c], st.u_cur[c]);
  std::vector<Vec> u_next(nc);
  for (int c = 0; c < nc; ++c) {
    const Vec acc = interior_accelerations(sys.cells[c], st.u_cur[c]);
    Vec& un = u_next[c];
    un.resize(acc.size());
    for (size_t i = 0; i < acc.size(); ++i)
      un[i] = 2.0 * st.u_cur[c][i] - st.u_prev[c][i] + dt2 * acc[i];
  }
  for (int f = 0; f < nf; ++f) {
    const Iface& cf = sys.ifaces[f];
    const int M = cf.M;
    const int oi = sys.off(cf.ci, cf.li);
    Vec phi(M);
    for (int i = 0; i < M; ++i) phi[i] = flux[cf.ci][oi + i];
    if (cf.cj >= 0) {
      const int oj = sys.off(cf.cj, cf.lj);
      for (int i = 0; i < M; ++i) phi[i] += flux[cf.cj][oj + i];
    }
    const int ro = sys.iface_row_off[f];
    for (int i = 0; i < M; ++i) phi[i] += source_value * g_col[static_cast<size_t>(ro + i) * g_stride];
    Vec acc(M);
    gemv(cf.mass.data(), M, phi.data(), acc.data());
    Vec nb(M);
    for (int i = 0; i < M; ++i)
      nb[i] = 2.0 * st.ubar_cur[f][i] - st.ubar_prev[f][i] + dt2 * acc[i];
    for (int i = 0; i < M; ++i) u_next[cf.ci][oi + i] = nb[i];
    if (cf.cj >= 0) {
      const int oj = sys.off(cf.cj, cf.lj);
      for (int i = 0; i < M; ++i) u_next[cf.cj][oj + i] = nb[i];
    }
    st.ubar_prev[f] = st.ubar_cur[f];
    st.ubar_cur[f] = std::move(nb);
  }
  // amp = max |u_cur| over all cells (msolver.cpp:185-190); any non-finite
  // entry makes the step unstable.
  double amp = 0.0;
  bool nonfinite = false;
  for (int c = 0; c < nc; ++c) {
    st.u_prev[c] = std::move(st.u_cur[c]);
    st.u_cur[c] = std::move(u_next[c]);
    for (double v : st.u_cur[c]) {
      if (!std::isfinite(v)) nonfinite = true;
      else amp = std::max(amp, std::abs(v));
    }
  }
  return nonfinite ? std::numeric_limits<double>::infinity() : amp;
}

bool unstable(double amp) { return !std::isfinite(amp) || amp > 1e12; }  // msolver.cpp:147-150

// corner_correct (msolver.cpp:196-227) for one source.
void corner_correct_one(const System& sys, State& st) {
  if (sys.corners.empty()) return;
  const int nf = static_cast<int>(sys.ifaces.size());
  std::vector<Vec> delta(nf);
  for (int f = 0; f < nf; ++f) delta[f].assign(sys.ifaces[f].M, 0.0);
  auto Srow = [&](int f, int row, int j) {
    return sys.basis[sys.basis_off[f] + row + static_cast<long>(j) * sys.iface_K[f]];
  };
  for (const auto& grp : sys.corners) {
    double num = 0.0, den = 0.0;
    std::vector<double> values(grp.size());
    for (size_t i = 0; i < grp.size(); ++i) {
      const CornerCopy& cp = grp[i];
      double v = 0.0;
      for (int j = 0; j < sys.ifaces[cp.iface].M; ++j) v += Srow(cp.iface, cp.row, j) * st.ubar_cur[cp.iface][j];
      values[i] = v;
      num += values[i] * cp.mass;
      den += cp.mass;
    }
    const double mean = den > 0.0 ? num / den : 0.0;
    for (size_t i = 0; i < grp.size(); ++i) {
      const CornerCopy& cp = grp[i];
      for (int j = 0; j < sys.ifaces[cp.iface].M; ++j)
        delta[cp.iface][j] += Srow(cp.iface, cp.row, j) * (mean - values[i]);
    }
  }
  for (int f = 0; f < nf; ++f) {
    double mx = 0.0;
    for (double v : delta[f]) mx = std::max(mx, std::abs(v));
    if (mx == 0.0) continue;
    const Iface& cf = sys.ifaces[f];
    for (int j = 0; j < cf.M; ++j) st.ubar_cur[f][j] += delta[f][j];
    const int oi = sys.off(cf.ci, cf.li);
    for (int j = 0; j < cf.M; ++j) st.u_cur[cf.ci][oi + j] = st.ubar_cur[f][j];
    if (cf.cj >= 0) {
      const int oj = sys.off(cf.cj, cf.lj);
      for (int j = 0; j < cf.M; ++j) st.u_cur[cf.cj][oj + j] = st.ubar_cur[f][j];
    }
  }
}

// sample() of run_simulation (msolver.cpp:405-411) for receiver r.
double sample_one(const System& sys, const State& st, int r) {
  double v = 0.0;
  for (int t = sys.rcv_ptr[r]; t < sys.rcv_ptr[r + 1]; ++t) {
    const int f = sys.term_iface[t];
    const double* q = sys.term_q.data() + sys.term_qoff[t];
    double d = 0.0;
    for (int i = 0; i < sys.ifaces[f].M; ++i) d += q[i] * st.ubar_cur[f][i];
    v += d;
  }
  return v;
}

// ---------------- FlatOps (msolver.cpp:233-345) for estimate_dt / energy ----
struct FlatOps {
  const System& sys;
  long n = 0;
  explicit FlatOps(const System& s) : sys(s) {
    for (const auto& f : sys.ifaces) n += f.M;
    for (const auto& c : sys.cells) n += static_cast<long>(c.m - 1) * c.kt;
  }
  std::vector<Vec> cells_of(const Vec& x) const {
    std::vector<Vec> u;
    for (const auto& c : sys.cells) u.emplace_back(static_cast<size_t>(c.m) * c.kt, 0.0);
    long off = 0;
    for (size_t f = 0; f < sys.ifaces.size(); ++f) {
      const Iface& cf = sys.ifaces[f];
      for (int i = 0; i < cf.M; ++i) u[cf.ci][sys.off(cf.ci, cf.li) + i] = x[off + i];
      if (cf.cj >= 0)
        for (int i = 0; i < cf.M; ++i) u[cf.cj][sys.off(cf.cj, cf.lj) + i] = x[off + i];
      off += cf.M;
    }
    for (size_t c = 0; c < sys.cells.size(); ++c) {
      const long tail = static_cast<long>(sys.cells[c].m - 1) * sys.cells[c].kt;
      for (long i = 0; i < tail; ++i) u[c][sys.cells[c].kt + i] = x[off + i];
      off += tail;
    }
    return u;
  }
  Vec acc(const Vec& x) const {
    const std::vector<Vec> u = cells_of(x);
    Vec out(n, 0.0);
    std::vector<Vec> flux(sys.cells.size());
    for (size_t c = 0; c < sys.cells.size(); ++c) flux[c] = first_layer_flux(sys.cells[c], u[c]);
    long off = 0;
    for (const auto& cf : sys.ifaces) {
      Vec phi(cf.M);
      for (int i = 0; i < cf.M; ++i) phi[i] = flux[cf.ci][sys.off(cf.ci, cf.li) + i];
      if (cf.cj >= 0)
        for (int i = 0; i < cf.M; ++i) phi[i] += flux[cf.cj][sys.off(cf.cj, cf.lj) + i];
      gemv(cf.mass.data(), cf.M, phi.data(), out.data() + off);
      off += cf.M;
    }
    for (size_t c = 0; c < sys.cells.size(); ++c) {
      const Vec a = interior_accelerations(sys.cells[c], u[c]);
      const long tail = static_cast<long>(sys.cells[c].m - 1) * sys.cells[c].kt;
      for (long i = 0; i < tail; ++i) out[off + i] = a[sys.cells[c].kt + i];
      off += tail;
    }
    return out;
  }
  Vec force(const Vec& x) const {
    const std::vector<Vec> u = cells_of(x);
    Vec out(n, 0.0);
    std::vector<Vec> flux(sys.cells.size());
    for (size_t c = 0; c < sys.cells.size(); ++c) flux[c] = first_layer_flux(sys.cells[c], u[c]);
    long off = 0;
    for (const auto& cf : sys.ifaces) {
      for (int i = 0; i < cf.M; ++i) out[off + i] = flux[cf.ci][sys.off(cf.ci, cf.li) + i];
      if (cf.cj >= 0)
        for (int i = 0; i < cf.M; ++i) out[off + i] += flux[cf.cj][sys.off(cf.cj, cf.lj) + i];
      off += cf.M;
    }
    for (size_t c = 0; c < sys.cells.size(); ++c) {
      const Cell& r = sys.cells[c];
      const int kt = r.kt;
      Vec d(kt), t1(kt), t2(kt);
      for (int k = 2; k <= r.m; ++k) {
        const double* uk = u[c].data() + static_cast<size_t>(k - 1) * kt;
        const double* ukm = u[c].data() + static_cast<size_t>(k - 2) * kt;
        for (int i = 0; i < kt; ++i) d[i] = uk[i] - ukm[i];
        gemv(r.L(k - 2), kt, d.data(), t1.data());
        if (k < r.m) {
          const double* ukp = u[c].data() + static_cast<size_t>(k) * kt;
          for (int i = 0; i < kt; ++i) d[i] = ukp[i] - uk[i];
        } else {
          for (int i = 0; i < kt; ++i) d[i] = -uk[i];
        }
        gemv(r.L(k - 1), kt, d.data(), t2.data());
        for (int i = 0; i < kt; ++i) out[off + i] = -t1[i] + t2[i];
        off += kt;
      }
    }
    return out;
  }
  Vec mass_apply(const Vec& x) const {
    Vec out(n, 0.0);
    long off = 0;
    for (const auto& cf : sys.ifaces) {
      gemv(cf.mass_form.data(), cf.M, x.data() + off, out.data() + off);
      off += cf.M;
    }
    for (const auto& r : sys.cells) {
      for (int k = 2; k <= r.m; ++k) {
        spd_solve(r.Lhat(k - 1), r.kt, x.data() + off, out.data() + off);
        off += r.kt;
      }
    }
    return out;
  }
  Vec flatten(const std::vector<Vec>& u_cells, const std::vector<Vec>& ubar) const {
    Vec x(n, 0.0);
    long off = 0;
    for (size_t f = 0; f < sys.ifaces.size(); ++f) {
      for (int i = 0; i < sys.ifaces[f].M; ++i) x[off + i] = ubar[f][i];
      off += sys.ifaces[f].M;
    }
    for (size_t c = 0; c < sys.cells.size(); ++c) {
      const long tail = static_cast<long>(sys.cells[c].m - 1) * sys.cells[c].kt;
      for (long i = 0; i < tail; ++i) x[off + i] = u_cells[c][sys.cells[c].kt + i];
      off += tail;
    }
    return x;
  }
};

double dot(const Vec& a, const Vec& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

// estimate_dt (msolver.cpp:349-385)
double estimate_dt(const System& sys, double safety) {
  FlatOps ops(sys);
  Vec x(ops.n);
  for (long i = 0; i < ops.n; ++i) x[i] = std::sin(1.3 * static_cast<double>(i) + 0.7) + 1e-3;
  double nrm = std::sqrt(dot(x, x));
  for (double& v : x) v /= nrm;
  double lambda = 0.0;
  bool converged = false;
  for (int it = 0; it < 500; ++it) {
    Vec y = ops.acc(x);
    for (double& v : y) v = -v;
    const double next = dot(x, y);
    const double delta = std::abs(next - lambda);
    lambda = next;
    const double norm = std::sqrt(dot(y, y));
    if (norm == 0.0) break;
    for (long i = 0; i < ops.n; ++i) x[i] = y[i] / norm;
    if (it > 16 && delta <= 1e-8 * std::abs(lambda)) {
      converged = true;
      break;
    }
  }
  if (!converged || !(lambda > 0.0)) {
    double bound = 0.0;
    std::vector<double> rowsum(ops.n, 0.0);
    Vec e(ops.n, 0.0);
    for (long j = 0; j < ops.n; ++j) {
      std::fill(e.begin(), e.end(), 0.0);
      e[j] = 1.0;
      const Vec col = ops.acc(e);
      for (long i = 0; i < ops.n; ++i) rowsum[i] += std::abs(col[i]);
    }
    for (double r : rowsum) bound = std::max(bound, r);
    lambda = std::max(lambda, bound);
    if (!(lambda > 0.0)) throw NumericalError("estimate_dt: could not bound the spectrum");
  }
  return safety * 2.0 / std::sqrt(lambda);
}

// energy (msolver.cpp:387-395)
double energy_one(const System& sys, const State& st, double dt) {
  FlatOps ops(sys);
  const Vec xc = ops.flatten(st.u_cur, st.ubar_cur);
  const Vec xp = ops.flatten(st.u_prev, st.ubar_prev);
  Vec d(ops.n);
  for (long i = 0; i < ops.n; ++i) d[i] = xc[i] - xp[i];
  const double kinetic = 0.5 * dot(d, ops.mass_apply(d)) / (dt * dt);
  const double potential = -0.5 * dot(xp, ops.force(xc));
  return kinetic + potential;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    g_err.clear();
    return MSW_OK;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return MSW_CONFIG_ERROR;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return MSW_NUMERICAL_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MSW_CONFIG_ERROR;
  }
}

// ------------------------------ fine grid ---------------------------------
struct Fine {
  int nd = 0;
  int dims[3] = {1, 1, 1};
  int idims[3] = {1, 1, 1};
  double h = 1.0;
  long n = 0;
  // CSC-like storage: per row, ordered (col, val) with ascending col --
  // symmetric matrix so row == column pattern (fine_grid.cpp:58-112).
  std::vector<long> ptr;
  std::vector<long> col;
  std::vector<double> val;
  std::vector<double> B;
};

// assemble_nd (fine_grid.cpp:58-112)
void fine_assemble(Fine& F, int nd, const int* dims, double h, const double* sigma,
                   const double* rho) {
  if (nd < 1 || nd > 3) throw ConfigError("medium must have 1-3 axes");
  if (h <= 0.0) throw ConfigError("grid step h must be positive");
  F.nd = nd;
  F.h = h;
  long nfull = 1;
  F.n = 1;
  for (int a = 0; a < nd; ++a) {
    if (dims[a] < 3) throw ConfigError("every axis needs at least 3 nodes (no interior otherwise)");
    F.dims[a] = dims[a];
    F.idims[a] = dims[a] - 2;
    F.n *= F.idims[a];
    nfull *= dims[a];
  }
  for (long g = 0; g < nfull; ++g) {
    if (sigma[g] < 0.0) throw ConfigError("sigma must be nonnegative");
    if (rho[g] <= 0.0) throw ConfigError("rho must be strictly positive");
  }
  const double inv_h2 = 1.0 / (h * h);
  auto node_id = [&](const int* c) {
    long id = 0;
    for (int a = 0; a < nd; ++a) id = id * F.dims[a] + c[a];
    return id;
  };
  F.B.assign(F.n, 0.0);
  F.ptr.assign(F.n + 1, 0);
  F.col.clear();
  F.val.clear();
  int c[3] = {0, 0, 0};
  for (long row = 0; row < F.n; ++row) {
    long r = row;
    for (int a = nd - 1; a >= 0; --a) {
      c[a] = 1 + static_cast<int>(r % F.idims[a]);
      r /= F.idims[a];
    }
    const long gid = node_id(c);
    F.B[row] = rho[gid];
    double diag = 0.0;
    std::vector<std::pair<long, double>> ents;
    for (int a = 0; a < nd; ++a) {
      for (int dir = -1; dir <= 1; dir += 2) {
        int nb[3] = {c[0], c[1], c[2]};
        nb[a] += dir;
        const double edge = 0.5 * (sigma[gid] + sigma[node_id(nb)]);
        diag -= edge * inv_h2;
        if (nb[a] >= 1 && nb[a] <= F.dims[a] - 2) {
          long cl = 0;
          for (int b = 0; b < nd; ++b) cl = cl * F.idims[b] + (nb[b] - 1);
          ents.emplace_back(cl, edge * inv_h2);
        }
      }
    }
    ents.emplace_back(row, diag);
    std::sort(ents.begin(), ents.end());
    for (auto& e : ents) {
      F.col.push_back(e.first);
      F.val.push_back(e.second);
    }
    F.ptr[row + 1] = static_cast<long>(F.col.size());
  }
}

}  // namespace

// =============================== C API ======================================
extern "C" {

typedef struct oracle_sys* oracle_handle;

const char* oracle_last_error(void) { return g_err.c_str(); }

int oracle_create(const msw_system_desc* d, oracle_handle* out) {
  return guard([&] {
    auto* s = new System();
    try {
      assemble(*s, d);
    } catch (...) {
      delete s;
      throw;
    }
    *out = reinterpret_cast<oracle_handle>(s);
  });
}

void oracle_destroy(oracle_handle h) { delete reinterpret_cast<System*>(h); }

int oracle_get_masses(oracle_handle h, double* mass, double* mass_form) {
  return guard([&] {
    System& s = *reinterpret_cast<System*>(h);
    long off = 0;
    for (const Iface& f : s.ifaces) {
      for (int k = 0; k < f.M * f.M; ++k) {
        if (mass) mass[off + k] = f.mass[k];
        if (mass_form) mass_form[off + k] = f.mass_form[k];
      }
      off += static_cast<long>(f.M) * f.M;
    }
  });
}

int oracle_set_sources(oracle_handle h, int S, const double* gproj) {
  return guard([&] {
    System& s = *reinterpret_cast<System*>(h);
    if (S < 1) throw ConfigError("need at least one source");
    s.S = S;
    s.gproj.assign(gproj, gproj + static_cast<size_t>(s.total_io) * S);
    s.has_state = false;
  });
}

int oracle_set_receivers(oracle_handle h, int R, const int* rcv_ptr, const int* term_iface,
                         const double* term_q) {
  return guard([&] {
    System& s = *reinterpret_cast<System*>(h);
    s.R = R;
    s.rcv_ptr.assign(rcv_ptr, rcv_ptr + R + 1);
    const int nt = rcv_ptr[R];
    s.term_iface.assign(term_iface, term_iface + nt);
    s.term_qoff.assign(nt, 0);
    long off = 0;
    for (int t = 0; t < nt; ++t) {
      s.term_qoff[t] = off;
      off += s.ifaces[term_iface[t]].M;
    }
    s.term_q.assign(term_q, term_q + off);
  });
}

int oracle_set_corners(oracle_handle h, int n_groups, const int* grp_ptr, const int* copy_iface,
                       const int* copy_row, const double* copy_mass, const int* iface_K,
                       const double* basis) {
  return guard([&] {
    System& s = *reinterpret_cast<System*>(h);
    s.corners.assign(n_groups, {});
    for (int g = 0; g < n_groups; ++g)
      for (int p = grp_ptr[g]; p < grp_ptr[g + 1]; ++p)
        s.corners[g].push_back(CornerCopy{copy_iface[p], copy_row[p], copy_mass[p]});
    const int nf = static_cast<int>(s.ifaces.size());
    s.iface_K.assign(iface_K, iface_K + nf);
    s.basis_off.assign(nf, 0);
    long off = 0;
    for (int f = 0; f < nf; ++f) {
      s.basis_off[f] = off;
      off += static_cast<long>(iface_K[f]) * s.ifaces[f].M;
    }
    s.basis.assign(basis, basis + off);
  });
}

int oracle_make_state(oracle_handle h, double dt) {
  return guard([&] { make_state(*reinterpret_cast<System*>(h), dt); });
}

int oracle_step(oracle_handle h, const double* source_values, int w_stride) {
  return guard([&] {
    System& s = *reinterpret_cast<System*>(h);
    if (!s.has_state) throw ConfigError("no state: call make_state");
    double amp = 0.0;
    for (int src = 0; src < s.S; ++src) {
      const double w = source_values[w_stride > 1 ? src : 0];
      amp = std::max(amp, step_one(s, s.st[src], s.gproj.data() + src, s.S, w, s.dt));
    }
    s.t += s.dt;
    ++s.step_index;
    if (unstable(amp))
      throw NumericalError("multiscale step: instability at step " + std::to_string(s.step_index));
  });
}

int oracle_corner_correct(oracle_handle h) {
  return guard([&] {
    System& s = *reinterpret_cast<System*>(h);
    for (State& st : s.st) corner_correct_one(s, st);
  });
}

// Layout [rows][S] (source fastest), as msw_get_state.
int oracle_get_state(oracle_handle h, double* u_cur, double* u_prev, double* ubar_cur,
                     double* ubar_prev, double* t, int64_t* step_index) {
  return guard([&] {
    System& s = *reinterpret_cast<System*>(h);
    if (!s.has_state) throw ConfigError("no state");
    const int S = s.S;
    for (int src = 0; src < S; ++src) {
      const State& st = s.st[src];
      long row = 0;
      for (size_t c = 0; c < s.cells.size(); ++c)
        for (size_t i = 0; i < st.u_cur[c].size(); ++i, ++row) {
          if (u_cur) u_cur[row * S + src] = st.u_cur[c][i];
          if (u_prev) u_prev[row * S + src] = st.u_prev[c][i];
        }
      row = 0;
      for (size_t f = 0; f < s.ifaces.size(); ++f)
        for (size_t i = 0; i < st.ubar_cur[f].size(); ++i, ++row) {
          if (ubar_cur) ubar_cur[row * S + src] = st.ubar_cur[f][i];
          if (ubar_prev) ubar_prev[row * S + src] = st.ubar_prev[f][i];
        }
    }
    if (t) *t = s.t;
    if (step_index) *step_index = s.step_index;
  });
}

int oracle_set_state(oracle_handle h, const double* u_cur, const double* u_prev,
                     const double* ubar_cur, const double* ubar_prev, double t,
                     int64_t step_index) {
  return guard([&] {
    System& s = *reinterpret_cast<System*>(h);
    if (!s.has_state) throw ConfigError("no state");
    const int S = s.S;
    for (int src = 0; src < S; ++src) {
      State& st = s.st[src];
      long row = 0;
      for (size_t c = 0; c < s.cells.size(); ++c)
        for (size_t i = 0; i < st.u_cur[c].size(); ++i, ++row) {
          st.u_cur[c][i] = u_cur[row * S + src];
          st.u_prev[c][i] = u_prev[row * S + src];
        }
      row = 0;
      for (size_t f = 0; f < s.ifaces.size(); ++f)
        for (size_t i = 0; i < st.ubar_cur[f].size(); ++i, ++row) {
          st.ubar_cur[f][i] = ubar_cur[row * S + src];
          st.ubar_prev[f][i] = ubar_prev[row * S + src];
        }
      // conjugation invariant: layer-1 blocks mirror ubar
      for (size_t f = 0; f < s.ifaces.size(); ++f) {
        const Iface& cf = s.ifaces[f];
        for (int i = 0; i < cf.M; ++i) {
          st.u_cur[cf.ci][s.off(cf.ci, cf.li) + i] = st.ubar_cur[f][i];
          st.u_prev[cf.ci][s.off(cf.ci, cf.li) + i] = st.ubar_prev[f][i];
          if (cf.cj >= 0) {
            st.u_cur[cf.cj][s.off(cf.cj, cf.lj) + i] = st.ubar_cur[f][i];
            st.u_prev[cf.cj][s.off(cf.cj, cf.lj) + i] = st.ubar_prev[f][i];
          }
        }
      }
    }
    s.t = t;
    s.step_index = step_index;
  });
}

// run_simulation loop (msolver.cpp:405-422) from the current state, with
// precomputed wavelet samples w[n * w_stride (+ s)].  Sources are
// independent single-source runs (the reference API is single-source);
// nthreads > 1 parallelises over sources (timing variant only).
int oracle_run(oracle_handle h, int64_t steps, const double* w, int w_stride,
               int corner_correction, double* traces, double* times, int64_t* bad_step,
               int nthreads) {
  return guard([&] {
    System& s = *reinterpret_cast<System*>(h);
    if (!s.has_state) throw ConfigError("no state: call make_state");
    const int S = s.S, R = s.R;
    std::vector<int64_t> bad(S, 0);
    const double t0 = s.t;
    const long si0 = s.step_index;
    if (times) {
      double t = t0;
      times[0] = t;
      for (int64_t n = 0; n < steps; ++n) {
        t += s.dt;
        times[n + 1] = t;
      }
    }
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int src = 0; src < S; ++src) {
      State& st = s.st[src];
      for (int r = 0; r < R; ++r) traces[static_cast<size_t>(r) * S + src] = sample_one(s, st, r);
      for (int64_t n = 0; n < steps; ++n) {
        const double amp =
            step_one(s, st, s.gproj.data() + src, S, w[n * w_stride + (w_stride > 1 ? src : 0)], s.dt);
        if (unstable(amp) && bad[src] == 0) bad[src] = si0 + n + 1;
        if (corner_correction) corner_correct_one(s, st);
        for (int r = 0; r < R; ++r)
          traces[(static_cast<size_t>(n + 1) * R + r) * S + src] = sample_one(s, st, r);
        if (bad[src]) break;
      }
    }
    int64_t first = 0;
    for (int64_t b : bad)
      if (b && (first == 0 || b < first)) first = b;
    double t = t0;
    for (int64_t n = 0; n < steps; ++n) t += s.dt;
    s.t = t;
    s.step_index = si0 + steps;
    if (bad_step) *bad_step = first;
    if (first)
      throw NumericalError("multiscale step: instability at step " + std::to_string(first));
  });
}

int oracle_estimate_dt(oracle_handle h, double safety, double* dt_out) {
  return guard([&] { *dt_out = estimate_dt(*reinterpret_cast<System*>(h), safety); });
}

// energy per source (msolver.cpp:387-395)
int oracle_energy(oracle_handle h, double* e_out) {
  return guard([&] {
    System& s = *reinterpret_cast<System*>(h);
    if (!s.has_state) throw ConfigError("no state");
    for (int src = 0; src < s.S; ++src) e_out[src] = energy_one(s, s.st[src], s.dt);
  });
}

// Wavelet::operator() (wavelet.cpp:9-19), kind 0 = GaussianDerivative,
// 1 = Gaussian, 2 = Ricker (extension: (1 - x^2) exp(-x^2/2), absent in the
// reference, wavelet.hpp:12).
double oracle_wavelet(int kind, double omega_cut, double width_factor, double delay_factor,
                      double t) {
  const double tau = width_factor / omega_cut;
  const double x = (t - delay_factor * tau) / tau;
  switch (kind) {
    case 0: return -x * std::exp(0.5 - 0.5 * x * x);
    case 1: return std::exp(-0.5 * x * x);
    case 2: return (1.0 - x * x) * std::exp(-0.5 * x * x);
  }
  return 0.0;
}

// ------------------------------- fine grid ----------------------------------
typedef struct oracle_fine* oracle_fine_handle;

int oracle_fine_create(int nd, const int* dims, double h, const double* sigma, const double* rho,
                       oracle_fine_handle* out) {
  return guard([&] {
    auto* F = new Fine();
    try {
      fine_assemble(*F, nd, dims, h, sigma, rho);
    } catch (...) {
      delete F;
      throw;
    }
    *out = reinterpret_cast<oracle_fine_handle>(F);
  });
}

// Generic pencil (A given as symmetric CSR with ascending columns, B diag).
int oracle_fine_create_csr(int64_t n, const int64_t* ptr, const int64_t* col, const double* val,
                           const double* B, oracle_fine_handle* out) {
  return guard([&] {
    auto* F = new Fine();
    F->n = n;
    F->ptr.assign(ptr, ptr + n + 1);
    F->col.assign(col, col + ptr[n]);
    F->val.assign(val, val + ptr[n]);
    F->B.assign(B, B + n);
    *out = reinterpret_cast<oracle_fine_handle>(F);
  });
}

void oracle_fine_destroy(oracle_fine_handle f) { delete reinterpret_cast<Fine*>(f); }

int64_t oracle_fine_size(oracle_fine_handle f) { return reinterpret_cast<Fine*>(f)->n; }

// Export the assembled pencil (CSR, ascending columns) for inspection.
int oracle_fine_export(oracle_fine_handle f, int64_t* ptr, int64_t* col, double* val, double* B) {
  return guard([&] {
    const Fine& F = *reinterpret_cast<Fine*>(f);
    if (ptr) std::copy(F.ptr.begin(), F.ptr.end(), ptr);
    if (col) std::copy(F.col.begin(), F.col.end(), col);
    if (val) std::copy(F.val.begin(), F.val.end(), val);
    if (B) std::copy(F.B.begin(), F.B.end(), B);
  });
}

int64_t oracle_fine_nnz(oracle_fine_handle f) { return reinterpret_cast<Fine*>(f)->ptr.back(); }

// y = A x in Eigen's col-major order: column j ascending, y_i += a_ij x_j.
// A is symmetric, so row i's entries (ascending column) are exactly the
// column-order contributions to y_i.
static void fine_spmv(const Fine& F, const double* x, double* y) {
  for (long i = 0; i < F.n; ++i) {
    double s = 0.0;
    for (long p = F.ptr[i]; p < F.ptr[i + 1]; ++p) s += F.val[p] * x[F.col[p]];
    y[i] = s;
  }
}

// fine_cfl (reference.cpp:24-47)
int oracle_fine_cfl(oracle_fine_handle f, double* dt_out) {
  return guard([&] {
    const Fine& F = *reinterpret_cast<Fine*>(f);
    const long n = F.n;
    Vec x(n), y(n);
    for (long i = 0; i < n; ++i) x[i] = std::sin(0.7 * static_cast<double>(i) + 0.3) + 1e-3;
    double nrm = std::sqrt(dot(x, x));
    for (double& v : x) v /= nrm;
    double lambda = 0.0;
    for (int it = 0; it < 5000; ++it) {
      fine_spmv(F, x.data(), y.data());
      for (long i = 0; i < n; ++i) y[i] = -y[i] / F.B[i];
      const double next = dot(x, y);
      const double delta = std::abs(next - lambda);
      lambda = next;
      const double norm = std::sqrt(dot(y, y));
      if (norm == 0.0) break;
      for (long i = 0; i < n; ++i) x[i] = y[i] / norm;
      if (it > 32 && delta <= 1e-7 * std::abs(lambda)) break;
    }
    if (!(lambda > 0.0)) {
      double bound = 0.0;
      for (long i = 0; i < n; ++i) {
        double ra = 0.0;
        for (long p = F.ptr[i]; p < F.ptr[i + 1]; ++p) ra += std::abs(F.val[p]);
        bound = std::max(bound, ra / F.B[i]);
      }
      lambda = bound;
    }
    if (!(lambda > 0.0)) throw NumericalError("fine_cfl: could not bound the spectrum");
    *dt_out = 2.0 / std::sqrt(lambda);
  });
}

// fine_leapfrog (reference.cpp:49-80) for S sources (independent runs) and
// R receivers; sparse g/q as CSR over interior rows.  t_s = s*dt.
int oracle_fine_leapfrog(oracle_fine_handle f, int S, const int* src_ptr, const int64_t* src_row,
                         const double* src_val, int R, const int* rcv_ptr, const int64_t* rcv_row,
                         const double* rcv_val, double dt, int64_t steps, const double* w,
                         int w_stride, double* traces, int64_t* bad_step, int nthreads) {
  return guard([&] {
    const Fine& F = *reinterpret_cast<Fine*>(f);
    if (dt <= 0.0) throw ConfigError("fine_leapfrog: dt must be positive");
    const long n = F.n;
    std::vector<int64_t> bad(S, 0);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int src = 0; src < S; ++src) {
      Vec u(n, 0.0), up(n, 0.0), un(n), g(n, 0.0), rhs(n);
      for (int p = src_ptr[src]; p < src_ptr[src + 1]; ++p) g[src_row[p]] = src_val[p];
      auto sample = [&](int64_t step) {
        for (int r = 0; r < R; ++r) {
          // q.dot(u) over the full vector == sum over q's support in
          // ascending row order (zeros elsewhere contribute exact zeros)
          double v = 0.0;
          for (int p = rcv_ptr[r]; p < rcv_ptr[r + 1]; ++p) v += rcv_val[p] * u[rcv_row[p]];
          traces[(static_cast<size_t>(step) * R + r) * S + src] = v;
        }
      };
      sample(0);
      for (int64_t s = 0; s < steps; ++s) {
        const double ws = w[s * w_stride + (w_stride > 1 ? src : 0)];
        fine_spmv(F, u.data(), rhs.data());
        for (long i = 0; i < n; ++i) rhs[i] = rhs[i] + ws * g[i];
        for (long i = 0; i < n; ++i) rhs[i] /= F.B[i];
        const double dt2 = dt * dt;
        double amp = 0.0;
        for (long i = 0; i < n; ++i) {
          un[i] = 2.0 * u[i] - up[i] + dt2 * rhs[i];
          const double a = std::abs(un[i]);
          if (std::isnan(a)) amp = std::numeric_limits<double>::infinity();
          else amp = std::max(amp, a);
        }
        up.swap(u);
        u.swap(un);
        if (!std::isfinite(amp) || amp > 1e12) {
          bad[src] = s + 1;
          sample(s + 1);
          break;
        }
        sample(s + 1);
      }
    }
    int64_t first = 0;
    for (int64_t b : bad)
      if (b && (first == 0 || b < first)) first = b;
    if (bad_step) *bad_step = first;
    if (first) throw NumericalError("fine_leapfrog: instability at step " + std::to_string(first));
  });
}

// compare_traces (trace_io.cpp:36-67): a_t/a_v (na), b_t/b_v (nb).
int oracle_compare_traces(const double* at, const double* av, int64_t na, const double* bt,
                          const double* bv, int64_t nb, double* max_abs, double* rel_l2) {
  return guard([&] {
    if (na == 0 || nb == 0) throw ConfigError("cannot compare empty traces");
    auto sample_b = [&](double t) {
      if (t <= bt[0]) return bv[0];
      if (t >= bt[nb - 1]) return bv[nb - 1];
      const double* it = std::upper_bound(bt, bt + nb, t);
      const long hi = it - bt;
      const long lo = hi - 1;
      const double w = (t - bt[lo]) / (bt[hi] - bt[lo]);
      return (1.0 - w) * bv[lo] + w * bv[hi];
    };
    double num2 = 0.0, den2 = 0.0, mx = 0.0;
    const double t_end = std::min(at[na - 1], bt[nb - 1]);
    for (int64_t i = 0; i < na; ++i) {
      if (at[i] > t_end + 1e-12) break;
      const double b = sample_b(at[i]);
      const double d = av[i] - b;
      mx = std::max(mx, std::abs(d));
      num2 += d * d;
      den2 += b * b;
    }
    *max_abs = mx;
    *rel_l2 = den2 > 0.0 ? std::sqrt(num2 / den2) : std::sqrt(num2);
  });
}

}  // extern "C"
