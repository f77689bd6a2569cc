// C++ drop-in check: the reference's own test cases (proj/tests/
// test_msolver.cpp, test_reference.cpp), written against the mirrored
// mswave:: API and linked to libmswave_b200.so -- what a reference user's
// code compiles to after switching libraries.  Needs a GPU; run by
// tests/test_cpp_mirror.py.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "mswave/msolver.hpp"
#include "mswave/trace_io.hpp"

using namespace mswave;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    if (cond) ++g_pass;                                                          \
    else {                                                                       \
      ++g_fail;                                                                  \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);                \
    }                                                                            \
  } while (0)
#define APPROX(a, b, rel) (std::abs((a) - (b)) <= (rel) * std::max(1.0, std::abs(b)) + 1e-300)

// test_helpers.hpp:48-76
static MultiscaleSystem scalar_oscillator(double lhat, double lmain) {
  SubdomainROM rom;
  rom.cell = 0;
  rom.m = 1;
  rom.ktilde = 1;
  rom.shift = -1.0;
  rom.iface_ids = {0};
  rom.iface_offsets = {0, 1};
  rom.ladder_hat = {Mat::Constant(1, 1, lhat)};
  rom.ladder = {Mat::Constant(1, 1, lmain)};
  rom.g_proj = {Vec::Ones(1)};
  rom.q_proj = {Vec::Ones(1)};
  CoupledInterface cf;
  cf.part_iface = 0;
  cf.ci = 0;
  cf.li = 0;
  cf.size = 1;
  cf.S = Mat::Identity(1, 1);
  cf.mass_form = Mat::Constant(1, 1, 1.0 / lhat);
  cf.mass = Mat::Constant(1, 1, lhat);
  cf.g_proj = Vec::Ones(1);
  cf.q_proj = Vec::Ones(1);
  MultiscaleSystem sys;
  sys.roms.push_back(rom);
  sys.ifaces.push_back(cf);
  return sys;
}

static void test_single_cell() {  // test_msolver.cpp:51-60
  MultiscaleSystem sys = scalar_oscillator(1.0, 4.0);
  WaveState st = make_state(sys, 0.1);
  st.ubar_cur[0][0] = st.ubar_prev[0][0] = 0.3;
  st.u_cur[0][0] = st.u_prev[0][0] = 0.3;
  step(sys, st, 0.0);
  CHECK(APPROX(st.ubar_cur[0][0], 0.3 + 0.01 * (-4.0 * 0.3), 1e-14));
  CHECK(st.u_cur[0][0] == st.ubar_cur[0][0]);
  CHECK(st.step_index == 1);
}

static void test_dispersion() {  // test_msolver.cpp:72-85
  MultiscaleSystem sys = scalar_oscillator(1.0, 4.0);
  const double dt = 0.2;
  WaveState st = make_state(sys, dt);
  step(sys, st, 1.0 / dt);
  CHECK(APPROX(st.ubar_cur[0][0], dt, 1e-14));
  const double wt = 2.0 / dt * std::asin(0.5 * 2.0 * dt);
  for (int n = 2; n <= 50; ++n) {
    step(sys, st, 0.0);
    const double expect = dt * std::sin(n * wt * dt) / std::sin(wt * dt);
    CHECK(APPROX(st.ubar_cur[0][0], expect, 1e-10));
  }
}

static void test_run_simulation() {
  // the same oscillator driven through run_simulation with an impulse-like
  // Gaussian; compare against step() by step()
  MultiscaleSystem sys = scalar_oscillator(1.0, 4.0);
  Wavelet w;
  w.kind = Wavelet::Kind::Ricker;
  w.omega_cut = 3.0;
  const double dt = 0.05;
  RunResult rr = run_simulation(sys, w, 10.0, dt);
  WaveState st = make_state(sys, dt);
  double err = 0.0;
  for (long s = 0; s < rr.steps; ++s) {
    step(sys, st, w(st.t));
    err = std::max(err, std::abs(st.ubar_cur[0][0] - rr.trace.values[s + 1]));
    CHECK(rr.trace.times[s + 1] == st.t);
  }
  CHECK(rr.trace.values.size() == static_cast<size_t>(rr.steps + 1));
  CHECK(err < 1e-13);
  Trace a = rr.trace, b = rr.trace;
  CHECK(compare_traces(a, b).rel_l2_error == 0.0);
}

static void test_estimate_dt_and_energy() {
  // test_msolver.cpp:51-60: estimate_dt(scalar_oscillator(1, 4), 1.0) == 1.0
  MultiscaleSystem sys = scalar_oscillator(1.0, 4.0);
  CHECK(APPROX(estimate_dt(sys, 1.0), 1.0, 1e-6));
  // energy_stride (msolver.cpp:415-420): same trace as without, energy
  // constant once the wavelet has died out
  Wavelet w;
  w.omega_cut = 3.0;
  const double dt = 0.05;
  RunResult a = run_simulation(sys, w, 40.0, dt);
  RunResult b = run_simulation(sys, w, 40.0, dt, false, 25);
  CHECK(a.trace.values == b.trace.values);
  CHECK(a.trace.times == b.trace.times);
  CHECK(b.energy_values.size() == static_cast<size_t>(a.steps / 25));
  CHECK(b.energy_times.size() == b.energy_values.size() && b.energy_times[0] == a.trace.times[25]);
  const double e_late = b.energy_values.back();
  CHECK(e_late > 0.0 && APPROX(b.energy_values[b.energy_values.size() - 2], e_late, 1e-9 * e_late));
  WaveState st = make_state(sys, dt);
  st.ubar_cur[0][0] = st.u_cur[0][0] = 0.3;
  st.ubar_prev[0][0] = st.u_prev[0][0] = 0.25;
  // 1x1 form: 0.5 (0.05)^2 (1/lhat) / dt^2 - 0.5 * 0.25 * (1/lhat) acc, acc = -4 * 0.3
  const double expect = 0.5 * 0.05 * 0.05 / (dt * dt) - 0.5 * 0.25 * (-4.0 * 0.3);
  CHECK(APPROX(energy(sys, st), expect, 1e-12));
}

static void test_instability() {  // test_msolver.cpp:416-426
  MultiscaleSystem sys = scalar_oscillator(1.0, 100.0);
  WaveState st = make_state(sys, 1.0);
  st.ubar_cur[0][0] = 1.0;
  st.u_cur[0][0] = 1.0;
  bool thrown = false;
  try {
    for (int s = 0; s < 200; ++s) step(sys, st, 0.0);
  } catch (const NumericalError& e) {
    thrown = std::string(e.what()).find("instability at step") != std::string::npos;
  }
  CHECK(thrown);
  bool cfg = false;
  try {
    make_state(sys, 0.0);
  } catch (const ConfigError&) {
    cfg = true;
  }
  CHECK(cfg);
}

static void test_corner_correction() {  // test_msolver.cpp:303-358
  for (int sub = 0; sub < 3; ++sub) {
    MultiscaleSystem sys;
    for (int f = 0; f < 2; ++f) {
      CoupledInterface cf;
      cf.part_iface = f;
      cf.ci = 0;
      cf.li = f;
      cf.size = 2;
      cf.S = Mat::Identity(2, 2);
      cf.mass = cf.mass_form = Mat::Identity(2, 2);
      cf.g_proj = cf.q_proj = Vec::Zero(2);
      sys.ifaces.push_back(cf);
    }
    SubdomainROM rom;
    rom.cell = 0;
    rom.m = 1;
    rom.ktilde = 4;
    rom.iface_ids = {0, 1};
    rom.iface_offsets = {0, 2, 4};
    rom.ladder = {Mat::Identity(4, 4)};
    rom.ladder_hat = {Mat::Identity(4, 4)};
    sys.roms.push_back(rom);
    CornerGroup grp;
    grp.parent = 0;
    grp.copies = {{0, 0, 1.0}, {1, 1, sub == 2 ? 3.0 : 1.0}};
    sys.corners.push_back(grp);
    WaveState st = make_state(sys, 0.1);
    if (sub == 0) {
      st.ubar_cur[0][0] = 2.5; st.ubar_cur[0][1] = 9.0;
      st.ubar_cur[1][0] = 7.0; st.ubar_cur[1][1] = 2.5;
    } else {
      st.ubar_cur[0][0] = 1.0; st.ubar_cur[0][1] = 0.0;
      st.ubar_cur[1][0] = 0.0; st.ubar_cur[1][1] = 3.0;
    }
    corner_correct(sys, st);
    if (sub == 0) {
      CHECK(st.ubar_cur[0][0] == 2.5 && st.ubar_cur[1][1] == 2.5 && st.ubar_cur[0][1] == 9.0);
    } else {
      const double e = sub == 1 ? 2.0 : 2.5;
      CHECK(APPROX(st.ubar_cur[0][0], e, 1e-14));
      CHECK(APPROX(st.ubar_cur[1][1], e, 1e-14));
    }
    CHECK(st.u_cur[0][0] == st.ubar_cur[0][0] && st.u_cur[0][3] == st.ubar_cur[1][1]);
  }
}

static void test_fine_unit_oscillator() {  // test_reference.cpp:25-48
  // dims {3}, h = 1, sigma = 0.5: one interior node, A = -1, B = 1
  GridMedium m = make_uniform_medium({3}, 1.0, 0.5);
  SparsePencil p = assemble_1d(m);
  Vec g = Vec::Ones(1), q = Vec::Ones(1);
  Wavelet w;
  w.kind = Wavelet::Kind::Gaussian;
  w.omega_cut = 350.0;
  const double tau = w.tau();
  const double amp = tau * std::sqrt(2.0 * M_PI) * std::exp(-0.5 * tau * tau);
  auto max_err = [&](double dt) {
    Trace t = fine_leapfrog(p, g, q, w, 10.0, dt);
    double e = 0.0;
    for (size_t i = 0; i < t.times.size(); ++i) {
      if (t.times[i] < w.delay() + 5.0 * tau) continue;
      e = std::max(e, std::abs(t.values[i] - amp * std::sin(t.times[i] - w.delay())));
    }
    return e / amp;
  };
  const double e1 = max_err(2e-3), e2 = max_err(1e-3);
  CHECK(e1 < 1e-4);
  CHECK(std::abs(e1 / e2 - 4.0) < 0.8);
}

static void test_fine_zero_and_instability() {  // test_reference.cpp:50-66
  GridMedium m = make_uniform_medium({9, 9}, 0.5, 1.0);
  SparsePencil p = assemble_nd(m);
  Vec g = Vec::Zero(p.n()), q = Vec::Zero(p.n());
  q[10] = 1.0;
  Wavelet w;
  Trace t = fine_leapfrog(p, g, q, w, 2.0, 0.05);
  bool zero = true;
  for (double v : t.values) zero &= v == 0.0;
  CHECK(zero);
  GridMedium m1 = make_uniform_medium({3}, 1.0, 50.0);  // A = -100
  SparsePencil p1 = assemble_1d(m1);
  bool thrown = false;
  try {
    Wavelet w10;
    w10.omega_cut = 10.0;
    fine_leapfrog(p1, Vec::Ones(1), Vec::Ones(1), w10, 50.0, 1.0);
  } catch (const NumericalError& e) {
    thrown = std::string(e.what()).find("fine_leapfrog: instability at step") != std::string::npos;
  }
  CHECK(thrown);
}

static void test_fine_cfl_known_spectra() {  // test_reference.cpp:68-85
  // 1D sigma = 1: lambda_max -> 4/h^2, dt_max -> h
  GridMedium m1 = make_uniform_medium({41}, 0.25, 1.0);
  SparsePencil p1 = assemble_1d(m1);
  const double d1 = fine_cfl(p1);
  CHECK(APPROX(d1, 0.25, 0.01));
  // scaling sigma by 4 halves the stable step
  GridMedium m4 = make_uniform_medium({41}, 0.25, 4.0);
  SparsePencil p4 = assemble_1d(m4);
  CHECK(std::abs(fine_cfl(p4) / d1 - 0.5) <= 0.01 * 0.5);
  // 2D: the reference compares with a dense eigensolve; for a uniform
  // medium the Dirichlet spectrum is known in closed form,
  // lambda_max = (4 sigma / h^2) * 2 sin^2(n pi / (2 (n + 1))), n = 19
  GridMedium m2 = make_uniform_medium({21, 21}, 0.5, 1.3);
  SparsePencil p2 = assemble_nd(m2);
  const double s = std::sin(19.0 * M_PI / 40.0);
  const double dt_exact = 2.0 / std::sqrt(4.0 * 1.3 / 0.25 * 2.0 * s * s);
  CHECK(APPROX(fine_cfl(p2), dt_exact, 0.01));
  // the matrix-free (GridMedium) path gives the same estimate
  CHECK(APPROX(fine_cfl(m2), fine_cfl(p2), 1e-6));
}

static void test_pencil_layout_and_paths() {
  // assemble_nd keeps the reference's A (fine_grid.cpp:58-112): 7-point rows,
  // diagonal = -(sum of all six edge stiffnesses incl. Dirichlet ones)
  std::vector<int> dims = {7, 6, 8};
  GridMedium m = make_uniform_medium(dims, 0.5, 1.0, 1.0);
  for (long i = 0; i < m.node_count(); ++i) {
    m.sigma[i] = 1.0 + 0.37 * std::sin(0.3 * static_cast<double>(i));
    m.rho[i] = 1.0 + 0.2 * std::cos(0.11 * static_cast<double>(i));
  }
  SparsePencil p = assemble_nd(m);
  CHECK(p.n() == 5 * 4 * 6 && p.A.cols() == p.n() && p.B.size() == p.n());
  long interior_rows = 0;
  for (long j = 0; j < p.A.outerSize(); ++j) {
    double sum = 0.0, diag = 0.0;
    int cnt = 0;
    for (SpMat::InnerIterator it(p.A, j); it; ++it) {
      ++cnt;
      if (it.row() == j) diag = it.value();
      else sum += it.value();
    }
    CHECK(diag < 0.0 && sum > 0.0 && -diag >= sum * (1.0 - 1e-14));
    if (cnt == 7) ++interior_rows;
  }
  CHECK(interior_rows == 3 * 2 * 4);
  // the pencil path (A on the device, CSR in column order) and the
  // matrix-free medium path agree bit for bit
  Vec g = Vec::Zero(p.n()), q1 = Vec::Zero(p.n()), q2 = Vec::Zero(p.n());
  g[p.node_of({3, 2, 4})] = 1.0;
  q1[p.node_of({3, 2, 4})] = 1.0;
  q2[p.node_of({4, 3, 5})] = 0.5;
  Wavelet w;
  w.omega_cut = 2.0;
  const double dt = 0.5 * fine_cfl(p);
  auto a = fine_leapfrog_batched(p, {g}, {q1, q2}, w, 20.0, dt);
  auto b = fine_leapfrog_batched(m, {g}, {q1, q2}, w, 20.0, dt);
  bool same = a.size() == 1 && b.size() == 1 && a[0].size() == 2;
  double amp = 0.0;
  for (int r = 0; r < 2 && same; ++r) {
    same = a[0][r].values.size() == b[0][r].values.size();
    for (size_t k = 0; same && k < a[0][r].values.size(); ++k) {
      same = a[0][r].values[k] == b[0][r].values[k];
      amp = std::max(amp, std::abs(a[0][r].values[k]));
    }
  }
  CHECK(same && amp > 0.0);
}

int main() {
  test_single_cell();
  test_dispersion();
  test_run_simulation();
  test_estimate_dt_and_energy();
  test_instability();
  test_corner_correction();
  test_fine_unit_oscillator();
  test_fine_zero_and_instability();
  test_fine_cfl_known_spectra();
  test_pencil_layout_and_paths();
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
