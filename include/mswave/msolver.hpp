// mswave/msolver.hpp -- B200 drop-in for proj/include/mswave/msolver.hpp.
//
// Same types and free functions as the reference (msolver.hpp:16-91).  The
// coupled system is uploaded once to device-resident storage on first use
// (MultiscaleSystem::device, an addition); step/run_simulation/corner_correct
// run as sm_100a kernels through the C ABI in mswave_b200.h.
//
// WaveState stays a host-visible struct as in the reference: step() and
// corner_correct() upload it, advance on the device and download it again,
// so callers may read or edit it between steps.  For
// throughput use run_simulation (or the batched run_simulation_batched),
// which keeps the state on the device for the whole loop.
#ifndef MSWAVE_MSOLVER_HPP
#define MSWAVE_MSOLVER_HPP

#include <memory>
#include <vector>

#include "mswave/partition.hpp"
#include "mswave/reference.hpp"
#include "mswave/romgen.hpp"
#include "mswave/types.hpp"
#include "mswave/wavelet.hpp"

namespace mswave {

struct CoupledInterface {
  int part_iface = -1;
  int ci = -1, cj = -1;
  int li = -1, lj = -1;
  int size = 0;
  Mat S;
  Mat mass;
  Mat mass_form;
  Vec g_proj, q_proj;
};

struct CornerGroup {
  struct Copy {
    int iface = -1;
    int row = -1;
    double mass = 0.0;
  };
  long parent = -1;
  std::vector<Copy> copies;
};

namespace detail {
struct DeviceSystem;  // owns the msw_handle
}

struct MultiscaleSystem {
  std::vector<SubdomainROM> roms;
  std::vector<CoupledInterface> ifaces;
  std::vector<CornerGroup> corners;

  int total_reduced_io() const;
  long reduced_dof() const;
  long flops_per_step() const;
};

// B200 addition: the device-resident copy of a system is created on first
// use and kept in a small library-side cache (MultiscaleSystem keeps the
// reference's layout); call invalidate_device(system) after editing the
// roms / interfaces / corners of a system that has already run in place.
void invalidate_device(const MultiscaleSystem& system);

MultiscaleSystem assemble_system(const Partition& partition, const BoundaryBasis& basis,
                                 std::vector<SubdomainROM> roms, const Vec& B_diag);

struct WaveState {
  std::vector<Vec> u_cur, u_prev;
  std::vector<Vec> ubar_cur, ubar_prev;
  double t = 0.0;
  double dt = 0.0;
  long step_index = 0;
};

WaveState make_state(const MultiscaleSystem& system, double dt);

void step(const MultiscaleSystem& system, WaveState& state, double source_value);

void corner_correct(const MultiscaleSystem& system, WaveState& state);

// msolver.hpp:75 / :78 -- evaluated on the device (msw_estimate_dt / msw_energy)
double estimate_dt(const MultiscaleSystem& system, double safety = 0.9);

double energy(const MultiscaleSystem& system, const WaveState& state);

struct RunResult {
  Trace trace;
  std::vector<double> energy_times, energy_values;
  long steps = 0;
};

RunResult run_simulation(const MultiscaleSystem& system, const Wavelet& wavelet, double t_final,
                         double dt, bool corner_correction = false, long energy_stride = 0);

// Batched extension: S sources (g_proj per source, [sum_f M_f] each) and
// R receivers (q_proj per receiver) in one device pass.  traces[r][s].
std::vector<std::vector<Trace>> run_simulation_batched(
    const MultiscaleSystem& system, const std::vector<std::vector<Vec>>& g_proj_per_source,
    const std::vector<std::vector<Vec>>& q_proj_per_receiver, const Wavelet& wavelet,
    double t_final, double dt, bool corner_correction = false);

}  // namespace mswave

#endif  // MSWAVE_MSOLVER_HPP
