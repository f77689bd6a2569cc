// mswave/romgen.hpp -- on-line subset of proj/include/mswave/romgen.hpp: the
// off-line products the stepper consumes (BoundaryBasis :13-19,
// SubdomainROM :23-45, RomOptions :120-127).  The off-line builders stay the
// reference's host setup (BASELINE north_star).
#ifndef MSWAVE_ROMGEN_HPP
#define MSWAVE_ROMGEN_HPP

#include <vector>

#include "mswave/types.hpp"

namespace mswave {

struct BoundaryBasis {
  double omega_max = 0.0;
  double epsilon = 0.0;
  std::vector<Mat> S;          // per interface, K_ij x M_ij
  std::vector<Vec> kept_eigs;  // descending
  std::vector<double> tail;
};

struct SubdomainROM {
  int cell = -1;
  int m = 0;       // number of layers
  int ktilde = 0;  // sum of interface block sizes
  double shift = 0.0;

  std::vector<int> iface_ids;      // ascending
  std::vector<int> iface_offsets;  // block offset per interface, plus total

  std::vector<Mat> ladder_hat;  // Lhat^1..Lhat^m, SPD
  std::vector<Mat> ladder;      // L^1..L^m, SPD
  std::vector<Vec> g_proj, q_proj;

  int block_offset(int local_iface) const { return iface_offsets[local_iface]; }
  int block_size(int local_iface) const {
    return iface_offsets[local_iface + 1] - iface_offsets[local_iface];
  }
};

struct RomOptions {
  int m = 4;
  double omega_max = 2.0 * 3.14159265358979323846;
  double epsilon_rel = 1e-6;
  int max_basis_per_interface = 0;
  double shift = 0.0;
  bool full_collar = false;
};

}  // namespace mswave

#endif  // MSWAVE_ROMGEN_HPP
