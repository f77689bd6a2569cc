// mswave/romgen.hpp -- mirror of proj/include/mswave/romgen.hpp: the off-line
// products the stepper consumes, member for member (BoundaryBasis :13-19,
// SubdomainROM :23-45, TruncatedBasis, ProjectedPencil, LanczosForm,
// Ladders, RomOptions :120-127).  The off-line builders stay the reference's
// host setup (BASELINE north_star); with -DMSWAVE_USE_EIGEN their
// declarations are present for the reference's own romgen.cpp.
#ifndef MSWAVE_ROMGEN_HPP
#define MSWAVE_ROMGEN_HPP

#include <vector>

#include "mswave/partition.hpp"
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

  // off-line intermediates (romgen.hpp:32-35): filled by the reference's
  // build_rom, not archived and never read by the on-line stage
  Mat V;
  Mat Am, Bm, Sm;
  Mat T;
  Mat beta1;
  std::vector<Mat> ladder_hat;  // Lhat^1..Lhat^m, SPD
  std::vector<Mat> ladder;      // L^1..L^m, SPD
  std::vector<Vec> g_proj, q_proj;

  int block_offset(int local_iface) const { return iface_offsets[local_iface]; }
  int block_size(int local_iface) const {
    return iface_offsets[local_iface + 1] - iface_offsets[local_iface];
  }
};

struct TruncatedBasis {
  Mat S;
  Vec kept;
  double tail;
};

struct ProjectedPencil {
  Mat Am, Bm, Sm;
};

struct LanczosForm {
  Mat T;
  Mat beta1;
  Mat Qb;
};

struct Ladders {
  std::vector<Mat> hat;   // Lhat^k
  std::vector<Mat> main;  // L^k
};

struct RomOptions {
  int m = 4;
  double omega_max = 2.0 * 3.14159265358979323846;
  double epsilon_rel = 1e-6;
  int max_basis_per_interface = 0;
  double shift = 0.0;
  bool full_collar = false;
};

// g~ = S_ij^T values (romgen.cpp:359-363); ConfigError on a size mismatch
Vec project_io(const Mat& S_ij, const Vec& values_on_iface);

#ifdef MSWAVE_USE_EIGEN
// off-line ROM construction: provided by the reference's romgen.cpp
std::vector<long> local_indices(const std::vector<long>& nodes, const std::vector<long>& subset);
CMat exact_transfer(const SubdomainSplit& split, const std::vector<long>& boundary_local, Cpx w2);
Mat boundary_gramian(const SpMat& A, const Vec& B, const std::vector<long>& iface_nodes,
                     double omega_max, const std::vector<long>& collar_nodes);
TruncatedBasis truncate_basis(const Mat& G, double epsilon, int max_cols = 0);
Mat rational_krylov(const SubdomainSplit& split, const Mat& PS, double s, int m);
ProjectedPencil project_pencil(const SubdomainSplit& split, const Mat& V, const Mat& PS);
LanczosForm block_lanczos(const Mat& Am, const Mat& Bm, const Mat& Sm, int m, int ktilde);
Ladders sfraction_coeffs(const Mat& T, const Mat& beta1, int m, int ktilde);
CMat evaluate_sfraction(const std::vector<Mat>& ladder_hat, const std::vector<Mat>& ladder, Cpx w2);
Mat evaluate_sfraction_real(const std::vector<Mat>& ladder_hat, const std::vector<Mat>& ladder,
                            double w2);
inline CMat evaluate_sfraction(const SubdomainROM& rom, Cpx w2) {
  return evaluate_sfraction(rom.ladder_hat, rom.ladder, w2);
}
CMat partial_fraction_transfer(const Mat& Am, const Mat& Bm, const Mat& Sm, Cpx w2);
CMat resolvent_transfer(const Mat& T, const Mat& beta1, Cpx w2);
BoundaryBasis build_boundary_basis(const SparsePencil& pencil, const Partition& partition,
                                   const RomOptions& opt);
SubdomainROM build_rom(int cell, const Partition& partition,
                       const std::vector<SubdomainSplit>& splits, const BoundaryBasis& basis,
                       const Vec& g, const Vec& q, const RomOptions& opt);
std::vector<SubdomainROM> build_all_roms(const Partition& partition,
                                         const std::vector<SubdomainSplit>& splits,
                                         const BoundaryBasis& basis, const Vec& g, const Vec& q,
                                         const RomOptions& opt, int threads = 1);
#endif

}  // namespace mswave

#endif  // MSWAVE_ROMGEN_HPP
