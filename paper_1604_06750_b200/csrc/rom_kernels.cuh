// On-line ROM step kernels for sm_100a (fp64).
//
// One leapfrog step of the coupled S-fraction ROM system
// (reference: proj/src/msolver.cpp:154-194) is two kernels:
//
//   K1 rom_cell_step   one CTA per (cell, source tile).  Gathers layer 1 of
//                      the cell from the shared interface values ubar
//                      (conjugation invariant, msolver.hpp:51-52), layers
//                      2..m from the cell state, forms
//                        D_k = L^k (U^{k+1} - U^k),  k = 1..m, U^{m+1} = 0,
//                      publishes D_1 restricted to each face (step 2.1,
//                      msolver.cpp:159-161) and advances layers 2..m
//                        U^k <- 2U^k - U^k_prev + dt^2 Lhat^k (D_k - D_{k-1})
//                      (step 2.2, msolver.cpp:163-168 with the interior flux
//                      of msolver.cpp:133-145 written as D_k - D_{k-1}).
//   K2 rom_iface_step  one CTA per (interface tile, source tile): the
//                      conjugated update of step 2.3 (msolver.cpp:170-183)
//                        ubar <- 2ubar - ubar_prev + dt^2 mass (D1_i + D1_j + w g~)
//                      plus in-kernel receiver sampling (msolver.cpp:405-411)
//                      for receivers supported on that interface.
//
// Both kernels fuse the instability guard (msolver.cpp:147-150,185-193):
// any |u| > 1e12 or non-finite entry records the step index with atomicMin.
//
// Layout (HBM): every state / source / flux array is [row][S], the source
// index fastest, so each row of a source tile is a contiguous, coalesced,
// 16-byte-vectorisable segment.  Ladders are per cell, column-major
// ktilde x ktilde as in the reference archive; which of them are resident is
// decided by the host (see rom_system.cu).
#pragma once

#include <cstdint>

namespace mswb {

constexpr double kGuard = 1e12;

struct CellMeta {
  int32_t kt;        // ktilde
  int32_t m;         // layers
  int32_t nif;       // local interfaces
  int32_t if_begin;  // index into CellIface array
  int64_t lad_off;   // doubles: L^1, L^2, Lhat^2, .., L^m, Lhat^m, each lstride doubles
  int64_t inter_row; // first row of layer 2 in the interior state arrays
  int32_t ld;        // ladder leading dimension (>= kt rounded to 4, bank-conflict free)
  int32_t lstride;   // doubles per ladder matrix: kt rounded to 4 columns (zero pad) x ld
  int64_t flux_row;  // first row of this cell's D_1 in the flux buffer (cell-local layout)
  // fused-layer operator (rom_cell_fused): per layer k >= 2 the kt x 2kt4
  // matrix [Lhat^k L^k | Lhat^k L^{k-1}] stored transposed (column n = output
  // row n), leading dimension ld2 = bank_stride(2 kt4); L^1 follows with ld2
  int64_t lad2_off;
  int32_t ld2;
  int32_t pad2;
  // K-streaming fused operator (rom_cell_fks): per layer k >= 2, P_k then
  // -Q_k column-major with the ladder layout (ld, lstride); ktilde > 64 only
  int64_t lad3_off;
};

// Source-tiled state layout: element (row, s) of an array with `rows` rows
// lives at ((s / ST) * rows + row) * ldst + s % ST.
struct Tiling {
  int32_t ST;
  int32_t ldst;
  int32_t n_st;
  int32_t S;  // user-visible sources (< n_st * ST)
  __host__ __device__ int64_t at(int64_t rows, int64_t row, int s) const {
    return ((s / ST) * rows + row) * ldst + (s % ST);
  }
};

struct CellIface {
  int32_t row_off;    // first ubar row of the interface
  int32_t block_off;  // block offset inside the cell's layer vector
  int32_t M;          // interface size
  int32_t side;       // 0: this cell is ci, 1: cj
};

struct IfaceMeta {
  int32_t row_off;
  int32_t M;
  int32_t two_sided;  // cj >= 0
  int32_t rcv_begin;  // single-interface receivers fused into K2: [rcv_begin, rcv_end)
  int32_t rcv_end;
  int32_t has_src;    // any nonzero g~ on this interface (else the g read is skipped)
  int64_t mass_off;   // doubles
  int64_t frow_i;     // first flux row of side i (cell-local D_1 layout)
  int64_t frow_j;     // first flux row of side j (-1: single-sided)
};

// Per-run parameters read by every kernel through one device pointer, so a
// captured CUDA graph can be replayed with new w / trace buffers and a new
// step base without re-instantiation.
struct StepParams {
  const double* w;     // [steps][w_stride]
  double* traces;      // [(steps+1)][R][S]
  int64_t base;        // global step index of graph node 0 (advanced in-graph)
  int64_t n0;          // global step index at the start of the run
  int64_t bad;         // first unstable step (INT64_MAX: none)
  double dt2;
  int32_t w_stride;
  int32_t pad;
};

struct RcvTerm {       // fused receiver on one interface
  int32_t rcv;         // receiver index
  int32_t q_off;       // offset in q array (M values)
};

// Leapfrog combination exactly as the reference evaluates it:
// (2.0 * u - u_prev) + dt2 * acc   (msolver.cpp:167,177), no FMA contraction.
__device__ __forceinline__ double leapfrog_rn(double u, double up, double dt2, double acc) {
  return __dadd_rn(__dsub_rn(__dmul_rn(2.0, u), up), __dmul_rn(dt2, acc));
}


}  // namespace mswb
