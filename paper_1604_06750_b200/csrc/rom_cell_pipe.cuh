// K1 rom_cell_pipe: persistent, warp-specialised cell kernel (sm_100a, fp64).
//
// Per work item (cell c, source tile of ST columns) it computes, exactly as
// msolver.cpp:126-168 (first_layer_flux + interior_accelerations + leapfrog)
//
//   D_k = L^k (U^{k+1} - U^k)            k = 1..m,  U^{m+1} = 0
//   D_1 restricted to every face  -> flux buffer (step 2.1, read by K2)
//   U^k <- (2 U^k - U^k_prev) + dt^2 Lhat^k (D_k - D_{k-1})    k = 2..m
//
// as 2m-1 small dense products C^T = X^T L on the fp64 tensor path
// (mma.sync m8n8k4 f64 -> DMMA.8x8x4; tcgen05 has no f64 kind).  The
// ladders are symmetric, so L is used directly as the col-major B operand.
//
// HBM layout (host-packed, see rom_system.cu):
//   ladders  per cell, in consumption order L^1, L^2, Lhat^2, ..., L^m,
//            Lhat^m; each kt columns with leading dimension ld(kt) (bank-
//            conflict-free stride, zero pad rows); a panel of NP columns is
//            one contiguous block;
//   state    source-tiled: [tile][row][ldst] with ldst = ST + pad, so the
//            rows of one cell layer (or one face) in one tile are contiguous.
// Every stage is therefore ONE cp.async.bulk (TMA 1-D) copy.
//
// Structure (one CTA per SM, grid-strided over items):
//   warps 0, 1   producers: one elected lane each streams, in consumption
//                order, the ladder panels (L2 evict_first: read once per
//                step) resp. the state tiles U^1..U^m, U_prev^k into two smem
//                rings; mbarrier expect_tx / complete_tx per slot;
//   warps 2..    consumers (NCW): DMMA from smem; A fragments (X = U^{k+1}-U^k or
//                D_k - D_{k-1}) are formed on the fly from two smem tiles;
//                D_k lives in a smem tile, u_prev is prefetched from HBM into
//                registers one GEMM ahead and u_next is stored straight from
//                the accumulator registers (64 B row segments, full sectors).
//   Slots are released through per-slot "empty" mbarriers (one arrive per
//   consumer warp), so HBM streaming of item i+1 overlaps compute of item i.
//
// smem strides make every fragment load bank-conflict free:
// 2*stride mod 32 words in {8, 24}  <=>  stride mod 16 in {4, 12} doubles.
#pragma once

#include <cstdint>

#include "rom_kernels.cuh"

namespace mswb {
namespace pipe {

constexpr int kMaxRing = 8;
// doubles of slack between the last smem tile and the barriers: the software
// pipelined k-loops read up to 4 rows past a tile (stride <= 128 doubles)
constexpr int kSmemTailPad = 4 * 128 + 64;

struct K1Geom {
  int ST;        // source tile width (8, 16, 32, 64)
  int n_stiles;  // source tiles
  int ldst;      // row stride of state / D tiles in HBM and smem (doubles)
  int NP;        // ladder panel width (columns, multiple of 8)
  int NL;        // ladder ring depth
  int NU;        // state ring depth
  int slot_lad;  // doubles per ladder slot (NP * max ld)
  int slot_st;   // doubles per state slot (kt4_max * ldst; kstream: 2 * KC * ldst)
  int slot_d;    // kstream: doubles per D tile (rows8(kt_max) * ldst)
  int WM, WN;    // consumer warp grid: WM source groups x WN row groups (= NCW)
  int n_items;   // n_cells * n_stiles
  int total_io;
  int64_t total_inter;
  int64_t total_frows;  // rows of the flux buffer per tile (sum_c kt_c)
  int dbg;       // diagnostics bit flags: 1 skip the math, 2 skip the copies, 4 skip the
                 // epilogues; 8 (with -DMSWB_K1_PROFILE): cycle breakdown into prof[0..3];
                 // 16 no L2 prefetch of the next item
  unsigned long long* prof;
  int l2hint;    // 1: K2 reads the D_1 faces with an L2 evict_first hint (dead after K2)
  int single;    // rom_cell_fused: every cell's layer is one ladder panel (NP >= ktilde_max),
                 // use the stage-ordered form (see rom_cell_fused.cuh)
  int pflead;    // rom_cell_kstream L2 prefetch: 0 = none (default, measured fastest at
                 // config 5), -1 = the whole next item at item start, > 0 = the ladder
                 // matrix pflead ahead (across the item boundary)
};

// Consumer cycle accounting (build with -DMSWB_K1_PROFILE and run with
// MSW_K1_DEBUG=3); compiled out by default.
#ifdef MSWB_K1_PROFILE
#define MSWB_TW(...)                \
  do {                              \
    const long long _t0 = clock64(); \
    __VA_ARGS__;                    \
    t_wait += clock64() - _t0;      \
  } while (0)
#define MSWB_TG(...)                \
  do {                              \
    const long long _t0 = clock64(); \
    __VA_ARGS__;                    \
    t_math += clock64() - _t0;      \
  } while (0)
#define MSWB_CLOCK() clock64()
#else
#define MSWB_TW(...) __VA_ARGS__
#define MSWB_TG(...) __VA_ARGS__
#define MSWB_CLOCK() 0ll
#endif

// Mark-to-mark cycle accounting of a consumer warp (rom_cell_fused, rom_cell_kstream;
// same diagnostic build, run with MSW_K1_DEBUG=8): cycles between marks are summed
// into pt[0..7] and added to G.prof at kernel end.
#ifdef MSWB_K1_PROFILE
#define MSWB_PDECL unsigned pt[8] = {0, 0, 0, 0, 0, 0, 0, 0}; unsigned pt0 = clock()
#define MSWB_PMARK(i) do { const unsigned _t = clock(); pt[i] += _t - pt0; pt0 = _t; } while (0)
#define MSWB_PUSE(x) do { if ((x) == 0x7fffffff) pt[7] += 1; } while (0)
#define MSWB_DBG(x) (G.dbg & (x))  // 1 skip the math, 2 skip the copies, 4 skip the epilogues
#else
#define MSWB_DBG(x) 0
#define MSWB_PDECL
#define MSWB_PMARK(i)
#define MSWB_PUSE(x)
#endif

// ---------------------------------------------------------------- PTX --------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Programmatic dependent launch (K2 -> K1 -> K2 inside a step sequence,
// rom_system.cu launch_step): every CTA lets the next kernel be scheduled at
// once; the ladder producer (warp 0) reads only static data (ladders, cell
// metadata), so it may stream before the previous kernel (K2) has finished,
// and every other warp waits for that kernel's completion and memory.  Both
// instructions are no-ops for a normal launch.
__device__ __forceinline__ void pdl_k1_gate(int warp) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (warp != 0) asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Producer-side wait: the thread is suspended in hardware until the phase
// completes (or the time hint elapses) instead of spinning, so a producer
// blocked on a full ring does not steal issue slots from the math warps.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAITS_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}

// TMA 1-D bulk copy global -> smem, completion counted on `bar` in bytes.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Fire-and-forget L2 prefetch of a contiguous block (no smem, no barrier):
// the producers run it one item ahead of the smem rings, so ring refills hit
// L2 and the rings' in-flight bytes no longer bound HBM throughput.
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void prefetch_l2_big(const void* src, uint64_t bytes) {
  const char* p = static_cast<const char*>(src);
  while (bytes > 0) {
    const uint32_t chunk = bytes > (1u << 20) ? (1u << 20) : static_cast<uint32_t>(bytes);
    prefetch_l2(p, chunk);
    p += chunk;
    bytes -= chunk;
  }
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct Ring {
  int slot = 0;
  uint32_t phase = 0;
  int depth;
  __device__ explicit Ring(int d) : depth(d) {}
  __device__ void advance() {
    if (++slot == depth) {
      slot = 0;
      phase ^= 1u;
    }
  }
};

// One warp's share of C = L X for one ladder panel (rows n of the panel,
// NTW x 8 source columns): A = L (symmetric: the panel's columns are its
// rows), B = X = scale*hi - lo (scale 1: U^{k+1} - U^k or D_k - D_{k-1};
// scale 0: -U^m; fma(s, a, -b) rounds once and s*a is exact, so both match
// the reference's subtraction).  Rows k in [kt, kt4) of the smem tiles hold
// stale finite data; the ladder pad rows in HBM are zero, so those products
// vanish without a predicate.  Row tiles beyond the panel are clamped to a
// valid column and their accumulators are never stored.
//
// KS > 1 splits the reduction: k-step kk accumulates into partial set kk % KS,
// so a warp carries KS x MTP x NTW independent DMMA chains (the DMMA
// dependent-issue latency, not the pipe, bounds long ktilde loops); the
// partial sums are added in a fixed order at the end.  Steps past ksteps are
// predicated to zero operands.
// DIFF = false: B = hi (a single smem operand; lo unused).
template <int MTP, int NTW, int KMAX, int KS = 1, bool DIFF = true>
__device__ __forceinline__ void gemm_tile(double (&acc)[MTP][NTW][2], const double* __restrict__ hi,
                                          double scale, const double* __restrict__ lo,
                                          const double* __restrict__ Ls, int ld, int ldst, int ksteps,
                                          int mtiles, int wr, int WR, int s_w, int g, int t4) {
#pragma unroll
  for (int i = 0; i < MTP; ++i)
#pragma unroll
    for (int j = 0; j < NTW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const double* pa[MTP];
#pragma unroll
  for (int i = 0; i < MTP; ++i) pa[i] = Ls + (min(wr + i * WR, mtiles - 1) * 8 + g) * ld + t4;
  const int off_b = t4 * ldst + s_w + g;
  const double* pb_hi = hi + off_b;
  const double* pb_lo = (DIFF ? lo : hi) + off_b;
  if constexpr (KS > 1) {
    double part[KS - 1][MTP][NTW][2];
#pragma unroll
    for (int p = 0; p < KS - 1; ++p)
#pragma unroll
      for (int i = 0; i < MTP; ++i)
#pragma unroll
        for (int j = 0; j < NTW; ++j) part[p][i][j][0] = part[p][i][j][1] = 0.0;
    const int step_b = 4 * ldst;
    for (int kb = 0; kb < ksteps; kb += KS) {
      double a[KS][MTP], b[KS][NTW];
#pragma unroll
      for (int p = 0; p < KS; ++p) {
        const bool ok = kb + p < ksteps;
#pragma unroll
        for (int i = 0; i < MTP; ++i) a[p][i] = ok ? pa[i][4 * (kb + p)] : 0.0;
#pragma unroll
        for (int j = 0; j < NTW; ++j)
          b[p][j] = ok ? fma(scale, pb_hi[(kb + p) * step_b + j * 8], -pb_lo[(kb + p) * step_b + j * 8]) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < MTP; ++i)
#pragma unroll
        for (int j = 0; j < NTW; ++j) dmma(acc[i][j], a[0][i], b[0][j]);
#pragma unroll
      for (int p = 1; p < KS; ++p)
#pragma unroll
        for (int i = 0; i < MTP; ++i)
#pragma unroll
          for (int j = 0; j < NTW; ++j) dmma(part[p - 1][i][j], a[p][i], b[p][j]);
    }
#pragma unroll
    for (int p = 0; p < KS - 1; ++p)
#pragma unroll
      for (int i = 0; i < MTP; ++i)
#pragma unroll
        for (int j = 0; j < NTW; ++j) {
          acc[i][j][0] += part[p][i][j][0];
          acc[i][j][1] += part[p][i][j][1];
        }
  } else if constexpr (KMAX > 0) {
    // fully unrolled over k (KMAX >= ksteps): immediate smem offsets, no
    // loop-carried register copies; fragments of step kk+1 load before the
    // DMMAs of step kk issue.
    const int step_b = 4 * ldst;
    double a[2][MTP], b[2][NTW];
#pragma unroll
    for (int i = 0; i < MTP; ++i) a[0][i] = pa[i][0];
#pragma unroll
    for (int j = 0; j < NTW; ++j) b[0][j] = DIFF ? fma(scale, pb_hi[j * 8], -pb_lo[j * 8]) : pb_hi[j * 8];
#pragma unroll
    for (int kk = 0; kk < KMAX; ++kk) {
      if (kk >= ksteps) break;
      const int cb = kk & 1, nb = cb ^ 1;
      if (kk + 1 < KMAX) {
#pragma unroll
        for (int i = 0; i < MTP; ++i) a[nb][i] = pa[i][4 * (kk + 1)];
#pragma unroll
        for (int j = 0; j < NTW; ++j)
          b[nb][j] = DIFF ? fma(scale, pb_hi[(kk + 1) * step_b + j * 8], -pb_lo[(kk + 1) * step_b + j * 8])
                          : pb_hi[(kk + 1) * step_b + j * 8];
      }
#pragma unroll
      for (int i = 0; i < MTP; ++i)
#pragma unroll
        for (int j = 0; j < NTW; ++j) dmma(acc[i][j], a[cb][i], b[cb][j]);
    }
  } else {
    const int step_b = 4 * ldst;
    // software pipeline: fragments of k-step kk+1 load while k-step kk issues
    double a[MTP], b[NTW];
#pragma unroll
    for (int i = 0; i < MTP; ++i) a[i] = pa[i][0];
#pragma unroll
    for (int j = 0; j < NTW; ++j) b[j] = DIFF ? fma(scale, pb_hi[j * 8], -pb_lo[j * 8]) : pb_hi[j * 8];
    for (int kk = 0; kk < ksteps; ++kk) {
      double an[MTP], bn[NTW];
      pb_hi += step_b;
      pb_lo += step_b;
      // the last iteration reads one k-step past the tiles (still inside the
      // smem allocation, see kSmemTailPad) and discards it: no predicate
#pragma unroll
      for (int i = 0; i < MTP; ++i) an[i] = pa[i][4 * (kk + 1)];
#pragma unroll
      for (int j = 0; j < NTW; ++j) bn[j] = DIFF ? fma(scale, pb_hi[j * 8], -pb_lo[j * 8]) : pb_hi[j * 8];
#pragma unroll
      for (int i = 0; i < MTP; ++i)
#pragma unroll
        for (int j = 0; j < NTW; ++j) dmma(acc[i][j], a[i], b[j]);
#pragma unroll
      for (int i = 0; i < MTP; ++i) a[i] = an[i];
#pragma unroll
      for (int j = 0; j < NTW; ++j) b[j] = bn[j];
    }
  }
}

// ------------------------------------------------------------- kernel -------

// NCW: consumer warps; NTW: 8-source N-tiles per consumer warp; MTP: max
// 8-row M-tiles per warp per ladder panel.  UPG: U_prev^k for the GEMM2
// epilogue is loaded from global memory into registers as the panel's GEMM
// starts (its latency hides under the k-loop) instead of riding the TMA
// state ring, which frees a ring slot and its smem write + read per layer.
// DREG (single-panel geometries with WN == 1, i.e. each warp owns all rows
// of its columns): D_{k-1} of the warp's fragments stays in registers and
// one smem tile holds dD_k = D_k - D_{k-1} (GEMM2's B operand, written and
// read by the same warp: no CTA barrier).  The difference rounds exactly as
// fma(1, D_k, -D_{k-1}), so results are bit-identical to the two-tile form.
template <int NCW, int NTW, int MTP, int MINB, int KMAX, int KS = 1, bool UPG = false, bool DREG = false>
__global__ void __launch_bounds__(32 * (NCW + 2), MINB) rom_cell_pipe(
    const CellMeta* __restrict__ cells, const CellIface* __restrict__ cif,
    const double* __restrict__ lad, double* ubar0, double* ubar1, double* inter0,
    double* inter1, double* __restrict__ flux, StepParams* P, int64_t n_local, K1Geom G) {
  extern __shared__ __align__(128) double smem[];
  double* lad_slots = smem;
  double* st_slots = lad_slots + G.NL * G.slot_lad;
  constexpr int ND = DREG ? 1 : 2;
  double* dbuf = st_slots + G.NU * G.slot_st;  // 2 D tiles (DREG: one dD tile)
  uint64_t* bars = reinterpret_cast<uint64_t*>(dbuf + ND * G.slot_st + kSmemTailPad);
  uint64_t* full_lad = bars;
  uint64_t* empty_lad = bars + kMaxRing;
  uint64_t* full_st = bars + 2 * kMaxRing;
  uint64_t* empty_st = bars + 3 * kMaxRing;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t n = P->base + n_local;
  const int cur = static_cast<int>(n & 1);
  const double* ubar_cur = cur ? ubar1 : ubar0;
  const double* inter_cur = cur ? inter1 : inter0;
  double* inter_nxt = cur ? inter0 : inter1;
  const double dt2 = P->dt2;
  const int64_t io_tile = static_cast<int64_t>(G.total_io) * G.ldst;  // doubles per tile
  const int64_t inter_tile = G.total_inter * G.ldst;

  // zero every slot once (B operands must be finite in padding rows), init barriers
  {
    const int total = G.NL * G.slot_lad + (G.NU + ND) * G.slot_st;
    for (int i = threadIdx.x; i < total; i += blockDim.x) smem[i] = 0.0;
    if (threadIdx.x == 0) {
      for (int i = 0; i < G.NL; ++i) {
        mbar_init(full_lad + i, 1);
        mbar_init(empty_lad + i, NCW);
      }
      for (int i = 0; i < G.NU; ++i) {
        mbar_init(full_st + i, 1);
        mbar_init(empty_st + i, NCW);
      }
    }
    // make the generic-proxy zero fill and barrier inits visible to TMA
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
  pdl_k1_gate(warp);

  if (warp < 2) {
    // ============================== producers ==============================
    // warp 0 lane 0 streams the ladder ring, warp 1 lane 0 the state ring;
    // separate threads so neither ring's back-pressure stalls the other.
    if (lane != 0) return;
    const bool ladders = warp == 0;
    const uint64_t pol = policy_evict_first();
    Ring rl(G.NL), rs(G.NU);
    for (int item = blockIdx.x; item < G.n_items; item += gridDim.x) {
      const int c = item / G.n_stiles;
      const int tile = item - c * G.n_stiles;
      const CellMeta cm = cells[c];
      const int kt = cm.kt, m = cm.m, ld = cm.ld;
      if (!(G.dbg & 16)) {  // L2 prefetch of this CTA's next item
        const int nitem = item + gridDim.x;
        if (nitem < G.n_items) {
          const int nc = nitem / G.n_stiles;
          const int ntile = nitem - nc * G.n_stiles;
          const CellMeta nm = cells[nc];
          if (ladders) {
            prefetch_l2_big(lad + nm.lad_off, static_cast<uint64_t>(2 * nm.m - 1) * nm.lstride * 8u);
          } else if (nm.m > 1) {
            const uint64_t b = static_cast<uint64_t>(nm.m - 1) * nm.kt * G.ldst * 8u;
            prefetch_l2_big(inter_cur + ntile * inter_tile + nm.inter_row * G.ldst, b);
            prefetch_l2_big(inter_nxt + ntile * inter_tile + nm.inter_row * G.ldst, b);
          }
        }
      }
      if (ladders) {
        // consumption order L^1, L^2, Lhat^2, ..., L^m, Lhat^m in NP-column panels
        const double* L0 = lad + cm.lad_off;
        for (int j = 0; j < 2 * m - 1; ++j) {
          const double* Lj = L0 + static_cast<int64_t>(j) * cm.lstride;
          for (int p0 = 0; p0 < kt; p0 += G.NP) {
            const int cols = min(G.NP, kt - p0);
            const uint32_t bytes = static_cast<uint32_t>(cols) * ld * 8u;
            mbar_wait_sleep(empty_lad + rl.slot, rl.phase ^ 1u);
            if (G.dbg & 2) {
              mbar_arrive(full_lad + rl.slot);
            } else {
              mbar_expect_tx(full_lad + rl.slot, bytes);
              bulk_g2s_hint(lad_slots + rl.slot * G.slot_lad, Lj + static_cast<int64_t>(p0) * ld, bytes,
                            full_lad + rl.slot, pol);
            }
            rl.advance();
          }
        }
      } else {
        // state ring order: U^1, U^2, then per k = 2..m: U^{k+1} (k < m), U_prev^k
        const uint32_t bytes = static_cast<uint32_t>(kt) * G.ldst * 8u;
        const double* cur_tile = inter_cur + tile * inter_tile + cm.inter_row * G.ldst;
        const double* prev_tile = inter_nxt + tile * inter_tile + cm.inter_row * G.ldst;
        auto push = [&](const double* src) {  // one contiguous layer block
          mbar_wait_sleep(empty_st + rs.slot, rs.phase ^ 1u);
          if (G.dbg & 2) {
            mbar_arrive(full_st + rs.slot);
          } else {
            mbar_expect_tx(full_st + rs.slot, bytes);
            bulk_g2s(st_slots + rs.slot * G.slot_st, src, bytes, full_st + rs.slot);
          }
          rs.advance();
        };
        // U^1: gathered from the interface values, one copy per face
        mbar_wait_sleep(empty_st + rs.slot, rs.phase ^ 1u);
        if (G.dbg & 2) mbar_arrive(full_st + rs.slot);
        else mbar_expect_tx(full_st + rs.slot, bytes);
        for (int li = 0; li < cm.nif && !(G.dbg & 2); ++li) {
          const CellIface ci = cif[cm.if_begin + li];
          bulk_g2s(st_slots + rs.slot * G.slot_st + ci.block_off * G.ldst,
                   ubar_cur + tile * io_tile + static_cast<int64_t>(ci.row_off) * G.ldst,
                   static_cast<uint32_t>(ci.M) * G.ldst * 8u, full_st + rs.slot);
        }
        rs.advance();
        if (m > 1) push(cur_tile);  // U^2
        for (int k = 2; k <= m; ++k) {
          if (k < m) push(cur_tile + static_cast<int64_t>(k - 1) * kt * G.ldst);  // U^{k+1}
          if (!UPG) push(prev_tile + static_cast<int64_t>(k - 2) * kt * G.ldst);  // U_prev^k
        }
      }
    }
    return;
  }

  // ================================ consumers ================================
  // warp grid: WS source groups (NTW x 8 columns each) x WR row groups
  const int cw = warp - 2;
  const int ws = cw % G.WM, wr = cw / G.WM;  // WM = WS, WN = WR
  const int WR = G.WN;
  const int s_w = ws * NTW * 8;
  const int g = lane >> 2, t4 = lane & 3;
  const int ldst = G.ldst;
  Ring rl(G.NL), rs(G.NU);
  bool bad = false;
  long long t_wait = 0, t_math = 0;
  const long long t_start = MSWB_CLOCK();
  int n_items_done = 0;

  for (int item = blockIdx.x; item < G.n_items; item += gridDim.x) {
    const int c = item / G.n_stiles;
    const int tile = item - c * G.n_stiles;
    const CellMeta cm = cells[c];
    const int kt = cm.kt, m = cm.m, ld = cm.ld;
    const int ksteps = (kt + 3) >> 2;
    // ring slots of U^k (cur) and U^{k+1} (nxt), taken in ring order
    int slot_k = rs.slot;
    uint32_t phase_k = rs.phase;
    rs.advance();
    MSWB_TW(mbar_wait(full_st + slot_k, phase_k));
    ++n_items_done;
    double* flux_c = flux + (static_cast<int64_t>(tile) * G.total_frows + cm.flux_row) * ldst;
    double dprev[DREG ? MTP : 1][DREG ? NTW : 1][2];  // D_{k-1} of this warp's fragments

    for (int k = 1; k <= m; ++k) {
      const double* Uk = st_slots + slot_k * G.slot_st;
      const double* Ukp = nullptr;
      int slot_n = -1;
      uint32_t phase_n = 0;
      if (k < m) {
        slot_n = rs.slot;
        phase_n = rs.phase;
        rs.advance();
        MSWB_TW(mbar_wait(full_st + slot_n, phase_n));
        Ukp = st_slots + slot_n * G.slot_st;
      }
      // U_prev^k (k >= 2) for the GEMM2 epilogue: next slot in ring order
      int slot_p = -1;
      uint32_t phase_p = 0;
      if (k >= 2 && !UPG) {
        slot_p = rs.slot;
        phase_p = rs.phase;
        rs.advance();
      }
      // layer-k rows of this tile in HBM (u_prev in, u_next out)
      double* lay = inter_nxt + tile * inter_tile + (cm.inter_row + static_cast<int64_t>(k - 2) * kt) * ldst;

      // ---- GEMM1: D_k = L^k (U^{k+1} - U^k), panels of the ladder ring ----
      double* Dk = dbuf + (DREG ? 0 : (k & 1) * G.slot_st);
      for (int p0 = 0; p0 < kt; p0 += G.NP) {
        const int mtiles = (min(G.NP, kt - p0) + 7) >> 3;
        MSWB_TW(mbar_wait(full_lad + rl.slot, rl.phase));
        const double* Ls = lad_slots + rl.slot * G.slot_lad;
        double acc[MTP][NTW][2];
        MSWB_TG(gemm_tile<MTP, NTW, KMAX, KS>(acc, Ukp ? Ukp : Uk, Ukp ? 1.0 : 0.0, Uk, Ls, ld, ldst,
                                    (G.dbg & 1) ? 0 : ksteps, mtiles, wr, WR, s_w, g, t4));
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_lad + rl.slot);
        rl.advance();
        // epilogue: D_k rows of this panel (+ D_1 -> flux), 16-byte stores
#pragma unroll
        for (int i = 0; i < MTP && !(G.dbg & 4); ++i) {
          const int mt = wr + i * WR;
          const int nr = p0 + mt * 8 + g;
          if (mt >= mtiles || nr >= kt) continue;
#pragma unroll
          for (int j = 0; j < NTW; ++j) {
            const int s = s_w + j * 8 + 2 * t4;
            const double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
            if constexpr (DREG) {
              if (k == 1) {
                *reinterpret_cast<double2*>(flux_c + nr * ldst + s) = v;
              } else {
                *reinterpret_cast<double2*>(Dk + nr * ldst + s) =
                    make_double2(__dsub_rn(v.x, dprev[i][j][0]), __dsub_rn(v.y, dprev[i][j][1]));
              }
              dprev[i][j][0] = v.x;
              dprev[i][j][1] = v.y;
            } else {
              *reinterpret_cast<double2*>(Dk + nr * ldst + s) = v;
              if (k == 1) *reinterpret_cast<double2*>(flux_c + nr * ldst + s) = v;
            }
          }
        }
      }
      // row-split warps read D rows written by other warps; source-split
      // warps own all rows of their columns and need no CTA-level sync
      if (WR > 1) named_sync(1, 32 * NCW);

      if (k >= 2) {
        // ---- GEMM2: acc = Lhat^k (D_k - D_{k-1}); u_next ----
        const double* Dp = dbuf + (DREG ? 0 : ((k - 1) & 1) * G.slot_st);
        const double* Up = nullptr;
        if (!UPG) {
          MSWB_TW(mbar_wait(full_st + slot_p, phase_p));
          Up = st_slots + slot_p * G.slot_st;
        }
        for (int p0 = 0; p0 < kt; p0 += G.NP) {
          const int mtiles = (min(G.NP, kt - p0) + 7) >> 3;
          double2 upv[UPG ? MTP : 1][UPG ? NTW : 1];
          if constexpr (UPG) {
#pragma unroll
            for (int i = 0; i < MTP; ++i) {
              const int mt = wr + i * WR;
              const int nr = p0 + mt * 8 + g;
#pragma unroll
              for (int j = 0; j < NTW; ++j)
                upv[i][j] = (mt < mtiles && nr < kt)
                                ? __ldcs(reinterpret_cast<const double2*>(lay + nr * ldst + s_w + j * 8 + 2 * t4))
                                : make_double2(0.0, 0.0);
            }
          }
          MSWB_TW(mbar_wait(full_lad + rl.slot, rl.phase));
          const double* Ls = lad_slots + rl.slot * G.slot_lad;
          double acc[MTP][NTW][2];
          if constexpr (DREG) {
            __syncwarp();  // this warp's dD rows are in smem
            MSWB_TG(gemm_tile<MTP, NTW, KMAX, KS, false>(acc, Dk, 1.0, nullptr, Ls, ld, ldst, (G.dbg & 1) ? 0 : ksteps,
                                                         mtiles, wr, WR, s_w, g, t4));
          } else {
            MSWB_TG(gemm_tile<MTP, NTW, KMAX, KS>(acc, Dk, 1.0, Dp, Ls, ld, ldst, (G.dbg & 1) ? 0 : ksteps, mtiles,
                                                  wr, WR, s_w, g, t4));
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(empty_lad + rl.slot);
          rl.advance();
          // branch-free: every tile's operands are loaded (rows clamped into
          // the slot), all leapfrogs computed, only the stores are predicated,
          // so the per-tile latency chains overlap (rom_cell_fused, same form)
          if (!(G.dbg & 4)) {
            bool okt[MTP];
            int nrt[MTP];
            double2 u[MTP][NTW], up[MTP][NTW];
#pragma unroll
            for (int i = 0; i < MTP; ++i) {
              const int mt = wr + i * WR;
              const int nr = p0 + mt * 8 + g;
              okt[i] = mt < mtiles && nr < kt;
              nrt[i] = okt[i] ? nr : 0;
#pragma unroll
              for (int j = 0; j < NTW; ++j) {
                const int s = s_w + j * 8 + 2 * t4;
                u[i][j] = *reinterpret_cast<const double2*>(Uk + nrt[i] * ldst + s);
                if constexpr (UPG) up[i][j] = upv[i][j];
                else up[i][j] = *reinterpret_cast<const double2*>(Up + nrt[i] * ldst + s);
              }
            }
#pragma unroll
            for (int i = 0; i < MTP; ++i)
#pragma unroll
              for (int j = 0; j < NTW; ++j) {
                const int s = s_w + j * 8 + 2 * t4;
                double2 v;
                v.x = leapfrog_rn(u[i][j].x, up[i][j].x, dt2, acc[i][j][0]);
                v.y = leapfrog_rn(u[i][j].y, up[i][j].y, dt2, acc[i][j][1]);
                if (okt[i]) *reinterpret_cast<double2*>(lay + nrt[i] * ldst + s) = v;
                bad |= okt[i] && (!(fabs(v.x) <= kGuard) || !(fabs(v.y) <= kGuard));
              }
          }
        }
        if (WR > 1) named_sync(1, 32 * NCW);  // D_{k-1} free for reuse
        __syncwarp();
        if (!UPG && lane == 0) mbar_arrive(empty_st + slot_p);
      }
      // U^k done
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_st + slot_k);
      slot_k = slot_n;
      phase_k = phase_n;
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0)
    atomicMin(reinterpret_cast<unsigned long long*>(&P->bad), static_cast<unsigned long long>(n + 1));
  if ((G.dbg & 8) && lane == 0 && G.prof) {
    atomicAdd(G.prof + 0, static_cast<unsigned long long>(t_wait));
    atomicAdd(G.prof + 1, static_cast<unsigned long long>(t_math));
    atomicAdd(G.prof + 2, static_cast<unsigned long long>(MSWB_CLOCK() - t_start));
    atomicAdd(G.prof + 3, static_cast<unsigned long long>(n_items_done));
  }
}


// --------------------------------------------------------------------------
// K1' rom_cell_pipe2: single-panel cells (ktilde <= 64), dual GEMMs.
//
// D_k depends only on the state and acc_k = Lhat^k (D_k - D_{k-1}) only on
// D_k, D_{k-1}, so GEMM2 of layer k and GEMM1 of layer k+1 are independent.
// Each phase therefore runs two products in one k-loop, doubling the
// independent DMMA accumulators per warp (DMMA latency is long, ~200 cycles)
// and cutting the phases per cell from 2m-1 to m:
//   phase 1 : D_1 = L^1 (U^2-U^1),      D_2 = L^2 (U^3-U^2)
//   phase k : acc_k = Lhat^k (D_k-D_{k-1}) -> U^k,   D_{k+1} = L^{k+1} (U^{k+2}-U^{k+1})
// Ladder ring order is unchanged (L^1, L^2, Lhat^2, L^3, ...); the state ring
// carries U^1, U^2, U^3, then per phase k: U^{k+2} (k+2 <= m), U_prev^k.
// Each warp owns whole columns (all rows), so it keeps D_k of its fragments
// in registers and writes dD_{k+1} = D_{k+1} - D_k (rounded exactly like
// fma(1, D_{k+1}, -D_k)) to a double-buffered smem tile, which is GEMM2's
// single B operand in the next phase; no CTA barriers.
template <int MT, int NTW, bool DIFF1>
__device__ __forceinline__ void gemm_dual(double (&acc1)[MT][NTW][2], double (&acc2)[MT][NTW][2],
                                          const double* __restrict__ L1s, const double* __restrict__ h1,
                                          double sc1, const double* __restrict__ l1,
                                          const double* __restrict__ L2s, const double* __restrict__ h2,
                                          double sc2, const double* __restrict__ l2, bool two, int ld,
                                          int ldst, int ksteps, int mtiles, int s_w, int g, int t4) {
  // product 1: B = DIFF1 ? sc1*h1 - l1 : h1;  product 2 (if two): B = sc2*h2 - l2.
  // Software pipelined like gemm_tile: fragments of k-step kk+1 load while
  // the 2 x MT x NTW independent DMMA chains of k-step kk issue.
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NTW; ++j) acc1[i][j][0] = acc1[i][j][1] = acc2[i][j][0] = acc2[i][j][1] = 0.0;
  const double* pa1[MT];
  const double* pa2[MT];
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int col = (min(i, mtiles - 1) * 8 + g) * ld + t4;
    pa1[i] = L1s + col;
    pa2[i] = L2s + col;
  }
  const int off_b = t4 * ldst + s_w + g;
  const double* b1h = h1 + off_b;
  const double* b1l = (DIFF1 ? l1 : h1) + off_b;
  const double* b2h = h2 + off_b;
  const double* b2l = l2 + off_b;
  const int step_b = 4 * ldst;
  double a1[MT], a2[MT], b1[NTW], b2[NTW];
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    a1[i] = pa1[i][0];
    a2[i] = two ? pa2[i][0] : 0.0;
  }
#pragma unroll
  for (int j = 0; j < NTW; ++j) {
    b1[j] = DIFF1 ? fma(sc1, b1h[j * 8], -b1l[j * 8]) : b1h[j * 8];
    b2[j] = two ? fma(sc2, b2h[j * 8], -b2l[j * 8]) : 0.0;
  }
  for (int kk = 0; kk < ksteps; ++kk) {
    double an1[MT], an2[MT], bn1[NTW], bn2[NTW];
    b1h += step_b;
    b1l += step_b;
    b2h += step_b;
    b2l += step_b;
    // one k-step of look-ahead; the last one reads past the tiles (inside
    // the smem allocation, see kSmemTailPad) and is discarded
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      an1[i] = pa1[i][4 * (kk + 1)];
      an2[i] = two ? pa2[i][4 * (kk + 1)] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < NTW; ++j) {
      bn1[j] = DIFF1 ? fma(sc1, b1h[j * 8], -b1l[j * 8]) : b1h[j * 8];
      bn2[j] = two ? fma(sc2, b2h[j * 8], -b2l[j * 8]) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NTW; ++j) dmma(acc1[i][j], a1[i], b1[j]);
    if (two) {
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NTW; ++j) dmma(acc2[i][j], a2[i], b2[j]);
    }
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      a1[i] = an1[i];
      a2[i] = an2[i];
    }
#pragma unroll
    for (int j = 0; j < NTW; ++j) {
      b1[j] = bn1[j];
      b2[j] = bn2[j];
    }
  }
}

template <int NCW, int NTW, int MT, int MINB>
__global__ void __launch_bounds__(32 * (NCW + 2), MINB) rom_cell_pipe2(
    const CellMeta* __restrict__ cells, const CellIface* __restrict__ cif,
    const double* __restrict__ lad, double* ubar0, double* ubar1, double* inter0,
    double* inter1, double* __restrict__ flux, StepParams* P, int64_t n_local, K1Geom G) {
  extern __shared__ __align__(128) double smem[];
  double* lad_slots = smem;
  double* st_slots = lad_slots + G.NL * G.slot_lad;
  double* dbuf = st_slots + G.NU * G.slot_st;  // 2 dD tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(dbuf + 2 * G.slot_st + kSmemTailPad);
  uint64_t* full_lad = bars;
  uint64_t* empty_lad = bars + kMaxRing;
  uint64_t* full_st = bars + 2 * kMaxRing;
  uint64_t* empty_st = bars + 3 * kMaxRing;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t n = P->base + n_local;
  const int cur = static_cast<int>(n & 1);
  const double* ubar_cur = cur ? ubar1 : ubar0;
  const double* inter_cur = cur ? inter1 : inter0;
  double* inter_nxt = cur ? inter0 : inter1;
  const double dt2 = P->dt2;
  const int64_t io_tile = static_cast<int64_t>(G.total_io) * G.ldst;
  const int64_t inter_tile = G.total_inter * G.ldst;

  {
    const int total = G.NL * G.slot_lad + (G.NU + 2) * G.slot_st;
    for (int i = threadIdx.x; i < total; i += blockDim.x) smem[i] = 0.0;
    if (threadIdx.x == 0) {
      for (int i = 0; i < G.NL; ++i) {
        mbar_init(full_lad + i, 1);
        mbar_init(empty_lad + i, NCW);
      }
      for (int i = 0; i < G.NU; ++i) {
        mbar_init(full_st + i, 1);
        mbar_init(empty_st + i, NCW);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
  pdl_k1_gate(warp);

  if (warp < 2) {
    if (lane != 0) return;
    const bool ladders = warp == 0;
    const uint64_t pol = policy_evict_first();
    Ring rl(G.NL), rs(G.NU);
    for (int item = blockIdx.x; item < G.n_items; item += gridDim.x) {
      const int c = item / G.n_stiles;
      const int tile = item - c * G.n_stiles;
      const CellMeta cm = cells[c];
      const int kt = cm.kt, m = cm.m, ld = cm.ld;
      {  // L2 prefetch of this CTA's next item
        const int nitem = item + gridDim.x;
        if (nitem < G.n_items) {
          const int nc = nitem / G.n_stiles;
          const int ntile = nitem - nc * G.n_stiles;
          const CellMeta nm = cells[nc];
          if (ladders) {
            prefetch_l2_big(lad + nm.lad_off, static_cast<uint64_t>(2 * nm.m - 1) * nm.lstride * 8u);
          } else if (nm.m > 1) {
            const uint64_t b = static_cast<uint64_t>(nm.m - 1) * nm.kt * G.ldst * 8u;
            prefetch_l2_big(inter_cur + ntile * inter_tile + nm.inter_row * G.ldst, b);
            prefetch_l2_big(inter_nxt + ntile * inter_tile + nm.inter_row * G.ldst, b);
          }
        }
      }
      if (ladders) {
        const double* L0 = lad + cm.lad_off;
        const uint32_t bytes = static_cast<uint32_t>(kt) * ld * 8u;
        for (int j = 0; j < 2 * m - 1; ++j) {
          mbar_wait_sleep(empty_lad + rl.slot, rl.phase ^ 1u);
          mbar_expect_tx(full_lad + rl.slot, bytes);
          bulk_g2s_hint(lad_slots + rl.slot * G.slot_lad, L0 + static_cast<int64_t>(j) * cm.lstride, bytes,
                        full_lad + rl.slot, pol);
          rl.advance();
        }
      } else {
        const uint32_t bytes = static_cast<uint32_t>(kt) * G.ldst * 8u;
        const double* cur_tile = inter_cur + tile * inter_tile + cm.inter_row * G.ldst;
        const double* prev_tile = inter_nxt + tile * inter_tile + cm.inter_row * G.ldst;
        auto push = [&](const double* src) {
          mbar_wait_sleep(empty_st + rs.slot, rs.phase ^ 1u);
          mbar_expect_tx(full_st + rs.slot, bytes);
          bulk_g2s(st_slots + rs.slot * G.slot_st, src, bytes, full_st + rs.slot);
          rs.advance();
        };
        mbar_wait_sleep(empty_st + rs.slot, rs.phase ^ 1u);  // U^1 from the faces
        mbar_expect_tx(full_st + rs.slot, bytes);
        for (int li = 0; li < cm.nif; ++li) {
          const CellIface ci = cif[cm.if_begin + li];
          bulk_g2s(st_slots + rs.slot * G.slot_st + ci.block_off * G.ldst,
                   ubar_cur + tile * io_tile + static_cast<int64_t>(ci.row_off) * G.ldst,
                   static_cast<uint32_t>(ci.M) * G.ldst * 8u, full_st + rs.slot);
        }
        rs.advance();
        auto layer = [&](int k) { return cur_tile + static_cast<int64_t>(k - 2) * kt * G.ldst; };
        if (m >= 2) push(layer(2));
        if (m >= 3) push(layer(3));
        for (int k = 2; k <= m; ++k) {
          if (k + 2 <= m) push(layer(k + 2));
          push(prev_tile + static_cast<int64_t>(k - 2) * kt * G.ldst);  // U_prev^k
        }
      }
    }
    return;
  }

  // ================================ consumers ================================
  const int cw = warp - 2;
  const int s_w = cw * NTW * 8;
  const int g = lane >> 2, t4 = lane & 3;
  const int ldst = G.ldst;
  Ring rl(G.NL), rs(G.NU);
  bool bad = false;

  for (int item = blockIdx.x; item < G.n_items; item += gridDim.x) {
    const int c = item / G.n_stiles;
    const int tile = item - c * G.n_stiles;
    const CellMeta cm = cells[c];
    const int kt = cm.kt, m = cm.m, ld = cm.ld;
    const int ksteps = (kt + 3) >> 2;
    const int mtiles = (kt + 7) >> 3;
    double* flux_c = flux + (static_cast<int64_t>(tile) * G.total_frows + cm.flux_row) * ldst;
    double* lay0 = inter_nxt + tile * inter_tile + cm.inter_row * ldst;
    // rolling window of state-ring slots: U^k, U^{k+1}, U^{k+2}
    int s0 = rs.slot;
    uint32_t q0 = rs.phase;
    rs.advance();
    int s1 = -1, s2 = -1;
    uint32_t q1 = 0, q2 = 0;
    if (m >= 2) {
      s1 = rs.slot;
      q1 = rs.phase;
      rs.advance();
    }
    if (m >= 3) {
      s2 = rs.slot;
      q2 = rs.phase;
      rs.advance();
    }
    mbar_wait(full_st + s0, q0);
    if (m >= 2) mbar_wait(full_st + s1, q1);
    if (m >= 3) mbar_wait(full_st + s2, q2);
    double dprev[MT][NTW][2];

    // ---- phase 1: D_1 (and D_2) ----
    {
      const double* U1 = st_slots + s0 * G.slot_st;
      const double* U2 = m >= 2 ? st_slots + s1 * G.slot_st : U1;
      const double* U3 = m >= 3 ? st_slots + s2 * G.slot_st : U2;
      const bool two = m >= 2;
      mbar_wait(full_lad + rl.slot, rl.phase);
      const double* La = lad_slots + rl.slot * G.slot_lad;
      const int sa = rl.slot;
      rl.advance();
      const double* Lb = La;
      int sb = -1;
      if (two) {
        mbar_wait(full_lad + rl.slot, rl.phase);
        Lb = lad_slots + rl.slot * G.slot_lad;
        sb = rl.slot;
        rl.advance();
      }
      double accA[MT][NTW][2], accB[MT][NTW][2];
      // D_1 = L^1 (U^2 - U^1)  [m == 1: -U^1];  D_2 = L^2 (U^3 - U^2)  [m == 2: -U^2]
      gemm_dual<MT, NTW, true>(accA, accB, La, m >= 2 ? U2 : U1, m >= 2 ? 1.0 : 0.0, U1, Lb, U3,
                               m >= 3 ? 1.0 : 0.0, U2, two, ld, ldst, ksteps, mtiles, s_w, g, t4);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(empty_lad + sa);
        if (two) mbar_arrive(empty_lad + sb);
        mbar_arrive(empty_st + s0);  // U^1 done
      }
      double* dD = dbuf;  // dD_2 in buffer 2 & 1 = 0
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int nr = i * 8 + g;
        const bool ok = i < mtiles && nr < kt;
#pragma unroll
        for (int j = 0; j < NTW; ++j) {
          const int s = s_w + j * 8 + 2 * t4;
          if (ok) *reinterpret_cast<double2*>(flux_c + nr * ldst + s) = make_double2(accA[i][j][0], accA[i][j][1]);
          if (two) {
            if (ok)
              *reinterpret_cast<double2*>(dD + nr * ldst + s) =
                  make_double2(__dsub_rn(accB[i][j][0], accA[i][j][0]), __dsub_rn(accB[i][j][1], accA[i][j][1]));
            dprev[i][j][0] = accB[i][j][0];
            dprev[i][j][1] = accB[i][j][1];
          }
        }
      }
    }
    // window after phase 1: U^2 (s1), U^3 (s2)
    s0 = s1;
    q0 = q1;
    s1 = s2;
    q1 = q2;

    // ---- phases k = 2..m ----
    for (int k = 2; k <= m; ++k) {
      // new state: U^{k+2} (k+2 <= m), then U_prev^k
      if (k + 2 <= m) {
        s2 = rs.slot;
        q2 = rs.phase;
        rs.advance();
      }
      const int sp = rs.slot;
      const uint32_t pp = rs.phase;
      rs.advance();
      const bool two = k < m;
      const double* Uk = st_slots + s0 * G.slot_st;
      const double* Ukp1 = two ? st_slots + s1 * G.slot_st : Uk;
      const double* Ukp2 = Ukp1;
      if (k + 2 <= m) {
        mbar_wait(full_st + s2, q2);
        Ukp2 = st_slots + s2 * G.slot_st;
      }
      const double* dDk = dbuf + (k & 1) * G.slot_st;
      double* dDn = dbuf + ((k + 1) & 1) * G.slot_st;
      mbar_wait(full_lad + rl.slot, rl.phase);  // Lhat^k
      const double* La = lad_slots + rl.slot * G.slot_lad;
      const int sa = rl.slot;
      rl.advance();
      const double* Lb = La;
      int sb = -1;
      if (two) {
        mbar_wait(full_lad + rl.slot, rl.phase);  // L^{k+1}
        Lb = lad_slots + rl.slot * G.slot_lad;
        sb = rl.slot;
        rl.advance();
      }
      double accA[MT][NTW][2], accB[MT][NTW][2];
      // acc_k = Lhat^k dD_k;  D_{k+1} = L^{k+1} (U^{k+2} - U^{k+1})  [k+1 == m: -U^m]
      gemm_dual<MT, NTW, false>(accA, accB, La, dDk, 1.0, nullptr, Lb, Ukp2, (k + 2 <= m) ? 1.0 : 0.0, Ukp1, two,
                                ld, ldst, ksteps, mtiles, s_w, g, t4);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(empty_lad + sa);
        if (two) mbar_arrive(empty_lad + sb);
      }
      mbar_wait(full_st + sp, pp);
      const double* Up = st_slots + sp * G.slot_st;
      double* lay = lay0 + static_cast<int64_t>(k - 2) * kt * ldst;
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int nr = i * 8 + g;
        const bool ok = i < mtiles && nr < kt;
#pragma unroll
        for (int j = 0; j < NTW; ++j) {
          const int s = s_w + j * 8 + 2 * t4;
          if (ok) {
            const double2 u = *reinterpret_cast<const double2*>(Uk + nr * ldst + s);
            const double2 up = *reinterpret_cast<const double2*>(Up + nr * ldst + s);
            double2 v;
            v.x = leapfrog_rn(u.x, up.x, dt2, accA[i][j][0]);
            v.y = leapfrog_rn(u.y, up.y, dt2, accA[i][j][1]);
            *reinterpret_cast<double2*>(lay + nr * ldst + s) = v;
            bad |= !(fabs(v.x) <= kGuard) || !(fabs(v.y) <= kGuard);
          }
          if (two) {
            if (ok)
              *reinterpret_cast<double2*>(dDn + nr * ldst + s) = make_double2(
                  __dsub_rn(accB[i][j][0], dprev[i][j][0]), __dsub_rn(accB[i][j][1], dprev[i][j][1]));
            dprev[i][j][0] = accB[i][j][0];
            dprev[i][j][1] = accB[i][j][1];
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(empty_st + sp);  // U_prev^k done
        mbar_arrive(empty_st + s0);  // U^k done
      }
      s0 = s1;
      q0 = q1;
      s1 = s2;
      q1 = q2;
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0)
    atomicMin(reinterpret_cast<unsigned long long*>(&P->bad), static_cast<unsigned long long>(n + 1));
}

}  // namespace pipe
}  // namespace mswb
