// K1'' rom_cell_kstream: K-streaming cell kernel for large ktilde (sm_100a, fp64).
//
// Same step as rom_cell_pipe (msolver.cpp:126-168): per (cell, source tile)
//   D_k = L^k (U^{k+1} - U^k),  k = 1..m,  U^{m+1} = 0,   D_1|faces -> flux
//   U^k <- (2 U^k - U_prev^k) + dt^2 Lhat^k (D_k - D_{k-1}),  k = 2..m
// but with every output row of the cell accumulated in registers while the
// reduction dimension streams through smem in chunks of KC:
//   ladder ring  KC columns of one ladder (all ktilde rows; col-major, so one
//                contiguous TMA copy; columns past ktilde are zero in HBM);
//   state ring   KC rows of U^{k+1} (hi) and U^k (lo) for GEMM1 (U^1 gathered
//                from the interface values face by face);
//   dD tile      D_k - D_{k-1} full height in smem (GEMM2's B operand); each
//                warp keeps D_{k-1} of its own fragments in registers, so the
//                difference rounds exactly as fma(1, D_k, -D_{k-1}) did;
//   U^k, U_prev^k for the GEMM2 epilogue follow through the state ring in
//                row chunks (TMA, prefetched while the GEMM2 k-loop runs).
// Only the dD tile is ktilde-high, so source tiles of 32-64 fit next to
// deep rings at ktilde ~ 100 (config 5), where the panel kernel's full-height
// state slots do not.  The k-order of every accumulation is the panel
// kernel's (ascending k-steps, one DMMA chain per output fragment), so both
// kernels produce identical bits.
#pragma once

#include "rom_cell_pipe.cuh"

namespace mswb {
namespace pipe {

// One warp's C += L[:, chunk] X[chunk, :] over `ksteps` k-steps of 4.
// A(n, k) = Ls[k * ld + n] (chunk columns are the k index), B = scale*hi - lo.
// MTA <= MTW: the warp's row tiles in use for this cell (the others would only
// recompute the last tile); the loops run over those alone.
template <int MTW, int NTW, bool DIFF = true, int MTA = MTW>
__device__ __forceinline__ void kchunk_t(double (&acc)[MTW][NTW][2], const double* __restrict__ hi,
                                         double scale, const double* __restrict__ lo,
                                         const double* __restrict__ Ls, int ld, int ldst, int ksteps,
                                         int rtiles, int wr, int WN, int s_w, int g, int t4) {
  const double* pa[MTA];
#pragma unroll
  for (int i = 0; i < MTA; ++i) pa[i] = Ls + t4 * ld + min(wr + i * WN, rtiles - 1) * 8 + g;
  const int off_b = t4 * ldst + s_w + g;
  const double* pb_hi = hi + off_b;
  const double* pb_lo = lo + off_b;
  const int step_a = 4 * ld, step_b = 4 * ldst;
  double a[MTA], b[NTW];
#pragma unroll
  for (int i = 0; i < MTA; ++i) a[i] = pa[i][0];
#pragma unroll
  for (int j = 0; j < NTW; ++j) b[j] = DIFF ? fma(scale, pb_hi[j * 8], -pb_lo[j * 8]) : pb_hi[j * 8];
  for (int kk = 0; kk < ksteps; ++kk) {
    double an[MTA], bn[NTW];
    pb_hi += step_b;
    pb_lo += step_b;
    // one k-step of look-ahead; the last one reads past the chunk (still
    // inside the smem allocation) and is discarded
#pragma unroll
    for (int i = 0; i < MTA; ++i) an[i] = pa[i][(kk + 1) * step_a];
#pragma unroll
    for (int j = 0; j < NTW; ++j) bn[j] = DIFF ? fma(scale, pb_hi[j * 8], -pb_lo[j * 8]) : pb_hi[j * 8];
#pragma unroll
    for (int i = 0; i < MTA; ++i)
#pragma unroll
      for (int j = 0; j < NTW; ++j) dmma(acc[i][j], a[i], b[j]);
#pragma unroll
    for (int i = 0; i < MTA; ++i) a[i] = an[i];
#pragma unroll
    for (int j = 0; j < NTW; ++j) b[j] = bn[j];
  }
}

// Dispatch on the warp's live row tiles `mta` (uniform per warp and cell):
// instances for MTW, MTW-1, MTW-2, MTW-3 tiles; fewer live tiles use the
// smallest of those (boundary cells of a regular grid have smaller ktilde, and
// 13 row tiles split 7 + 6 over two row groups).
template <int MTW, int NTW, bool DIFF = true, int MTA = MTW>
__device__ __forceinline__ void kchunk(double (&acc)[MTW][NTW][2], const double* __restrict__ hi,
                                       double scale, const double* __restrict__ lo,
                                       const double* __restrict__ Ls, int ld, int ldst, int ksteps,
                                       int rtiles, int wr, int WN, int s_w, int g, int t4, int mta) {
  if constexpr (MTA > 1 && MTA > MTW - 3) {
    if (mta < MTA) {
      kchunk<MTW, NTW, DIFF, MTA - 1>(acc, hi, scale, lo, Ls, ld, ldst, ksteps, rtiles, wr, WN, s_w, g, t4, mta);
      return;
    }
  }
  kchunk_t<MTW, NTW, DIFF, MTA>(acc, hi, scale, lo, Ls, ld, ldst, ksteps, rtiles, wr, WN, s_w, g, t4);
}

// The epilogue warps share the fp64 pipe with the consumers' DMMA stream, so
// their update uses as few fp64 instructions as the reference's roundings allow:
// 2u is exact, so fma(2, u, -u_prev) rounds exactly like (2.0 * u) - u_prev
// (leapfrog_rn, msolver.cpp:167,177); the instability guard !(|v| <= kGuard)
// is an integer compare of the magnitude bits (NaN and inf compare above).
__device__ __forceinline__ double leapfrog_lean(double u, double up, double dt2, double acc) {
  return __dadd_rn(__fma_rn(2.0, u, -up), __dmul_rn(dt2, acc));
}
__device__ __forceinline__ bool beyond_guard(double v) {
  return (static_cast<unsigned long long>(__double_as_longlong(v)) & 0x7fffffffffffffffull) >
         static_cast<unsigned long long>(__double_as_longlong(kGuard));
}

// 256-bit global accesses (sm_100: LDG.256 / STG.256), 32-byte aligned
__device__ __forceinline__ void ldg256(double (&v)[4], const double* p) {
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}
__device__ __forceinline__ void stg256(double* p, const double (&v)[4]) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
               : "memory");
}

// G.NP is the chunk width KC (multiple of 4); G.slot_st = 2 * KC * ldst
// (hi rows, then lo rows); G.slot_d = rows8(ktilde_max) * ldst (one dD tile).
// DREG: D_{k-1} of each warp's fragments in registers and one dD tile in
// smem (deeper rings); false: D_k and D_{k-1} tiles in smem (fewer registers).
// EPW > 0: EPW epilogue warps (after the consumers) do the leapfrog update.  The
// consumers hand GEMM2's accumulators over through the D tile that is dead
// after GEMM2(k) (acc_full / acc_empty mbarriers) and go straight on to layer
// k+1; the epilogue warps read U^k, U_prev^k from global memory with many loads
// in flight and store u_next, all under the next layer's GEMMs.  The state
// ring then carries GEMM1 operands only.  Same arithmetic, same bits.
template <int NCW, int NTW, int MTW, int MINB, bool DREG = true, int EPW = 0>
__global__ void __launch_bounds__(32 * (NCW + 2 + EPW), MINB) rom_cell_kstream(
    const CellMeta* __restrict__ cells, const CellIface* __restrict__ cif,
    const double* __restrict__ lad, double* ubar0, double* ubar1, double* inter0,
    double* inter1, double* __restrict__ flux, StepParams* P, int64_t n_local, K1Geom G) {
  extern __shared__ __align__(128) double smem[];
  double* lad_slots = smem;
  double* st_slots = lad_slots + G.NL * G.slot_lad;
  double* dbuf = st_slots + G.NU * G.slot_st;  // dD tile (DREG) or D_k, D_{k-1} tiles
  constexpr bool EPI = EPW > 0;
  // DREG with epilogue warps: the second tile is the accumulator hand-over tile (own
  // tile: the epilogue warps have a whole layer to finish); without DREG the
  // accumulators borrow the D tile that is dead after GEMM2(k)
  constexpr bool ACC_OWN = EPI && DREG;
  constexpr int ND = DREG && !EPI ? 1 : 2;
  uint64_t* bars = reinterpret_cast<uint64_t*>(dbuf + ND * G.slot_d + kSmemTailPad);
  uint64_t* full_lad = bars;
  uint64_t* empty_lad = bars + kMaxRing;
  uint64_t* full_st = bars + 2 * kMaxRing;
  uint64_t* empty_st = bars + 3 * kMaxRing;
  uint64_t* acc_full = bars + 4 * kMaxRing;  // EPW > 0: accumulator tile handed to the epilogue warps
  uint64_t* acc_empty = acc_full + 1;        // ... and consumed by them

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t n = P->base + n_local;
  const int cur = static_cast<int>(n & 1);
  const double* ubar_cur = cur ? ubar1 : ubar0;
  const double* inter_cur = cur ? inter1 : inter0;
  double* inter_nxt = cur ? inter0 : inter1;
  const double dt2 = P->dt2;
  const int KC = G.NP;
  const int64_t io_tile = static_cast<int64_t>(G.total_io) * G.ldst;
  const int64_t inter_tile = G.total_inter * G.ldst;

  {
    const int total = G.NL * G.slot_lad + G.NU * G.slot_st + ND * G.slot_d + kSmemTailPad;
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
      if (EPI) {
        mbar_init(acc_full, NCW);
        mbar_init(acc_empty, EPW);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
  pdl_k1_gate(warp);

  if (warp < 2) {
    // ============================== producers ==============================
    if (lane != 0) return;
    const bool ladders = warp == 0;
    const uint64_t pol = policy_evict_first();
    Ring rl(G.NL), rs(G.NU);
    for (int item = blockIdx.x; item < G.n_items; item += gridDim.x) {
      const int c = item / G.n_stiles;
      const int tile = item - c * G.n_stiles;
      const CellMeta cm = cells[c];
      const int kt = cm.kt, m = cm.m, ld = cm.ld;
      const int kt4 = (kt + 3) & ~3;
      // L2 prefetch of this CTA's next item (pflead = -1 only): at config 5 a
      // whole-item lead keeps ~90-115 MB of prefetched lines in flight, the L2
      // evicts them before the TMA reads them (DRAM reads 3.04 -> 4.31 GB per
      // K1 at S = 32) and K1 is 12% slower at S <= 8 (profiles/r01/k1_prefetch_c5.log)
      if (G.pflead < 0 && !(G.dbg & 16)) {
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
        // L^1, L^2, Lhat^2, ..., L^m, Lhat^m, each in KC-column chunks
        const double* L0 = lad + cm.lad_off;
        const int nmat = 2 * m - 1;
        const int nitem = item + gridDim.x;
        const bool window = G.pflead > 0 && !(G.dbg & 16);
        const CellMeta* nmp = window && nitem < G.n_items ? cells + nitem / G.n_stiles : nullptr;
        for (int j = 0; j < nmat; ++j) {
          if (window) {
            // windowed L2 prefetch: the matrix pflead ahead in this CTA's
            // stream (measured slower than none at every config 5 S)
            const int jj = j + G.pflead;
            if (jj < nmat) {
              prefetch_l2_big(L0 + static_cast<int64_t>(jj) * cm.lstride, static_cast<uint64_t>(cm.lstride) * 8u);
            } else if (nmp && jj - nmat < 2 * nmp->m - 1) {
              prefetch_l2_big(lad + nmp->lad_off + static_cast<int64_t>(jj - nmat) * nmp->lstride,
                              static_cast<uint64_t>(nmp->lstride) * 8u);
            }
          }
          const double* Lj = L0 + static_cast<int64_t>(j) * cm.lstride;
          for (int k0 = 0; k0 < kt4; k0 += KC) {
            const uint32_t bytes = static_cast<uint32_t>(min(KC, kt4 - k0)) * ld * 8u;
            mbar_wait_sleep(empty_lad + rl.slot, rl.phase ^ 1u);
            mbar_expect_tx(full_lad + rl.slot, bytes);
            bulk_g2s_hint(lad_slots + rl.slot * G.slot_lad, Lj + static_cast<int64_t>(k0) * ld, bytes,
                          full_lad + rl.slot, pol);
            rl.advance();
          }
        }
      } else {
        // GEMM1(k), k = 1..m: per chunk [U^{k+1} rows | U^k rows]; then for
        // k >= 2 the GEMM2 epilogue's operands, per row chunk [U^k | U_prev^k]
        const double* cur_tile = inter_cur + tile * inter_tile + cm.inter_row * G.ldst;
        const double* prev_tile = inter_nxt + tile * inter_tile + cm.inter_row * G.ldst;
        const double* ub_tile = ubar_cur + tile * io_tile;
        for (int k = 1; k <= m; ++k) {
          // epilogue warps read U_prev^k from global memory after GEMM2(k): start
          // it towards L2 now, two GEMMs ahead (U^k itself was just streamed)
          if (EPI && k >= 2 && !(G.dbg & 16))
            prefetch_l2_big(prev_tile + static_cast<int64_t>(k - 2) * kt * G.ldst,
                            static_cast<uint64_t>(kt) * G.ldst * 8u);
          for (int k0 = 0; k0 < kt4; k0 += KC) {
            const int rows = min(KC, kt - k0);
            double* dst = st_slots + rs.slot * G.slot_st;
            // byte count first (the barrier must expect before any complete_tx lands)
            uint32_t tx = k < m ? static_cast<uint32_t>(rows) * G.ldst * 8u : 0u;
            if (k == 1) {
              for (int li = 0; li < cm.nif; ++li) {
                const CellIface ci = cif[cm.if_begin + li];
                const int a = max(ci.block_off, k0), b = min(ci.block_off + ci.M, k0 + rows);
                if (a < b) tx += static_cast<uint32_t>(b - a) * G.ldst * 8u;
              }
            } else {
              tx += static_cast<uint32_t>(rows) * G.ldst * 8u;
            }
            mbar_wait_sleep(empty_st + rs.slot, rs.phase ^ 1u);
            mbar_expect_tx(full_st + rs.slot, tx);
            if (k < m)
              bulk_g2s(dst, cur_tile + (static_cast<int64_t>(k - 1) * kt + k0) * G.ldst,
                       static_cast<uint32_t>(rows) * G.ldst * 8u, full_st + rs.slot);
            double* lo = dst + KC * G.ldst;
            if (k == 1) {
              // layer 1 = interface values, face blocks [block_off, block_off + M)
              for (int li = 0; li < cm.nif; ++li) {
                const CellIface ci = cif[cm.if_begin + li];
                const int a = max(ci.block_off, k0), b = min(ci.block_off + ci.M, k0 + rows);
                if (a >= b) continue;
                bulk_g2s(lo + (a - k0) * G.ldst,
                         ub_tile + static_cast<int64_t>(ci.row_off + (a - ci.block_off)) * G.ldst,
                         static_cast<uint32_t>(b - a) * G.ldst * 8u, full_st + rs.slot);
              }
            } else {
              bulk_g2s(lo, cur_tile + (static_cast<int64_t>(k - 2) * kt + k0) * G.ldst,
                       static_cast<uint32_t>(rows) * G.ldst * 8u, full_st + rs.slot);
            }
            rs.advance();
          }
          if (k >= 2 && !EPI) {
            for (int k0 = 0; k0 < kt; k0 += KC) {
              const uint32_t bytes = static_cast<uint32_t>(min(KC, kt - k0)) * G.ldst * 8u;
              double* dst = st_slots + rs.slot * G.slot_st;
              mbar_wait_sleep(empty_st + rs.slot, rs.phase ^ 1u);
              mbar_expect_tx(full_st + rs.slot, 2 * bytes);
              bulk_g2s(dst, cur_tile + (static_cast<int64_t>(k - 2) * kt + k0) * G.ldst, bytes, full_st + rs.slot);
              bulk_g2s(dst + KC * G.ldst, prev_tile + (static_cast<int64_t>(k - 2) * kt + k0) * G.ldst, bytes,
                       full_st + rs.slot);
              rs.advance();
            }
          }
        }
      }
    }
    return;
  }

  if (EPI && warp >= 2 + NCW) {
    // ============================ epilogue warps ============================
    // u_next = leapfrog(U^k, U_prev^k, dt^2 acc) for layers 2..m of every item,
    // row-major over the tile (one double2 per lane, coalesced), UNR row
    // chunks of loads in flight per lane
    // loads in flight per lane, within the kernel's register cap
    constexpr int UNR = (NCW + 2 + EPW) * MINB <= 12 ? 7 : (NCW + 2 + EPW) * MINB <= 16 ? 5 : 3;
    const int ew = warp - 2 - NCW;
    const int ldst = G.ldst;
    const int c4n = G.ST >> 2;             // 32-byte groups per row (a power of two)
    const int c4s = 31 - __clz(c4n);
    uint32_t par = 0;
    bool bad = false;
    for (int item = blockIdx.x; item < G.n_items; item += gridDim.x) {
      const int c = item / G.n_stiles;
      const int tile = item - c * G.n_stiles;
      const CellMeta cm = cells[c];
      const int kt = cm.kt, m = cm.m;
      const int total = kt << c4s;
      for (int k = 2; k <= m; ++k) {
        const int64_t lay = tile * inter_tile + (cm.inter_row + static_cast<int64_t>(k - 2) * kt) * ldst;
        const double* uk = inter_cur + lay;
        double* un = inter_nxt + lay;  // U_prev^k in, u_next out (in place)
        const double* At = DREG ? dbuf + G.slot_d : dbuf + ((k - 1) & 1) * G.slot_d;
        bool waited = false;
        for (int i0 = ew * 32 + lane; i0 < total; i0 += EPW * 32 * UNR) {
          // operands first (256-bit loads, 2 * UNR in flight per lane): they do
          // not depend on the accumulators
          double u[UNR][4], up[UNR][4];
          int off[UNR];
#pragma unroll
          for (int q = 0; q < UNR; ++q) {
            const int idx = i0 + q * EPW * 32;
            off[q] = idx < total ? (idx >> c4s) * ldst + 4 * (idx & (c4n - 1)) : -1;
            if (off[q] >= 0) {
              ldg256(u[q], uk + off[q]);
              ldg256(up[q], un + off[q]);
            }
          }
          if (!waited) {  // first chunk of the layer: now the accumulators
            mbar_wait(acc_full, par);
            waited = true;
          }
#pragma unroll
          for (int q = 0; q < UNR; ++q) {
            if (off[q] < 0) continue;
            const double2 a0 = *reinterpret_cast<const double2*>(At + off[q]);
            const double2 a1 = *reinterpret_cast<const double2*>(At + off[q] + 2);
            double v[4];
            v[0] = leapfrog_lean(u[q][0], up[q][0], dt2, a0.x);
            v[1] = leapfrog_lean(u[q][1], up[q][1], dt2, a0.y);
            v[2] = leapfrog_lean(u[q][2], up[q][2], dt2, a1.x);
            v[3] = leapfrog_lean(u[q][3], up[q][3], dt2, a1.y);
            stg256(un + off[q], v);
            bad |= beyond_guard(v[0]) || beyond_guard(v[1]) || beyond_guard(v[2]) || beyond_guard(v[3]);
          }
        }
        if (!waited) mbar_wait(acc_full, par);
        par ^= 1u;
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty);
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0)
      atomicMin(reinterpret_cast<unsigned long long*>(&P->bad), static_cast<unsigned long long>(n + 1));
    return;
  }

  // ================================ consumers ================================
  const int cw = warp - 2;
  const int ws = cw % G.WM, wr = cw / G.WM;
  const int WN = G.WN;
  const int s_w = ws * NTW * 8;
  const int g = lane >> 2, t4 = lane & 3;
  const int ldst = G.ldst;
  Ring rl(G.NL), rs(G.NU);
  bool bad = false;
  // D tile hand-over between consumer warps: with one row group (WN == 1) a warp
  // reads only the source columns it wrote itself, so the warps never wait for
  // each other there (they stay coupled through the rings only)
  auto cons_sync = [&]() {
    if (WN > 1)
      named_sync(1, 32 * NCW);
    else
      __syncwarp();
  };
  uint32_t epi_par = 0;      // EPW > 0: parity of the next acc_empty completion
  bool epi_pending = false;  // ... an accumulator tile is with the epilogue warps
  // cycle accounting (diagnostic build): 0 item metadata, 1 GEMM1 ring waits, 2 GEMM1
  // issue, 3 D tile hand-over (barriers, smem / flux stores), 4 GEMM2 ladder waits,
  // 5 GEMM2 issue, 6 leapfrog operand waits, 7 leapfrog epilogue
  MSWB_PDECL;

  for (int item = blockIdx.x; item < G.n_items; item += gridDim.x) {
    const int c = item / G.n_stiles;
    const int tile = item - c * G.n_stiles;
    const CellMeta cm = cells[c];
    const int kt = cm.kt, m = cm.m, ld = cm.ld;
    const int kt4 = (kt + 3) & ~3;
    const int rtiles = (kt + 7) >> 3;
    const int mta = max(1, (rtiles - wr + WN - 1) / WN);  // this warp's live row tiles
    double* flux_c = flux + (static_cast<int64_t>(tile) * G.total_frows + cm.flux_row) * ldst;
    double* nxt_lay = inter_nxt + tile * inter_tile + cm.inter_row * ldst;
    MSWB_PUSE(kt + m + ld);
    MSWB_PMARK(0);

    double dprev[DREG ? MTW : 1][DREG ? NTW : 1][2];  // D_{k-1} of this warp's fragments
    for (int k = 1; k <= m; ++k) {
      double acc[MTW][NTW][2];
#pragma unroll
      for (int i = 0; i < MTW; ++i)
#pragma unroll
        for (int j = 0; j < NTW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      // ---- GEMM1: D_k = L^k (U^{k+1} - U^k) ----
      for (int k0 = 0; k0 < kt4; k0 += KC) {
        const int ksteps = min(KC, kt4 - k0) >> 2;
        mbar_wait(full_lad + rl.slot, rl.phase);
        mbar_wait(full_st + rs.slot, rs.phase);
        MSWB_PMARK(1);
        const double* hi = st_slots + rs.slot * G.slot_st;
        kchunk<MTW, NTW>(acc, hi, k < m ? 1.0 : 0.0, hi + KC * ldst, lad_slots + rl.slot * G.slot_lad, ld,
                         ldst, (G.dbg & 1) ? 0 : ksteps, rtiles, wr, WN, s_w, g, t4, mta);
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(empty_lad + rl.slot);
          mbar_arrive(empty_st + rs.slot);
        }
        rl.advance();
        rs.advance();
        MSWB_PMARK(2);
      }
      if constexpr (DREG) {
        if (k == 1) {
  #pragma unroll
          for (int i = 0; i < MTW; ++i) {
            const int nr = (wr + i * WN) * 8 + g;
  #pragma unroll
            for (int j = 0; j < NTW; ++j) {
              // compact rows (ldst < 8, S < 8): columns >= ldst are not stored
              if (wr + i * WN < rtiles && nr < kt && s_w + j * 8 + 2 * t4 < ldst)
                *reinterpret_cast<double2*>(flux_c + nr * ldst + s_w + j * 8 + 2 * t4) =
                    make_double2(acc[i][j][0], acc[i][j][1]);
              dprev[i][j][0] = acc[i][j][0];
              dprev[i][j][1] = acc[i][j][1];
            }
          }
          MSWB_PMARK(3);
          continue;
        }
        // every warp is done reading the previous dD (GEMM2 of layer k-1)
        if constexpr (EPI && !ACC_OWN) {
          if (epi_pending) {
            mbar_wait(acc_empty, epi_par);
            epi_par ^= 1u;
            epi_pending = false;
          }
        } else {
          cons_sync();
        }
  #pragma unroll
        for (int i = 0; i < MTW; ++i) {
          const int nr = (wr + i * WN) * 8 + g;
          const bool ok = wr + i * WN < rtiles && nr < kt;
  #pragma unroll
          for (int j = 0; j < NTW; ++j) {
            const int s = s_w + j * 8 + 2 * t4;
            const double2 v = make_double2(__dsub_rn(acc[i][j][0], dprev[i][j][0]),
                                           __dsub_rn(acc[i][j][1], dprev[i][j][1]));
            if (ok && s < ldst) *reinterpret_cast<double2*>(dbuf + nr * ldst + s) = v;
            dprev[i][j][0] = acc[i][j][0];
            dprev[i][j][1] = acc[i][j][1];
          }
        }
        cons_sync();  // dD_k complete
        MSWB_PMARK(3);
      } else {
        double* Dk = dbuf + (k & 1) * G.slot_d;
        // every warp is done reading the buffer D_k overwrites (see above)
        if constexpr (EPI) {
          if (epi_pending) {
            mbar_wait(acc_empty, epi_par);
            epi_par ^= 1u;
            epi_pending = false;
          }
        } else {
          cons_sync();
        }
#pragma unroll
        for (int i = 0; i < MTW; ++i) {
          const int nr = (wr + i * WN) * 8 + g;
          if (wr + i * WN >= rtiles || nr >= kt) continue;
#pragma unroll
          for (int j = 0; j < NTW; ++j) {
            const int s = s_w + j * 8 + 2 * t4;
            if (s >= ldst) continue;
            const double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
            *reinterpret_cast<double2*>(Dk + nr * ldst + s) = v;
            if (k == 1) *reinterpret_cast<double2*>(flux_c + nr * ldst + s) = v;
          }
        }
        cons_sync();  // D_k complete
        MSWB_PMARK(3);
        if (k < 2) continue;
      }

      // ---- GEMM2: acc = Lhat^k (D_k - D_{k-1}); u_next ----
#pragma unroll
      for (int i = 0; i < MTW; ++i)
#pragma unroll
        for (int j = 0; j < NTW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      for (int k0 = 0; k0 < kt4; k0 += KC) {
        const int ksteps = min(KC, kt4 - k0) >> 2;
        mbar_wait(full_lad + rl.slot, rl.phase);
        MSWB_PMARK(4);
        if constexpr (DREG)
          kchunk<MTW, NTW, false>(acc, dbuf + k0 * ldst, 1.0, nullptr, lad_slots + rl.slot * G.slot_lad, ld,
                                  ldst, (G.dbg & 1) ? 0 : ksteps, rtiles, wr, WN, s_w, g, t4, mta);
        else
          kchunk<MTW, NTW>(acc, dbuf + (k & 1) * G.slot_d + k0 * ldst, 1.0,
                           dbuf + ((k - 1) & 1) * G.slot_d + k0 * ldst, lad_slots + rl.slot * G.slot_lad, ld,
                           ldst, (G.dbg & 1) ? 0 : ksteps, rtiles, wr, WN, s_w, g, t4, mta);
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_lad + rl.slot);
        rl.advance();
        MSWB_PMARK(5);
      }
      // epilogue: U^k, U_prev^k arrive through the state ring in row chunks
      // (TMA, prefetched during the k-loop above); row tiles never straddle
      // a chunk (KC is a multiple of 8)
      if constexpr (EPI) {
        if constexpr (ACC_OWN) {
          // the hand-over tile is back from the epilogue warps
          if (epi_pending) {
            mbar_wait(acc_empty, epi_par);
            epi_par ^= 1u;
          }
        } else {
          // every warp is done reading the tile the accumulators go to
          cons_sync();
        }
        MSWB_PMARK(6);
        double* At = DREG ? dbuf + G.slot_d : dbuf + ((k - 1) & 1) * G.slot_d;
#pragma unroll
        for (int i = 0; i < MTW; ++i) {
          const int nr = (wr + i * WN) * 8 + g;
          if (wr + i * WN >= rtiles || nr >= kt) continue;
#pragma unroll
          for (int j = 0; j < NTW; ++j)
            *reinterpret_cast<double2*>(At + nr * ldst + s_w + j * 8 + 2 * t4) =
                make_double2(acc[i][j][0], acc[i][j][1]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_full);
        epi_pending = true;
        MSWB_PMARK(7);
        continue;
      }
      double* un = nxt_lay + static_cast<int64_t>(k - 2) * kt * ldst;
      for (int k0 = 0; k0 < kt; k0 += KC) {
        mbar_wait(full_st + rs.slot, rs.phase);
        MSWB_PMARK(6);
        const double* eu = st_slots + rs.slot * G.slot_st;
        const double* ep = eu + KC * ldst;
#pragma unroll
        for (int i = 0; i < MTW; ++i) {
          const int rt = wr + i * WN;
          const int nr = rt * 8 + g;
          if (rt >= rtiles || rt * 8 < k0 || rt * 8 >= k0 + KC || nr >= kt) continue;
#pragma unroll
          for (int j = 0; j < NTW; ++j) {
            const int s = s_w + j * 8 + 2 * t4;
            if (s >= ldst) continue;
            const double2 u = *reinterpret_cast<const double2*>(eu + (nr - k0) * ldst + s);
            const double2 up = *reinterpret_cast<const double2*>(ep + (nr - k0) * ldst + s);
            double2 v;
            v.x = leapfrog_rn(u.x, up.x, dt2, acc[i][j][0]);
            v.y = leapfrog_rn(u.y, up.y, dt2, acc[i][j][1]);
            *reinterpret_cast<double2*>(un + nr * ldst + s) = v;
            bad |= !(fabs(v.x) <= kGuard) || !(fabs(v.y) <= kGuard);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_st + rs.slot);
        rs.advance();
        MSWB_PMARK(7);
      }
    }
  }
#ifdef MSWB_K1_PROFILE
  if ((G.dbg & 8) && lane == 0 && G.prof)
    for (int i = 0; i < 8; ++i) atomicAdd(G.prof + i, static_cast<unsigned long long>(pt[i]));
#endif
  if (__any_sync(0xffffffffu, bad) && lane == 0)
    atomicMin(reinterpret_cast<unsigned long long*>(&P->bad), static_cast<unsigned long long>(n + 1));
}

}  // namespace pipe
}  // namespace mswb
