// K1'''' rom_cell_fks: K-streaming fused-layer cell kernel for large ktilde
// (sm_100a, fp64).
//
// The fused-layer algebra of rom_cell_fused.cuh (acc_k = P_k X_k - Q_k X_{k-1},
// X_k = U^{k+1} - U^k, P_k = Lhat^k L^k, Q_k = Lhat^k L^{k-1}) in the stage
// order, with the reduction dimension streamed as in rom_cell_kstream.cuh:
//   stage j = 1..m: for each KC-row chunk of X_j (state ring: U^{j+1} rows |
//   U^j rows, the kstream GEMM1 feed), the ladder ring delivers the matching
//   KC-column chunks of A1 = (j == 1 ? L^1 : P_j) and A2 = -Q_{j+1} (j < m);
//   every warp accumulates acc1 += A1 X_j, acc2 += A2 X_j for the output rows
//   and sources it owns.  After the stage, acc1 is D_1 (-> faces) or the
//   finished acc_j (-> leapfrog epilogue, U^j / U_prev^j row chunks through
//   the state ring, the kstream epilogue feed); acc2 becomes acc1.
// Every output row lives in one warp's registers, so there are no D tiles,
// no named barriers and no cross-warp exchange; each B fragment (one DFMA)
// feeds two DMMA chains.  Operator: L^1 from the ladder array, P_k and -Q_k
// column-major in lad3 (rom_fuse_ladders_cm), same bytes as the reference's
// 2m - 1 ladders.  The accumulation order (-Q_k X_{k-1}, then P_k X_k, each
// over ascending k) is the single-panel rom_cell_fused order.
#pragma once

#include "rom_cell_kstream.cuh"

namespace mswb {
namespace pipe {

// lad3 (per cell, per layer k >= 2): P_k then -Q_k, column-major (element
// (n, j) at j * ld + n), lstride doubles each, zero padded like the ladders.
__global__ void rom_fuse_ladders_cm(const CellMeta* __restrict__ cells, int nc, const double* __restrict__ lad,
                                    double* __restrict__ lad3) {
  const int c = blockIdx.x;
  if (c >= nc) return;
  const CellMeta cm = cells[c];
  const int kt = cm.kt, ld = cm.ld;
  const int kt4 = (kt + 3) & ~3;
  for (int k = 2; k <= cm.m; ++k) {
    const double* H = lad + cm.lad_off + static_cast<int64_t>(2 * k - 2) * cm.lstride;   // Lhat^k
    const double* Lk = lad + cm.lad_off + static_cast<int64_t>(2 * k - 3) * cm.lstride;  // L^k
    const double* Lm = lad + cm.lad_off + (k == 2 ? 0 : static_cast<int64_t>(2 * k - 5) * cm.lstride);  // L^{k-1}
    double* dP = lad3 + cm.lad3_off + static_cast<int64_t>(2 * (k - 2)) * cm.lstride;
    double* dQ = dP + cm.lstride;
    for (int e = threadIdx.x; e < kt4 * ld; e += blockDim.x) {
      const int j = e / ld, n = e - j * ld;  // column j, row n
      double p = 0.0, q = 0.0;
      if (n < kt && j < kt) {
        for (int l = 0; l < kt; ++l) {
          const double h = H[n + static_cast<int64_t>(l) * ld];
          p = fma(h, Lk[j + static_cast<int64_t>(l) * ld], p);
          q = fma(h, Lm[j + static_cast<int64_t>(l) * ld], q);
        }
      }
      dP[e] = p;
      dQ[e] = -q;
    }
  }
}

// acc1 += A1[:, chunk] X, acc2 += A2[:, chunk] X (TWO), X = scale*hi - lo,
// over `ksteps` k-steps; A(n, k) = A[k * ld + n].
template <int MTW, int NTW, bool TWO>
__device__ __forceinline__ void kchunk2(double (&acc1)[MTW][NTW][2], double (&acc2)[MTW][NTW][2],
                                        const double* __restrict__ hi, double scale, const double* __restrict__ lo,
                                        const double* __restrict__ A1, const double* __restrict__ A2, int ld,
                                        int ldst, int ksteps, int rtiles, int wr, int WN, int s_w, int g, int t4) {
  const double* pa1[MTW];
  const double* pa2[MTW];
#pragma unroll
  for (int i = 0; i < MTW; ++i) {
    const int off = t4 * ld + min(wr + i * WN, rtiles - 1) * 8 + g;
    pa1[i] = A1 + off;
    pa2[i] = A2 + off;
  }
  const int off_b = t4 * ldst + s_w + g;
  const double* pb_hi = hi + off_b;
  const double* pb_lo = lo + off_b;
  const int step_a = 4 * ld, step_b = 4 * ldst;
  double a1[MTW], a2[MTW], b[NTW];
#pragma unroll
  for (int i = 0; i < MTW; ++i) {
    a1[i] = pa1[i][0];
    if (TWO) a2[i] = pa2[i][0];
  }
#pragma unroll
  for (int j = 0; j < NTW; ++j) b[j] = fma(scale, pb_hi[j * 8], -pb_lo[j * 8]);
  for (int kk = 0; kk < ksteps; ++kk) {
    double an1[MTW], an2[MTW], bn[NTW];
    pb_hi += step_b;
    pb_lo += step_b;
    // one k-step of look-ahead; the last one reads past the chunk (inside
    // the smem allocation) and is discarded
#pragma unroll
    for (int i = 0; i < MTW; ++i) {
      an1[i] = pa1[i][(kk + 1) * step_a];
      if (TWO) an2[i] = pa2[i][(kk + 1) * step_a];
    }
#pragma unroll
    for (int j = 0; j < NTW; ++j) bn[j] = fma(scale, pb_hi[j * 8], -pb_lo[j * 8]);
#pragma unroll
    for (int i = 0; i < MTW; ++i)
#pragma unroll
      for (int j = 0; j < NTW; ++j) {
        dmma(acc1[i][j], a1[i], b[j]);
        if (TWO) dmma(acc2[i][j], a2[i], b[j]);
      }
#pragma unroll
    for (int i = 0; i < MTW; ++i) {
      a1[i] = an1[i];
      if (TWO) a2[i] = an2[i];
    }
#pragma unroll
    for (int j = 0; j < NTW; ++j) b[j] = bn[j];
  }
}

// G.NP = KC (multiple of 8); G.slot_lad = 2 * KC * ld_max (A1 chunk, then A2
// chunk); G.slot_st = 2 * KC * ldst.
template <int NCW, int NTW, int MTW, int MINB>
__global__ void __launch_bounds__(32 * (NCW + 2), MINB) rom_cell_fks(
    const CellMeta* __restrict__ cells, const CellIface* __restrict__ cif,
    const double* __restrict__ lad, const double* __restrict__ lad3, double* ubar0, double* ubar1,
    double* inter0, double* inter1, double* __restrict__ flux, StepParams* P, int64_t n_local, K1Geom G) {
  extern __shared__ __align__(128) double smem[];
  double* lad_slots = smem;
  double* st_slots = lad_slots + G.NL * G.slot_lad;
  uint64_t* bars = reinterpret_cast<uint64_t*>(st_slots + G.NU * G.slot_st + kSmemTailPad);
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
  const int KC = G.NP;
  const int64_t io_tile = static_cast<int64_t>(G.total_io) * G.ldst;
  const int64_t inter_tile = G.total_inter * G.ldst;

  {
    const int total = G.NL * G.slot_lad + G.NU * G.slot_st + kSmemTailPad;
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
      if (ladders) {
        // stage j: [A1 chunk | A2 chunk] per KC columns
        for (int j = 1; j <= m; ++j) {
          const double* A1 = j == 1 ? lad + cm.lad_off
                                    : lad3 + cm.lad3_off + static_cast<int64_t>(2 * (j - 2)) * cm.lstride;
          const double* A2 = j < m ? lad3 + cm.lad3_off + static_cast<int64_t>(2 * (j - 1) + 1) * cm.lstride
                                   : nullptr;
          for (int k0 = 0; k0 < kt4; k0 += KC) {
            const uint32_t bytes = static_cast<uint32_t>(min(KC, kt4 - k0)) * ld * 8u;
            mbar_wait_sleep(empty_lad + rl.slot, rl.phase ^ 1u);
            mbar_expect_tx(full_lad + rl.slot, A2 ? 2 * bytes : bytes);
            double* dst = lad_slots + rl.slot * G.slot_lad;
            bulk_g2s_hint(dst, A1 + static_cast<int64_t>(k0) * ld, bytes, full_lad + rl.slot, pol);
            if (A2) bulk_g2s_hint(dst + KC * ld, A2 + static_cast<int64_t>(k0) * ld, bytes, full_lad + rl.slot, pol);
            rl.advance();
          }
        }
      } else {
        // the rom_cell_kstream state feed: per stage [U^{j+1} rows | U^j rows]
        // chunks; for j >= 2 then the epilogue's [U^j | U_prev^j] row chunks
        const double* cur_tile = inter_cur + tile * inter_tile + cm.inter_row * G.ldst;
        const double* prev_tile = inter_nxt + tile * inter_tile + cm.inter_row * G.ldst;
        const double* ub_tile = ubar_cur + tile * io_tile;
        for (int k = 1; k <= m; ++k) {
          for (int k0 = 0; k0 < kt4; k0 += KC) {
            const int rows = min(KC, kt - k0);
            double* dst = st_slots + rs.slot * G.slot_st;
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
          if (k >= 2) {
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

  // ================================ consumers ================================
  const int cw = warp - 2;
  const int ws = cw % G.WM, wr = cw / G.WM;
  const int WN = G.WN;
  const int s_w = ws * NTW * 8;
  const int g = lane >> 2, t4 = lane & 3;
  const int ldst = G.ldst;
  Ring rl(G.NL), rs(G.NU);
  bool bad = false;

  for (int item = blockIdx.x; item < G.n_items; item += gridDim.x) {
    const int c = item / G.n_stiles;
    const int tile = item - c * G.n_stiles;
    const CellMeta cm = cells[c];
    const int kt = cm.kt, m = cm.m, ld = cm.ld;
    const int kt4 = (kt + 3) & ~3;
    const int rtiles = (kt + 7) >> 3;
    double* flux_c = flux + (static_cast<int64_t>(tile) * G.total_frows + cm.flux_row) * ldst;
    double* nxt_lay = inter_nxt + tile * inter_tile + cm.inter_row * ldst;

    double acc1[MTW][NTW][2], acc2[MTW][NTW][2];
#pragma unroll
    for (int i = 0; i < MTW; ++i)
#pragma unroll
      for (int j = 0; j < NTW; ++j) acc1[i][j][0] = acc1[i][j][1] = acc2[i][j][0] = acc2[i][j][1] = 0.0;
    for (int jst = 1; jst <= m; ++jst) {
      for (int k0 = 0; k0 < kt4; k0 += KC) {
        const int ksteps = min(KC, kt4 - k0) >> 2;
        mbar_wait(full_lad + rl.slot, rl.phase);
        mbar_wait(full_st + rs.slot, rs.phase);
        const double* hi = st_slots + rs.slot * G.slot_st;
        const double* A1 = lad_slots + rl.slot * G.slot_lad;
        if (jst < m)
          kchunk2<MTW, NTW, true>(acc1, acc2, hi, 1.0, hi + KC * ldst, A1, A1 + KC * ld, ld, ldst, ksteps, rtiles,
                                  wr, WN, s_w, g, t4);
        else
          kchunk2<MTW, NTW, false>(acc1, acc2, hi, 0.0, hi + KC * ldst, A1, A1, ld, ldst, ksteps, rtiles, wr, WN,
                                   s_w, g, t4);
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(empty_lad + rl.slot);
          mbar_arrive(empty_st + rs.slot);
        }
        rl.advance();
        rs.advance();
      }
      if (jst == 1) {
        // D_1 -> faces (step 2.1)
#pragma unroll
        for (int i = 0; i < MTW; ++i) {
          const int nr = (wr + i * WN) * 8 + g;
          if (wr + i * WN >= rtiles || nr >= kt) continue;
#pragma unroll
          for (int j = 0; j < NTW; ++j) {
            const int s = s_w + j * 8 + 2 * t4;
            if (s >= ldst) continue;  // compact rows
            *reinterpret_cast<double2*>(flux_c + nr * ldst + s) = make_double2(acc1[i][j][0], acc1[i][j][1]);
          }
        }
      } else {
        // epilogue of layer jst: U^j, U_prev^j in row chunks through the state ring
        double* un = nxt_lay + static_cast<int64_t>(jst - 2) * kt * ldst;
        for (int k0 = 0; k0 < kt; k0 += KC) {
          mbar_wait(full_st + rs.slot, rs.phase);
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
              v.x = leapfrog_rn(u.x, up.x, dt2, acc1[i][j][0]);
              v.y = leapfrog_rn(u.y, up.y, dt2, acc1[i][j][1]);
              *reinterpret_cast<double2*>(un + nr * ldst + s) = v;
              bad |= !(fabs(v.x) <= kGuard) || !(fabs(v.y) <= kGuard);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(empty_st + rs.slot);
          rs.advance();
        }
      }
#pragma unroll
      for (int i = 0; i < MTW; ++i)
#pragma unroll
        for (int j = 0; j < NTW; ++j) {
          acc1[i][j][0] = acc2[i][j][0];
          acc1[i][j][1] = acc2[i][j][1];
          acc2[i][j][0] = acc2[i][j][1] = 0.0;
        }
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0)
    atomicMin(reinterpret_cast<unsigned long long*>(&P->bad), static_cast<unsigned long long>(n + 1));
}

}  // namespace pipe
}  // namespace mswb
