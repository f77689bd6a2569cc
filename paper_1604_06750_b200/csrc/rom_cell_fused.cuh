// K1''' rom_cell_fused: fused-layer cell kernel (sm_100a, fp64).
//
// The interior acceleration of layer k (msolver.cpp:133-145)
//   acc_k = Lhat^k ( L^k (U^{k+1} - U^k) - L^{k-1} (U^k - U^{k-1}) )
// is applied as ONE product with a doubled reduction dimension,
//   acc_k = [P_k | Q_k] [U^{k+1} - U^k ; U^{k-1} - U^k],
//   P_k = Lhat^k L^k,  Q_k = Lhat^k L^{k-1}   (precomputed once, rom_fuse_ladders)
// so a cell is m products (D_1 = L^1 (U^2 - U^1) for the faces, then one per
// layer) instead of 2m-1 short ones, with no D tiles in smem, no D epilogues
// and no CTA barriers even when warps split the rows.  Same flops and the
// same operator bytes (L^1 + (m-1) 2 ktilde^2 = (2m-1) ktilde^2); the
// re-association rounds differently from the reference's order (about one
// unit roundoff per product), well inside the 1e-10 trace gate, so this
// family is opt-in for bit-reproducibility (MSW_K1_FUSED=1) and bitwise equal
// only to itself.
//
// Rings: ladder ring = L^1 panels (leading dimension ld), then for each layer
// the transposed [P_k | Q_k] panels (column n = output row n, ld2 rows:
// [0, kt4) P part, [kt4, 2 kt4) Q part); state ring = U^1 (gathered from the
// faces), U^2, then per layer k >= 2: U^{k+1} (k < m), U_prev^k -- the
// rom_cell_pipe order; U^{k-1} is simply held one layer longer.
#pragma once

#include "rom_cell_pipe.cuh"

namespace mswb {
namespace pipe {

// Stage-form cycle accounting (diagnostic build -DMSWB_K1_PROFILE, run with
// MSW_K1_DEBUG=8): per consumer warp, cycles between marks summed into
// prof[0..7]: 0 cell metadata load, 1 first-slot waits of a cell, 2 GEMM issue,
// 3 accumulator drain, 4 stage-top ring waits, 5 U_prev wait, 6 epilogues and
// releases, 7 everything else.  MSWB_PUSE(x) makes the in-order issue wait for x.
// (macros MSWB_PDECL / MSWB_PMARK / MSWB_PUSE / MSWB_DBG: rom_cell_pipe.cuh)

// acc += A-panel x (scale*hi - lo) over ksteps k-steps (no zeroing): the
// rom_cell_pipe k-loop with an explicit A row offset.
template <int MTP, int NTW>
__device__ __forceinline__ void gemm_acc(double (&acc)[MTP][NTW][2], const double* __restrict__ hi,
                                         double scale, const double* __restrict__ lo,
                                         const double* __restrict__ Ls, int ld, int krow0, int ldst, int ksteps,
                                         int mtiles, int wr, int WR, int s_w, int g, int t4) {
  const double* pa[MTP];
#pragma unroll
  for (int i = 0; i < MTP; ++i) pa[i] = Ls + (min(wr + i * WR, mtiles - 1) * 8 + g) * ld + krow0 + t4;
  const int off_b = t4 * ldst + s_w + g;
  const double* pb_hi = hi + off_b;
  const double* pb_lo = lo + off_b;
  const int step_b = 4 * ldst;
  double a[MTP], b[NTW];
#pragma unroll
  for (int i = 0; i < MTP; ++i) a[i] = pa[i][0];
#pragma unroll
  for (int j = 0; j < NTW; ++j) b[j] = fma(scale, pb_hi[j * 8], -pb_lo[j * 8]);
  for (int kk = 0; kk < ksteps; ++kk) {
    double an[MTP], bn[NTW];
    pb_hi += step_b;
    pb_lo += step_b;
#pragma unroll
    for (int i = 0; i < MTP; ++i) an[i] = pa[i][4 * (kk + 1)];
#pragma unroll
    for (int j = 0; j < NTW; ++j) bn[j] = fma(scale, pb_hi[j * 8], -pb_lo[j * 8]);
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

// One X-stage of the single-panel form: B = scale*hi - lo (= X_j) is formed
// once per k-step and multiplies two A panels -- acc1 += A1 X_j (L^1 or P_j,
// finishing layer j) and, if TWO, acc2 += A2 X_j (-Q_{j+1}, starting layer
// j+1): 2 x MTP chains per warp sharing each B fragment.
//
// PK (packed last row tile): when the last row tile of a panel holds at most
// 4 valid rows (ktilde mod 8 in 1..4, e.g. 36 = 4 x 8 + 4) and the warp owns
// every row tile, the last tiles of BOTH panels share one DMMA: lanes of row
// half h1 (g >> 2 == h1) carry A1's leftover rows base + (g & 3), the other
// half A2's, into acc1[MTP-1] (acc2[MTP-1] is unused).  Every output element
// still accumulates the same products in the same k order (a DMMA output
// element depends only on its own A row), so the bits are those of the
// unpacked form; 2 MTP - 1 DMMAs per k-step instead of 2 MTP.
// MFA <= MF full-chain tiles and PKA (packed chain) are the ones this cell uses:
// the unrolled loops skip the others at compile time (they would only recompute
// a tile, or idle the packed chain in a cell without packable rows).
template <int MTP, int NTW, bool TWO, bool PK, int MFA, bool PKA>
__device__ __forceinline__ void gemm_stage_t(double (&acc1)[MTP][NTW][2], double (&acc2)[MTP][NTW][2],
                                             const double* __restrict__ hi, double scale,
                                             const double* __restrict__ lo, const double* __restrict__ A1, int ld1,
                                             const double* __restrict__ A2, int ld2, int ldst, int ksteps,
                                             int mtiles, int wr, int WR, int s_w, int g, int t4, int h1,
                                             int base) {
  constexpr int MF = PK ? MTP - 1 : MTP;  // tiles with one chain per panel
  static_assert(MFA <= MF, "live tiles");
  auto live = [](int i) { return i < MFA || (PK && PKA && i == MTP - 1); };
  const double* pa1[MTP];
  const double* pa2[MTP];
#pragma unroll
  for (int i = 0; i < MFA; ++i) {
    const int row = min(wr + i * WR, mtiles - 1) * 8 + g;
    pa1[i] = A1 + row * ld1 + t4;
    pa2[i] = A2 + row * ld2 + t4;
  }
  if (PK && PKA) {
    const int row = base + (g & 3);
    pa1[MTP - 1] = (!TWO || (g >> 2) == h1) ? A1 + row * ld1 + t4 : A2 + row * ld2 + t4;
  }
  const int off_b = t4 * ldst + s_w + g;
  const double* pb_hi = hi + off_b;
  const double* pb_lo = lo + off_b;
  const int step_b = 4 * ldst;
  double a1[MTP], a2[MTP], b[NTW];
#pragma unroll
  for (int i = 0; i < MTP; ++i) {
    if (!live(i)) continue;
    a1[i] = pa1[i][0];
    if (TWO && i < MFA) a2[i] = pa2[i][0];
  }
#pragma unroll
  for (int j = 0; j < NTW; ++j) b[j] = fma(scale, pb_hi[j * 8], -pb_lo[j * 8]);
  for (int kk = 0; kk < ksteps; ++kk) {
    double an1[MTP], an2[MTP], bn[NTW];
    pb_hi += step_b;
    pb_lo += step_b;
#pragma unroll
    for (int i = 0; i < MTP; ++i) {
      if (!live(i)) continue;
      an1[i] = pa1[i][4 * (kk + 1)];
      if (TWO && i < MFA) an2[i] = pa2[i][4 * (kk + 1)];
    }
#pragma unroll
    for (int j = 0; j < NTW; ++j) bn[j] = fma(scale, pb_hi[j * 8], -pb_lo[j * 8]);
#pragma unroll
    for (int i = 0; i < MTP; ++i) {
      if (!live(i)) continue;
#pragma unroll
      for (int j = 0; j < NTW; ++j) {
        dmma(acc1[i][j], a1[i], b[j]);
        if (TWO && i < MFA) dmma(acc2[i][j], a2[i], b[j]);
      }
    }
#pragma unroll
    for (int i = 0; i < MTP; ++i) {
      if (!live(i)) continue;
      a1[i] = an1[i];
      if (TWO && i < MFA) a2[i] = an2[i];
    }
#pragma unroll
    for (int j = 0; j < NTW; ++j) b[j] = bn[j];
  }
}

// Dispatch on the warp's live full-chain tiles `mfa` and on whether the cell
// packs its last row tile (both uniform per warp and cell): instances for MF,
// MF-1, MF-2 tiles, each with and without the packed chain.
template <int MTP, int NTW, bool TWO, bool PK, int MFA = (PK ? MTP - 1 : MTP)>
__device__ __forceinline__ void gemm_stage(double (&acc1)[MTP][NTW][2], double (&acc2)[MTP][NTW][2],
                                           const double* __restrict__ hi, double scale,
                                           const double* __restrict__ lo, const double* __restrict__ A1, int ld1,
                                           const double* __restrict__ A2, int ld2, int ldst, int ksteps,
                                           int mtiles, int wr, int WR, int s_w, int g, int t4, int h1, int base,
                                           int mfa, bool pka) {
  constexpr int MF = PK ? MTP - 1 : MTP;
  // the packed instances (config 3 at S = 64) keep the single full-size loop: with
  // the dispatch their step measured 3% slower (0.2674 -> 0.2753 ms), while the
  // small-tile instances gain 8-14% (config 2 0.0236 -> 0.0203 ms, config 3 S = 16
  // 0.132 -> 0.122 ms; profiles/r02/t/k1_live_tiles_ab.log)
  if constexpr (PK) {
    gemm_stage_t<MTP, NTW, TWO, PK, MF, true>(acc1, acc2, hi, scale, lo, A1, ld1, A2, ld2, ldst, ksteps, mtiles, wr,
                                              WR, s_w, g, t4, h1, base);
    return;
  }
  if constexpr (MFA > 1 && MFA > MF - 2) {
    if (mfa < MFA) {
      gemm_stage<MTP, NTW, TWO, PK, MFA - 1>(acc1, acc2, hi, scale, lo, A1, ld1, A2, ld2, ldst, ksteps, mtiles, wr,
                                             WR, s_w, g, t4, h1, base, mfa, pka);
      return;
    }
  }
  if (PK && !pka)
    gemm_stage_t<MTP, NTW, TWO, PK, MFA, false>(acc1, acc2, hi, scale, lo, A1, ld1, A2, ld2, ldst, ksteps, mtiles,
                                                wr, WR, s_w, g, t4, h1, base);
  else
    gemm_stage_t<MTP, NTW, TWO, PK, MFA, true>(acc1, acc2, hi, scale, lo, A1, ld1, A2, ld2, ldst, ksteps, mtiles,
                                               wr, WR, s_w, g, t4, h1, base);
}

// one-time precompute: lad2 (per cell, per layer k >= 2) = [P_k | Q_k]^T
// with P_k(n, j) = sum_l Lhat^k(n, l) L^k(l, j), Q_k likewise with L^{k-1};
// the ladders are symmetric, so L(l, j) = L(j, l) is read coalesced along j.
__global__ void rom_fuse_ladders(const CellMeta* __restrict__ cells, int nc, const double* __restrict__ lad,
                                 double* __restrict__ lad2) {
  const int c = blockIdx.x;
  if (c >= nc) return;
  const CellMeta cm = cells[c];
  const int kt = cm.kt, ld = cm.ld, ld2 = cm.ld2;
  const int kt4 = (kt + 3) & ~3;
  for (int k = 2; k <= cm.m; ++k) {
    const double* H = lad + cm.lad_off + static_cast<int64_t>(2 * k - 2) * cm.lstride;   // Lhat^k
    const double* Lk = lad + cm.lad_off + static_cast<int64_t>(2 * k - 3) * cm.lstride;  // L^k
    const double* Lm = lad + cm.lad_off + (k == 2 ? 0 : static_cast<int64_t>(2 * k - 5) * cm.lstride);  // L^{k-1}
    double* dst = lad2 + cm.lad2_off + static_cast<int64_t>(k - 2) * kt4 * ld2;
    for (int e = threadIdx.x; e < kt4 * ld2; e += blockDim.x) {
      const int n = e / ld2, kp = e - n * ld2;
      double v = 0.0;
      if (n < kt) {
        const double* L = nullptr;
        int j = -1;
        if (kp < kt) {
          L = Lk;
          j = kp;
        } else if (kp >= kt4 && kp - kt4 < kt) {
          L = Lm;
          j = kp - kt4;
        }
        if (L)
          for (int l = 0; l < kt; ++l) v = fma(H[n + static_cast<int64_t>(l) * ld], L[j + static_cast<int64_t>(l) * ld], v);
        if (kp >= kt4) v = -v;  // stored as -Q_k (exact), multiplied by X_{k-1} = U^k - U^{k-1}
      }
      dst[static_cast<int64_t>(n) * ld2 + kp] = v;
    }
  }
}

// Re-association sensitivity of the fused family, once per system: for every
// cell and layer k >= 2 the ratios ||Lhat^k||_F ||L^k||_F / ||P_k||_F and
// ||Lhat^k||_F ||L^{k-1}||_F / ||Q_k||_F (P_k = Lhat^k L^k, Q_k = Lhat^k L^{k-1}).
// They bound how much larger the rounding of the fused products is than the
// products themselves; well-conditioned ladders give O(1), the deep layers of
// real off-line ROMs give 10^3..10^5, where the fused form's traces drift from
// the reference order by far more than the problem's own rounding sensitivity
// (DESIGN.md §2).  The maximum (a positive double, ordered as its bit pattern)
// is atomically folded into *kappa.
__global__ void rom_fuse_sensitivity(const CellMeta* __restrict__ cells, int nc, const double* __restrict__ lad,
                                     const double* __restrict__ lad2, unsigned long long* kappa) {
  const int c = blockIdx.x;
  if (c >= nc) return;
  const CellMeta cm = cells[c];
  const int kt = cm.kt, ld = cm.ld, ld2 = cm.ld2;
  const int kt4 = (kt + 3) & ~3;
  __shared__ double red[5][256];
  double worst = 0.0;
  for (int k = 2; k <= cm.m; ++k) {
    const double* H = lad + cm.lad_off + static_cast<int64_t>(2 * k - 2) * cm.lstride;
    const double* Lk = lad + cm.lad_off + static_cast<int64_t>(2 * k - 3) * cm.lstride;
    const double* Lm = lad + cm.lad_off + (k == 2 ? 0 : static_cast<int64_t>(2 * k - 5) * cm.lstride);
    const double* PQ = lad2 + cm.lad2_off + static_cast<int64_t>(k - 2) * kt4 * ld2;
    double a[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int e = threadIdx.x; e < kt * kt; e += blockDim.x) {
      const int i = e / kt, j = e - i * kt;
      const double h = H[i + static_cast<int64_t>(j) * ld], l = Lk[i + static_cast<int64_t>(j) * ld];
      const double lm = Lm[i + static_cast<int64_t>(j) * ld];
      const double p = PQ[static_cast<int64_t>(i) * ld2 + j], q = PQ[static_cast<int64_t>(i) * ld2 + kt4 + j];
      a[0] += h * h;
      a[1] += l * l;
      a[2] += lm * lm;
      a[3] += p * p;
      a[4] += q * q;
    }
    for (int t = 0; t < 5; ++t) red[t][threadIdx.x] = a[t];
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w)
        for (int t = 0; t < 5; ++t) red[t][threadIdx.x] += red[t][threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const double nh = sqrt(red[0][0]), nl = sqrt(red[1][0]), nm = sqrt(red[2][0]);
      const double np = sqrt(red[3][0]), nq = sqrt(red[4][0]);
      worst = fmax(worst, np > 0.0 ? nh * nl / np : 0.0);
      worst = fmax(worst, nq > 0.0 ? nh * nm / nq : 0.0);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicMax(kappa, __double_as_longlong(worst));
}

template <int NCW, int NTW, int MTP, int MINB, bool PK = false>
__global__ void __launch_bounds__(32 * (NCW + 2), MINB) rom_cell_fused(
    const CellMeta* __restrict__ cells, const CellIface* __restrict__ cif,
    const double* __restrict__ lad, const double* __restrict__ lad2, double* ubar0, double* ubar1,
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
      const int kt = cm.kt, m = cm.m, ld = cm.ld, ld2 = cm.ld2;
      const int kt4 = (kt + 3) & ~3;
      {  // L2 prefetch of this CTA's next item
        const int nitem = item + gridDim.x;
        if (nitem < G.n_items) {
          const int nc = nitem / G.n_stiles;
          const int ntile = nitem - nc * G.n_stiles;
          const CellMeta nm = cells[nc];
          if (ladders) {
            prefetch_l2_big(lad + nm.lad_off, static_cast<uint64_t>(nm.lstride) * 8u);
            if (nm.m > 1)
              prefetch_l2_big(lad2 + nm.lad2_off,
                              static_cast<uint64_t>(nm.m - 1) * ((nm.kt + 3) & ~3) * nm.ld2 * 8u);
          } else if (nm.m > 1) {
            const uint64_t b = static_cast<uint64_t>(nm.m - 1) * nm.kt * G.ldst * 8u;
            prefetch_l2_big(inter_cur + ntile * inter_tile + nm.inter_row * G.ldst, b);
            prefetch_l2_big(inter_nxt + ntile * inter_tile + nm.inter_row * G.ldst, b);
          }
        }
      }
      if (ladders) {
        auto push = [&](const double* src, uint32_t bytes) {
          mbar_wait_sleep(empty_lad + rl.slot, rl.phase ^ 1u);
          if (MSWB_DBG(2)) {
            mbar_arrive(full_lad + rl.slot);
          } else {
            mbar_expect_tx(full_lad + rl.slot, bytes);
            bulk_g2s_hint(lad_slots + rl.slot * G.slot_lad, src, bytes, full_lad + rl.slot, pol);
          }
          rl.advance();
        };
        for (int p0 = 0; p0 < kt; p0 += G.NP)  // L^1 panels
          push(lad + cm.lad_off + static_cast<int64_t>(p0) * ld, static_cast<uint32_t>(min(G.NP, kt - p0)) * ld * 8u);
        for (int k = 2; k <= m; ++k) {  // [P_k | Q_k]^T panels
          const double* Mk = lad2 + cm.lad2_off + static_cast<int64_t>(k - 2) * kt4 * ld2;
          for (int p0 = 0; p0 < kt; p0 += G.NP)
            push(Mk + static_cast<int64_t>(p0) * ld2, static_cast<uint32_t>(min(G.NP, kt - p0)) * ld2 * 8u);
        }
      } else {
        const uint32_t bytes = static_cast<uint32_t>(kt) * G.ldst * 8u;
        const double* cur_tile = inter_cur + tile * inter_tile + cm.inter_row * G.ldst;
        const double* prev_tile = inter_nxt + tile * inter_tile + cm.inter_row * G.ldst;
        auto push = [&](const double* src) {
          mbar_wait_sleep(empty_st + rs.slot, rs.phase ^ 1u);
          if (MSWB_DBG(2)) {
            mbar_arrive(full_st + rs.slot);
          } else {
            mbar_expect_tx(full_st + rs.slot, bytes);
            bulk_g2s(st_slots + rs.slot * G.slot_st, src, bytes, full_st + rs.slot);
          }
          rs.advance();
        };
        mbar_wait_sleep(empty_st + rs.slot, rs.phase ^ 1u);  // U^1 from the faces
        if (MSWB_DBG(2)) mbar_arrive(full_st + rs.slot);
        else mbar_expect_tx(full_st + rs.slot, bytes);
        for (int li = 0; li < cm.nif && !MSWB_DBG(2); ++li) {
          const CellIface ci = cif[cm.if_begin + li];
          bulk_g2s(st_slots + rs.slot * G.slot_st + ci.block_off * G.ldst,
                   ubar_cur + tile * io_tile + static_cast<int64_t>(ci.row_off) * G.ldst,
                   static_cast<uint32_t>(ci.M) * G.ldst * 8u, full_st + rs.slot);
        }
        rs.advance();
        if (m > 1) push(cur_tile);  // U^2
        for (int k = 2; k <= m; ++k) {
          if (k < m) push(cur_tile + static_cast<int64_t>(k - 1) * kt * G.ldst);  // U^{k+1}
          push(prev_tile + static_cast<int64_t>(k - 2) * kt * G.ldst);          // U_prev^k
        }
      }
    }
    return;
  }

  // ================================ consumers ================================
  const int cw = warp - 2;
  const int ws = cw % G.WM, wr = cw / G.WM;
  const int WR = G.WN;
  const int s_w = ws * NTW * 8;
  const int g = lane >> 2, t4 = lane & 3;
  const int ldst = G.ldst;
  Ring rl(G.NL), rs(G.NU);
  bool bad = false;
  MSWB_PDECL;

  auto take = [&](int& slot, uint32_t& phase) {
    slot = rs.slot;
    phase = rs.phase;
    rs.advance();
  };
  auto release_st = [&](int slot) {
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_st + slot);
  };
  for (int item = blockIdx.x; item < G.n_items; item += gridDim.x) {
    const int c = item / G.n_stiles;
    const int tile = item - c * G.n_stiles;
    const CellMeta cm = cells[c];
    const int kt = cm.kt, m = cm.m, ld = cm.ld, ld2 = cm.ld2;
    const int kt4 = (kt + 3) & ~3;
    const int ksteps = MSWB_DBG(1) ? 0 : kt4 >> 2;
    double* flux_c = flux + (static_cast<int64_t>(tile) * G.total_frows + cm.flux_row) * ldst;
    MSWB_PMARK(7);
    MSWB_PUSE(kt + ld2);
    MSWB_PMARK(0);

    if (G.single && m > 1) {
      // ==== stage-ordered single-panel form (every layer is one ladder panel) ====
      // Stage j forms X_j = U^{j+1} - U^j once (X_m = -U^m) and multiplies it
      // by two panels: L^1 (j = 1, D_1) or P_j (finishing acc_j), and -Q_{j+1}
      // (starting acc_{j+1}).  acc_k = (-Q_k) X_{k-1} + P_k X_k, in that order.
      const int mtiles = (kt + 7) >> 3;
      // packed last row tile (see gemm_stage_t): layer k's leftover rows live
      // in row half (k & 1) of acc*[MTP-1]
      // (PK instances: WR == 1 and ktilde_max <= 8 (MTP - 1) + 4, so a cell
      // either packs or fits the MTP - 1 full tiles and the packed chain idles)
      const int base = (mtiles - 1) * 8;
      const bool pk = PK && kt - base <= 4;
      const int nfull = pk ? mtiles - 1 : mtiles;
      const int mfa = max(1, (nfull - wr + WR - 1) / WR);  // this warp's live full-chain tiles
      const int half = g >> 2;
      auto take_lad = [&](int& slot, uint32_t& phase) {
        slot = rl.slot;
        phase = rl.phase;
        rl.advance();
        mbar_wait(full_lad + slot, phase);
      };
      auto release_lad = [&](int slot) {
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_lad + slot);
      };
      int sU0, sU1, sU2 = -1, sP;  // U^j, U^{j+1}, U^{j+2}, U_prev^j
      uint32_t pU0, pU1, pU2 = 0, pP;
      int lc, ln;  // ladder slots: current stage's first panel, next layer's panel
      uint32_t plc, pln;
      double accA[MTP][NTW][2], accB[MTP][NTW][2];
#pragma unroll
      for (int i = 0; i < MTP; ++i)
#pragma unroll
        for (int j = 0; j < NTW; ++j) accA[i][j][0] = accA[i][j][1] = accB[i][j][0] = accB[i][j][1] = 0.0;
      take(sU0, pU0);
      mbar_wait(full_st + sU0, pU0);
      take(sU1, pU1);
      mbar_wait(full_st + sU1, pU1);
      take_lad(lc, plc);  // L^1
      take_lad(ln, pln);  // [P_2 | -Q_2]
      MSWB_PMARK(1);
      // ---- stage 1: D_1 = L^1 X_1 -> faces; acc_2 = -Q_2 X_1 ----
      gemm_stage<MTP, NTW, true, PK>(accA, accB, st_slots + sU1 * G.slot_st, 1.0, st_slots + sU0 * G.slot_st,
                                       lad_slots + lc * G.slot_lad, ld, lad_slots + ln * G.slot_lad + kt4, ld2,
                                       ldst, ksteps, nfull, wr, WR, s_w, g, t4, 1, base, mfa, pk);
      MSWB_PMARK(2);
      MSWB_PUSE(__double2hiint(accA[0][0][0]) + __double2hiint(accB[MTP - 2][0][1]));
      MSWB_PMARK(3);
      release_lad(lc);
      release_st(sU0);  // U^1
      if (!MSWB_DBG(4)) {
#pragma unroll
        for (int i = 0; i < MTP; ++i) {
          const int mt = wr + i * WR;
          const bool pki = PK && i == MTP - 1;
          const int nr = pki ? base + (g & 3) : mt * 8 + g;
          if (pki ? (!pk || half != 1 || nr >= kt) : (mt >= nfull || nr >= kt)) continue;
#pragma unroll
          for (int j = 0; j < NTW; ++j) {
            const int s = s_w + j * 8 + 2 * t4;
            if (s >= ldst) continue;
            *reinterpret_cast<double2*>(flux_c + nr * ldst + s) = make_double2(accA[i][j][0], accA[i][j][1]);
          }
        }
      }
      lc = ln;
      plc = pln;
      MSWB_PMARK(6);
      // ---- stages k = 2..m: acc_k += P_k X_k (then its leapfrog); acc_{k+1} = -Q_{k+1} X_k ----
      for (int k = 2; k <= m; ++k) {
        if (k < m) {
          take(sU2, pU2);  // U^{k+1}
          mbar_wait(full_st + sU2, pU2);
        }
        take(sP, pP);  // U_prev^k
#pragma unroll
        for (int i = 0; i < MTP; ++i)
#pragma unroll
          for (int j = 0; j < NTW; ++j) {
            if (PK && i == MTP - 1) {
              // the packed tile stays put: layer k's half keeps its -Q_k X_{k-1}
              // part, layer k-1's half (finished) restarts as layer k+1's
              if (half == ((k + 1) & 1)) accA[i][j][0] = accA[i][j][1] = 0.0;
            } else {
              accA[i][j][0] = accB[i][j][0];
              accA[i][j][1] = accB[i][j][1];
            }
            accB[i][j][0] = accB[i][j][1] = 0.0;
          }
        const double* Uk = st_slots + sU1 * G.slot_st;
        if (k < m) {
          take_lad(ln, pln);  // [P_{k+1} | -Q_{k+1}]
          MSWB_PMARK(4);
          gemm_stage<MTP, NTW, true, PK>(accA, accB, st_slots + sU2 * G.slot_st, 1.0, Uk,
                                           lad_slots + lc * G.slot_lad, ld2, lad_slots + ln * G.slot_lad + kt4, ld2,
                                           ldst, ksteps, nfull, wr, WR, s_w, g, t4, k & 1, base, mfa, pk);
        } else {
          MSWB_PMARK(4);
          gemm_stage<MTP, NTW, false, PK>(accA, accB, Uk, 0.0, Uk, lad_slots + lc * G.slot_lad, ld2,
                                            lad_slots + lc * G.slot_lad, ld2, ldst, ksteps, nfull, wr, WR, s_w, g,
                                            t4, k & 1, base, mfa, pk);
        }
        MSWB_PMARK(2);
        MSWB_PUSE(__double2hiint(accA[0][0][0]) + __double2hiint(accA[MTP - 1][0][1]));
        MSWB_PMARK(3);
        release_lad(lc);
        mbar_wait(full_st + sP, pP);
        MSWB_PMARK(5);
        const double* Up = st_slots + sP * G.slot_st;
        double* lay = inter_nxt + tile * inter_tile + (cm.inter_row + static_cast<int64_t>(k - 2) * kt) * ldst;
        // branch-free: every tile's operands are loaded (rows clamped into
        // the slot), all leapfrogs computed, only the stores are predicated --
        // the per-tile latency chains overlap instead of running back to back
        if (!MSWB_DBG(4)) {
          bool okt[MTP];
          int nrt[MTP];
          double2 u[MTP][NTW], up[MTP][NTW];
#pragma unroll
          for (int i = 0; i < MTP; ++i) {
            const int mt = wr + i * WR;
            const bool pki = PK && i == MTP - 1;
            const int nr = pki ? base + (g & 3) : mt * 8 + g;
            okt[i] = !(pki ? (!pk || half != (k & 1) || nr >= kt) : (mt >= nfull || nr >= kt));
            nrt[i] = okt[i] ? nr : 0;
#pragma unroll
            for (int j = 0; j < NTW; ++j) {
              const int s = min(s_w + j * 8 + 2 * t4, ldst - 2);
              u[i][j] = *reinterpret_cast<const double2*>(Uk + nrt[i] * ldst + s);
              up[i][j] = *reinterpret_cast<const double2*>(Up + nrt[i] * ldst + s);
            }
          }
#pragma unroll
          for (int i = 0; i < MTP; ++i)
#pragma unroll
            for (int j = 0; j < NTW; ++j) {
              const int s = s_w + j * 8 + 2 * t4;
              double2 v;
              v.x = leapfrog_rn(u[i][j].x, up[i][j].x, dt2, accA[i][j][0]);
              v.y = leapfrog_rn(u[i][j].y, up[i][j].y, dt2, accA[i][j][1]);
              const bool st = okt[i] && s < ldst;
              if (st) *reinterpret_cast<double2*>(lay + nrt[i] * ldst + s) = v;
              bad |= st && (!(fabs(v.x) <= kGuard) || !(fabs(v.y) <= kGuard));
            }
        }
        release_st(sU1);  // U^k
        release_st(sP);   // U_prev^k
        sU1 = sU2;
        pU1 = pU2;
        lc = ln;
        plc = pln;
        MSWB_PMARK(6);
      }
      continue;
    }

    int sA, sB = -1, sC = -1;  // U^{k-1}, U^k, U^{k+1}
    uint32_t pA, pB = 0, pC = 0;
    take(sA, pA);
    mbar_wait(full_st + sA, pA);
    if (m > 1) {
      take(sB, pB);
      mbar_wait(full_st + sB, pB);
    }
    // ---- D_1 = L^1 (U^2 - U^1)  [m == 1: -U^1] -> faces (step 2.1) ----
    {
      const double* U1 = st_slots + sA * G.slot_st;
      const double* U2 = m > 1 ? st_slots + sB * G.slot_st : U1;
      for (int p0 = 0; p0 < kt; p0 += G.NP) {
        const int mtiles = (min(G.NP, kt - p0) + 7) >> 3;
        mbar_wait(full_lad + rl.slot, rl.phase);
        double acc[MTP][NTW][2];
#pragma unroll
        for (int i = 0; i < MTP; ++i)
#pragma unroll
          for (int j = 0; j < NTW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        gemm_acc<MTP, NTW>(acc, U2, m > 1 ? 1.0 : 0.0, U1, lad_slots + rl.slot * G.slot_lad, ld, 0, ldst, ksteps,
                           mtiles, wr, WR, s_w, g, t4);
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_lad + rl.slot);
        rl.advance();
#pragma unroll
        for (int i = 0; i < MTP; ++i) {
          const int mt = wr + i * WR;
          const int nr = p0 + mt * 8 + g;
          if (mt >= mtiles || nr >= kt) continue;
#pragma unroll
          for (int j = 0; j < NTW; ++j) {
            const int s = s_w + j * 8 + 2 * t4;
            if (s >= ldst) continue;  // compact rows (ldst < 8, S < 8)
            *reinterpret_cast<double2*>(flux_c + nr * ldst + s) = make_double2(acc[i][j][0], acc[i][j][1]);
          }
        }
      }
    }
    if (m == 1) {
      release_st(sA);
      continue;
    }
    // ---- layers k = 2..m: acc_k = [P_k | Q_k] [U^{k+1} - U^k ; U^{k-1} - U^k] ----
    for (int k = 2; k <= m; ++k) {
      if (k < m) {
        take(sC, pC);
        mbar_wait(full_st + sC, pC);
      }
      int sP;
      uint32_t pP;
      take(sP, pP);
      const double* Ukm = st_slots + sA * G.slot_st;
      const double* Uk = st_slots + sB * G.slot_st;
      const double* Ukp = k < m ? st_slots + sC * G.slot_st : Uk;
      double* lay = inter_nxt + tile * inter_tile + (cm.inter_row + static_cast<int64_t>(k - 2) * kt) * ldst;
      bool up_ready = false;
      for (int p0 = 0; p0 < kt; p0 += G.NP) {
        const int mtiles = (min(G.NP, kt - p0) + 7) >> 3;
        mbar_wait(full_lad + rl.slot, rl.phase);
        const double* Ls = lad_slots + rl.slot * G.slot_lad;
        double acc[MTP][NTW][2];
#pragma unroll
        for (int i = 0; i < MTP; ++i)
#pragma unroll
          for (int j = 0; j < NTW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        gemm_acc<MTP, NTW>(acc, Ukp, k < m ? 1.0 : 0.0, Uk, Ls, ld2, 0, ldst, ksteps, mtiles, wr, WR, s_w, g, t4);
        gemm_acc<MTP, NTW>(acc, Uk, 1.0, Ukm, Ls, ld2, kt4, ldst, ksteps, mtiles, wr, WR, s_w, g, t4);
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_lad + rl.slot);
        rl.advance();
        if (!up_ready) {
          mbar_wait(full_st + sP, pP);
          up_ready = true;
        }
        const double* Up = st_slots + sP * G.slot_st;
#pragma unroll
        for (int i = 0; i < MTP; ++i) {
          const int mt = wr + i * WR;
          const int nr = p0 + mt * 8 + g;
          if (mt >= mtiles || nr >= kt) continue;
#pragma unroll
          for (int j = 0; j < NTW; ++j) {
            const int s = s_w + j * 8 + 2 * t4;
            if (s >= ldst) continue;
            const double2 u = *reinterpret_cast<const double2*>(Uk + nr * ldst + s);
            const double2 up = *reinterpret_cast<const double2*>(Up + nr * ldst + s);
            double2 v;
            v.x = leapfrog_rn(u.x, up.x, dt2, acc[i][j][0]);
            v.y = leapfrog_rn(u.y, up.y, dt2, acc[i][j][1]);
            *reinterpret_cast<double2*>(lay + nr * ldst + s) = v;
            bad |= !(fabs(v.x) <= kGuard) || !(fabs(v.y) <= kGuard);
          }
        }
      }
      release_st(sP);  // U_prev^k
      release_st(sA);  // U^{k-1}
      sA = sB;
      pA = pB;
      sB = sC;
      pB = pC;
    }
    release_st(sA);  // U^m
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0)
    atomicMin(reinterpret_cast<unsigned long long*>(&P->bad), static_cast<unsigned long long>(n + 1));
#ifdef MSWB_K1_PROFILE
  MSWB_PMARK(7);
  if ((G.dbg & 8) && lane == 0 && G.prof)
    for (int i = 0; i < 8; ++i) atomicAdd(G.prof + i, static_cast<unsigned long long>(pt[i]));
#endif
}

}  // namespace pipe
}  // namespace mswb
