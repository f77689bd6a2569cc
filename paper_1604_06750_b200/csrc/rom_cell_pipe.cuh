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
//   warp 0       producer: one elected lane streams, in consumption order,
//                the ladder panels (L2 evict_first: read once per step) and
//                the state tiles U^1..U^m into two smem rings;
//                mbarrier expect_tx / complete_tx per slot;
//   warps 1..4   consumers: DMMA from smem; A fragments (X = U^{k+1}-U^k or
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

constexpr int kConsumerWarps = 4;
constexpr int kThreads = 32 * (kConsumerWarps + 1);
constexpr int kMaxRing = 8;

struct K1Geom {
  int ST;        // source tile width (8, 16, 32, 64)
  int n_stiles;  // source tiles
  int ldst;      // row stride of state / D tiles in HBM and smem (doubles)
  int NP;        // ladder panel width (columns, multiple of 8)
  int NL;        // ladder ring depth
  int NU;        // state ring depth
  int slot_lad;  // doubles per ladder slot (NP * max ld)
  int slot_st;   // doubles per state slot (kt4_max * ldst)
  int WM, WN;    // consumer warp grid (WM * WN = 4)
  int n_items;   // n_cells * n_stiles
  int total_io;
  int64_t total_inter;
};

// ---------------------------------------------------------------- PTX --------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
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

// ------------------------------------------------------------- kernel -------

// MTW: M-tiles (8-source groups) per consumer warp; NTP: max N-tiles per warp
// per ladder panel; NTA: max N-tiles per warp over the whole ktilde.
template <int MTW, int NTP, int NTA>
__global__ void __launch_bounds__(kThreads, 1) rom_cell_pipe(
    const CellMeta* __restrict__ cells, const CellIface* __restrict__ cif,
    const double* __restrict__ lad, double* ubar0, double* ubar1, double* inter0,
    double* inter1, double* __restrict__ flux, StepParams* P, int64_t n_local, K1Geom G) {
  extern __shared__ __align__(128) double smem[];
  double* lad_slots = smem;
  double* st_slots = lad_slots + G.NL * G.slot_lad;
  double* dbuf = st_slots + G.NU * G.slot_st;  // 2 D tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(dbuf + 2 * G.slot_st);
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
    const int total = G.NL * G.slot_lad + (G.NU + 2) * G.slot_st;
    for (int i = threadIdx.x; i < total; i += blockDim.x) smem[i] = 0.0;
    if (threadIdx.x == 0) {
      for (int i = 0; i < G.NL; ++i) {
        mbar_init(full_lad + i, 1);
        mbar_init(empty_lad + i, kConsumerWarps);
      }
      for (int i = 0; i < G.NU; ++i) {
        mbar_init(full_st + i, 1);
        mbar_init(empty_st + i, kConsumerWarps);
      }
    }
    // make the generic-proxy zero fill and barrier inits visible to TMA
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }

  if (warp == 0) {
    // =============================== producer ==============================
    if (lane != 0) return;
    const uint64_t pol = policy_evict_first();
    Ring rl(G.NL), rs(G.NU);
    for (int item = blockIdx.x; item < G.n_items; item += gridDim.x) {
      const int c = item / G.n_stiles;
      const int tile = item - c * G.n_stiles;
      const CellMeta cm = cells[c];
      const int kt = cm.kt, m = cm.m, ld = cm.ld;
      const double* L0 = lad + cm.lad_off;
      auto push_state = [&](int k) {  // U^k (1-based)
        mbar_wait(empty_st + rs.slot, rs.phase ^ 1u);
        double* dst = st_slots + rs.slot * G.slot_st;
        const uint32_t bytes = static_cast<uint32_t>(kt) * G.ldst * 8u;
        mbar_expect_tx(full_st + rs.slot, bytes);
        if (k == 1) {
          for (int li = 0; li < cm.nif; ++li) {
            const CellIface ci = cif[cm.if_begin + li];
            bulk_g2s(dst + ci.block_off * G.ldst,
                     ubar_cur + tile * io_tile + static_cast<int64_t>(ci.row_off) * G.ldst,
                     static_cast<uint32_t>(ci.M) * G.ldst * 8u, full_st + rs.slot);
          }
        } else {
          bulk_g2s(dst, inter_cur + tile * inter_tile + (cm.inter_row + static_cast<int64_t>(k - 2) * kt) * G.ldst,
                   bytes, full_st + rs.slot);
        }
        rs.advance();
      };
      auto push_ladder = [&](int j) {  // j-th matrix in consumption order
        const double* Lj = L0 + static_cast<int64_t>(j) * kt * ld;
        for (int p0 = 0; p0 < kt; p0 += G.NP) {
          const int cols = min(G.NP, kt - p0);
          const uint32_t bytes = static_cast<uint32_t>(cols) * ld * 8u;
          mbar_wait(empty_lad + rl.slot, rl.phase ^ 1u);
          mbar_expect_tx(full_lad + rl.slot, bytes);
          bulk_g2s_hint(lad_slots + rl.slot * G.slot_lad, Lj + static_cast<int64_t>(p0) * ld, bytes,
                        full_lad + rl.slot, pol);
          rl.advance();
        }
      };
      push_state(1);
      if (m > 1) push_state(2);
      push_ladder(0);  // L^1
      for (int k = 2; k <= m; ++k) {
        if (k < m) push_state(k + 1);
        push_ladder(2 * k - 3);  // L^k
        push_ladder(2 * k - 2);  // Lhat^k
      }
    }
    return;
  }

  // ================================ consumers ================================
  const int cw = warp - 1;
  const int wm = cw % G.WM, wn = cw / G.WM;
  const int s_w = wm * MTW * 8;  // first tile-local source column of this warp
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
    // ring slots of U^k (cur) and U^{k+1} (nxt), taken in ring order
    int slot_k = rs.slot;
    uint32_t phase_k = rs.phase;
    rs.advance();
    mbar_wait(full_st + slot_k, phase_k);

    for (int k = 1; k <= m; ++k) {
      const double* Uk = st_slots + slot_k * G.slot_st;
      const double* Ukp = nullptr;
      int slot_n = -1;
      uint32_t phase_n = 0;
      if (k < m) {
        slot_n = rs.slot;
        phase_n = rs.phase;
        rs.advance();
        mbar_wait(full_st + slot_n, phase_n);
        Ukp = st_slots + slot_n * G.slot_st;
      }
      // layer-k rows of this tile in HBM (u_prev in, u_next out)
      double* lay = inter_nxt + tile * inter_tile + (cm.inter_row + static_cast<int64_t>(k - 2) * kt) * ldst;

      // prefetch u_prev^k (k >= 2) for the GEMM2 epilogue
      double up[NTA][MTW][2];
      if (k >= 2) {
#pragma unroll
        for (int a = 0; a < NTA; ++a) {
          const int pan = a / NTP, j = a - pan * NTP;
          const int nn = pan * G.NP + (wn + j * G.WN) * 8 + 2 * t4;
          const bool in_panel = (wn + j * G.WN) * 8 < G.NP;
#pragma unroll
          for (int mt = 0; mt < MTW; ++mt) {
            const int s = s_w + mt * 8 + g;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int nr = nn + i;
              up[a][mt][i] = (in_panel && nr < kt) ? lay[nr * ldst + s] : 0.0;
            }
          }
        }
      }

      // ---- GEMM1: D_k = L^k (U^{k+1} - U^k), panels of the ladder ring ----
      double* Dk = dbuf + (k & 1) * G.slot_st;
      for (int p0 = 0; p0 < kt; p0 += G.NP) {
        const int cols = min(G.NP, kt - p0);
        const int ntiles = (cols + 7) >> 3;
        mbar_wait(full_lad + rl.slot, rl.phase);
        const double* Ls = lad_slots + rl.slot * G.slot_lad;
        double acc[NTP][MTW][2];
#pragma unroll
        for (int j = 0; j < NTP; ++j)
#pragma unroll
          for (int mt = 0; mt < MTW; ++mt) acc[j][mt][0] = acc[j][mt][1] = 0.0;
        for (int kk = 0; kk < ksteps; ++kk) {
          const int kr = 4 * kk + t4;
          double a[MTW];
#pragma unroll
          for (int mt = 0; mt < MTW; ++mt) {
            const int s = s_w + mt * 8 + g;
            const double ub = Uk[kr * ldst + s];
            const double ua = Ukp ? Ukp[kr * ldst + s] : 0.0;
            a[mt] = kr < kt ? ua - ub : 0.0;
          }
#pragma unroll
          for (int j = 0; j < NTP; ++j) {
            const int nt = wn + j * G.WN;
            if (nt < ntiles) {
              const double b = Ls[(nt * 8 + g) * ld + kr];
#pragma unroll
              for (int mt = 0; mt < MTW; ++mt) dmma(acc[j][mt], a[mt], b);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_lad + rl.slot);
        rl.advance();
        // epilogue: D_k tile (+ D_1 -> faces)
#pragma unroll
        for (int j = 0; j < NTP; ++j) {
          const int nt = wn + j * G.WN;
          if (nt >= ntiles) continue;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int nr = p0 + nt * 8 + 2 * t4 + i;
            if (nr >= kt) continue;
            int64_t frow = 0;
            if (k == 1) {
              int li = 0;
              while (li + 1 < cm.nif && cif[cm.if_begin + li + 1].block_off <= nr) ++li;
              const CellIface ci = cif[cm.if_begin + li];
              frow = (static_cast<int64_t>(ci.side) * G.n_stiles + tile) * io_tile +
                     static_cast<int64_t>(ci.row_off + nr - ci.block_off) * ldst;
            }
#pragma unroll
            for (int mt = 0; mt < MTW; ++mt) {
              const int s = s_w + mt * 8 + g;
              Dk[nr * ldst + s] = acc[j][mt][i];
              if (k == 1) flux[frow + s] = acc[j][mt][i];
            }
          }
        }
      }
      named_sync(1, 32 * kConsumerWarps);  // D_k complete (all rows, all warps)

      if (k >= 2) {
        // ---- GEMM2: acc = Lhat^k (D_k - D_{k-1}); u_next ----
        const double* Dp = dbuf + ((k - 1) & 1) * G.slot_st;
        constexpr int NPAN = NTA / NTP;
#pragma unroll
        for (int pan = 0; pan < NPAN; ++pan) {
          const int p0 = pan * G.NP;
          if (p0 >= kt) break;
          const int cols = min(G.NP, kt - p0);
          const int ntiles = (cols + 7) >> 3;
          mbar_wait(full_lad + rl.slot, rl.phase);
          const double* Ls = lad_slots + rl.slot * G.slot_lad;
          double acc[NTP][MTW][2];
#pragma unroll
          for (int j = 0; j < NTP; ++j)
#pragma unroll
            for (int mt = 0; mt < MTW; ++mt) acc[j][mt][0] = acc[j][mt][1] = 0.0;
          for (int kk = 0; kk < ksteps; ++kk) {
            const int kr = 4 * kk + t4;
            double a[MTW];
#pragma unroll
            for (int mt = 0; mt < MTW; ++mt) {
              const int s = s_w + mt * 8 + g;
              a[mt] = kr < kt ? Dk[kr * ldst + s] - Dp[kr * ldst + s] : 0.0;
            }
#pragma unroll
            for (int j = 0; j < NTP; ++j) {
              const int nt = wn + j * G.WN;
              if (nt < ntiles) {
                const double b = Ls[(nt * 8 + g) * ld + kr];
#pragma unroll
                for (int mt = 0; mt < MTW; ++mt) dmma(acc[j][mt], a[mt], b);
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(empty_lad + rl.slot);
          rl.advance();
#pragma unroll
          for (int j = 0; j < NTP; ++j) {
            const int nt = wn + j * G.WN;
            if (nt >= ntiles) continue;
#pragma unroll
            for (int mt = 0; mt < MTW; ++mt) {
              const int s = s_w + mt * 8 + g;
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                const int nr = p0 + nt * 8 + 2 * t4 + i;
                if (nr < kt) {
                  const double v = leapfrog_rn(Uk[nr * ldst + s], up[pan * NTP + j][mt][i], dt2, acc[j][mt][i]);
                  lay[nr * ldst + s] = v;
                  bad |= !(fabs(v) <= kGuard);
                }
              }
            }
          }
        }
        named_sync(1, 32 * kConsumerWarps);  // D_{k-1} free for reuse
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
}

}  // namespace pipe
}  // namespace mswb
