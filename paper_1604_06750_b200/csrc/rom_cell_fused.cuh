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

// Consumer cycle accounting of the stage form (build with -DMSWB_K1_PROFILE,
// run with MSW_K1_DEBUG=8): prof[0] state-ring waits, [1] ladder-ring waits,
// [2] GEMM issue, [3] epilogues (D_1 stores, leapfrog), [4] per-item total,
// [5] items -- summed over consumer warps (lane 0).
#ifdef MSWB_K1_PROFILE
#define MSWB_FP(slot, ...)            \
  do {                                \
    const long long _t0 = clock64();  \
    __VA_ARGS__;                      \
    fprof[slot] += clock64() - _t0;   \
  } while (0)
#else
#define MSWB_FP(slot, ...) \
  do {                     \
    __VA_ARGS__;           \
  } while (0)
#endif

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
template <int MTP, int NTW, bool TWO>
__device__ __forceinline__ void gemm_stage(double (&acc1)[MTP][NTW][2], double (&acc2)[MTP][NTW][2],
                                           const double* __restrict__ hi, double scale,
                                           const double* __restrict__ lo, const double* __restrict__ A1, int ld1,
                                           const double* __restrict__ A2, int ld2, int ldst, int ksteps,
                                           int mtiles, int wr, int WR, int s_w, int g, int t4) {
  const double* pa1[MTP];
  const double* pa2[MTP];
#pragma unroll
  for (int i = 0; i < MTP; ++i) {
    const int row = min(wr + i * WR, mtiles - 1) * 8 + g;
    pa1[i] = A1 + row * ld1 + t4;
    pa2[i] = A2 + row * ld2 + t4;
  }
  const int off_b = t4 * ldst + s_w + g;
  const double* pb_hi = hi + off_b;
  const double* pb_lo = lo + off_b;
  const int step_b = 4 * ldst;
  double a1[MTP], a2[MTP], b[NTW];
#pragma unroll
  for (int i = 0; i < MTP; ++i) {
    a1[i] = pa1[i][0];
    if (TWO) a2[i] = pa2[i][0];
  }
#pragma unroll
  for (int j = 0; j < NTW; ++j) b[j] = fma(scale, pb_hi[j * 8], -pb_lo[j * 8]);
  for (int kk = 0; kk < ksteps; ++kk) {
    double an1[MTP], an2[MTP], bn[NTW];
    pb_hi += step_b;
    pb_lo += step_b;
#pragma unroll
    for (int i = 0; i < MTP; ++i) {
      an1[i] = pa1[i][4 * (kk + 1)];
      if (TWO) an2[i] = pa2[i][4 * (kk + 1)];
    }
#pragma unroll
    for (int j = 0; j < NTW; ++j) bn[j] = fma(scale, pb_hi[j * 8], -pb_lo[j * 8]);
#pragma unroll
    for (int i = 0; i < MTP; ++i)
#pragma unroll
      for (int j = 0; j < NTW; ++j) {
        dmma(acc1[i][j], a1[i], b[j]);
        if (TWO) dmma(acc2[i][j], a2[i], b[j]);
      }
#pragma unroll
    for (int i = 0; i < MTP; ++i) {
      a1[i] = an1[i];
      if (TWO) a2[i] = an2[i];
    }
#pragma unroll
    for (int j = 0; j < NTW; ++j) b[j] = bn[j];
  }
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

// ---- interface step fused into the cell kernel (IFUSE) --------------------
// K2 (rom_iface_step) needs D_1 of both cells of an interface, so it ran as a
// second kernel after every cell's D_1 was written.  With IFUSE, two extra
// "interface warps" per CTA finish each interface inside K1: after a cell's
// consumers have stored its D_1 faces (and fenced them), the interface warps
// bump a per-(interface, source tile) arrival counter; the cell that arrives
// second (or the only cell of a single-sided interface) performs the
// interface update -- the same arithmetic, in the same order, as K2, so the
// results are bitwise those of the K1 + K2 pair -- while the consumers go on
// with the cell's interior layers.  The D_1 face round trip through DRAM and
// the separate launch go away; the partner's D_1 is usually an L2 hit.
// Counters only ever increase (two arrivals per step), so no reset is needed.
constexpr int kIfSlots = 8;     // cells in flight between consumers and interface warps
constexpr int kMaxCellIf = 32;  // interfaces per cell handled by the fused path
constexpr int kFastIf = 8;      // interfaces per cell on the register path (M <= 6)

struct IfuseArgs {
  const IfaceMeta* ifs;
  const double* mass;
  const double* g;
  const RcvTerm* rterms;
  const double* q;
  unsigned* cnt;        // [n_ifaces][n_stiles] arrival counters
  int R;
  int M_max;
  int fuse_rcv;
  int total_io;
  int S;                // user-visible sources
};

// smem bytes the IFUSE path adds after the ring barriers
__host__ __device__ constexpr size_t ifuse_smem_bytes(int M_max, int ST) {
  return 2 * kIfSlots * sizeof(uint64_t) + kIfSlots * (kMaxCellIf + 1) * sizeof(int) + 16 +
         static_cast<size_t>(2) * M_max * ST * sizeof(double) + kFastIf * 36 * sizeof(double) +
         kFastIf * sizeof(IfaceMeta);
}

// One (interface, source tile) update with NT threads (tid in [0, NT)),
// rom_iface_step's operations: phi = D1_i + D1_j (+ w g), ubar_next =
// (2 ubar - ubar_prev) + dt^2 mass phi, fused single-interface receivers.
template <int NT>
__device__ __forceinline__ bool iface_update(const IfuseArgs& A, int f, int tile, int ST, int ldst,
                                             int64_t total_frows, const double* __restrict__ flux,
                                             const double* ub, double* ubn, double* phi, double* un,
                                             StepParams* P, int64_t n, int tid, int bar_id) {
  const IfaceMeta im = A.ifs[f];
  const int M = im.M;
  const bool full = ldst >= ST;
  const int H = full ? ST / 2 : ldst / 2;
  const int MH = M * H;
  const double dt2 = P->dt2;
  const int64_t wi = (n - P->n0) * P->w_stride;
  const int64_t base = (static_cast<int64_t>(tile) * A.total_io + im.row_off) * ldst;
  const int64_t ft = static_cast<int64_t>(tile) * total_frows;
  for (int idx = tid; idx < MH; idx += NT) {
    const int r = idx / H, sp = 2 * (idx - r * H);
    double2 v = __ldcg(reinterpret_cast<const double2*>(flux + (ft + im.frow_i + r) * ldst + sp));
    if (im.two_sided) {
      const double2 vj = __ldcg(reinterpret_cast<const double2*>(flux + (ft + im.frow_j + r) * ldst + sp));
      v.x = v.x + vj.x;
      v.y = v.y + vj.y;
    }
    if (im.has_src) {
      const int gs = tile * ST + sp;
      const double2 gg = *reinterpret_cast<const double2*>(A.g + base + static_cast<int64_t>(r) * ldst + sp);
      const double w0 = P->w[wi + (P->w_stride > 1 ? min(gs, A.S - 1) : 0)];
      const double w1 = P->w[wi + (P->w_stride > 1 ? min(gs + 1, A.S - 1) : 0)];
      v.x = v.x + __dmul_rn(w0, gg.x);
      v.y = v.y + __dmul_rn(w1, gg.y);
    }
    *reinterpret_cast<double2*>(phi + r * ST + sp) = v;
  }
  named_sync(bar_id, NT);
  bool bad = false;
  const double* Mm = A.mass + im.mass_off;
  for (int idx = tid; idx < MH; idx += NT) {
    const int r = idx / H, sp = 2 * (idx - r * H);
    double a0 = 0.0, a1 = 0.0;
    for (int j = 0; j < M; ++j) {
      const double mj = __ldg(Mm + r + j * M);
      const double2 pj = *reinterpret_cast<const double2*>(phi + j * ST + sp);
      a0 = fma(mj, pj.x, a0);
      a1 = fma(mj, pj.y, a1);
    }
    const int64_t e = base + static_cast<int64_t>(r) * ldst + sp;
    const double2 u = *reinterpret_cast<const double2*>(ub + e);
    const double2 up = *reinterpret_cast<const double2*>(ubn + e);
    double2 v;
    v.x = leapfrog_rn(u.x, up.x, dt2, a0);
    v.y = leapfrog_rn(u.y, up.y, dt2, a1);
    *reinterpret_cast<double2*>(ubn + e) = v;
    bad |= !(fabs(v.x) <= kGuard) || !(fabs(v.y) <= kGuard);
    *reinterpret_cast<double2*>(un + r * ST + sp) = v;
  }
  named_sync(bar_id, NT);
  if (A.fuse_rcv && P->traces && im.rcv_end > im.rcv_begin) {  // msolver.cpp:405-411
    const int nr = im.rcv_end - im.rcv_begin;
    double* tr = P->traces + static_cast<size_t>(n - P->n0 + 1) * A.R * A.S;
    for (int idx = tid; idx < nr * ST; idx += NT) {
      const int t = idx / ST, sp = idx - t * ST;
      const int gs = tile * ST + sp;
      if (gs >= A.S) continue;
      const RcvTerm rt = A.rterms[im.rcv_begin + t];
      double d = 0.0;
      for (int i = 0; i < M; ++i) d = fma(__ldg(A.q + rt.q_off + i), un[i * ST + sp], d);
      tr[static_cast<size_t>(rt.rcv) * A.S + gs] = d;
    }
  }
  named_sync(bar_id, NT);  // phi / un are reused by the next interface
  return bad;
}

// Register form for small interfaces (M <= MR): one thread owns one source
// pair of one interface and computes all M rows -- phi, mass * phi, the
// leapfrog and the fused receivers -- with every global load of the column
// issued up front and no shared memory or barrier.  Same operations, in the
// same order, as rom_iface_step.
template <int MR>
__device__ __forceinline__ bool iface_column(const IfuseArgs& A, const IfaceMeta& im, const double* Mm, int tile,
                                             int sp, int ST, int ldst, int64_t total_frows,
                                             const double* __restrict__ flux, const double* __restrict__ ub,
                                             double* __restrict__ ubn, StepParams* P, int64_t n) {
  const int M = im.M;
  const int64_t wi = (n - P->n0) * P->w_stride;
  const int64_t base = (static_cast<int64_t>(tile) * A.total_io + im.row_off) * ldst + sp;
  const int64_t ft = static_cast<int64_t>(tile) * total_frows;
  double2 phi[MR], pj[MR], u[MR], up[MR];
  const bool two = im.two_sided != 0;
#pragma unroll
  for (int r = 0; r < MR; ++r) {  // every load of the column issued together
    if (r < M) {
      phi[r] = __ldcg(reinterpret_cast<const double2*>(flux + (ft + im.frow_i + r) * ldst + sp));
      if (two) pj[r] = __ldcg(reinterpret_cast<const double2*>(flux + (ft + im.frow_j + r) * ldst + sp));
      u[r] = *reinterpret_cast<const double2*>(ub + base + static_cast<int64_t>(r) * ldst);
      up[r] = *reinterpret_cast<const double2*>(ubn + base + static_cast<int64_t>(r) * ldst);
    }
  }
  if (two) {
#pragma unroll
    for (int r = 0; r < MR; ++r)
      if (r < M) {
        phi[r].x = phi[r].x + pj[r].x;
        phi[r].y = phi[r].y + pj[r].y;
      }
  }
  if (im.has_src) {
    const int gs = tile * ST + sp;
    const double w0 = P->w[wi + (P->w_stride > 1 ? min(gs, A.S - 1) : 0)];
    const double w1 = P->w[wi + (P->w_stride > 1 ? min(gs + 1, A.S - 1) : 0)];
#pragma unroll
    for (int r = 0; r < MR; ++r)
      if (r < M) {
        const double2 gg = *reinterpret_cast<const double2*>(A.g + base + static_cast<int64_t>(r) * ldst);
        phi[r].x = phi[r].x + __dmul_rn(w0, gg.x);
        phi[r].y = phi[r].y + __dmul_rn(w1, gg.y);
      }
  }
  const double dt2 = P->dt2;
  bool bad = false;
  double2 un[MR];
#pragma unroll
  for (int r = 0; r < MR; ++r) {
    if (r >= M) continue;
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int j = 0; j < MR; ++j)
      if (j < M) {
        const double mj = __ldg(Mm + r + j * M);
        a0 = fma(mj, phi[j].x, a0);
        a1 = fma(mj, phi[j].y, a1);
      }
    un[r].x = leapfrog_rn(u[r].x, up[r].x, dt2, a0);
    un[r].y = leapfrog_rn(u[r].y, up[r].y, dt2, a1);
    *reinterpret_cast<double2*>(ubn + base + static_cast<int64_t>(r) * ldst) = un[r];
    bad |= !(fabs(un[r].x) <= kGuard) || !(fabs(un[r].y) <= kGuard);
  }
  if (A.fuse_rcv && P->traces && im.rcv_end > im.rcv_begin) {  // msolver.cpp:405-411
    double* tr = P->traces + static_cast<size_t>(n - P->n0 + 1) * A.R * A.S;
    const int gs = tile * ST + sp;
    for (int t = im.rcv_begin; t < im.rcv_end; ++t) {
      const RcvTerm rt = A.rterms[t];
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int i = 0; i < MR; ++i)
        if (i < M) {
          const double qi = __ldg(A.q + rt.q_off + i);
          d0 = fma(qi, un[i].x, d0);
          d1 = fma(qi, un[i].y, d1);
        }
      if (gs < A.S) tr[static_cast<size_t>(rt.rcv) * A.S + gs] = d0;
      if (gs + 1 < A.S) tr[static_cast<size_t>(rt.rcv) * A.S + gs + 1] = d1;
    }
  }
  return bad;
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

template <int NCW, int NTW, int MTP, int MINB, bool IFUSE = false>
__global__ void __launch_bounds__(32 * (NCW + 2 + (IFUSE ? 2 : 0)), MINB) rom_cell_fused(
    const CellMeta* __restrict__ cells, const CellIface* __restrict__ cif,
    const double* __restrict__ lad, const double* __restrict__ lad2, double* ubar0, double* ubar1,
    double* inter0, double* inter1, double* __restrict__ flux, StepParams* P, int64_t n_local, K1Geom G,
    IfuseArgs IF) {
  extern __shared__ __align__(128) double smem[];
  double* lad_slots = smem;
  double* st_slots = lad_slots + G.NL * G.slot_lad;
  uint64_t* bars = reinterpret_cast<uint64_t*>(st_slots + G.NU * G.slot_st + kSmemTailPad);
  uint64_t* full_lad = bars;
  uint64_t* empty_lad = bars + kMaxRing;
  uint64_t* full_st = bars + 2 * kMaxRing;
  uint64_t* empty_st = bars + 3 * kMaxRing;
  // IFUSE: D_1-stored / slot-free barriers, per-slot lists of the interfaces
  // this CTA finishes, and the interface warps' phi / ubar_next tiles
  uint64_t* d1_full = bars + 4 * kMaxRing;
  uint64_t* d1_empty = d1_full + kIfSlots;
  int* if_list = reinterpret_cast<int*>(d1_empty + kIfSlots);
  double* if_phi = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(if_list + kIfSlots * (kMaxCellIf + 1)) + 15) & ~uintptr_t(15));
  double* if_un = if_phi + IF.M_max * G.ST;
  double* if_mass = if_un + IF.M_max * G.ST;                       // kFastIf x 6 x 6
  IfaceMeta* if_meta = reinterpret_cast<IfaceMeta*>(if_mass + kFastIf * 36);  // kFastIf

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
      if (IFUSE)
        for (int i = 0; i < kIfSlots; ++i) {
          mbar_init(d1_full + i, NCW);
          mbar_init(d1_empty + i, 1);
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
  pdl_k1_gate(warp);

  if (IFUSE && warp >= NCW + 2) {
    // ============================ interface warps ============================
    const int tid = threadIdx.x - 32 * (NCW + 2);
    const int64_t n = P->base + n_local;
    const int cur = static_cast<int>(n & 1);
    const double* ub = cur ? ubar1 : ubar0;
    double* ubn = cur ? ubar0 : ubar1;  // holds ubar_prev, overwritten with ubar_next
    bool bad = false;
    uint32_t k = 0;
    for (int item = blockIdx.x; item < G.n_items; item += gridDim.x, ++k) {
      const int slot = k & (kIfSlots - 1);
      const uint32_t phase = (k / kIfSlots) & 1u;
      const int c = item / G.n_stiles;
      const int tile = item - c * G.n_stiles;
      int* lst = if_list + slot * (kMaxCellIf + 1);
      const bool fast = IF.M_max <= 6;
      if (tid < 32) {
        // one lane per interface of the cell; its static metadata is loaded
        // before the wait, the counter updates run concurrently.  This
        // cell's D_1 stores were fenced by their writers before d1_full; the
        // fence orders the counter updates after them (the
        // threadFenceReduction pattern across CTAs)
        const CellMeta cm = cells[c];
        const int nif = min(cm.nif, kMaxCellIf);
        int f = -1;
        IfaceMeta im{};
        if (tid < nif) {
          f = cif[cm.if_begin + tid].f;
          im = IF.ifs[f];
        }
        mbar_wait(d1_full + slot, phase);
        bool last = false;
        if (tid < nif) {
          __threadfence();
          const unsigned old = atomicAdd(IF.cnt + static_cast<int64_t>(f) * G.n_stiles + tile, 1u);
          last = !im.two_sided || (old & 1u);
          __threadfence();  // the partner's fenced D_1 is visible to the loads below
        }
        const unsigned mask = __ballot_sync(0xffffffffu, last);
        const int pos = __popc(mask & ((1u << tid) - 1u));
        if (last) {
          lst[1 + pos] = f;
          if (fast && pos < kFastIf) if_meta[pos] = im;
        }
        if (tid == 0) lst[0] = __popc(mask);
      } else {
        mbar_wait(d1_full + slot, phase);
      }
      named_sync(2, 64);
      const int nl = lst[0];
      if (fast && nl <= kFastIf) {
        // every (interface, source pair) column of the cell's finished
        // interfaces at once: all loads of a column in flight together
        const int H = (G.ldst >= G.ST ? G.ST : G.ldst) / 2;
        for (int idx = tid; idx < nl * H; idx += 64) {
          const int i = idx / H;
          bad |= iface_column<6>(IF, if_meta[i], IF.mass + if_meta[i].mass_off, tile, 2 * (idx - i * H), G.ST,
                                 G.ldst, G.total_frows, flux, ub, ubn, P, n);
        }
        named_sync(2, 64);  // the list slot is read until here
        if (tid == 0) mbar_arrive(d1_empty + slot);
      } else {
        for (int i = 0; i < nl; ++i)
          bad |= iface_update<64>(IF, lst[1 + i], tile, G.ST, G.ldst, G.total_frows, flux, ub, ubn, if_phi, if_un,
                                  P, n, tid, 2);
        if (tid == 0) mbar_arrive(d1_empty + slot);
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0)
      atomicMin(reinterpret_cast<unsigned long long*>(&P->bad), static_cast<unsigned long long>(n + 1));
    return;
  }

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
          mbar_expect_tx(full_lad + rl.slot, bytes);
          bulk_g2s_hint(lad_slots + rl.slot * G.slot_lad, src, bytes, full_lad + rl.slot, pol);
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
        if (m > 1) push(cur_tile);  // U^2
        const bool upg = G.upg && G.single && m > 1;  // consumers read U_prev^k themselves
        for (int k = 2; k <= m; ++k) {
          if (k < m) push(cur_tile + static_cast<int64_t>(k - 1) * kt * G.ldst);  // U^{k+1}
          if (!upg) push(prev_tile + static_cast<int64_t>(k - 2) * kt * G.ldst);  // U_prev^k
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
#ifdef MSWB_K1_PROFILE
  long long fprof[6] = {0, 0, 0, 0, 0, 0};
#define MSWB_FT0 const long long _te = clock64()
#define MSWB_FT1(slot) fprof[slot] += clock64() - _te
#else
#define MSWB_FT0
#define MSWB_FT1(slot)
#endif

  auto take = [&](int& slot, uint32_t& phase) {
    slot = rs.slot;
    phase = rs.phase;
    rs.advance();
  };
  auto release_st = [&](int slot) {
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_st + slot);
  };

  // IFUSE: after a cell's D_1 stores, each consumer warp fences them and
  // signals the interface warps (slot = the CTA-local item count mod kIfSlots)
  auto d1_signal = [&](uint32_t kk) {
    if (!IFUSE) return;
    __threadfence();
    __syncwarp();
    if (lane == 0) {
      const int slot = kk & (kIfSlots - 1);
      mbar_wait(d1_empty + slot, ((kk / kIfSlots) & 1u) ^ 1u);
      mbar_arrive(d1_full + slot);
    }
  };
  if (G.stagger > 0 && cw >= NCW / 2) {
    const long long t0 = clock64();
    while (clock64() - t0 < G.stagger) __nanosleep(32);
  }
  uint32_t kk = 0;
  for (int item = blockIdx.x; item < G.n_items; item += gridDim.x, ++kk) {
    const int c = item / G.n_stiles;
    const int tile = item - c * G.n_stiles;
    const CellMeta cm = cells[c];
    const int kt = cm.kt, m = cm.m, ld = cm.ld, ld2 = cm.ld2;
    const int kt4 = (kt + 3) & ~3;
    const int ksteps = kt4 >> 2;
    double* flux_c = flux + (static_cast<int64_t>(tile) * G.total_frows + cm.flux_row) * ldst;

    if (G.single && m > 1) {
#ifdef MSWB_K1_PROFILE
      const long long _titem = clock64();
#endif
      // ==== stage-ordered single-panel form (every layer is one ladder panel) ====
      // Stage j forms X_j = U^{j+1} - U^j once (X_m = -U^m) and multiplies it
      // by two panels: L^1 (j = 1, D_1) or P_j (finishing acc_j), and -Q_{j+1}
      // (starting acc_{j+1}).  acc_k = (-Q_k) X_{k-1} + P_k X_k, in that order.
      const int mtiles = (kt + 7) >> 3;
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
      MSWB_FP(0, mbar_wait(full_st + sU0, pU0));
      take(sU1, pU1);
      MSWB_FP(0, mbar_wait(full_st + sU1, pU1));
      MSWB_FP(1, take_lad(lc, plc));  // L^1
      MSWB_FP(1, take_lad(ln, pln));  // [P_2 | -Q_2]
      // ---- stage 1: D_1 = L^1 X_1 -> faces; acc_2 = -Q_2 X_1 ----
      MSWB_FP(2, gemm_stage<MTP, NTW, true>(accA, accB, st_slots + sU1 * G.slot_st, 1.0, st_slots + sU0 * G.slot_st,
                                 lad_slots + lc * G.slot_lad, ld, lad_slots + ln * G.slot_lad + kt4, ld2, ldst,
                                 (G.dbg & 1) ? 0 : ksteps, mtiles, wr, WR, s_w, g, t4));
      release_lad(lc);
      release_st(sU0);  // U^1
      {
      MSWB_FT0;
#pragma unroll
      for (int i = 0; i < MTP; ++i) {
        const int mt = wr + i * WR;
        const int nr = mt * 8 + g;
        if (mt >= mtiles || nr >= kt) continue;
#pragma unroll
        for (int j = 0; j < NTW; ++j) {
          const int s = s_w + j * 8 + 2 * t4;
          if (s >= ldst) continue;
          *reinterpret_cast<double2*>(flux_c + nr * ldst + s) = make_double2(accA[i][j][0], accA[i][j][1]);
        }
      }
      MSWB_FT1(3);
      }
      lc = ln;
      plc = pln;
      // ---- stages k = 2..m: acc_k += P_k X_k (then its leapfrog); acc_{k+1} = -Q_{k+1} X_k ----
      const bool upg = G.upg != 0;
      for (int k = 2; k <= m; ++k) {
        double* lay = inter_nxt + tile * inter_tile + (cm.inter_row + static_cast<int64_t>(k - 2) * kt) * ldst;
        // upg: this thread's U_prev^k elements, loaded now and consumed by the
        // epilogue after the GEMM (the same addresses the epilogue overwrites)
        double2 upr[MTP][NTW];
        if (upg) {
#pragma unroll
          for (int i = 0; i < MTP; ++i) {
            const int mt = wr + i * WR;
            const int nr = mt * 8 + g;
#pragma unroll
            for (int j = 0; j < NTW; ++j) {
              const int s = s_w + j * 8 + 2 * t4;
              upr[i][j] = (mt < mtiles && nr < kt && s < ldst)
                              ? *reinterpret_cast<const double2*>(lay + nr * ldst + s)
                              : make_double2(0.0, 0.0);
            }
          }
        }
        if (k < m) {
          take(sU2, pU2);  // U^{k+1}
          MSWB_FP(0, mbar_wait(full_st + sU2, pU2));
        }
        if (!upg) take(sP, pP);  // U_prev^k
#pragma unroll
        for (int i = 0; i < MTP; ++i)
#pragma unroll
          for (int j = 0; j < NTW; ++j) {
            accA[i][j][0] = accB[i][j][0];
            accA[i][j][1] = accB[i][j][1];
            accB[i][j][0] = accB[i][j][1] = 0.0;
          }
        const double* Uk = st_slots + sU1 * G.slot_st;
        if (k < m) {
          MSWB_FP(1, take_lad(ln, pln));  // [P_{k+1} | -Q_{k+1}]
          MSWB_FP(2, gemm_stage<MTP, NTW, true>(accA, accB, st_slots + sU2 * G.slot_st, 1.0, Uk, lad_slots + lc * G.slot_lad,
                                     ld2, lad_slots + ln * G.slot_lad + kt4, ld2, ldst, (G.dbg & 1) ? 0 : ksteps,
                                     mtiles, wr, WR,
                                     s_w, g, t4));
        } else {
          MSWB_FP(2, gemm_stage<MTP, NTW, false>(accA, accB, Uk, 0.0, Uk, lad_slots + lc * G.slot_lad, ld2,
                                      lad_slots + lc * G.slot_lad, ld2, ldst, (G.dbg & 1) ? 0 : ksteps, mtiles, wr,
                                      WR, s_w, g, t4));
        }
        release_lad(lc);
        // IFUSE: signal the interface warps one stage after the D_1 stores,
        // when they have long drained, so the release fence costs nothing
        if (k == 2) d1_signal(kk);
        if (!upg) MSWB_FP(0, mbar_wait(full_st + sP, pP));
        const double* Up = st_slots + (upg ? 0 : sP) * G.slot_st;
        {
        MSWB_FT0;
#pragma unroll
        for (int i = 0; i < MTP; ++i) {
          const int mt = wr + i * WR;
          const int nr = mt * 8 + g;
          if (mt >= mtiles || nr >= kt) continue;
#pragma unroll
          for (int j = 0; j < NTW; ++j) {
            const int s = s_w + j * 8 + 2 * t4;
            if (s >= ldst) continue;
            const double2 u = *reinterpret_cast<const double2*>(Uk + nr * ldst + s);
            const double2 up = upg ? upr[i][j] : *reinterpret_cast<const double2*>(Up + nr * ldst + s);
            double2 v;
            v.x = leapfrog_rn(u.x, up.x, dt2, accA[i][j][0]);
            v.y = leapfrog_rn(u.y, up.y, dt2, accA[i][j][1]);
            *reinterpret_cast<double2*>(lay + nr * ldst + s) = v;
            bad |= !(fabs(v.x) <= kGuard) || !(fabs(v.y) <= kGuard);
          }
        }
        MSWB_FT1(3);
        }
        release_st(sU1);  // U^k
        if (!upg) release_st(sP);  // U_prev^k
        sU1 = sU2;
        pU1 = pU2;
        lc = ln;
        plc = pln;
      }
#ifdef MSWB_K1_PROFILE
      fprof[4] += clock64() - _titem;
      fprof[5] += 1;
#endif
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
    d1_signal(kk);
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
  if ((G.dbg & 8) && G.prof && lane == 0)
    for (int i = 0; i < 6; ++i) atomicAdd(G.prof + i, static_cast<unsigned long long>(fprof[i]));
#endif
}

}  // namespace pipe
}  // namespace mswb
