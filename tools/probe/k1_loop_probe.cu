// Micro-probe for the config-3 cell kernel's inner loop (not part of the
// product): how fast can an m8n8k4.f64 loop with operands in shared memory
// run on one SM, as a function of the warp tile, warps per SM, the A-fragment
// load width, and whether DFMA work runs beside it?
//
// The loop emulates one stage of rom_cell_fused's stage form at config 3:
// two A panels (P_j, -Q_{j+1}) of 40 output rows x 36 k, B = X_j (36 k x 64
// sources, formed as hi - lo), kt4 = 36 -> 9 k-steps of 4.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

constexpr int KT4 = 36, KSTEPS = 9, LDA = 76, LDB = 68, ROWS = 40;

// NWG warps per group cover 64 sources with NT col tiles each (NWG*NT = 8);
// MT row tiles per warp (MT = 5: all rows).  FRAG: A stored in fragment
// order (lane-contiguous per (tile, k-step pair)) and loaded 16 bytes at a
// time (two k-steps per LDS.128).
template <int NT, int MT, bool TWO, bool FRAG>
__global__ void __launch_bounds__(512) loop_probe(double* out, int reps, int groups) {
  extern __shared__ double sm[];
  double* A1 = sm;                    // ROWS x LDA (or fragment order)
  double* A2 = A1 + ROWS * LDA;
  double* Bh = A2 + ROWS * LDA;       // KT4 x LDB
  double* Bl = Bh + KT4 * LDB;
  const int tid = threadIdx.x;
  for (int i = tid; i < 2 * ROWS * LDA + 2 * KT4 * LDB; i += blockDim.x) sm[i] = 1e-3 * (i % 97) - 0.03;
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int ws = warp % (8 / NT);          // source group
  const int s_w = ws * NT * 8;
  double acc1[MT][NT][2], acc2[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc1[i][j][0] = acc1[i][j][1] = acc2[i][j][0] = acc2[i][j][1] = 0.0;
  for (int r = 0; r < reps; ++r) {
    const double* pa1[MT];
    const double* pa2[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      if (FRAG) {
        pa1[i] = A1 + (i * (KSTEPS + 1) / 2) * 64 + lane * 2;
        pa2[i] = A2 + (i * (KSTEPS + 1) / 2) * 64 + lane * 2;
      } else {
        pa1[i] = A1 + (i * 8 + g) * LDA + t4;
        pa2[i] = A2 + (i * 8 + g) * LDA + t4;
      }
    }
    const double* ph = Bh + t4 * LDB + s_w + g;
    const double* pl = Bl + t4 * LDB + s_w + g;
    if (FRAG) {
#pragma unroll 1
      for (int kk = 0; kk < KSTEPS; kk += 2) {
        double2 a1[MT], a2[MT];
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          a1[i] = *reinterpret_cast<const double2*>(pa1[i] + (kk / 2) * 64);
          if (TWO) a2[i] = *reinterpret_cast<const double2*>(pa2[i] + (kk / 2) * 64);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (kk + h >= KSTEPS) break;
          double b[NT];
#pragma unroll
          for (int j = 0; j < NT; ++j) b[j] = ph[(kk + h) * 4 * LDB + j * 8] - pl[(kk + h) * 4 * LDB + j * 8];
#pragma unroll
          for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) {
              dmma(acc1[i][j], h ? a1[i].y : a1[i].x, b[j]);
              if (TWO) dmma(acc2[i][j], h ? a2[i].y : a2[i].x, b[j]);
            }
        }
      }
    } else {
      double a1[MT], a2[MT], b[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        a1[i] = pa1[i][0];
        if (TWO) a2[i] = pa2[i][0];
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = ph[j * 8] - pl[j * 8];
#pragma unroll 4
      for (int kk = 0; kk < KSTEPS; ++kk) {
        double an1[MT], an2[MT], bn[NT];
        const int kn = kk + 1 < KSTEPS ? kk + 1 : kk;
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          an1[i] = pa1[i][4 * kn];
          if (TWO) an2[i] = pa2[i][4 * kn];
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) bn[j] = ph[kn * 4 * LDB + j * 8] - pl[kn * 4 * LDB + j * 8];
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            dmma(acc1[i][j], a1[i], b[j]);
            if (TWO) dmma(acc2[i][j], a2[i], b[j]);
          }
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          a1[i] = an1[i];
          if (TWO) a2[i] = an2[i];
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) b[j] = bn[j];
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) s += acc1[i][j][0] + acc1[i][j][1] + acc2[i][j][0] + acc2[i][j][1];
  if (s == 1234.5678) out[blockIdx.x] = s;
}

// DFMA work beside the DMMA loop: `dfma_warps` extra warps per CTA run an
// 8-chain DFMA loop while the others run the smem DMMA loop.
__global__ void __launch_bounds__(512) mixed_probe(double* out, int reps, int dmma_warps, int dfma_iters) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= dmma_warps) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = lane * 1e-3 + i;
    for (int it = 0; it < dfma_iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 1.0000001, 1e-9);
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
    return;
  }
  double a = lane * 1e-3, b = 1.0 - lane * 1e-4;
  double c[10][2];
#pragma unroll
  for (int i = 0; i < 10; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < reps; ++it)
#pragma unroll
    for (int i = 0; i < 10; ++i) dmma(c[i], a, b);
  double s = 0;
#pragma unroll
  for (int i = 0; i < 10; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int NT, int MT, bool TWO, bool FRAG>
int run(const char* name, int warps, int ctas_per_sm, int sms, double* out) {
  auto k = loop_probe<NT, MT, TWO, FRAG>;
  const size_t smem = (2 * ROWS * LDA + 2 * KT4 * LDB) * 8;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int reps = 4000;
  k<<<sms * ctas_per_sm, 32 * warps, smem>>>(out, 10, 1);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<sms * ctas_per_sm, 32 * warps, smem>>>(out, reps, 1);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dmmas = (double)sms * ctas_per_sm * warps * reps * KSTEPS * MT * NT * (TWO ? 2 : 1);
  printf("{\"probe\": \"%s\", \"warps_per_cta\": %d, \"ctas_per_sm\": %d, \"tflops\": %.2f}\n", name, warps,
         ctas_per_sm, dmmas * 512 / ms / 1e9);
  return 0;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount;
  double* out;
  CK(cudaMalloc(&out, 8 * sms * 8));
  // the production shape: 8 warps, 5x1 tiles, two panels
  run<1, 5, true, false>("5x1x2 lds64", 8, 1, sms, out);
  run<1, 5, true, false>("5x1x2 lds64", 8, 2, sms, out);
  run<1, 5, true, false>("5x1x2 lds64", 16, 1, sms, out);
  run<1, 5, true, true>("5x1x2 frag128", 8, 1, sms, out);
  run<1, 5, true, true>("5x1x2 frag128", 16, 1, sms, out);
  run<2, 5, true, false>("5x2x2 lds64", 4, 1, sms, out);
  run<2, 5, true, false>("5x2x2 lds64", 8, 1, sms, out);
  run<2, 5, true, true>("5x2x2 frag128", 4, 1, sms, out);
  run<2, 5, true, true>("5x2x2 frag128", 8, 1, sms, out);
  run<1, 5, false, false>("5x1x1 lds64", 8, 1, sms, out);
  run<2, 5, false, false>("5x2x1 lds64", 8, 1, sms, out);
  run<4, 5, false, false>("5x4x1 lds64", 4, 1, sms, out);
  // DMMA + DFMA concurrency: 8 DMMA warps alone, then with 8 DFMA warps beside
  for (int dfw : {0, 4, 8}) {
    const int warps = 8 + dfw, reps = 20000, dfi = 40000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    mixed_probe<<<sms, 32 * warps>>>(out, 10, 8, 10);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    mixed_probe<<<sms, 32 * warps>>>(out, reps, 8, dfw ? dfi : 0);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double f_dmma = (double)sms * 8 * reps * 10 * 512;
    const double f_dfma = (double)sms * dfw * 32 * dfi * 8 * 2;
    printf("{\"probe\": \"dmma8+dfma%d\", \"ms\": %.3f, \"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f, \"total\": %.2f}\n",
           dfw, ms, f_dmma / ms / 1e9, f_dfma / ms / 1e9, (f_dmma + f_dfma) / ms / 1e9);
  }
  return 0;
}
