// Probe: DMMA throughput vs consumer warps per SM with smem-fed fragments,
// the inner loop shape of rom_cell_pipe (MT M-tiles x NT N-tiles per warp).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int MT, int NT>
__global__ void k(double* out, int iters, int ksteps) {
  __shared__ double X[64 * 68];
  __shared__ double L[40 * 44];
  for (int i = threadIdx.x; i < 64 * 68; i += blockDim.x) X[i] = 1e-3 * i;
  for (int i = threadIdx.x; i < 40 * 44; i += blockDim.x) L[i] = 1e-4 * i;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  double acc[NT][MT][2] = {};
  for (int it = 0; it < iters; ++it) {
    for (int kk = 0; kk < ksteps; ++kk) {
      const int kr = 4 * kk + t4;
      double a[MT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int s = (warp * MT + mt) * 8 % 64 + g;
        a[mt] = X[kr * 68 + s] - X[(kr + 1) * 68 + s];
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const double b = L[(j * 8 + g) * 44 + kr];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) dmma(acc[j][mt], a[mt], b);
      }
    }
  }
  double s = 0;
  for (int j = 0; j < NT; ++j) for (int mt = 0; mt < MT; ++mt) s += acc[j][mt][0] + acc[j][mt][1];
  if (s == 1.2345) out[0] = s;
}

template <int MT, int NT>
void run(int warps, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 200, ksteps = 9;
  k<MT, NT><<<148, warps * 32>>>(out, 10, ksteps);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  k<MT, NT><<<148, warps * 32>>>(out, iters, ksteps);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 256 * MT * NT * ksteps * (double)iters * warps * 148;
  printf("{\"MT\": %d, \"NT\": %d, \"warps_per_sm\": %d, \"tflops\": %.2f}\n", MT, NT, warps, flops / ms / 1e9);
}

int main() {
  double* out; cudaMalloc(&out, 8);
  for (int w : {4, 8, 12, 16}) { run<2, 5>(w, out); run<1, 5>(w, out); run<2, 2>(w, out); }
  return 0;
}
