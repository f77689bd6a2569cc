// Micro-probe: fp64 DFMA and DMMA (mma.sync m8n8k4 f64) peak on this GPU,
// plus a streaming copy bandwidth check.  Used to fill the fp64 roof that
// MEASURED_PEAKS.json lacks.  Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

int main(int argc, char** argv) {
  const bool dmma_only = argc > 1 && argv[1][0] == 'd';  // bench.py: the fp64 roof only
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("{\"name\": \"%s\", \"sms\": %d, \"l2\": %d, \"smem_optin\": %zu}\n", p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int blocksPerSm : {4, 8}) {
    if (dmma_only && blocksPerSm == 4) continue;
    int iters = 20000;
    dim3 grid(sms * blocksPerSm), block(256);
    float ms = 0.f;
    double flops = 0.0;
    if (!dmma_only) {
      dfma_kernel<<<grid, block>>>(out, 100, 1.0000001, 1e-9);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dfma_kernel<<<grid, block>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 8 * iters * (double)grid.x * block.x;
      printf("{\"probe\": \"dfma\", \"blocks_per_sm\": %d, \"tflops\": %.2f}\n", blocksPerSm, flops / ms / 1e9);
    }
    dmma_kernel<<<grid, block>>>(out, 100);
    CK(cudaDeviceSynchronize());
    iters = 5000;
    cudaEventRecord(e0);
    dmma_kernel<<<grid, block>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 256 * 8 * iters * (double)grid.x * (block.x / 32);
    printf("{\"probe\": \"dmma_m8n8k4\", \"blocks_per_sm\": %d, \"tflops\": %.2f}\n", blocksPerSm, flops / ms / 1e9);
  }
  if (dmma_only) return 0;
  size_t n = (size_t)1 << 28;  // 2^28 double2 = 4 GiB each
  double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
  cudaMemset(a, 0, n * 16);
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    copy_kernel<<<sms * 8, 512>>>(a, b, n);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"probe\": \"copy\", \"gbs\": %.1f}\n", 2.0 * n * 16 / ms / 1e6);
  }
  return 0;
}
