// fp64 peak microbenchmarks (sm_100a): DFMA issue throughput with independent chains per thread.
// Built and timed by scripts/fp64_peak.py (not part of the library).
#include <cuda_runtime.h>

extern "C" __global__ void dfma_kernel(double* out, int iters, double a, double b) {
  // 8 independent FMA chains per thread: enough ILP to cover the DFMA latency
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-9, x2 = x0 + 2e-9, x3 = x0 + 3e-9;
  double x4 = x0 + 4e-9, x5 = x0 + 5e-9, x6 = x0 + 6e-9, x7 = x0 + 7e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[blockIdx.x] = s;  // keeps the chains alive
}

extern "C" int run_dfma(int blocks, int threads, int iters, float* ms) {
  double* out = nullptr;
  cudaMalloc(&out, sizeof(double) * blocks);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);  // warm-up
  cudaEventRecord(e0);
  dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms, e0, e1);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// DMMA (mma.sync m8n8k4 f64) issue throughput: 4 independent accumulator tiles per warp
extern "C" __global__ void dmma_kernel(double* out, int iters, double a0, double b0) {
  double a = a0 + threadIdx.x * 1e-12, b = b0 - threadIdx.x * 1e-12;
  double c[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) c[t][0] = c[t][1] = t * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int t = 0; t < 4; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                     : "+d"(c[t][0]), "+d"(c[t][1])
                     : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[blockIdx.x] = s;
}

extern "C" int run_dmma(int blocks, int threads, int iters, float* ms) {
  double* out = nullptr;
  cudaMalloc(&out, sizeof(double) * blocks);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dmma_kernel<<<blocks, threads>>>(out, iters, 1e-3, 1e-3);
  cudaEventRecord(e0);
  dmma_kernel<<<blocks, threads>>>(out, iters, 1e-3, 1e-3);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms, e0, e1);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
