// DFMA latency / throughput microbenchmark (B200): K independent dependent-chains per thread,
// W warps per CTA, one CTA per SM.  Prints cycles per chain step and DFMA per SM per cycle.
#include <cstdio>
#include <cuda_runtime.h>
template <int K>
__global__ void chain(double* out, int iters, long long* cyc) {
  double a[K];
#pragma unroll
  for (int k = 0; k < K; ++k) a[k] = threadIdx.x * 1e-3 + k;
  const double m = 0.999999, c = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int k = 0; k < K; ++k) a[k] = fma(a[k], m, c);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
// LDS latency: pointer chase in shared memory
__global__ void lds_lat(int iters, long long* cyc, int* out) {
  __shared__ int buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i + 33) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = buf[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <int K>
void run(int warps) {
  double* o; long long* c; long long h;
  cudaMalloc(&o, 148 * 1024 * 8); cudaMalloc(&c, 8);
  const int iters = 2000;
  chain<K><<<148, warps * 32>>>(o, iters, c);
  chain<K><<<148, warps * 32>>>(o, iters, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  double steps = iters * 8.0;
  printf("K=%d warps/SM=%2d: %.2f cycles per chain step, %.1f DFMA/SM/cycle\n", K, warps, h / steps,
         warps * 32.0 * K * steps / h);
  cudaFree(o); cudaFree(c);
}
int main() {
  for (int w : {1, 4, 8, 12, 16}) { run<1>(w); run<2>(w); run<4>(w); run<8>(w); }
  long long* c; int* o; long long h;
  cudaMalloc(&c, 8); cudaMalloc(&o, 4096);
  lds_lat<<<1, 32>>>(10000, c, o); lds_lat<<<1, 32>>>(10000, c, o);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("LDS latency %.1f cycles\n", h / 10000.0);
  return 0;
}
