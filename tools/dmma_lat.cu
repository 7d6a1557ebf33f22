// DMMA m8n8k4 latency / throughput microbenchmark (one warp per SMSP or one warp total).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, int n, long long* cyc) {
  double c[CH][2];
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* o; long long* cy; cudaMalloc(&o, 1 << 24); cudaMallocManaged(&cy, 8);
  const int n = 4096;
  auto run = [&](auto kern, int ch, int blocks, int threads) {
    kern<<<blocks, threads>>>(o, 16, cy); cudaDeviceSynchronize();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); kern<<<blocks, threads>>>(o, n, cy); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double dmmas = (double)n * ch * blocks * (threads / 32);
    printf("chains %d blocks %d threads %d: %.1f cycles per iteration (warp 0), %.2f TFLOP/s\n", ch, blocks, threads,
           (double)*cy / n, dmmas * 512 / ms / 1e9);
  };
  run(k<1>, 1, 1, 32);
  run(k<2>, 2, 1, 32);
  run(k<4>, 4, 1, 32);
  run(k<8>, 8, 1, 32);
  run(k<1>, 1, 1, 128);
  run(k<4>, 4, 1, 128);
  run(k<4>, 4, 148, 128);
  run(k<8>, 8, 148, 128);
  run(k<4>, 4, 148 * 4, 128);
  run(k<8>, 8, 148 * 2, 256);
}
