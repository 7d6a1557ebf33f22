// FP64 peak microbenchmark for B200 (sm_100a): DFMA, DMMA (mma.sync m8n8k4 f64),
// and the per-interaction cost of the kernel functions used by the P2P kernels.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 123.456) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0001;
  double c[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) { c[t][0] = t; c[t][1] = -t; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  if (s == 123.456) out[0] = s;
}

template <int K>
__device__ __forceinline__ double kfun(double r2) {
  if (K == 0) return rsqrt(r2);
  if (K == 1) return 0.5 * log(r2);
  if (K == 2) return exp(-sqrt(r2));
  return 1.0 / sqrt(r2);
}

template <int K>
__global__ void kern_kernel(double* out, int iters) {
  double acc[4] = {0, 0, 0, 0};
  double x[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) x[c] = 0.5 + threadIdx.x * 1e-5 + c * 0.1;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) { acc[c] += kfun<K>(x[c]); x[c] += 1e-7; }
  }
  double s = acc[0] + acc[1] + acc[2] + acc[3];
  if (s == 123.456) out[0] = s;
}

int main() {
  double* d; CK(cudaMalloc(&d, 8));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  printf("device %s sms %d clock %d kHz\n", p.name, sms, p.clockRate);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const int iters = 1 << 16;
  for (int blocksPerSm : {4, 8}) {
    int grid = sms * blocksPerSm, block = 256;
    dfma_kernel<8><<<grid, block>>>(d, 64, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_kernel<8><<<grid, block>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)grid * block;
    printf("DFMA blocks/SM %d: %.2f TFLOP/s (%.3f ms)\n", blocksPerSm, flops / ms / 1e9, ms);
  }
  {
    int grid = sms * 8, block = 128;
    dmma_kernel<<<grid, block>>>(d, 64);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_kernel<<<grid, block>>>(d, iters / 4);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 4 * (double)(iters / 4) * grid * (block / 32);
    printf("DMMA m8n8k4: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  const char* names[4] = {"rsqrt", "0.5*log(r2)", "exp(-sqrt(r2))", "1/sqrt(r2)"};
  for (int k = 0; k < 4; ++k) {
    int grid = sms * 8, block = 256;
    auto run = [&](int it) {
      if (k == 0) kern_kernel<0><<<grid, block>>>(d, it);
      if (k == 1) kern_kernel<1><<<grid, block>>>(d, it);
      if (k == 2) kern_kernel<2><<<grid, block>>>(d, it);
      if (k == 3) kern_kernel<3><<<grid, block>>>(d, it);
    };
    run(16); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); run(iters / 16); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double evals = 4.0 * (iters / 16) * (double)grid * block;
    printf("kernel %-16s %.2f Geval/s (%.3f ms)\n", names[k], evals / ms / 1e6, ms);
  }
  return 0;
}
