// Latency probe (one warp / one CTA): dependent DFMA, DADD, DDIV, DSQRT, double SHFL,
// redux.sync, __syncthreads with 9 warps, LDS of a double.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[64];
  double x = a + threadIdx.x * 1e-9, y = b;
  if (threadIdx.x < 64) sm[threadIdx.x] = x;
  __syncthreads();
  long long t[10];
  t[0] = clock64();
  for (int i = 0; i < n; ++i) x = __fma_rn(x, y, 1e-3);
  t[1] = clock64();
  for (int i = 0; i < n; ++i) x = __ddiv_rn(x, y) + 1e-3;
  t[2] = clock64();
  for (int i = 0; i < n; ++i) x = __dsqrt_rn(x) + 1.0;
  t[3] = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) * 1.0000001;
  t[4] = clock64();
  unsigned u = (unsigned)threadIdx.x;
  for (int i = 0; i < n; ++i) u = __reduce_max_sync(0xffffffffu, u) + threadIdx.x;
  t[5] = clock64();
  for (int i = 0; i < n; ++i) { __syncthreads(); x += 1e-9; }
  t[6] = clock64();
  int idx = threadIdx.x & 63;
  for (int i = 0; i < n; ++i) { x = sm[idx] + x * 1e-9; idx = ((int)x & 1) + (idx ^ 1) & 63; }
  t[7] = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / x + 1.0;
  t[8] = clock64();
  out[threadIdx.x] = x + u;
  if (threadIdx.x == 0)
    for (int j = 0; j < 8; ++j) cyc[j] = t[j + 1] - t[j];
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 8192); cudaMallocManaged(&c, 128);
  const int n = 256;
  k<<<1, 288>>>(o, c, 1.5, 0.999, n); cudaDeviceSynchronize();
  k<<<1, 288>>>(o, c, 1.5, 0.999, n); cudaDeviceSynchronize();
  const char* names[8] = {"dfma", "ddiv_rn", "dsqrt_rn", "shfl f64", "redux u32", "syncthreads(9w)", "lds f64", "1.0/x"};
  for (int j = 0; j < 8; ++j) printf("%-18s %.1f cycles/iter\n", names[j], (double)c[j] / n);
  return 0;
}
