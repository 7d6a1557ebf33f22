// GPU dense oracle: z = K(X, Y) q streamed over source tiles, never stored --
// the exact-product checker of smash.bench.dense_matvec (smash/bench.py:284-296)
// at sizes where the CPU oracle takes hours (2^20 .. 2^21 points).  Not on the
// compressed hot path; used by tests / tools to measure the matvec's error
// against the exact product.
#include "kernels.cuh"

namespace smash {

namespace {

constexpr int DT = 128;  // targets per CTA = sources per staged tile

template <int KER, int D, int RC>
__global__ void __launch_bounds__(DT) k_dense(const double* X, int64_t nx, const double* Y,
                                              int64_t ny, const double* q, int64_t ldq, int64_t c0,
                                              double dx, double* z, int64_t ldz) {
  __shared__ double ys[DT * D];
  __shared__ double qs[DT * RC];
  const int64_t i = blockIdx.x * (int64_t)DT + threadIdx.x;
  double x[D];
#pragma unroll
  for (int a = 0; a < D; ++a) x[a] = i < nx ? X[i * D + a] : 0.0;
  double acc[RC];
#pragma unroll
  for (int c = 0; c < RC; ++c) acc[c] = 0.0;
  for (int64_t j0 = 0; j0 < ny; j0 += DT) {
    __syncthreads();
    const int64_t j = j0 + threadIdx.x;
    if (j < ny) {
#pragma unroll
      for (int a = 0; a < D; ++a) ys[threadIdx.x * D + a] = Y[j * D + a];
#pragma unroll
      for (int c = 0; c < RC; ++c) qs[threadIdx.x * RC + c] = q[j * ldq + c0 + c];
    }
    __syncthreads();
    const int nt = (int)(ny - j0 < DT ? ny - j0 : DT);
    if (i < nx)
      for (int t = 0; t < nt; ++t) {
        const double k = kval<KER, D>(x, ys + t * D, dx);
#pragma unroll
        for (int c = 0; c < RC; ++c) acc[c] = fma(k, qs[t * RC + c], acc[c]);
      }
  }
  if (i < nx)
#pragma unroll
    for (int c = 0; c < RC; ++c) z[i * ldz + c0 + c] = acc[c];
}

template <int KER, int D>
void dense_chunks(const double* X, int64_t nx, const double* Y, int64_t ny, const double* q,
                  int64_t nrhs, double dx, double* z, cudaStream_t s) {
  const unsigned grid = cdiv(nx, DT);
  int64_t c0 = 0;
  while (c0 < nrhs) {
    const int64_t rem = nrhs - c0;
    if (rem >= 8) {
      k_dense<KER, D, 8><<<grid, DT, 0, s>>>(X, nx, Y, ny, q, nrhs, c0, dx, z, nrhs);
      c0 += 8;
    } else if (rem >= 4) {
      k_dense<KER, D, 4><<<grid, DT, 0, s>>>(X, nx, Y, ny, q, nrhs, c0, dx, z, nrhs);
      c0 += 4;
    } else {
      k_dense<KER, D, 1><<<grid, DT, 0, s>>>(X, nx, Y, ny, q, nrhs, c0, dx, z, nrhs);
      c0 += 1;
    }
  }
}

}  // namespace

void dense_matvec(int kernel, double dx, int dim, const double* X, int64_t nx, const double* Y,
                  int64_t ny, const double* q, int64_t nrhs, double* z, cudaStream_t s) {
  SMASH_CHECK(nx >= 0 && ny >= 0 && nrhs >= 0, SMASH_ERR_INVALID, "bad shape");
  if (nx == 0 || nrhs == 0) return;
  if (ny == 0) {
    SMASH_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * nx * nrhs, s));
    return;
  }
  dispatch_kernel_dim(kernel, dim, [&]<int KER, int D>() {
    dense_chunks<KER, D>(X, nx, Y, ny, q, nrhs, dx, z, s);
  });
  SMASH_CUDA(cudaGetLastError());
}

}  // namespace smash
