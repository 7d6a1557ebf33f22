// Device building blocks of the column-pivoted Householder QR shared by the
// sRRQR kernel (compress.cu) and the HSS truncated-SVD kernel (svd.cu).
// Semantics follow LAPACK dlaqp2 / dlarfg / dlarf (see compress.cu).
#pragma once

#include "common.cuh"

namespace smash {
namespace qr {

constexpr double TOL3Z = 1.0536712127723509e-08;  // sqrt(dlamch('E')), dlaqp2

struct Shared {
  double* vn1;
  double* vn2;
  double* vh;
  double* rdiag;
  double* nodes;  // [3][MAX_M_AXIS_1D]
  double* redv;   // [32]
  int* redi;      // [32]
  double* misc;   // [8]
  int* imisc;     // [8]
  int* jpvt;
  double* panel;
};

__device__ __forceinline__ void argmax_combine(double& v, int& i, double ov, int oi) {
  if (ov > v || (ov == v && oi < i)) { v = ov; i = oi; }
}

// Block-wide (max value, smallest index) reduction; result broadcast to all threads.
__device__ __forceinline__ void block_argmax(double& v, int& i, Shared& S) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int off = 16; off; off >>= 1) {
    double ov = __shfl_down_sync(0xffffffffu, v, off);
    int oi = __shfl_down_sync(0xffffffffu, i, off);
    argmax_combine(v, i, ov, oi);
  }
  __syncthreads();  // protect redv/redi reuse
  if (lane == 0) { S.redv[wid] = v; S.redi[wid] = i; }
  __syncthreads();
  if (wid == 0) {
    v = lane < nw ? S.redv[lane] : -1.0;
    i = lane < nw ? S.redi[lane] : 0x7fffffff;
    for (int off = 16; off; off >>= 1) {
      double ov = __shfl_down_sync(0xffffffffu, v, off);
      int oi = __shfl_down_sync(0xffffffffu, i, off);
      argmax_combine(v, i, ov, oi);
    }
    if (lane == 0) { S.redv[0] = v; S.redi[0] = i; }
  }
  __syncthreads();
  v = S.redv[0];
  i = S.redi[0];
}

// Sum of squares of column j over rows [r0, r1), sequential in row order.  The
// loads of a chunk are issued before its FMAs so a global/L2-resident panel
// keeps CH requests in flight (the accumulation order is unchanged).
template <int CH = 8>
// Block-wide argmax with a single barrier: each warp reduces with shuffles and
// publishes one partial; after the barrier every thread reduces the partials
// itself (the (max value, smallest index) rule makes the order irrelevant).
// The caller must separate two calls by another barrier (partials are reused).
__device__ __forceinline__ int block_argmax_1bar(double v, int i, Shared& S) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int off = 16; off; off >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, off);
    int oi = __shfl_xor_sync(0xffffffffu, i, off);
    argmax_combine(v, i, ov, oi);
  }
  if (lane == 0) { S.redv[wid] = v; S.redi[wid] = i; }
  __syncthreads();
  v = S.redv[0];
  i = S.redi[0];
  for (int w = 1; w < nw; ++w) argmax_combine(v, i, S.redv[w], S.redi[w]);
  return i;
}

template <int CH = 8>
__device__ __forceinline__ double col_sumsq(const double* __restrict__ P, int ld, int j, int r0,
                                            int r1) {
  double s = 0.0;
  for (int row = r0; row < r1; row += CH) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = row + c < r1 ? P[(row + c) * ld + j] : 0.0;
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (row + c < r1) s = __fma_rn(x[c], x[c], s);
  }
  return s;
}

__device__ __forceinline__ double dlapy2(double x, double y) {
  double xa = fabs(x), ya = fabs(y);
  double w = fmax(xa, ya), z = fmin(xa, ya);
  if (z == 0.0 || w > 1.7976931348623157e308) return w;
  double q = __ddiv_rn(z, w);
  return __dmul_rn(w, __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(q, q))));
}

// Householder reflector on column i (dlarfg), done by warp 0; result in panel,
// tau in S.misc[0], v (rows > i) in S.vh.
__device__ __forceinline__ void householder(double* P, int ld, int m, int i, Shared& S) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  double alpha = P[i * ld + i];
  double ss = 0.0;
  for (int row = i + 1 + lane; row < m; row += 32) {
    double x = P[row * ld + i];
    ss = __fma_rn(x, x, ss);
  }
  for (int off = 16; off; off >>= 1) ss = __dadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, off));
  double xnorm = __dsqrt_rn(ss);
  double tau = 0.0;
  if (m - i > 1 && xnorm != 0.0) {
    double beta = -copysign(dlapy2(alpha, xnorm), alpha);
    tau = __ddiv_rn(__dsub_rn(beta, alpha), beta);
    double scal = __ddiv_rn(1.0, __dsub_rn(alpha, beta));
    for (int row = i + 1 + lane; row < m; row += 32) {
      double x = __dmul_rn(scal, P[row * ld + i]);
      P[row * ld + i] = x;
      S.vh[row] = x;
    }
    if (lane == 0) P[i * ld + i] = beta;
  }
  if (lane == 0) {
    S.misc[0] = tau;
    S.rdiag[i] = P[i * ld + i];
  }
}

// Apply H_i^T = I - tau v v^T (v_i = 1) to column j > i (dlarf: w = C^T v; C -= tau v w^T).
// Chunked like col_sumsq: each chunk's loads are independent, the FMA order is
// the sequential row order.
template <int CH = 8>
__device__ __forceinline__ void apply_reflector(double* __restrict__ P, int ld, int m, int i, int j,
                                                double tau, const double* __restrict__ vh) {
  double w = P[i * ld + j];
  for (int row = i + 1; row < m; row += CH) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = row + c < m ? P[(row + c) * ld + j] : 0.0;
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (row + c < m) w = __fma_rn(vh[row + c], x[c], w);
  }
  double t = -__dmul_rn(tau, w);
  P[i * ld + j] = __dadd_rn(P[i * ld + j], t);
  for (int row = i + 1; row < m; row += CH) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = row + c < m ? P[(row + c) * ld + j] : 0.0;
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (row + c < m) P[(row + c) * ld + j] = __fma_rn(t, vh[row + c], x[c]);
  }
}

// Four-chain variants (the compression default; SMASH_QR_CHAINS=1 selects the sequential
// ones above): the same sums split over four independent accumulators (rows round-robin,
// combined (0+1)+(2+3)), a quarter of the dependent FMA latency per pivot step.  Neither
// order is OpenBLAS's (dgemv / x87 dnrm2); the pivots and ranks are the reference's either
// way on every fixture and full-size node (tests/test_fullsize_parity.py).
template <int CH = 8>
__device__ __forceinline__ double col_sumsq4(const double* __restrict__ P, int ld, int j, int r0,
                                             int r1) {
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  int row = r0;
  for (; row + 4 <= r1; row += 4) {
    double x[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) x[c] = P[(row + c) * ld + j];
#pragma unroll
    for (int c = 0; c < 4; ++c) s[c] = __fma_rn(x[c], x[c], s[c]);
  }
  for (int c = 0; row < r1; ++row, ++c) {
    const double x = P[row * ld + j];
    s[c] = __fma_rn(x, x, s[c]);
  }
  return __dadd_rn(__dadd_rn(s[0], s[1]), __dadd_rn(s[2], s[3]));
}

template <int CH = 8>
__device__ __forceinline__ void apply_reflector4(double* __restrict__ P, int ld, int m, int i, int j,
                                                 double tau, const double* __restrict__ vh) {
  double w[4] = {P[i * ld + j], 0.0, 0.0, 0.0};
  int row = i + 1;
  for (; row + 4 <= m; row += 4) {
    double x[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) x[c] = P[(row + c) * ld + j];
#pragma unroll
    for (int c = 0; c < 4; ++c) w[c] = __fma_rn(vh[row + c], x[c], w[c]);
  }
  for (int c = 0; row < m; ++row, ++c) w[c] = __fma_rn(vh[row], P[row * ld + j], w[c]);
  const double t = -__dmul_rn(tau, __dadd_rn(__dadd_rn(w[0], w[1]), __dadd_rn(w[2], w[3])));
  P[i * ld + j] = __dadd_rn(P[i * ld + j], t);
  for (row = i + 1; row < m; row += CH) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = row + c < m ? P[(row + c) * ld + j] : 0.0;
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (row + c < m) P[(row + c) * ld + j] = __fma_rn(t, vh[row + c], x[c]);
  }
}

}  // namespace qr
}  // namespace smash
