// Kernel functions K(x, y) evaluated in registers (smash/kernel.py:278-310 for the
// real 1-D Cauchy kernel; log|x-y|, 1/|x-y|, exp(-|x-y|) are the BASELINE kernels,
// SURVEY.md 8(c)).  Coincident points (r^2 == 0, or x - y == 0 for Cauchy) take the
// KernelSpec.dx value, except exp whose diagonal is the natural exp(0) = 1.
#pragma once

#include "common.cuh"

namespace smash {

// Branch-free fp64 1/sqrt: MUFU approximation (~2^-20) + two Newton steps
// (measured max relative error 2.7e-16 vs 2.2e-16 for CUDA's rsqrt(), which
// carries a special-case branch that breaks instruction-level parallelism
// across the unrolled target tiles of the P2P kernels; tools/rsqrt_test.cu).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double h = x * y;
    const double e = fma(-h, y, 1.0);
    y = fma(0.5 * y, e, y);
  }
  return y;
}

template <int KER, int D>
__device__ __forceinline__ double kval(const double* x, const double* y, double dx) {
  if (KER == SMASH_KERNEL_CAUCHY) {
    double d = x[0] - y[0];
    return d == 0.0 ? dx : 1.0 / d;
  }
  double r2 = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double t = x[a] - y[a];
    r2 = fma(t, t, r2);
  }
  if (KER == SMASH_KERNEL_LOG) return r2 == 0.0 ? dx : 0.5 * log(r2);
  if (KER == SMASH_KERNEL_INV_R) {
    const double v = rsqrt_nr(r2);
    return r2 == 0.0 ? dx : v;
  }
  // exp(-r): r = sqrt(r2); exp(0) = 1 on the diagonal
  return exp(-sqrt(r2));
}

// runtime dispatch helper: f.template operator()<KER, D>()
template <typename F>
void dispatch_kernel_dim(int ker, int dim, F&& f) {
  switch (ker * 4 + dim) {
    case SMASH_KERNEL_LOG * 4 + 1: f.template operator()<SMASH_KERNEL_LOG, 1>(); break;
    case SMASH_KERNEL_LOG * 4 + 2: f.template operator()<SMASH_KERNEL_LOG, 2>(); break;
    case SMASH_KERNEL_LOG * 4 + 3: f.template operator()<SMASH_KERNEL_LOG, 3>(); break;
    case SMASH_KERNEL_INV_R * 4 + 1: f.template operator()<SMASH_KERNEL_INV_R, 1>(); break;
    case SMASH_KERNEL_INV_R * 4 + 2: f.template operator()<SMASH_KERNEL_INV_R, 2>(); break;
    case SMASH_KERNEL_INV_R * 4 + 3: f.template operator()<SMASH_KERNEL_INV_R, 3>(); break;
    case SMASH_KERNEL_EXP * 4 + 1: f.template operator()<SMASH_KERNEL_EXP, 1>(); break;
    case SMASH_KERNEL_EXP * 4 + 2: f.template operator()<SMASH_KERNEL_EXP, 2>(); break;
    case SMASH_KERNEL_EXP * 4 + 3: f.template operator()<SMASH_KERNEL_EXP, 3>(); break;
    case SMASH_KERNEL_CAUCHY * 4 + 1: f.template operator()<SMASH_KERNEL_CAUCHY, 1>(); break;
    default: throw Error(SMASH_ERR_INVALID, "unsupported kernel / dimension combination");
  }
}

}  // namespace smash
