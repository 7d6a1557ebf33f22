// Kernel functions K(x, y) evaluated in registers (smash/kernel.py:278-310 for the
// real 1-D Cauchy kernel; log|x-y|, 1/|x-y|, exp(-|x-y|) are the BASELINE kernels,
// SURVEY.md 8(c)).  Coincident points (r^2 == 0, or x - y == 0 for Cauchy) take the
// KernelSpec.dx value, except exp whose diagonal is the natural exp(0) = 1.
#pragma once

#include "common.cuh"

namespace smash {

// Branch-free fp64 1/sqrt: MUFU.RSQ64H approximation (max rel. error 9.2e-7),
// one residual e = 1 - x y0^2 and the quadratic correction
// y = y0 (1 + e/2 + 3e^2/8) (truncation ~(5/16)e^3 < 2^-60): 5 FP64 ops instead
// of the 8 of two Newton steps, measured max rel. error 2.65e-16 (CUDA's
// rsqrt(): 2.2e-16, but with a special-case branch that breaks the ILP across
// the unrolled target tiles of the P2P kernels; tools/rsqrt_test.cu).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
  const double h = x * y0;
  const double e = fma(-h, y0, 1.0);
  const double p = fma(e, 0.375, 0.5);
  return fma(y0 * e, p, y0);
}

// Branch-free fp64 reciprocal: MUFU.RCP64H approximation, e = 1 - x y0,
// y = y0 (1 + e + e^2) (truncation e^3 < 2^-59).
__device__ __forceinline__ double rcp_nr(double x) {
  double y0;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
  const double e = fma(-x, y0, 1.0);
  return fma(y0, fma(e, e, e), y0);
}

// x == +-0.0 tested on the integer pipe (keeps DSETP off the FP64 pipe)
__device__ __forceinline__ bool is_zero(double x) {
  return ((__double2hiint(x) & 0x7fffffff) | __double2loint(x)) == 0;
}

// Branch-free 0.5 * log(x) for positive normal x (the log kernel's 0.5 log r^2):
// x = 2^e m, m in [sqrt(1/2), sqrt(2)), f = (m-1)/(m+1), 0.5 log m = atanh f =
// f (1 + f^2/3 + f^4/5 + ...), |f| <= 0.1716: 10 terms (truncation s^10/21 < 3e-17,
// s = f^2), the halving folded into the series and the ln2 split (e ln2 / 2).
__device__ __forceinline__ double log_half_pos(double x) {
  int hi = __double2hiint(x);
  const int lo = __double2loint(x);
  int e = (hi >> 20) - 1023;
  int mh = (hi & 0x000fffff) | 0x3ff00000;
  const bool big = mh > 0x3ff6a09e;  // m > sqrt(2) -> m / 2
  mh = big ? mh - 0x00100000 : mh;
  e = big ? e + 1 : e;
  const double m = __hiloint2double(mh, lo);
  const double f = (m - 1.0) * rcp_nr(m + 1.0);
  const double s = f * f;
  double p = 1.0 / 21;
  p = fma(p, s, 1.0 / 19); p = fma(p, s, 1.0 / 17);
  p = fma(p, s, 1.0 / 15); p = fma(p, s, 1.0 / 13); p = fma(p, s, 1.0 / 11);
  p = fma(p, s, 1.0 / 9); p = fma(p, s, 1.0 / 7); p = fma(p, s, 1.0 / 5);
  p = fma(p, s, 1.0 / 3);
  const double lm = fma(f * s, p, f);
  const double de = (double)e;
  return fma(de, 3.46573590184561908245e-01, fma(de, 9.54107464635293850010e-11, lm));
}

// Table-driven 0.5 * log(x) for the matvec kernels (coupling / nearfield P2P, where the
// evaluation count decides the run time): x = 2^e m, m in [1, 2); the top 5 mantissa bits
// pick c_j = 1 + (j + 0.5) / 32 and the entry {ic_j = fl(1 / c_j), lc_j = fl(-0.5 log ic_j)};
// u = fma(m, ic_j, -1) is exact to its own rounding and |u| <= 2^-6, so
// 0.5 log m = lc_j + 0.5 log1p(u) with the series to u^9 (remainder u^10 / 20 < 1e-19).
// lc_j belongs to the ROUNDED ic_j: no table bias.  11 FP64 operations after the table read
// against 21 for the atanh series of log_half_pos (no reciprocal); measured against an 80-bit
// reference the absolute error stays below 2.3e-16 (tools/gen_logtab.py).  The table lives in
// shared memory, 8 copies of each 16-byte entry side by side (copy = lane & 7): the 8 lanes
// of an LDS.128 quarter-warp read different bank groups whatever their entries, so the read
// is conflict-free.
static __device__ const double2 g_logtab[32] = {
    {0x1.f81f81f81f820p-1, 0x1.fc0a8b0fc03c4p-8},  {0x1.e9131abf0b767p-1, 0x1.77458f632dcffp-6},
    {0x1.dae6076b981dbp-1, 0x1.341d7961bd1d0p-5},  {0x1.cd85689039b0bp-1, 0x1.a926d3a4ad562p-5},
    {0x1.c0e070381c0e0p-1, 0x1.0d77e7cd08e5bp-4},  {0x1.b4e81b4e81b4fp-1, 0x1.44d2b6ccb7d1cp-4},
    {0x1.a98ef606a63bep-1, 0x1.7ab890210d907p-4},  {0x1.9ec8e951033d9p-1, 0x1.af3c94e80bff3p-4},
    {0x1.948b0fcd6e9e0p-1, 0x1.e27076e2af2e8p-4},  {0x1.8acb90f6bf3aap-1, 0x1.0a324e27390e2p-3},
    {0x1.8181818181818p-1, 0x1.22941fbcf7966p-3},  {0x1.78a4c8178a4c8p-1, 0x1.3a64c556945eap-3},
    {0x1.702e05c0b8170p-1, 0x1.51aad872df82ep-3},  {0x1.6816816816817p-1, 0x1.686c81e9b14adp-3},
    {0x1.6058160581606p-1, 0x1.7eaf83b82afc2p-3},  {0x1.58ed2308158edp-1, 0x1.947941c2116fbp-3},
    {0x1.51d07eae2f815p-1, 0x1.a9cec9a9a084ap-3},  {0x1.4afd6a052bf5bp-1, 0x1.beb4d9da71b7ap-3},
    {0x1.446f86562d9fbp-1, 0x1.d32fe7e00ebd5p-3},  {0x1.3e22cbce4a902p-1, 0x1.e744261d68789p-3},
    {0x1.3813813813814p-1, 0x1.faf588f78f31dp-3},  {0x1.323e34a2b10bfp-1, 0x1.0723e5c1cdf41p-2},
    {0x1.2c9fb4d812ca0p-1, 0x1.109f39e2d4c96p-2},  {0x1.27350b8812735p-1, 0x1.19ee6b467c96fp-2},
    {0x1.21fb78121fb78p-1, 0x1.23130d7bebf43p-2},  {0x1.1cf06ada2811dp-1, 0x1.2c0e9ed448e8cp-2},
    {0x1.1811811811812p-1, 0x1.34e289d9ce1d2p-2},  {0x1.135c81135c811p-1, 0x1.3d9026a7156fbp-2},
    {0x1.0ecf56be69c90p-1, 0x1.4618bc21c5ec2p-2},  {0x1.0a6810a6810a7p-1, 0x1.4e7d811b75bb0p-2},
    {0x1.0624dd2f1a9fcp-1, 0x1.56bf9d5b3f399p-2},  {0x1.0204081020408p-1, 0x1.5ee02a9241676p-2},
};
constexpr int LOGTAB_BYTES = 32 * 8 * 16;  // shared-memory copy: entry j, copy c at [j * 8 + c]
constexpr int KERTAB_BYTES = LOGTAB_BYTES;  // the exp table below has the same footprint

__device__ __forceinline__ void logtab_fill(double2* tab) {
  for (int e = threadIdx.x; e < 32 * 8; e += blockDim.x) tab[e] = g_logtab[e >> 3];
}

__device__ __forceinline__ double log_half_tab(double x, const double2* tab, int copy) {
  const int hi = __double2hiint(x);
  const int e = (hi >> 20) - 1023;
  const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, __double2loint(x));
  const double2 t = tab[((hi >> 15) & 31) * 8 + copy];
  const double u = fma(m, t.x, -1.0);
  double q = 1.0 / 18;  // 0.5 * (-1/2, 1/3, ..., 1/9), Horner from the u^9 term
  q = fma(q, u, -1.0 / 16); q = fma(q, u, 1.0 / 14); q = fma(q, u, -1.0 / 12);
  q = fma(q, u, 1.0 / 10); q = fma(q, u, -1.0 / 8); q = fma(q, u, 1.0 / 6);
  q = fma(q, u, -0.25);
  // 0.5 log1p(u) = u (0.5 + u q); e ln2 / 2 with the constant in one piece: its representation
  // error |e| 2^-55 stays below 2.3e-16 absolute for |e| <= 80 (measured, tools/gen_logtab.py)
  const double lm = fma(u, fma(u, q, 0.5), t.y);
  return fma((double)e, 3.4657359027997264e-01, lm);
}

// Branch-free exp for x <= 0 (exp(-r) kernel): n = rint(x / ln2),
// t = x - n ln2 (|t| <= 0.347, Cody-Waite), Taylor to degree 13, scale by 2^n.
__device__ __forceinline__ double exp_neg(double x) {
  const bool under = x < -708.0;
  x = under ? -708.0 : x;
  const double sh = 6755399441055744.0;  // 1.5 * 2^52: round to nearest integer
  const double kd = fma(x, 1.4426950408889634, sh);
  const int n = __double2loint(kd);
  const double nd = kd - sh;
  double t = fma(-nd, 6.93147180369123816490e-01, x);
  t = fma(-nd, 1.90821492927058770002e-10, t);
  double p = 1.0 / 6227020800.0;  // 1/13!
  p = fma(p, t, 1.0 / 479001600.0); p = fma(p, t, 1.0 / 39916800.0);
  p = fma(p, t, 1.0 / 3628800.0); p = fma(p, t, 1.0 / 362880.0);
  p = fma(p, t, 1.0 / 40320.0); p = fma(p, t, 1.0 / 5040.0); p = fma(p, t, 1.0 / 720.0);
  p = fma(p, t, 1.0 / 120.0); p = fma(p, t, 1.0 / 24.0); p = fma(p, t, 1.0 / 6.0);
  p = fma(p, t, 0.5); p = fma(p, t, 1.0); p = fma(p, t, 1.0);
  const double sc = __hiloint2double((n + 1023) << 20, 0);
  return under ? 0.0 : p * sc;
}

template <int KER, int D>
__device__ __forceinline__ double kval(const double* x, const double* y, double dx) {
  if (KER == SMASH_KERNEL_CAUCHY) {
    const double d = x[0] - y[0];
    const double v = rcp_nr(d);
    return is_zero(d) ? dx : v;
  }
  double r2 = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double t = x[a] - y[a];
    r2 = fma(t, t, r2);
  }
  if (KER == SMASH_KERNEL_LOG) {
    const double v = log_half_pos(r2);
    return is_zero(r2) ? dx : v;
  }
  if (KER == SMASH_KERNEL_INV_R) {
    const double v = rsqrt_nr(r2);
    return is_zero(r2) ? dx : v;
  }
  // exp(-r): r = r2 * rsqrt(r2) (0 on the diagonal, exp(0) = 1)
  const double r = r2 * rsqrt_nr(r2);
  return exp_neg(is_zero(r2) ? 0.0 : -r);
}

// Table-driven exp(x), x <= 0, for the matvec kernels: k = rint(32 x / ln2), x = k ln2 / 32 + t,
// |t| <= ln2 / 64, exp(x) = 2^(k >> 5) * 2^((k & 31) / 32) * exp(t) with exp(t) to t^6 (remainder
// t^7 / 5040 < 4e-18): 12 FP64 operations against 19 for the degree-13 Taylor sum of exp_neg;
// relative error <= 3.2e-16 against an 80-bit reference (tools/gen_logtab.py).  The 32 doubles
// 2^(j/32) sit in shared memory as 16 copies side by side (copy = lane & 15): the 16 lanes of an
// LDS.64 half-warp read different banks whatever their entries.
static __device__ const double g_exptab[32] = {
    0x1.0000000000000p+0, 0x1.059b0d3158574p+0, 0x1.0b5586cf9890fp+0, 0x1.11301d0125b51p+0,
    0x1.172b83c7d517bp+0, 0x1.1d4873168b9aap+0, 0x1.2387a6e756238p+0, 0x1.29e9df51fdee1p+0,
    0x1.306fe0a31b715p+0, 0x1.371a7373aa9cbp+0, 0x1.3dea64c123422p+0, 0x1.44e086061892dp+0,
    0x1.4bfdad5362a27p+0, 0x1.5342b569d4f82p+0, 0x1.5ab07dd485429p+0, 0x1.6247eb03a5585p+0,
    0x1.6a09e667f3bcdp+0, 0x1.71f75e8ec5f74p+0, 0x1.7a11473eb0187p+0, 0x1.82589994cce13p+0,
    0x1.8ace5422aa0dbp+0, 0x1.93737b0cdc5e5p+0, 0x1.9c49182a3f090p+0, 0x1.a5503b23e255dp+0,
    0x1.ae89f995ad3adp+0, 0x1.b7f76f2fb5e47p+0, 0x1.c199bdd85529cp+0, 0x1.cb720dcef9069p+0,
    0x1.d5818dcfba487p+0, 0x1.dfc97337b9b5fp+0, 0x1.ea4afa2a490dap+0, 0x1.f50765b6e4540p+0,
};

__device__ __forceinline__ void exptab_fill(double* tab) {
  for (int e = threadIdx.x; e < 32 * 16; e += blockDim.x) tab[e] = g_exptab[e >> 4];
}

__device__ __forceinline__ double exp_neg_tab(double x, const double* tab, int copy) {
  const bool under = x < -708.0;
  x = under ? -708.0 : x;
  const double sh = 6755399441055744.0;  // 1.5 * 2^52: round to nearest integer
  const double kd = fma(x, 46.16624130844683, sh);  // 32 / ln2
  const int k = __double2loint(kd);
  const double nd = kd - sh;
  double t = fma(-nd, 0x1.62e42fef80000p-6, x);  // ln2 / 32, high part (35 bits: k * hi exact)
  t = fma(-nd, 0x1.1cf79ac000000p-41, t);
  const double tj = tab[(k & 31) * 16 + copy];
  double p = 1.0 / 720.0;
  p = fma(p, t, 1.0 / 120.0); p = fma(p, t, 1.0 / 24.0); p = fma(p, t, 1.0 / 6.0);
  p = fma(p, t, 0.5); p = fma(p, t, 1.0); p = fma(p, t, 1.0);
  const double sc = __hiloint2double(((k >> 5) + 1023) << 20, 0);
  return under ? 0.0 : (tj * p) * sc;
}

// kval for the matvec kernels: the log and exp kernels read their shared-memory table (tab:
// KERTAB_BYTES, filled by kertab_fill), every other kernel is kval itself.
template <int KER>
constexpr bool kertab_used() { return KER == SMASH_KERNEL_LOG || KER == SMASH_KERNEL_EXP; }

template <int KER>
__device__ __forceinline__ void kertab_fill(double2* tab) {
  if constexpr (KER == SMASH_KERNEL_LOG) logtab_fill(tab);
  if constexpr (KER == SMASH_KERNEL_EXP) exptab_fill(reinterpret_cast<double*>(tab));
}

template <int KER, int D>
__device__ __forceinline__ double kval_mv(const double* x, const double* y, double dx, const double2* tab,
                                          int lane) {
  if constexpr (KER == SMASH_KERNEL_LOG || KER == SMASH_KERNEL_EXP) {
    double r2 = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      double t = x[a] - y[a];
      r2 = fma(t, t, r2);
    }
    if constexpr (KER == SMASH_KERNEL_LOG) {
      const double v = log_half_tab(r2, tab, lane & 7);
      return is_zero(r2) ? dx : v;
    } else {
      // exp(-r): r = r2 * rsqrt(r2) (0 on the diagonal, exp(0) = 1)
      const double r = r2 * rsqrt_nr(r2);
      return exp_neg_tab(is_zero(r2) ? 0.0 : -r, reinterpret_cast<const double*>(tab), lane & 15);
    }
  } else {
    return kval<KER, D>(x, y, dx);
  }
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
