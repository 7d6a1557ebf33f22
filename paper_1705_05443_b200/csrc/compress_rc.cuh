// K3 + K4, register-column variant (instantiated per point dimension by compress_rc_d{1,2,3}.cu).
//
// Same algorithm and the same floating-point operation order as k_compress (pivots,
// ranks, swap decisions and G are bit-identical to it), with a different home for the
// panel: thread j owns ibar column j for the whole node.  The last RR rows of the
// column live in registers, the rows above them in shared memory (row-major, one column
// per thread, conflict free).  Consequences:
//  * a 64 x 256 panel needs 64 KB of shared memory instead of 128 KB: two CTAs per SM
//    with everything on chip (k_compress ran such nodes from global/L2 panels or alone
//    on an SM), and four times less shared-memory traffic per pivot step;
//  * columns are never swapped physically: dlaqp2's column order is a position kept per
//    thread (pos) and the position -> column table jpvt; the first-maximum pivot rule is
//    evaluated on positions;
//  * register rows are indexed statically, so every step runs over all RR register
//    rows with the reflector zero-padded above the pivot row (adds exact zeros); the
//    four accumulation chains are assigned by row mod 4 and combined in the rotation
//    that reproduces k_compress's (row - i - 1) mod 4 chains bit for bit;
//  * the pivot column is published to shared memory for warp 0's dlarfg, which keeps
//    the lane-strided norm of k_compress.
// Used for size classes of at most 256 columns (one column per thread, CTAs of 64 / 128 /
// 256 threads); wider panels and the single-call compr stay on k_compress.

#pragma once

#include <cooperative_groups.h>

#include "compress_common.cuh"

namespace smash {
namespace {

using namespace qr;
using namespace cmn;
namespace cg = cooperative_groups;

struct RcShared {
  double* vh0;     // reflector of the current step, zero at rows <= i   [vhn]
  double* vh1;     // the same with a one at row i (dlarf's v)           [vhn]
  double* colbuf;  // published register rows of the pivot column       [vhn]
  double* rdiag;   // [mmax]
  double* nodes;   // Chebyshev nodes per axis, [D][rc_nodes_stride(D)]
  double* redv;    // [32]
  double* misc;    // [8]
  double* r11;     // R11 [kcap][kld], or a block of four of its rows (streaming variants)
  double* panel;   // [srows][NT]
  int* redi;       // [32]
  int* imisc;      // [8]
  int* jpvt;       // position -> column, [NT] (clusters: a global slice of CS * NT)
};

// The same shared arrays in every CTA of the cluster (CS = 1: the CTA itself).  Wide nodes
// (|ibar| <= CS * NT) are spread over a thread-block cluster, NT columns per CTA: the pivot
// candidates, the reflector and the streamed R11 rows are written into every CTA's shared
// memory (DSMEM), and the barriers that order them become cluster barriers.
template <int CS>
struct RcPeers {
  double* vh0[CS];
  double* vh1[CS];
  double* misc[CS];
  double* rdiag[CS];
  double* redv[CS];
  double* r11[CS];
  int* redi[CS];
  int* imisc[CS];
  int crank = 0;
  __device__ __forceinline__ void sync() const {
    if constexpr (CS > 1) cg::this_cluster().sync();
    else __syncthreads();
  }
};

// x[s] for a CTA-uniform s: a tree of selects per block of 16 registers instead of a
// dynamically indexed array (a dense switch measured slower: cfg5 build 30.9 -> 37.6 ms).
__device__ __forceinline__ double rc_sel16(const double* x, int s) {
  double a[8], b[4], c[2];
#pragma unroll
  for (int t = 0; t < 8; ++t) a[t] = (s & 1) ? x[2 * t + 1] : x[2 * t];
#pragma unroll
  for (int t = 0; t < 4; ++t) b[t] = (s & 2) ? a[2 * t + 1] : a[2 * t];
#pragma unroll
  for (int t = 0; t < 2; ++t) c[t] = (s & 4) ? b[2 * t + 1] : b[2 * t];
  return (s & 8) ? c[1] : c[0];
}
template <int RR>
__device__ __forceinline__ double rc_sel(const double (&x)[RR], int s) {
  static_assert(RR % 4 == 0 && RR >= 16 && RR <= 48, "register rows");
  // blocks [0,16), [16,32), [RR-16,RR) (the last one may overlap the second)
  double r = rc_sel16(&x[0], s & 15);
  if (RR > 16) {
    const double r1 = rc_sel16(&x[RR >= 32 ? 16 : RR - 16], RR >= 32 ? (s & 15) : s - (RR - 16));
    r = s >= 16 ? r1 : r;
  }
  if (RR > 32) {
    const double r2 = rc_sel16(&x[RR - 16], s - (RR - 16));
    r = s >= 32 ? r2 : r;
  }
  return r;
}

// (max value, smallest index) over the CTA with one barrier; two calls must be separated
// by another barrier.  Candidates are non-negative doubles (norms, |W| entries) or -1 for
// "none": their bit patterns order like unsigned integers, so each warp reduces with three
// redux.sync operations (high word, low word among the leaders, smallest index among the
// equals) instead of five shuffle rounds.  Returns the index, the value through v.
template <int NT, int CS>
__device__ __forceinline__ int rc_argmax(double& v, int i, RcShared& S, const RcPeers<CS>& P) {
  constexpr int NW = NT / 32;
  static_assert(CS * NW <= 32, "one lane per warp partial of the cluster");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool valid = v >= 0.0;
  const unsigned long long key = valid ? (unsigned long long)__double_as_longlong(v) : 0ULL;
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  const unsigned mi = __reduce_min_sync(0xffffffffu, (valid && hi == mh && lo == ml) ? (unsigned)i : 0x7fffffffu);
  if constexpr (CS == 1) {
    if (lane == 0) {
      reinterpret_cast<unsigned long long*>(S.redv)[wid] = ((unsigned long long)mh << 32) | ml;
      S.redi[wid] = (int)mi;
    }
    __syncthreads();
    unsigned long long bk = reinterpret_cast<const unsigned long long*>(S.redv)[0];
    int bi = S.redi[0];
#pragma unroll
    for (int w = 1; w < NW; ++w) {
      const unsigned long long ok = reinterpret_cast<const unsigned long long*>(S.redv)[w];
      const int oi = S.redi[w];
      if (ok > bk || (ok == bk && oi < bi)) { bk = ok; bi = oi; }
    }
    v = bi == 0x7fffffff ? -1.0 : __longlong_as_double((long long)bk);
    return bi;
  } else {
    // every warp's partial goes to every CTA; after the cluster barrier one lane per
    // partial and three more redux operations
    const int slot = P.crank * NW + wid;
#pragma unroll
    for (int q = 0; q < CS; ++q)  // (static peer index: the pointer arrays stay in registers)
      if (lane == q) {
        reinterpret_cast<unsigned long long*>(P.redv[q])[slot] = ((unsigned long long)mh << 32) | ml;
        P.redi[q][slot] = (int)mi;
      }
    P.sync();
    const bool on = lane < CS * NW;
    const unsigned long long k2 = on ? reinterpret_cast<const unsigned long long*>(S.redv)[lane] : 0ULL;
    const int i2 = on ? S.redi[lane] : 0x7fffffff;
    const unsigned h2 = (unsigned)(k2 >> 32), l2 = (unsigned)k2;
    const unsigned gh = __reduce_max_sync(0xffffffffu, h2);
    const unsigned gl = __reduce_max_sync(0xffffffffu, h2 == gh ? l2 : 0u);
    const unsigned gi = __reduce_min_sync(0xffffffffu, (h2 == gh && l2 == gl) ? (unsigned)i2 : 0x7fffffffu);
    v = gi == 0x7fffffffu ? -1.0 : __longlong_as_double((long long)(((unsigned long long)gh << 32) | gl));
    return (int)gi;
  }
}

// dlarfg on the published pivot column c at step i, by one warp (the owner's), as
// qr::householder: the lane-strided sum of squares, beta / tau / scal, the scaled
// reflector to vh0 / vh1.
template <int NT, int CS>
__device__ __forceinline__ void rc_householder(const double* __restrict__ Ps, int rbase, int m, int i,
                                               int c, RcShared& S, const RcPeers<CS>& P) {
  const int lane = threadIdx.x & 31;
  const double* __restrict__ pc = Ps + c;
  const double* __restrict__ cb = S.colbuf;
  const double alpha = i < rbase ? pc[i * NT] : cb[i];
  double ss = 0.0;
#pragma unroll 1
  for (int row = i + 1 + lane; row < m; row += 32) {
    const double x = row < rbase ? pc[row * NT] : cb[row];
    ss = __fma_rn(x, x, ss);
  }
  for (int off = 16; off; off >>= 1) ss = __dadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, off));
  const double xnorm = __dsqrt_rn(ss);
  double tau = 0.0, diag = alpha;
  if (m - i > 1 && xnorm != 0.0) {
    const double beta = -copysign(dlapy2(alpha, xnorm), alpha);
    tau = __ddiv_rn(__dsub_rn(beta, alpha), beta);
    const double scal = __ddiv_rn(1.0, __dsub_rn(alpha, beta));
#pragma unroll 1
    for (int row = i + 1 + lane; row < m; row += 32) {
      const double x = __dmul_rn(scal, row < rbase ? pc[row * NT] : cb[row]);
#pragma unroll
      for (int q = 0; q < CS; ++q) { P.vh0[q][row] = x; P.vh1[q][row] = x; }
    }
    diag = beta;
  }
#pragma unroll
  for (int q = 0; q < CS; ++q)
    if (lane == q) {
      P.vh0[q][i] = 0.0;
      P.vh1[q][i] = 1.0;
      if (i > 0) P.vh1[q][i - 1] = 0.0;
      P.misc[q][0] = tau;
      P.rdiag[q][i] = diag;
    }
}

template <int D, int NT, int RR, bool R11G, int CS>
__device__ __forceinline__ void rc_node(const CompressArgs& A, RcShared& S, const RcPeers<CS>& P, int v,
                                        int n, int m, const NodeSrc& src, int vhn, int kld) {
  static_assert(CS == 1 || R11G, "clusters stream R11");
  const int tid = threadIdx.x;
  const int gcol = P.crank * NT + tid;  // the own column of ibar
  const int rbase = max(0, rc_round4(m - RR));
  double* __restrict__ Ps = S.panel;
#ifdef SMASH_COMPRESS_PROF
  long long pt0 = clock64();
#define RC_MARK(k) if (tid == 0) { long long pt1 = clock64(); atomicAdd(A.prof + (k), (unsigned long long)(pt1 - pt0)); pt0 = pt1; }
#else
#define RC_MARK(k)
#endif
  const bool have = gcol < n;
  double xr[RR];

  // ---- own column of the panel (smash/lowrank.py:103-144; HSS rows hss.py:287)
  auto build_col = [&]() {
    const int r = A.r;
    const int mt = A.tab.m;
    double x[D];
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = src.base[(size_t)a * src.stride + gcol];
    const int kp = m - r;
    const double* sv = kp > 0 ? A.sv + A.sv_off[v] + (size_t)gcol * kp : nullptr;
    if (D == 1) {
      const double* nd = S.nodes;
      bool exact = false;
      for (int k = 0; k < mt; ++k) exact |= (__dsub_rn(x[0], nd[k]) == 0.0);
      double Ssum = 1.0;
      if (!exact)
        Ssum = np_pairwise_sum(mt, [&](int k) { return __ddiv_rn(A.tab.wv[k], __dsub_rn(x[0], nd[k])); });
      auto val = [&](int q) -> double {
        if (q >= r) return q < m ? sv[q - r] : 0.0;
        const double dx = __dsub_rn(x[0], nd[q]);
        if (exact) return dx == 0.0 ? 1.0 : 0.0;
        return __ddiv_rn(__ddiv_rn(A.tab.wv[q], dx), Ssum);
      };
      for (int q = 0; q < rbase; ++q) Ps[q * NT + tid] = val(q);
#pragma unroll
      for (int t = 0; t < RR; ++t) xr[t] = val(rbase + t);
    } else {
      double L[D][MAX_M_AXIS_ND];
#pragma unroll
      for (int a = 0; a < D; ++a) lagrange_axis(x[a], S.nodes + a * rc_nodes_stride(D), A.tab.wv, mt, L[a]);
      auto val = [&](int q) -> double {
        if (q >= r) return q < m ? sv[q - r] : 0.0;
        const int* o = A.tab.order + 3 * q;
        double pv = __dmul_rn(L[0][o[0]], L[1][o[1]]);
        if (D == 3) pv = __dmul_rn(pv, L[D - 1][o[2]]);
        return pv;
      };
      for (int q = 0; q < rbase; ++q) Ps[q * NT + tid] = val(q);
#pragma unroll
      for (int t = 0; t < RR; ++t) xr[t] = val(rbase + t);
    }
  };
  // sum of squares of the own column over rows > i0, chains by (row - i0 - 1) mod 4
  auto sumsq_after = [&](int i0) -> double {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (int g = (i0 + 1) & ~3; g < rbase; g += 4) {
      const double x0 = g + 0 > i0 ? Ps[(g + 0) * NT + tid] : 0.0;
      const double x1 = g + 1 > i0 ? Ps[(g + 1) * NT + tid] : 0.0;
      const double x2 = g + 2 > i0 ? Ps[(g + 2) * NT + tid] : 0.0;
      const double x3 = g + 3 > i0 ? Ps[(g + 3) * NT + tid] : 0.0;
      s0 = __fma_rn(x0, x0, s0); s1 = __fma_rn(x1, x1, s1);
      s2 = __fma_rn(x2, x2, s2); s3 = __fma_rn(x3, x3, s3);
    }
#pragma unroll
    for (int t = 0; t < RR; t += 4) {
      const double x0 = rbase + t + 0 > i0 ? xr[t + 0] : 0.0;
      const double x1 = rbase + t + 1 > i0 ? xr[t + 1] : 0.0;
      const double x2 = rbase + t + 2 > i0 ? xr[t + 2] : 0.0;
      const double x3 = rbase + t + 3 > i0 ? xr[t + 3] : 0.0;
      s0 = __fma_rn(x0, x0, s0); s1 = __fma_rn(x1, x1, s1);
      s2 = __fma_rn(x2, x2, s2); s3 = __fma_rn(x3, x3, s3);
    }
    return ((i0 + 1) & 1) ? __dadd_rn(__dadd_rn(s1, s2), __dadd_rn(s3, s0))
                          : __dadd_rn(__dadd_rn(s0, s1), __dadd_rn(s2, s3));
  };
  // own entry of row i (uniform i)
  auto own_row = [&](int i) -> double { return i < rbase ? Ps[i * NT + tid] : rc_sel<RR>(xr, i - rbase); };
  auto publish_col = [&]() {
#pragma unroll
    for (int t = 0; t < RR; t += 2)
      *reinterpret_cast<double2*>(S.colbuf + rbase + t) = make_double2(xr[t], xr[t + 1]);
  };

  for (int e = tid; e < vhn; e += NT) { S.vh0[e] = 0.0; S.vh1[e] = 0.0; S.colbuf[e] = 0.0; }
  if (have) {
    build_col();
    S.jpvt[gcol] = gcol;
  } else {
#pragma unroll
    for (int t = 0; t < RR; ++t) xr[t] = 0.0;
  }
  int pos = have ? gcol : 0x7fffffff;
  double vn1 = 0.0, vn2 = 0.0;
  double cv = -1.0;
  int cp = 0x7fffffff;
  if (have) {
    const double nr = __dsqrt_rn(sumsq_after(-1));
    vn1 = nr;
    vn2 = nr;
    if (nr > cv) { cv = nr; cp = pos; }
  }
  const int kmax = min(m, n);
  RC_MARK(0)
  // ---- dgeqp3 / dlaqp2 (two barriers per pivot step: pivot choice, reflector)
  for (int i = 0; i < kmax; ++i) {
    int pp = rc_argmax<NT, CS>(cv, cp, S, P);
    if (pp >= n) pp = i;  // (all candidates NaN)
    RC_MARK(1)
    // the column at position pp becomes pivot i, the column at position i takes its place
    // (each of the two threads records itself in the position -> column table)
    const bool owner = have && pos == pp;
    if (have && pos == i) { pos = pp; S.jpvt[pp] = gcol; }
    if (owner) { pos = i; S.jpvt[i] = gcol; }
    const unsigned own_mask = __ballot_sync(0xffffffffu, owner);
    if (own_mask) {  // the owner's warp: publish the register rows, then dlarfg
      if (owner) publish_col();
      __syncwarp();
      rc_householder<NT, CS>(Ps, rbase, m, i, (tid & ~31) + (__ffs(own_mask) - 1), S, P);
    }
    RC_MARK(2)
    P.sync();
    RC_MARK(3)
    cv = -1.0;
    cp = 0x7fffffff;
    if (have && pos > i) {
      const double tau = S.misc[0];
      // the norm-downdate divisions do not depend on the reflector: issue them first
      double v1 = vn1;
      const double rv1 = 1.0 / v1;
      const double q2 = v1 / vn2;
      const double xi = own_row(i);
      double pij = xi;
      if (tau != 0.0) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        {
          const int a = (i + 1) & 3;
          s0 = a == 0 ? xi : 0.0; s1 = a == 1 ? xi : 0.0; s2 = a == 2 ? xi : 0.0; s3 = a == 3 ? xi : 0.0;
        }
#pragma unroll 2
        for (int g = (i + 1) & ~3; g < rbase; g += 4) {
          const double2 va = *reinterpret_cast<const double2*>(S.vh0 + g);
          const double2 vb = *reinterpret_cast<const double2*>(S.vh0 + g + 2);
          const double x0 = Ps[(g + 0) * NT + tid], x1 = Ps[(g + 1) * NT + tid];
          const double x2 = Ps[(g + 2) * NT + tid], x3 = Ps[(g + 3) * NT + tid];
          s0 = __fma_rn(va.x, x0, s0); s1 = __fma_rn(va.y, x1, s1);
          s2 = __fma_rn(vb.x, x2, s2); s3 = __fma_rn(vb.y, x3, s3);
        }
#pragma unroll
        for (int t = 0; t < RR; t += 4) {
          const double2 va = *reinterpret_cast<const double2*>(S.vh0 + rbase + t);
          const double2 vb = *reinterpret_cast<const double2*>(S.vh0 + rbase + t + 2);
          s0 = __fma_rn(va.x, xr[t + 0], s0); s1 = __fma_rn(va.y, xr[t + 1], s1);
          s2 = __fma_rn(vb.x, xr[t + 2], s2); s3 = __fma_rn(vb.y, xr[t + 3], s3);
        }
        const double w = ((i + 1) & 1) ? __dadd_rn(__dadd_rn(s1, s2), __dadd_rn(s3, s0))
                                       : __dadd_rn(__dadd_rn(s0, s1), __dadd_rn(s2, s3));
        const double tt = -__dmul_rn(tau, w);
        pij = __dadd_rn(xi, tt);
#pragma unroll 2
        for (int g = i & ~3; g < rbase; g += 4) {
          const double2 va = *reinterpret_cast<const double2*>(S.vh1 + g);
          const double2 vb = *reinterpret_cast<const double2*>(S.vh1 + g + 2);
          const double x0 = Ps[(g + 0) * NT + tid], x1 = Ps[(g + 1) * NT + tid];
          const double x2 = Ps[(g + 2) * NT + tid], x3 = Ps[(g + 3) * NT + tid];
          Ps[(g + 0) * NT + tid] = __fma_rn(tt, va.x, x0);
          Ps[(g + 1) * NT + tid] = __fma_rn(tt, va.y, x1);
          Ps[(g + 2) * NT + tid] = __fma_rn(tt, vb.x, x2);
          Ps[(g + 3) * NT + tid] = __fma_rn(tt, vb.y, x3);
        }
#pragma unroll
        for (int t = 0; t < RR; t += 4) {
          const double2 va = *reinterpret_cast<const double2*>(S.vh1 + rbase + t);
          const double2 vb = *reinterpret_cast<const double2*>(S.vh1 + rbase + t + 2);
          xr[t + 0] = __fma_rn(tt, va.x, xr[t + 0]); xr[t + 1] = __fma_rn(tt, va.y, xr[t + 1]);
          xr[t + 2] = __fma_rn(tt, vb.x, xr[t + 2]); xr[t + 3] = __fma_rn(tt, vb.y, xr[t + 3]);
        }
      }
      if (v1 != 0.0) {
        double q = fabs(pij) * rv1;
        double temp = fmax(1.0 - q * q, 0.0);
        double temp2 = temp * (q2 * q2);
        if (temp2 <= TOL3Z) {
          double nv = i + 1 < m ? __dsqrt_rn(sumsq_after(i)) : 0.0;
          vn1 = nv;
          vn2 = nv;
          v1 = nv;
        } else {
          v1 = __dmul_rn(v1, __dsqrt_rn(temp));
          vn1 = v1;
        }
      }
      if (v1 > cv) { cv = v1; cp = pos; }
    }
    RC_MARK(4)
#ifdef SMASH_COMPRESS_PROF
    if (tid == 0) atomicAdd(A.prof + 7, 1ULL);
#endif
  }
  __syncthreads();
  // ---- numerical rank (count semantics, lowrank.py:163-167)
  if (tid == 0) {
    int k = 0;
    double r0 = fabs(S.rdiag[0]);
    if (r0 != 0.0) {
      double thr = __dmul_rn(A.rtol, r0);
      for (int i = 0; i < kmax; ++i) k += fabs(S.rdiag[i]) > thr ? 1 : 0;
    }
    S.imisc[0] = min(k, kmax);
  }
  __syncthreads();
  const int k = S.imisc[0];
  const int ktop = min(k, rbase);  // rows of R below it are register rows
  // ---- bounded-entry swap loop (lowrank.py:191-202)
  int swaps = 0;
  while (k > 0 && k < n) {
    const int nk = n - k;
    // R11 as a [a][c] array, zero outside the strict upper triangle (so the solve's aligned
    // groups need no bounds: out-of-range terms multiply by zero).  Resident variants hold
    // all of it in shared memory; streaming variants (R11G) a block of four rows at a time,
    // written by the thread at position c for every c (zero where R11 has no entry).
    {
      const int tot = R11G ? 4 * kld : k * kld;
      for (int e = tid; e < tot; e += NT) S.r11[e] = 0.0;
    }
    if (!R11G) {
      __syncthreads();
      if (have && pos < k) {
        const int top = min(pos, rbase);
        for (int a = 0; a < top; ++a) S.r11[a * kld + pos] = Ps[a * NT + tid];
#pragma unroll
        for (int t = 0; t < RR; ++t)
          if (rbase + t < pos) S.r11[(rbase + t) * kld + pos] = xr[t];
      }
      __syncthreads();
    }
    double bv = -1.0;
    int bi = 0x7fffffff;
    const bool solver = have && pos >= k;
    const bool writer = have && pos < kld;
    // W = R11^-1 R12 by back substitution on the own column, the same FMA sequence as
    // k_compress (terms k-1 .. a+1 of row a on four chains by (k-1-c) mod 4)
    const bool odd = (k - 1) & 1;
    if (rbase < k) {
#pragma unroll
      for (int t = RR - 1; t >= 0; --t) {
        const int a = rbase + t;
        if (R11G && (t & 3) == 3 && a - 3 < k) {  // next block of four register rows
          P.sync();
          if (writer) {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const double val = (pos > a - 3 + r && pos < k) ? xr[t - 3 + r] : 0.0;
#pragma unroll
              for (int q = 0; q < CS; ++q) P.r11[q][r * kld + pos] = val;
            }
          }
          P.sync();
        }
        if (a < k && solver) {
          double s[4] = {0.0, 0.0, 0.0, 0.0};
          const double* __restrict__ Rr = S.r11 + (R11G ? (t & 3) : a) * kld + rbase;
#pragma unroll
          for (int p2 = RR / 2 - 1; 2 * p2 + 1 > t; --p2) {
            const double2 rr = *reinterpret_cast<const double2*>(Rr + 2 * p2);
            s[(2 * p2 + 1) & 3] = __fma_rn(-xr[2 * p2 + 1], rr.y, s[(2 * p2 + 1) & 3]);
            if (2 * p2 > t) s[(2 * p2) & 3] = __fma_rn(-xr[2 * p2], rr.x, s[(2 * p2) & 3]);
          }
          const double comb = odd ? __dadd_rn(__dadd_rn(s[0], s[1]), __dadd_rn(s[2], s[3]))
                                  : __dadd_rn(__dadd_rn(s[1], s[2]), __dadd_rn(s[3], s[0]));
          const double x = __ddiv_rn(__dadd_rn(xr[t], comb), S.rdiag[a]);
          xr[t] = x;
          argmax_combine(bv, bi, fabs(x), a * nk + (pos - k));
        }
      }
    }
    for (int a = ktop - 1; a >= 0; --a) {
      if (R11G && ((a & 3) == 3 || a == ktop - 1)) {  // next block of four shared rows
        const int a0 = a & ~3;
        P.sync();
        if (writer) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const double val = (a0 + r < ktop && pos > a0 + r && pos < k) ? Ps[(a0 + r) * NT + tid] : 0.0;
#pragma unroll
            for (int q = 0; q < CS; ++q) P.r11[q][r * kld + pos] = val;
          }
        }
        P.sync();
      }
      if (solver) {
        double s[4] = {0.0, 0.0, 0.0, 0.0};
        const double* __restrict__ Ra = S.r11 + (R11G ? (a & 3) : a) * kld;
        if (rbase < k) {
#pragma unroll
          for (int p2 = RR / 2 - 1; p2 >= 0; --p2) {
            const double2 rr = *reinterpret_cast<const double2*>(Ra + rbase + 2 * p2);
            s[(2 * p2 + 1) & 3] = __fma_rn(-xr[2 * p2 + 1], rr.y, s[(2 * p2 + 1) & 3]);
            s[(2 * p2) & 3] = __fma_rn(-xr[2 * p2], rr.x, s[(2 * p2) & 3]);
          }
        }
#pragma unroll 2
        for (int g = (ktop - 1) & ~3; g + 3 > a; g -= 4) {
          const double2 r01 = *reinterpret_cast<const double2*>(Ra + g);
          const double2 r23 = *reinterpret_cast<const double2*>(Ra + g + 2);
          const double x0 = Ps[(g + 0) * NT + tid], x1 = Ps[(g + 1) * NT + tid];
          const double x2 = Ps[(g + 2) * NT + tid], x3 = Ps[(g + 3) * NT + tid];
          s[3] = __fma_rn(-x3, r23.y, s[3]); s[2] = __fma_rn(-x2, r23.x, s[2]);
          s[1] = __fma_rn(-x1, r01.y, s[1]); s[0] = __fma_rn(-x0, r01.x, s[0]);
        }
        const double comb = odd ? __dadd_rn(__dadd_rn(s[0], s[1]), __dadd_rn(s[2], s[3]))
                                : __dadd_rn(__dadd_rn(s[1], s[2]), __dadd_rn(s[3], s[0]));
        const double x = __ddiv_rn(__dadd_rn(Ps[a * NT + tid], comb), S.rdiag[a]);
        Ps[a * NT + tid] = x;
        argmax_combine(bv, bi, fabs(x), a * nk + (pos - k));
      }
    }
    bi = rc_argmax<NT, CS>(bv, bi, S, P);
    RC_MARK(5)
    if (!(bv > A.s_bound)) break;
    if (swaps >= MAX_SWAPS) {
      if (tid == 0) atomicOr(A.err, DEV_SWAP_CAP);
      break;
    }
    {
      const int sa = bi / nk, sj = bi % nk;
      const int ca = S.jpvt[sa], cb = S.jpvt[k + sj];
      P.sync();  // every thread has read the two table entries
      if (gcol == 0) { S.jpvt[sa] = cb; S.jpvt[k + sj] = ca; }
      for (int e = tid; e < vhn; e += NT) { S.vh0[e] = 0.0; S.vh1[e] = 0.0; }
      P.sync();
      if (gcol == ca) pos = k + sj;
      if (gcol == cb) pos = sa;
    }
    ++swaps;
    if (have) build_col();
    // unpivoted QR (dgeqr2) of the permuted panel; rows < k of R suffice.  Sequential
    // dot-product order, as k_compress's refactorisation.
    for (int i = 0; i < k; ++i) {
      const int c = S.jpvt[i];
      if ((gcol >> 5) == (c >> 5)) {  // the owner's warp (of the owner's CTA)
        if (gcol == c) publish_col();
        __syncwarp();
        rc_householder<NT, CS>(Ps, rbase, m, i, c - P.crank * NT, S, P);
      }
      P.sync();
      const double tau = S.misc[0];
      if (have && pos > i && tau != 0.0) {
        const double xi = own_row(i);
        double w = xi;
        for (int row = i + 1; row < rbase; ++row) w = __fma_rn(S.vh0[row], Ps[row * NT + tid], w);
#pragma unroll
        for (int t = 0; t < RR; ++t) w = __fma_rn(S.vh0[rbase + t], xr[t], w);
        const double tt = -__dmul_rn(tau, w);
        for (int row = i; row < rbase; ++row)
          Ps[row * NT + tid] = __fma_rn(tt, S.vh1[row], Ps[row * NT + tid]);
#pragma unroll
        for (int t = 0; t < RR; ++t) xr[t] = __fma_rn(tt, S.vh1[rbase + t], xr[t]);
      }
      P.sync();  // the next reflector overwrites vh0 / vh1
    }
    RC_MARK(6)
  }
  __syncthreads();
  // ---- outputs
  if (gcol == 0) {
    A.rank[v] = k;
    if (swaps) atomicAdd(A.swaps, (unsigned long long)swaps);
  }
  const int64_t io = A.ib_off[v];
  if (have) A.perm[io + gcol] = S.jpvt[gcol];
  if (k > 0 && k < n && have && pos >= k) {
    double* __restrict__ G = A.G + A.g_off[v] + (size_t)(pos - k) * k;
    for (int a = 0; a < ktop; ++a) G[a] = Ps[a * NT + tid];
#pragma unroll
    for (int t = 0; t < RR; ++t)
      if (rbase + t < k) G[rbase + t] = xr[t];
  }
  if (A.tmp_lab) {
    const int64_t lo = io - A.ib_level_base;
    if (gcol < k) {
      const int pc = S.jpvt[gcol];
      A.tmp_lab[lo + gcol] = src.lab ? src.lab[pc] : src.lab0 + pc;
      for (int d = 0; d < D; ++d)
        A.tmp_pts[(size_t)d * A.tmp_stride + lo + gcol] = src.base[(size_t)d * src.stride + pc];
    }
  }
  __syncthreads();
}

template <int D, int NT, int RR, bool R11G, int CS>
__global__ void __launch_bounds__(NT, RR > 32 ? 1 : (65536 / (NT * 128) > 16 ? 16 : 65536 / (NT * 128)))
k_compress_rc(CompressArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int vhn = rc_vhn(A.mmax, RR);
  const int kcap = rc_kcap(A.mmax, NT);
  const int kld = rc_kld(A.mmax, RR);
  const int srows = rc_srows(A.mmax, RR);
  RcShared S;
  {
    double* d = reinterpret_cast<double*>(smem_raw);
    S.vh0 = d; d += vhn;
    S.vh1 = d; d += vhn;
    S.colbuf = d; d += vhn;
    S.r11 = d; d += R11G ? (size_t)4 * kld : (size_t)kcap * kld;
    S.panel = d; d += (size_t)srows * NT;
    S.rdiag = d; d += rc_round4(A.mmax);
    S.nodes = d; d += D * rc_nodes_stride(D);
    S.redv = d; d += 32;
    S.misc = d; d += 8;
    int* ip = reinterpret_cast<int*>(d);
    S.redi = ip; ip += 32;
    S.imisc = ip; ip += 8;
    S.jpvt = ip;
  }
  RcPeers<CS> P;
  if constexpr (CS > 1) {
    cg::cluster_group cl = cg::this_cluster();
    P.crank = (int)cl.block_rank();
#pragma unroll
    for (int q = 0; q < CS; ++q) {
      P.vh0[q] = cl.map_shared_rank(S.vh0, q);
      P.vh1[q] = cl.map_shared_rank(S.vh1, q);
      P.misc[q] = cl.map_shared_rank(S.misc, q);
      P.rdiag[q] = cl.map_shared_rank(S.rdiag, q);
      P.redv[q] = cl.map_shared_rank(S.redv, q);
      P.r11[q] = cl.map_shared_rank(S.r11, q);
      P.redi[q] = cl.map_shared_rank(S.redi, q);
      P.imisc[q] = cl.map_shared_rank(S.imisc, q);
    }
    // position -> column table of the cluster's node: a global slice
    S.jpvt = reinterpret_cast<int*>(A.gws) + (size_t)(blockIdx.x / CS) * (CS * NT);
  } else {
    P.vh0[0] = S.vh0; P.vh1[0] = S.vh1; P.misc[0] = S.misc; P.rdiag[0] = S.rdiag;
    P.redv[0] = S.redv; P.r11[0] = S.r11; P.redi[0] = S.redi; P.imisc[0] = S.imisc;
  }
  const int tid = threadIdx.x;
  const int nteams = (int)gridDim.x / CS;  // CTAs (clusters) claiming nodes
  auto next_node = [&]() {
    P.sync();
    if (P.crank == 0 && tid == 0) {
      const int nv = A.lb + nteams + atomicAdd(A.next, 1);
#pragma unroll
      for (int q = 0; q < CS; ++q) P.imisc[q][4] = nv;
    }
    P.sync();
    return S.imisc[4];
  };
  for (int v = A.lb + (int)blockIdx.x / CS; v < A.le;) {
    const int n = A.nib[v];
    if (n <= A.n_lo || n > A.n_hi) {  // another launch of this level takes this size class
      v = next_node();
      continue;
    }
    if (n == 0) {
      if (P.crank == 0 && tid == 0) A.rank[v] = 0;
      v = next_node();
      continue;
    }
    const int m = A.r + (A.keep ? A.keep[v] : 0);
    SMASH_DASSERT(n <= CS * NT && m <= A.mmax);
    const NodeSrc src = node_src(A, v);
    // ---- padded box + Chebyshev nodes (hss.py:39-45, lowrank.py:103-105,127-134)
    if (tid == 0) {
      double plo[3], phi[3];
      double scale = 1.0;
      for (int a = 0; a < D; ++a) {
        double lo = A.lo[(size_t)v * D + a], hi = A.hi[(size_t)v * D + a];
        if (__dsub_rn(hi, lo) < A.pad) {
          lo = __dsub_rn(lo, A.half_pad);
          hi = __dadd_rn(hi, A.half_pad);
        }
        plo[a] = lo; phi[a] = hi;
        scale = fmax(scale, __dsub_rn(hi, lo));
      }
      int bad = 0;
      for (int a = 0; a < D; ++a)
        if (!(__dsub_rn(phi[a], plo[a]) > __dmul_rn(1e-14, scale))) bad = 1;
      if (bad) atomicOr(A.err, DEV_DEGENERATE_BOX);
      for (int a = 0; a < D; ++a) { S.misc[2 + a] = plo[a]; S.misc[5 + a] = phi[a]; }
    }
    __syncthreads();
    {
      const int mt = A.tab.m;
      for (int e = tid; e < D * mt; e += NT) {
        int a = e / mt, k = e % mt;
        double lo = S.misc[2 + a], hi = S.misc[5 + a];
        double t1 = __dmul_rn(0.5, __dadd_rn(lo, hi));
        double t2 = __dmul_rn(0.5, __dsub_rn(hi, lo));
        S.nodes[a * rc_nodes_stride(D) + k] = __dadd_rn(t1, __dmul_rn(t2, A.tab.cosv[k]));
      }
    }
    __syncthreads();
    rc_node<D, NT, RR, R11G, CS>(A, S, P, v, n, m, src, vhn, kld);
    v = next_node();
  }
  P.sync();  // (clusters: no CTA leaves while a peer may still write into its shared memory)
}

}  // namespace

// ---------------------------------------------------------------------------
// launch (one translation unit per point dimension: compress_rc_d{1,2,3}.cu)
// ---------------------------------------------------------------------------
template <int D>
void launch_compress_rc_dim(const CompressArgs& a, const RcVariant& v, int grid, size_t smem, cudaStream_t s) {
  auto go = [&](auto kern) {
    SMASH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (v.cs > 1) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)grid);
      cfg.blockDim = dim3((unsigned)v.nt);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = (unsigned)v.cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      SMASH_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    } else {
      kern<<<grid, v.nt, smem, s>>>(a);
    }
  };
  if (v.cs == 4 && v.nt == 256 && v.rr == 48 && v.r11g) go(k_compress_rc<D, 256, 48, true, 4>);
  else if (v.cs != 1) SMASH_CHECK(false, SMASH_ERR_INVALID, "no register-column cluster kernel for this launch shape");
  else if (v.nt == 32 && v.rr == 32 && v.r11g) go(k_compress_rc<D, 32, 32, true, 1>);
  else if (v.nt == 32 && v.rr == 48 && v.r11g) go(k_compress_rc<D, 32, 48, true, 1>);
  else if (v.nt == 64 && v.rr == 32 && v.r11g) go(k_compress_rc<D, 64, 32, true, 1>);
  else if (v.nt == 64 && v.rr == 48 && v.r11g) go(k_compress_rc<D, 64, 48, true, 1>);
  else if (v.nt == 128 && v.rr == 32 && !v.r11g) go(k_compress_rc<D, 128, 32, false, 1>);
  else if (v.nt == 128 && v.rr == 32 && v.r11g) go(k_compress_rc<D, 128, 32, true, 1>);
  else if (v.nt == 256 && v.rr == 32 && !v.r11g) go(k_compress_rc<D, 256, 32, false, 1>);
  else if (v.nt == 256 && v.rr == 48 && v.r11g) go(k_compress_rc<D, 256, 48, true, 1>);
  else if (v.nt == 320 && v.rr == 44 && v.r11g) go(k_compress_rc<D, 320, 44, true, 1>);
  else SMASH_CHECK(false, SMASH_ERR_INVALID, "no register-column kernel for this launch shape");
  SMASH_CUDA(cudaGetLastError());
}

}  // namespace smash
