// K5 device code (included by svd.cu and the per-kernel svd_<kernel>.cu units).
// K5: HSS nearfield block-row assembly + batched truncated SVD -- replaces the
// per-node `block(ibar, near columns)` + `truncated_svd` of build_hss
// (smash/hss.py:279-299, smash/lowrank.py:265-276).
//
// One CTA per node.  The left singular subspace of A (|ibar| x n_near, generated from the
// kernel on the fly) is computed as
//   A P = Q1 R      column-pivoted Householder QR, stopped once |R_ii| falls a few bits
//                   below the fp64 noise floor (2^-57 |R_00| internal nodes, 2^-56 leaves;
//                   SMASH_SVD_FLOOR / _LEAF): the discarded block perturbs the singular
//                   values by about sqrt(n) 2^-56 sigma_1, the order of LAPACK's own
//                   rounding.  Stopping AT the noise floor (2^-53) made the kept vectors
//                   near the eps_svd cut ~10x less accurate (cfg 4 full size: 21 rank
//                   flips vs 1 for a LAPACK restatement; 2^-57 .. 2^-63 all give the LAPACK
//                   restatement's counts on every fixture, profiles/hss_skeleton_census_r02.txt).
//                   Panels up to 128 x 256 are factored on chip by the group-column QR
//                   (group_qr below); larger ones by the swap-based QR on a shared or
//                   L2-resident panel;
//   R_k^T = Q2 R2   unpivoted QR of the k' leading rows (transposed), one barrier per step;
//   L V = W         one-sided (Hestenes) Jacobi on the columns of L = R2^T (k' x k'),
//                   round-robin pair order, one 8-lane group per pair;
// so sigma_j = ||W_j|| and U(A) = Q1[:, :k'] W diag(1/sigma).  keep = #{sigma >= eps
// sigma_1} (lowrank.py:275) and S = U[:, kept] (descending sigma) is handed to the
// compression kernel as extra panel rows.  Column order and signs of S do not
// change the pivoted QR of [U_basis, S]^T in exact arithmetic.
// Wide levels of large panels (config 4's leaves) run as two launches per chunk of nodes:
// the QR at one CTA per SM (255 registers, the whole SM's shared memory), the later phases
// at two CTAs per SM; panel, k' and taus pass through a per-node workspace.
#pragma once

#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"
#include "qr_device.cuh"
#include "svd.cuh"

namespace smash {
namespace svdk {

using namespace qr;

constexpr int SVD_THREADS = 256;
constexpr int MAX_NEAR = 64;
// The shared-memory work area (SvdArgs::big doubles) holds the panel A while it is
// factored, then B = R_k^T, then J, then the back-transform Y: about 96 KB where two CTAs
// share an SM, up to the whole SM on levels of few nodes and in the HYB kernel.
constexpr size_t SVD_SMEM_MAX = 227 * 1024;
// doubles the unconditional register-row loads may run past the end of a matrix in the work
// area (32 rows x 8 lanes + a pivot offset)
constexpr int SVD_SLACK = 272;

struct IbarSide {
  const int* nib;       // |ibar| per BFS node (valid for the current + deeper levels)
  const int* rank;
  const int* pt_a;      // leaf point range start
  const int* pt_b;
  const double* P;      // tree-ordered points SoA
  int64_t P_stride;
  const double* Sk;     // compact skeleton points SoA
  int64_t S_stride;
  const int* skel_off;
};

struct SvdArgs {
  int lb, le, dim, kernel;
  double dx, eps_svd;
  double floor_rel, floor_leaf;  // QR truncation |R_ii| <= floor |R_00| (internal / leaf nodes)
  int transpose;  // 0: K(target, source) (row pass); 1: K(source, target) (column pass)
  const int* nchild;
  const int* child_first;
  const int* near_ptr;
  const int* near_idx;
  IbarSide self, other;
  // outputs
  int* keep;
  const int64_t* sv_off;
  double* sv;
  int* nn_out;
  // workspace
  double* gws;
  int64_t gws_stride;  // doubles per CTA
  int nmax, nnmax;
  int big;  // doubles in the shared-memory work area
  int gq0;  // all-shared group-column QR allowed (SMASH_SVD_GQ0)
  // split launch (wide HYB levels): mode 1 = assembly + pivoted QR only (HYB kernel, one CTA
  // per SM), mode 2 = the later phases only (two CTAs per SM); the panel, kp and the taus of
  // each node pass through a per-node workspace.  mode 0 = everything in one launch.
  // Jacobi split (wide levels): mode 3 = everything up to L = R2^T in the per-node workspace
  // (the QR too unless prefac: done by a mode-1 launch), then k_jacobi rotates L in place at
  // four CTAs per SM (it needs 36 KB of shared memory, not the 96 KB work area), then
  // mode 4 = singular values, selection and back-transform.
  int mode, ws_lb, prefac;
  int* kp_g;
  double* taus_g;
  int64_t* joff_g;  // mode 3: offset of L in the node's workspace
  int* err;
  long long* dbg;  // SMASH_SVD_DBG: phase cycle counts of block 0's first nodes
};

__device__ __forceinline__ int ibar_size(const IbarSide& s, const int* nchild, const int* child_first,
                                         int j) {
  if (nchild[j] == 0) return s.pt_b[j] - s.pt_a[j];
  int n = 0;
  for (int c = 0; c < nchild[j]; ++c) n += s.rank[child_first[j] + c];
  return n;
}

__device__ __forceinline__ const double* ibar_base(const IbarSide& s, const int* nchild,
                                                   const int* child_first, int j, int64_t* stride) {
  if (nchild[j] == 0) {
    *stride = s.P_stride;
    return s.P + s.pt_a[j];
  }
  *stride = s.S_stride;
  return s.Sk + s.skel_off[child_first[j]];
}


// Column work by 8-lane groups: a column of the panel (column-major, stride 1) is
// split over the group's lanes (rows gl, gl + 8, ...), each lane keeping up to
// GR rows in registers between the dot product and the update; sums are
// combined by a 3-level butterfly (identical in every lane of the group).
constexpr int GR = 16;  // register-cached rows per lane (covers 128 rows below the pivot)

__device__ __forceinline__ double grp_sum(double x, unsigned gm) {
  x += __shfl_xor_sync(gm, x, 4);
  x += __shfl_xor_sync(gm, x, 2);
  x += __shfl_xor_sync(gm, x, 1);
  return x;
}

// The same butterfly with the full-warp mask, for call sites every lane of the warp reaches
// together: a shuffle under a computed 8-lane mask compiles to a WARPSYNC / collective
// sequence per shuffle, under the constant full mask to a single SHFL.BFLY.
__device__ __forceinline__ double grp_sum_w(double x) {
  x += __shfl_xor_sync(0xffffffffu, x, 4);
  x += __shfl_xor_sync(0xffffffffu, x, 2);
  x += __shfl_xor_sync(0xffffffffu, x, 1);
  return x;
}

__device__ __forceinline__ double grp_sumsq(const double* c, int r0, int r1, int gl, unsigned gm) {
  double s0 = 0.0, s1 = 0.0;
  int r = r0 + gl;
  for (; r + 8 < r1; r += 16) {
    const double a = c[r], b = c[r + 8];
    s0 = fma(a, a, s0);
    s1 = fma(b, b, s1);
  }
  if (r < r1) s0 = fma(c[r], c[r], s0);
  return grp_sum(s0 + s1, gm);
}

// H_i^T applied to column c (rows i..m-1; v_i = 1, v_r = vh[r] below): the
// group's rows i+1.. are loaded once (registers), w = c_i + v^T c, c -= tau w v.
// Returns the updated c_i in every lane; x[] keeps the updated rows (row
// i + 1 + gl + 8q) for a following norm recomputation.
__device__ __forceinline__ double grp_reflect(double* c, int m, int i, double tau, const double* vh,
                                              int gl, unsigned gm, double (&x)[GR], bool store) {
  const int rb = i + 1 + gl;
#pragma unroll
  for (int q = 0; q < GR; ++q) x[q] = rb + 8 * q < m ? c[rb + 8 * q] : 0.0;
  const double ci = c[i];
  if (tau == 0.0) return ci;
  double w0 = 0.0, w1 = 0.0;
#pragma unroll
  for (int q = 0; q < GR; q += 2) {
    if (rb + 8 * q < m) w0 = fma(vh[rb + 8 * q], x[q], w0);
    if (rb + 8 * q + 8 < m) w1 = fma(vh[rb + 8 * q + 8], x[q + 1], w1);
  }
  for (int r = rb + 8 * GR; r < m; r += 8) w0 = fma(vh[r], c[r], w0);
  const double w = ci + grp_sum(w0 + w1, gm);
  const double t = -tau * w;
#pragma unroll
  for (int q = 0; q < GR; ++q) {
    const int r = rb + 8 * q;
    if (r < m) {
      x[q] = fma(t, vh[r], x[q]);
      if (store) c[r] = x[q];
    }
  }
  for (int r = rb + 8 * GR; r < m; r += 8)
    if (store) c[r] = fma(t, vh[r], c[r]);
  return ci + t;
}

// ---- Group-column pivoted QR (panels of at most 128 x 256).  The 8-lane group g owns the
// physical columns g + 32 k (k < 8) for the whole factorisation, lane gl rows gl + 8 q
// (q < NQ): columns k < KR live in registers, the others in shared memory (column stride
// = 8 mod 16 doubles: the four groups of a warp fall on the two halves of the banks).
// KR = 2 holds config 4's 128 x 256 leaf blocks (256 KB) on chip with one CTA per SM;
// KR = 0 is the all-shared layout of the smaller panels (two CTAs per SM).
// No column ever moves: the pivot order is a position per column (posof).  Every update
// also leaves the EXACT squared norm of each column's remaining rows in vn1 and its next
// row entry in arow, so a pivot step needs no reduction for the reflector: with the pivot
// known, every thread forms beta = -sign(alpha) sqrt(norm^2), tau and the scaling itself,
// reads the raw pivot column straight from its shared-memory home (a register column is
// staged by its owner first) and updates its group's columns two at a time (independent
// dot products and reductions interleaved).  Two barriers per step: after the update and
// inside the argmax; dlaqp2's norm downdating (divisions, square roots, re-summing under
// cancellation) is not needed.  The owner writes the scaled reflector and beta into the
// pivot column after the update barrier, when nobody reads the raw column any more.  At the
// end the columns are written to W in position order, the layout the later phases expect.
constexpr int HQ_KC = 8;
constexpr int HQ_ROWS = 128;
constexpr int HQ_LDC = 136;
constexpr int HQ_BIG = (HQ_KC - 2) * 32 * HQ_LDC;  // doubles of shared column storage, KR = 2

template <int NQ>
__device__ __forceinline__ double grp_sel(const double (&x)[NQ], int sq) {
  // x[sq] for a CTA-uniform sq: a tree of selects on the bits of sq (a chain of compares
  // is turned into a dynamically indexed local array by the compiler)
  static_assert(NQ <= 16, "select tree over 16 register rows");
  double a[8], b[4], c[2];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const double lo = 2 * t < NQ ? x[2 * t < NQ ? 2 * t : 0] : 0.0;
    const double hi = 2 * t + 1 < NQ ? x[2 * t + 1 < NQ ? 2 * t + 1 : 0] : 0.0;
    a[t] = (sq & 1) ? hi : lo;
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) b[t] = (sq & 2) ? a[2 * t + 1] : a[2 * t];
#pragma unroll
  for (int t = 0; t < 2; ++t) c[t] = (sq & 4) ? b[2 * t + 1] : b[2 * t];
  return (sq & 8) ? c[1] : c[0];
}

template <int K, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (K > 0) {
    static_for<K - 1>(f);
    f(std::integral_constant<int, K - 1>{});
  }
}

template <int KER, int D, int KR, int NQ>
__device__ __forceinline__ int group_qr(const SvdArgs& A, Shared& S, double* sh, int ldc, double* arow,
                                        double* W, double* taus, int n, int nn, int nnear,
                                        const int* near_start, const double* const* near_base,
                                        const int64_t* near_stride, const double* tb, int64_t ts,
                                        double floor_v) {
  static_assert(KR == 0 || KR == 2, "register columns are the two named arrays below");
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int g8 = tid >> 3, gl = tid & 7;
  const unsigned gm = 0xffu << (lane & ~7);
  int* posof = S.jpvt;
  double cr0[NQ], cr1[NQ];
  // column k of the group: registers (k < KR) or shared memory
  auto col_load = [&](auto kc, double (&x)[NQ]) __attribute__((always_inline)) {
    constexpr int k = decltype(kc)::value;
    if constexpr (k < KR && k == 0) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) x[q] = cr0[q];
    } else if constexpr (k < KR && k == 1) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) x[q] = cr1[q];
    } else {
      const double* c = sh + (size_t)((k - KR) * 32 + g8) * ldc;
#pragma unroll
      for (int q = 0; q < NQ; ++q) x[q] = c[gl + 8 * q];
    }
  };
  auto col_store = [&](auto kc, const double (&x)[NQ]) __attribute__((always_inline)) {
    constexpr int k = decltype(kc)::value;
    if constexpr (k < KR && k == 0) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) cr0[q] = x[q];
    } else if constexpr (k < KR && k == 1) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) cr1[q] = x[q];
    } else {
      double* c = sh + (size_t)((k - KR) * 32 + g8) * ldc;
#pragma unroll
      for (int q = 0; q < NQ; ++q) c[gl + 8 * q] = x[q];
    }
  };
  // the same for a CTA-uniform runtime k (the pivot's owner): a pointer for the shared
  // columns, selects between the register columns
  auto col_load_dyn = [&](int k, double (&x)[NQ]) __attribute__((always_inline)) {
    if (k >= KR) {
      const double* c = sh + (size_t)((k - KR) * 32 + g8) * ldc;
#pragma unroll
      for (int q = 0; q < NQ; ++q) x[q] = c[gl + 8 * q];
    } else if constexpr (KR > 0) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) x[q] = k == 0 ? cr0[q] : cr1[q];
    }
  };
  auto col_store_dyn = [&](int k, const double (&x)[NQ]) __attribute__((always_inline)) {
    if (k >= KR) {
      double* c = sh + (size_t)((k - KR) * 32 + g8) * ldc;
#pragma unroll
      for (int q = 0; q < NQ; ++q) c[gl + 8 * q] = x[q];
    } else if constexpr (KR > 0) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        cr0[q] = k == 0 ? x[q] : cr0[q];
        cr1[q] = k == 0 ? cr1[q] : x[q];
      }
    }
  };
  // (max norm, smallest column) over the CTA: warp shuffles, one partial per warp, the
  // caller's barrier, then every thread folds the partials
  auto argmax_put = [&](double bv, int bi) __attribute__((always_inline)) {
    for (int off = 16; off; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      argmax_combine(bv, bi, ov, oi);
    }
    if (lane == 0) { S.redv[wid] = bv; S.redi[wid] = bi; }
  };
  auto argmax_get = [&]() __attribute__((always_inline)) {
    double bv = S.redv[0];
    int bi = S.redi[0];
    for (int w = 1; w < nw; ++w) argmax_combine(bv, bi, S.redv[w], S.redi[w]);
    return bi;
  };
  // ---- assemble the group's columns, initial norms
  static_for<HQ_KC>([&](auto kc) __attribute__((always_inline)) {
    constexpr int k = decltype(kc)::value;
    const int j = g8 + 32 * k;
    if (32 * k >= nn && k >= KR) return;
    double x[NQ];
    double s0 = 0.0;
    if (j < nn) {
      int g = 0;
      while (g + 1 < nnear && near_start[g + 1] <= j) ++g;
      const int bl = j - near_start[g];
      double y[D];
#pragma unroll
      for (int d = 0; d < D; ++d) y[d] = near_base[g][(int64_t)d * near_stride[g] + bl];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int r = gl + 8 * q;
        double xr[D];
#pragma unroll
        for (int d = 0; d < D; ++d) xr[d] = tb[(int64_t)d * ts + min(r, n - 1)];
        const double val = A.transpose ? kval<KER, D>(y, xr, A.dx) : kval<KER, D>(xr, y, A.dx);
        x[q] = r < n ? val : 0.0;
        s0 = fma(x[q], x[q], s0);
      }
    } else {
#pragma unroll
      for (int q = 0; q < NQ; ++q) x[q] = 0.0;
    }
    col_store(kc, x);
    const double nr2 = grp_sum(s0, gm);
    if (gl == 0 && j < nn) {
      S.vn1[j] = nr2;  // squared norm of the remaining rows
      arow[j] = x[0];
    }
  });
  if (tid < nn) posof[tid] = -1;
  __syncthreads();
  argmax_put(tid < nn ? S.vn1[tid] : -1.0, tid < nn ? tid : 0x7fffffff);
  __syncthreads();
  int pvt = argmax_get();
  // a register pivot column is staged raw in S.vh by its owner
  auto stage_pivot = [&]() __attribute__((always_inline)) {
    if constexpr (KR > 0) {
      if (pvt < 32 * KR) {  // CTA-uniform
        if (g8 == (pvt & 31)) {
          double x[NQ];
          col_load_dyn(pvt >> 5, x);
#pragma unroll
          for (int q = 0; q < NQ; ++q)
            if (gl + 8 * q < n) S.vh[gl + 8 * q] = x[q];
        }
        __syncthreads();
      }
    }
  };
  stage_pivot();
  const int kmax = min(n, nn);
  int kp = 0, nsteps = 0;
  double r0 = 0.0;
  const bool gdbg = A.dbg && blockIdx.x == 0 && tid == 0;
  long long gt0 = 0, gt1 = 0, gt2 = 0;
  for (int i = 0; i < kmax; ++i) {
    if (gdbg) gt0 = clock64();
    // ---- dlarfg scalars of the pivot column, by every thread
    const int og = pvt & 31, ok = pvt >> 5;
    const double alpha = arow[pvt], n2 = S.vn1[pvt];
    double tau = 0.0, beta = alpha, scal = 0.0;
    if (n - i > 1 && n2 > alpha * alpha) {
      beta = -copysign(__dsqrt_rn(n2), alpha);
      tau = __ddiv_rn(__dsub_rn(beta, alpha), beta);
      scal = __ddiv_rn(1.0, __dsub_rn(alpha, beta));
    }
    asm volatile("" : "+d"(tau), "+d"(beta), "+d"(scal));  // (no rematerialisation in the loops below)
    if (i == 0) r0 = fabs(beta);
    if (g8 == og && gl == 0) {
      posof[pvt] = i;
      taus[i] = tau;
    }
    __syncwarp(gm);
    nsteps = i + 1;
    if (r0 == 0.0 || !(fabs(beta) > floor_v * r0)) {
      // the column stays unscaled: the later phases read the first kp = i rows only
      break;
    }
    kp = i + 1;
    double vv[NQ];
    {
      const double* pc = (KR > 0 && pvt < 32 * KR) ? S.vh : sh + (size_t)(pvt - 32 * KR) * ldc;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int r = gl + 8 * q;
        const double pq = pc[r];  // (unconditional load: a column slot holds all 8 NQ rows)
        vv[q] = (tau != 0.0 && r > i && r < n) ? pq * scal : (r == i ? 1.0 : 0.0);
      }
    }
    // ---- H_i applied to the group's columns, two at a time; exact remaining norms
    static_for<HQ_KC / 2>([&](auto bc) __attribute__((always_inline)) {
      constexpr int k0 = 2 * decltype(bc)::value;
      if (32 * k0 >= nn) return;  // CTA-uniform: no column of this pair exists
      const std::integral_constant<int, k0> ka;
      const std::integral_constant<int, k0 + 1> kb;
      const int ja = g8 + 32 * k0, jb = ja + 32;
      const bool acta = ja < nn && posof[ja] < 0, actb = jb < nn && posof[jb] < 0;
      // (no group-level exit: the warp stays converged, the shuffles take the full mask)
      double xa[NQ], xb[NQ];
      col_load(ka, xa);
      if (32 * (k0 + 1) < nn) {  // CTA-uniform: the pair's second column slot exists
        col_load(kb, xb);
      } else {
#pragma unroll
        for (int q = 0; q < NQ; ++q) xb[q] = 0.0;
      }
      double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
      for (int q = 0; q + 1 < NQ; q += 2) {
        a0 = fma(vv[q], xa[q], a0);
        b0 = fma(vv[q], xb[q], b0);
        a1 = fma(vv[q + 1], xa[q + 1], a1);
        b1 = fma(vv[q + 1], xb[q + 1], b1);
      }
      if constexpr (NQ & 1) {
        a0 = fma(vv[NQ - 1], xa[NQ - 1], a0);
        b0 = fma(vv[NQ - 1], xb[NQ - 1], b0);
      }
      double wa = a0 + a1, wb = b0 + b1;
      wa += __shfl_xor_sync(0xffffffffu, wa, 4);
      wb += __shfl_xor_sync(0xffffffffu, wb, 4);
      wa += __shfl_xor_sync(0xffffffffu, wa, 2);
      wb += __shfl_xor_sync(0xffffffffu, wb, 2);
      wa += __shfl_xor_sync(0xffffffffu, wa, 1);
      wb += __shfl_xor_sync(0xffffffffu, wb, 1);
      const double ta = acta ? -tau * wa : 0.0, tb2 = actb ? -tau * wb : 0.0;
      a0 = a1 = b0 = b1 = 0.0;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        xa[q] = fma(ta, vv[q], xa[q]);
        xb[q] = fma(tb2, vv[q], xb[q]);
        const bool below = gl + 8 * q > i;
        const double ya = below ? xa[q] : 0.0, yb = below ? xb[q] : 0.0;
        if (q & 1) {
          a1 = fma(ya, ya, a1);
          b1 = fma(yb, yb, b1);
        } else {
          a0 = fma(ya, ya, a0);
          b0 = fma(yb, yb, b0);
        }
      }
      if (acta) col_store(ka, xa);
      if (actb) col_store(kb, xb);
      double na = a0 + a1, nb = b0 + b1;
      na += __shfl_xor_sync(0xffffffffu, na, 4);
      nb += __shfl_xor_sync(0xffffffffu, nb, 4);
      na += __shfl_xor_sync(0xffffffffu, na, 2);
      nb += __shfl_xor_sync(0xffffffffu, nb, 2);
      na += __shfl_xor_sync(0xffffffffu, na, 1);
      nb += __shfl_xor_sync(0xffffffffu, nb, 1);
      if (gl == ((i + 1) & 7)) {
        if (acta) {
          arow[ja] = grp_sel<NQ>(xa, (i + 1) >> 3);
          S.vn1[ja] = na;
        }
        if (actb) {
          arow[jb] = grp_sel<NQ>(xb, (i + 1) >> 3);
          S.vn1[jb] = nb;
        }
      }
    });
    __syncthreads();
    if (gdbg) gt1 = clock64();
    // ---- the owner stores the scaled reflector and beta in the pivot column
    if (g8 == og && tau != 0.0) {
      double x[NQ];
      col_load_dyn(ok, x);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int r = gl + 8 * q;
        x[q] = r > i ? vv[q] : (r == i ? beta : x[q]);
      }
      col_store_dyn(ok, x);
    }
    if (i + 1 == kmax) break;
    // ---- next pivot: largest remaining norm
    const bool live = tid < nn && posof[tid] < 0;
    argmax_put(live ? S.vn1[tid] : -1.0, live ? tid : 0x7fffffff);
    __syncthreads();
    pvt = argmax_get();
    stage_pivot();
    if (gdbg) {
      gt2 = clock64();
      A.dbg[40] += gt1 - gt0; A.dbg[42] += gt2 - gt1; A.dbg[43] += 1;
    }
  }
  __syncthreads();
  // ---- positions of the columns never chosen (after the pivoted ones, in column order)
  {
    const bool rest = tid < nn && posof[tid] < 0;
    const unsigned bal = __ballot_sync(0xffffffffu, rest);
    if (lane == 0) S.redi[wid] = __popc(bal);
    __syncthreads();
    int base = nsteps;
    for (int w = 0; w < wid; ++w) base += S.redi[w];
    if (rest) posof[tid] = base + __popc(bal & ((1u << lane) - 1u));
    __syncthreads();
  }
  static_for<HQ_KC>([&](auto kc) __attribute__((always_inline)) {
    constexpr int k = decltype(kc)::value;
    const int j = g8 + 32 * k;
    if (j >= nn) return;
    double x[NQ];
    col_load(kc, x);
    double* dst = W + (size_t)posof[j] * n;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int r = gl + 8 * q;
      if (r < n) dst[r] = x[q];
    }
  });
  __syncthreads();
  return kp;
}

// One-sided Jacobi sweeps on the kp x kp column-major J (see k_svd); NJ register rows per
// lane (8 covers kp <= 64).  Returns the number of sweeps.
template <int NJ>
__device__ __forceinline__ int jacobi_sweeps(double* J, int kp, double* nrm, Shared& S, long long* gdbg,
                                             bool dbg) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int g8 = tid >> 3, gl = tid & 7, ngr = blockDim.x >> 3;
  const unsigned gm = 0xffu << (lane & ~7);
    const int np = kp + (kp & 1);  // round-robin over an even count (dummy = kp)
  int sweeps_done = 0;
    for (int sweep = 0; sweep < 40; ++sweep) {
      sweeps_done = sweep + 1;
      for (int c = g8; c < kp; c += ngr) {  // exact squared norms
        double s2 = 0.0;
        for (int r = gl; r < kp; r += 8) s2 = fma(J[(size_t)c * kp + r], J[(size_t)c * kp + r], s2);
        s2 = grp_sum(s2, gm);
        if (gl == 0) nrm[c] = s2;
      }
      if (tid == 0) S.imisc[2] = 0;
      __syncthreads();
      for (int rnd = 0; rnd < np - 1; ++rnd) {
        for (int pr0 = 0; pr0 < np / 2; pr0 += ngr) {
          // circle method: position 0 fixed, others rotate.  The loop is warp-uniform (a
          // group without a pair works on a clamped one and stores nothing), so the
          // reductions shuffle under the full mask.
          const int pr = min(pr0 + g8, np / 2 - 1);
          int a = pr == 0 ? 0 : 1 + (pr - 1 + rnd) % (np - 1);
          int b = 1 + (np - 2 - pr + rnd) % (np - 1);
          const bool pair_ok = pr0 + g8 < np / 2 && a < kp && b < kp;
          a = min(a, kp - 1);
          b = min(b, kp - 1);
          double* ja = J + (size_t)a * kp;
          double* jb = J + (size_t)b * kp;
          long long jt0 = 0, jt1 = 0, jt2 = 0;
          if (dbg) jt0 = clock64();
          double xa[NJ], xb[NJ];
#pragma unroll
          for (int q = 0; q < NJ; ++q) {
            const int r = gl + 8 * q;
            const double va = ja[r], vb = jb[r];  // (unconditional: the work area has slack past J)
            xa[q] = r < kp ? va : 0.0;
            xb[q] = r < kp ? vb : 0.0;
          }
          double g0 = 0.0, g1 = 0.0;
#pragma unroll
          for (int q = 0; q < NJ; q += 2) {
            g0 = fma(xa[q], xb[q], g0);
            g1 = fma(xa[q + 1], xb[q + 1], g1);
          }
          for (int r = gl + 8 * NJ; r < kp; r += 8) g0 = fma(ja[r], jb[r], g0);
          const double ga = grp_sum_w(g0 + g1);
          if (dbg) jt1 = clock64();
          const double al = nrm[a], be = nrm[b];
          if (pair_ok && ga * ga > 1e-30 * (al * be) && ga != 0.0) {
            // t = tan of the rotation angle, the smaller root: sign(d) 2g / (|d| + sqrt(d^2 + 4 g^2))
            const double d = be - al, g2 = ga + ga;
            const double t = copysign(g2, d * ga) / (fabs(d) + sqrt(fma(d, d, g2 * g2)));
            double c = rsqrt_nr(fma(t, t, 1.0)), s = c * t;
            // (pin c and s: under the 128-register cap ptxas rematerialised the whole
            // reciprocal square root at every one of the 2 NJ stores of the rotation)
            asm volatile("" : "+d"(c), "+d"(s));
            if (dbg) jt2 = clock64();
#pragma unroll
            for (int q = 0; q < NJ; ++q) {
              const int r = gl + 8 * q;
              if (r < kp) {
                ja[r] = c * xa[q] - s * xb[q];
                jb[r] = s * xa[q] + c * xb[q];
              }
            }
            for (int r = gl + 8 * NJ; r < kp; r += 8) {
              const double x = ja[r], y = jb[r];
              ja[r] = c * x - s * y;
              jb[r] = s * x + c * y;
            }
            if (gl == 0) {
              nrm[a] = fmax(al - t * ga, 0.0);
              nrm[b] = be + t * ga;
              S.imisc[2] = 1;
            }
            if (dbg && tid == 0) {
              const long long jt3 = clock64();
              gdbg[34] += jt1 - jt0; gdbg[35] += jt2 - jt1; gdbg[36] += jt3 - jt2; gdbg[38] += 1;
            }
          }
        }
        long long jb0 = 0;
        if (dbg && tid == 0) jb0 = clock64();
        __syncthreads();
        if (dbg && tid == 0) { gdbg[37] += clock64() - jb0; gdbg[39] += 1; }
      }
      if (S.imisc[2] == 0) break;
      __syncthreads();
    }
  return sweeps_done;
}

template <int KER, int D, bool HYB>
__global__ void __launch_bounds__(SVD_THREADS, HYB ? 1 : 2) k_svd(SvdArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Shared S;
  double* taus;
  double* sig;
  double* rrow;
  int* near_start;
  const double** near_base;
  int64_t* near_stride;
  int* order;
  double* big;
  {
    double* d = reinterpret_cast<double*>(smem_raw);
    S.vn1 = d; d += A.nnmax;
    S.vn2 = d; d += A.nnmax;
    S.vh = d; d += max(A.nmax, A.nnmax);
    S.rdiag = d; d += max(A.nmax, A.nnmax);
    taus = d; d += A.nmax;
    sig = d; d += A.nmax;
    rrow = d; d += A.nnmax;
    S.nodes = nullptr;
    S.redv = d; d += 32;
    S.misc = d; d += 8;
    near_base = reinterpret_cast<const double**>(d); d += MAX_NEAR;
    near_stride = reinterpret_cast<int64_t*>(d); d += MAX_NEAR;
    int* ip = reinterpret_cast<int*>(d);
    S.redi = ip; ip += 32;
    S.imisc = ip; ip += 8;
    near_start = ip; ip += MAX_NEAR + 1;
    order = ip; ip += A.nmax;
    S.jpvt = ip; ip += A.nnmax;
    // (offset arithmetic on smem_raw itself: a uintptr_t round trip makes the pointer generic,
    // and every access of the work area a branch-guarded LD instead of a predicated LDS)
    const unsigned off = ((unsigned)(reinterpret_cast<unsigned char*>(ip) - smem_raw) + 15u) & ~15u;
    big = reinterpret_cast<double*>(smem_raw + off);
  }
  const int tid = threadIdx.x, NT = blockDim.x;
  const int lane = tid & 31;
  // 8-lane groups: one column (or Jacobi pair) per group
  const int g8 = tid >> 3, gl = tid & 7, ngr = NT >> 3;
  const unsigned gm = 0xffu << (lane & ~7);
  int dbg_n = 0;
  for (int v = A.lb + blockIdx.x; v < A.le; v += gridDim.x) {
    double* W = A.gws + (size_t)(A.mode ? v - A.ws_lb : blockIdx.x) * A.gws_stride;
    const int n = A.self.nib[v];
    const int e0 = A.near_ptr[v], e1 = A.near_ptr[v + 1];
    if (tid == 0) {
      int acc = 0, cnt = 0;
      for (int e = e0; e < e1 && cnt < MAX_NEAR; ++e) {
        const int j = A.near_idx[e];
        const int sz = ibar_size(A.other, A.nchild, A.child_first, j);
        if (sz == 0) continue;  // hss.py:283 drops empty neighbour sets
        near_start[cnt] = acc;
        near_base[cnt] = ibar_base(A.other, A.nchild, A.child_first, j, &near_stride[cnt]);
        acc += sz;
        ++cnt;
      }
      near_start[cnt] = acc;
      S.imisc[0] = cnt;
      S.imisc[1] = acc;
      if (e1 - e0 > MAX_NEAR) atomicOr(A.err, DEV_CAPACITY);
    }
    __syncthreads();
    const int nnear = S.imisc[0], nn = S.imisc[1];
    if (n == 0 || nn == 0) {
      if (tid == 0) A.keep[v] = 0;
      __syncthreads();
      continue;
    }
    const bool dbg = A.dbg && blockIdx.x < 4 && tid == 0 && dbg_n == 0;  // first node of blocks 0-3
    long long tsv[6];
    if (dbg) tsv[0] = clock64();
    // ---- assemble A (n x nn), column-major in W (one column per nearfield point)
    int64_t ts;
    const double* tb = ibar_base(A.self, A.nchild, A.child_first, v, &ts);
    const int ldp = n;
    // the panel is factored in shared memory when it fits (copied out to W afterwards:
    // the reflectors and R_k are read again by the later phases)
    // group-column QR (on-chip columns, no swaps) when the node fits one of its shapes:
    // HYB kernel: up to 128 x 256 with two register columns per group; otherwise up to
    // 80 rows with every column in the shared work area
    const int slots = (nn + 31) & ~31;
    // all-shared layout: NQ = 9 (n <= 72) or 10 register rows per lane; the column stride
    // covers all 8 NQ rows a group touches (72; 88, or 80 where 88 does not fit)
    const int ldc0 = n <= 72 ? 72 : (slots * 88 <= A.big ? 88 : 80);
    const bool gq2 = HYB && n <= HQ_ROWS && nn <= 32 * HQ_KC;
    const bool gq0 = !HYB && A.gq0 && n <= 80 && nn <= 32 * HQ_KC && slots * ldc0 <= A.big;
    const bool psm = !gq2 && !gq0 && n * nn <= A.big;
    double* P = psm ? big : W;
    const double floor_v = A.nchild[v] ? A.floor_rel : A.floor_leaf;
    const int kmax = min(n, nn);
    int kp = 0;
    const bool loaded = A.mode == 2 || A.mode == 4 || (A.mode == 3 && A.prefac);
    if (loaded) {  // factored by an earlier launch
      kp = A.kp_g[v - A.ws_lb];
      for (int i = tid; i < kp; i += NT) taus[i] = A.taus_g[(size_t)(v - A.ws_lb) * A.nmax + i];
      P = W;
      __syncthreads();
      if (dbg) tsv[1] = tsv[0];
    } else if (gq2 || gq0) {
      if constexpr (HYB)
        kp = group_qr<KER, D, 2, 16>(A, S, big, HQ_LDC, rrow, W, taus, n, nn, nnear, near_start, near_base,
                                     near_stride, tb, ts, floor_v);
      else if (n <= 72)
        kp = group_qr<KER, D, 0, 9>(A, S, big, ldc0, rrow, W, taus, n, nn, nnear, near_start, near_base,
                                    near_stride, tb, ts, floor_v);
      else
        kp = group_qr<KER, D, 0, 10>(A, S, big, ldc0, rrow, W, taus, n, nn, nnear, near_start, near_base,
                                     near_stride, tb, ts, floor_v);
      P = W;
      if (dbg) tsv[1] = tsv[0];
    } else {
      {
        int g = 0;
        for (int b = tid / n, a = tid % n; b < nn;) {
          while (g + 1 < nnear && near_start[g + 1] <= b) ++g;
          const int bl = b - near_start[g];
          double x[D], y[D];
  #pragma unroll
          for (int d = 0; d < D; ++d) {
            x[d] = tb[(int64_t)d * ts + a];
            y[d] = near_base[g][(int64_t)d * near_stride[g] + bl];
          }
          P[(size_t)b * ldp + a] = A.transpose ? kval<KER, D>(y, x, A.dx) : kval<KER, D>(x, y, A.dx);
          a += NT;
          while (a >= n) { a -= n; ++b; }
        }
      }
      __syncthreads();
      if (dbg) tsv[1] = clock64();
      // ---- column-pivoted QR of A, truncated at the noise floor
      for (int j = g8; j < nn; j += ngr) {
        const double nr = __dsqrt_rn(grp_sumsq(P + (size_t)j * ldp, 0, n, gl, gm));
        if (gl == 0) {
          S.vn1[j] = nr;
          S.vn2[j] = nr;
        }
      }
      __syncthreads();
      kp = 0;
      for (int i = 0; i < kmax; ++i) {
        double bv = -1.0;
        int bi = 0x7fffffff;
        for (int j = i + tid; j < nn; j += NT)
          if (S.vn1[j] > bv) { bv = S.vn1[j]; bi = j; }
        const int pvt = block_argmax_1bar(bv, bi, S);
        if (pvt != i) {
          double* ci = P + (size_t)i * ldp;
          double* cp = P + (size_t)pvt * ldp;
          for (int row = tid; row < n; row += NT) {
            const double t = cp[row];
            cp[row] = ci[row];
            ci[row] = t;
          }
          if (tid == 0) {
            S.vn1[pvt] = S.vn1[i];
            S.vn2[pvt] = S.vn2[i];
          }
        }
        __syncthreads();
        householder(P + (size_t)i * ldp - i, 1, n, i, S);  // column i (stride 1)
        __syncthreads();
        const double tau = S.misc[0];
        if (tid == 0) taus[i] = tau;
        const double r0 = fabs(S.rdiag[0]);
        if (r0 == 0.0 || !(fabs(S.rdiag[i]) > floor_v * r0)) break;
        kp = i + 1;
        for (int j = i + 1 + g8; j < nn; j += ngr) {
          double* c = P + (size_t)j * ldp;
          double x[GR];
          const double rij = grp_reflect(c, n, i, tau, S.vh, gl, gm, x, true);
          if (gl == 0 && tau != 0.0) c[i] = rij;
          // norm downdate (dlaqp2), exact recomputation when cancellation is severe
          const double v1 = S.vn1[j];
          if (v1 != 0.0) {
            const double q = fabs(rij) / v1;
            const double temp = fmax(1.0 - q * q, 0.0);
            const double q2 = v1 / S.vn2[j];
            if (temp * (q2 * q2) <= TOL3Z) {
              double s0 = 0.0;
  #pragma unroll
              for (int qq = 0; qq < GR; ++qq) s0 = fma(x[qq], x[qq], s0);
              for (int r = i + 1 + gl + 8 * GR; r < n; r += 8) s0 = fma(c[r], c[r], s0);
              const double nv = i + 1 < n ? sqrt(grp_sum(s0, gm)) : 0.0;
              if (gl == 0) {
                S.vn1[j] = nv;
                S.vn2[j] = nv;
              }
            } else if (gl == 0) {
              S.vn1[j] = v1 * sqrt(temp);
            }
          }
        }
        __syncthreads();
      }
      __syncthreads();
    }
    if (psm && kp > 0 && !loaded) {
      for (int e = tid; e < n * nn; e += NT) W[e] = P[e];
      __syncthreads();
      P = W;
    }
    if (A.mode == 1) {
      if (tid == 0) A.kp_g[v - A.ws_lb] = kp;
      for (int i = tid; i < kp; i += NT) A.taus_g[(size_t)(v - A.ws_lb) * A.nmax + i] = taus[i];
      __syncthreads();
      continue;
    }
    if (kp == 0) {
      if (tid == 0) {
        A.keep[v] = 0;
        if (A.mode == 3) A.kp_g[v - A.ws_lb] = 0;
      }
      __syncthreads();
      continue;
    }
    if (dbg) tsv[2] = clock64();
    // ---- B = R_k^T (nn x kp, column-major), unpivoted QR -> R2 (kp x kp); B in
    // shared memory when it fits
    const bool pre = A.mode == 3, post = A.mode == 4;
    const bool bsm = nn * kp + SVD_SLACK <= A.big;  // (+ slack: unconditional row loads run past a column)
    double* B = bsm ? big : W + (size_t)n * nn;
    double* T = W + (size_t)n * nn;  // global staging (free once B is in shared memory / consumed)
    const int ldb = nn;
    // L stays in the workspace when k_jacobi rotates it (modes 3 / 4)
    const bool jsm = !pre && !post && kp * kp + SVD_SLACK <= A.big;
    double* J = jsm ? big : W + (size_t)n * nn + (size_t)nn * kp;
    double* nrm = sig;  // squared column norms (reuses the sigma scratch)
    int sweeps_done = 0;
    if (!post) {
    for (int e = tid; e < nn * kp; e += NT) {
      const int j = e / nn, b = e - j * nn;
      B[(size_t)j * ldb + b] = b >= j ? P[(size_t)b * ldp + j] : 0.0;
    }
    __syncthreads();
    // One barrier per step: the group that updates column i + 1 also leaves its next
    // diagonal entry and the exact squared norm of its remaining rows in S.misc, so every
    // thread forms dlarfg's beta / tau / scaling for step i + 1 itself and applies the
    // reflector from the RAW column (v = scal * column); only beta is stored back (Q2 and
    // the scaled reflectors are never used: R2 is the upper triangle).
    // (instantiated for the shared-memory and the global B: LDS / LDG instead of generic loads)
    auto qr2 = [&](double* Bq) __attribute__((always_inline)) {
      if (g8 == 0) {
        const double s2 = grp_sumsq(Bq, 0, nn, gl, gm);
        if (gl == 0) {
          S.misc[2] = Bq[0];
          S.misc[3] = s2;
        }
      }
      __syncthreads();
      for (int i = 0; i < kp; ++i) {
        long long q0 = 0, q1 = 0, q2 = 0;
        if (dbg) q0 = clock64();
        double* ci = Bq + (size_t)i * ldb;
        const double alpha = S.misc[2 + 2 * (i & 1)], n2 = S.misc[3 + 2 * (i & 1)];
        double tau = 0.0, beta = alpha, scal = 0.0;
        if (nn - i > 1 && n2 > alpha * alpha) {
          beta = -copysign(__dsqrt_rn(n2), alpha);
          tau = __ddiv_rn(__dsub_rn(beta, alpha), beta);
          scal = __ddiv_rn(1.0, __dsub_rn(alpha, beta));
        }
        asm volatile("" : "+d"(tau), "+d"(beta), "+d"(scal));  // (no rematerialisation in the loops below)
        if (dbg) q1 = clock64();
        const int jn = i + 1;  // the next pivot column
        for (int j = i + 1 + g8; j < kp; j += ngr) {
          double* c = Bq + (size_t)j * ldb;
          // rows i+1.. of the group: row i + 1 + gl + 8 q in x[q]
          const int rb = i + 1 + gl;
          double x[GR];
  #pragma unroll
          for (int q = 0; q < GR; ++q) {
            const double cq = c[rb + 8 * q];  // (unconditional: the work area has slack past B)
            x[q] = rb + 8 * q < nn ? cq : 0.0;
          }
          if (tau != 0.0) {
            double vq[GR];
  #pragma unroll
            for (int q = 0; q < GR; ++q) vq[q] = ci[rb + 8 * q];
            double w0 = 0.0, w1 = 0.0;
  #pragma unroll
            for (int q = 0; q < GR; q += 2) {
              w0 = fma(vq[q], x[q], w0);  // x is zero past the last row
              w1 = fma(vq[q + 1], x[q + 1], w1);
            }
            for (int r = rb + 8 * GR; r < nn; r += 8) w0 = fma(ci[r], c[r], w0);
            const double cii = c[i];
            const double w = fma(scal, grp_sum(w0 + w1, gm), cii);
            const double t = -tau * w, ts2 = t * scal;
  #pragma unroll
            for (int q = 0; q < GR; ++q) {
              const int r = rb + 8 * q;
              if (r < nn) {
                x[q] = fma(ts2, vq[q], x[q]);
                c[r] = x[q];
              }
            }
            for (int r = rb + 8 * GR; r < nn; r += 8) c[r] = fma(ts2, ci[r], c[r]);
            if (gl == 0) c[i] = cii + t;
          }
          if (j == jn) {  // next step's alpha and remaining norm
            double s0 = 0.0, s1 = 0.0;
  #pragma unroll
            for (int q = 0; q < GR; q += 2) {
              s0 = (gl == 0 && q == 0) ? s0 : fma(x[q], x[q], s0);
              s1 = fma(x[q + 1], x[q + 1], s1);
            }
            __syncwarp(gm);
            for (int r = rb + 8 * GR; r < nn; r += 8) s0 = fma(c[r], c[r], s0);
            const double a2 = __shfl_sync(gm, x[0], lane & ~7);
            const double s2 = grp_sum(s0 + s1, gm);
            if (gl == 0) {
              S.misc[2 + 2 * (jn & 1)] = a2;
              S.misc[3 + 2 * (jn & 1)] = fma(a2, a2, s2);
            }
          }
        }
        if (dbg) q2 = clock64();
        __syncthreads();
        if (dbg && blockIdx.x == 0) {
          A.dbg[44] += q1 - q0; A.dbg[45] += q2 - q1; A.dbg[46] += clock64() - q2; A.dbg[47] += 1;
        }
        if (tid == 0) ci[i] = beta;
      }
      __syncthreads();
    };
    if (bsm) qr2(big);
    else qr2(W + (size_t)n * nn);
    // ---- one-sided (Hestenes) Jacobi on the columns of L = R2^T (kp x kp lower triangle,
    // column-major J[c*kp + r]).  R_k = L Q2^T, so the left singular vectors of A are
    // Q1 times those of L: L V = W gives them as the normalised columns of W and V is
    // never formed.  L^T L = R2 R2^T is one more LR step towards diagonal than the
    // R2^T R2 of the columns of R2 (Drmac / Veselic preconditioning), so fewer sweeps.
    // A pair's two columns are loaded once into registers (rows gl + 8q of the 8-lane
    // group), the dot product, the rotation and the stores all work from them.  Column
    // norms are carried through the rotations and refreshed exactly at every sweep.
    if (bsm && jsm) {
      for (int e = tid; e < kp * kp; e += NT) {
        const int c = e / kp, r = e - c * kp;
        T[e] = c <= r ? B[(size_t)r * ldb + c] : 0.0;
      }
      __syncthreads();
      for (int e = tid; e < kp * kp; e += NT) J[e] = T[e];
    } else {
      for (int e = tid; e < kp * kp; e += NT) {
        const int c = e / kp, r = e - c * kp;
        J[e] = c <= r ? B[(size_t)r * ldb + c] : 0.0;
      }
    }
    __syncthreads();
    if (pre) {  // k_jacobi takes over
      if (tid == 0) {
        A.kp_g[v - A.ws_lb] = kp;
        A.joff_g[v - A.ws_lb] = (int64_t)n * nn + (int64_t)nn * kp;
      }
      for (int i = tid; i < kp; i += NT) A.taus_g[(size_t)(v - A.ws_lb) * A.nmax + i] = taus[i];
      __syncthreads();
      continue;
    }
    if (dbg) tsv[3] = clock64();
    // (the shared-memory case is instantiated on the work area itself: LDS, not generic loads)
    sweeps_done = jsm ? (kp <= 64   ? jacobi_sweeps<8>(big, kp, nrm, S, A.dbg, dbg)
                         : kp <= 80 ? jacobi_sweeps<10>(big, kp, nrm, S, A.dbg, dbg)
                                    : jacobi_sweeps<16>(big, kp, nrm, S, A.dbg, dbg))
                      : jacobi_sweeps<16>(J, kp, nrm, S, A.dbg, dbg);
    }  // !post
    if (dbg && post) tsv[2] = tsv[3] = clock64();
    if (dbg) tsv[4] = clock64();
    if (A.dbg && tid == 0) {  // every node: max sweeps, nodes at the sweep cap
      atomicMax(reinterpret_cast<unsigned long long*>(A.dbg + 32), (unsigned long long)sweeps_done);
      if (sweeps_done >= 40) atomicAdd(reinterpret_cast<unsigned long long*>(A.dbg + 33), 1ull);
    }
    // ---- singular values, keep count, descending order
    for (int c = g8; c < kp; c += ngr) {
      double s2 = 0.0;
      for (int r = gl; r < kp; r += 8) s2 = fma(J[(size_t)c * kp + r], J[(size_t)c * kp + r], s2);
      s2 = grp_sum(s2, gm);
      if (gl == 0) sig[c] = sqrt(s2);
    }
    __syncthreads();
    if (tid == 0) {
      double smax = 0.0;
      for (int c = 0; c < kp; ++c) smax = fmax(smax, sig[c]);
      int keep = 0;
      if (smax > 0.0) {
        // selection of sigma >= eps * sigma_1 in descending order
        for (int c = 0; c < kp; ++c) order[c] = c;
        for (int c = 1; c < kp; ++c) {  // insertion sort by sigma descending (kp small)
          int x = order[c];
          int p = c - 1;
          while (p >= 0 && sig[order[p]] < sig[x]) { order[p + 1] = order[p]; --p; }
          order[p + 1] = x;
        }
        const double thr = A.eps_svd * smax;
        for (int c = 0; c < kp; ++c) keep += sig[c] >= thr ? 1 : 0;
      }
      S.imisc[3] = keep;
      A.keep[v] = keep;
    }
    __syncthreads();
    const int keep = S.imisc[3];
    if (keep == 0) continue;
    // ---- U = Q1[:, :kp] (W[:, kept] / sigma)  (n x keep).  Up to 128 rows: the kp
    // reflectors are staged once in the shared work area and every 8-lane group carries
    // one column of U in registers through all of them (no barrier between reflectors).
    // Otherwise: U staged in shared memory when it fits, one barrier pair per reflector.
    double* Yg = A.sv + A.sv_off[v];
    // kept columns of W (descending sigma), normalised -> T (global staging: the work area is reused)
    for (int e = tid; e < kp * keep; e += NT) {
      const int a = e / keep, c = e - a * keep;
      T[e] = J[(size_t)order[c] * kp + a] / sig[order[c]];
    }
    __syncthreads();
    if (n <= 8 * GR && kp * n + SVD_SLACK <= A.big) {
      double* Vs = big;  // reflector i at Vs[i * n + row], rows > i
      for (int e = tid; e < kp * n; e += NT) {
        const int i = e / n, row = e - i * n;
        Vs[e] = row > i ? P[(size_t)i * ldp + row] : 0.0;
      }
      __syncthreads();
      for (int c0 = 0; c0 < keep; c0 += ngr) {  // (warp-uniform passes: full-mask shuffles)
        const bool cok = c0 + g8 < keep;
        const int c = min(c0 + g8, keep - 1);
        double y[GR];
#pragma unroll
        for (int q = 0; q < GR; ++q) {
          const int r = gl + 8 * q;
          const double tq = T[min(r, kp - 1) * keep + c];
          y[q] = r < kp ? tq : 0.0;
        }
        for (int i = kp - 1; i >= 0; --i) {
          const double tau = taus[i];
          if (tau == 0.0) continue;
          const double* vi = Vs + (size_t)i * n;
          double vr[GR];
          double w0 = 0.0, w1 = 0.0;
#pragma unroll
          for (int q = 0; q < GR; ++q) {
            const int r = gl + 8 * q;
            const double vq = vi[r];  // (unconditional load: slack past the last reflector)
            vr[q] = r < n ? (r == i ? 1.0 : vq) : 0.0;
          }
#pragma unroll
          for (int q = 0; q < GR; q += 2) {
            w0 = fma(vr[q], y[q], w0);
            w1 = fma(vr[q + 1], y[q + 1], w1);
          }
          const double t = -tau * grp_sum_w(w0 + w1);
#pragma unroll
          for (int q = 0; q < GR; ++q) y[q] = fma(t, vr[q], y[q]);
        }
#pragma unroll
        for (int q = 0; q < GR; ++q) {
          const int r = gl + 8 * q;
          if (cok && r < n) Yg[(size_t)r * keep + c] = y[q];
        }
      }
      __syncthreads();
    } else {
      const bool ysm = n * (keep | 1) <= A.big;
      double* Y = ysm ? big : Yg;
      const int ldy = ysm ? (keep | 1) : keep;
      for (int e = tid; e < n * ldy; e += NT) {
        const int a = e / ldy, c = e - a * ldy;
        Y[e] = (a < kp && c < keep) ? T[a * keep + c] : 0.0;
      }
      __syncthreads();
      for (int i = kp - 1; i >= 0; --i) {
        const double tau = taus[i];
        if (tau == 0.0) continue;
        for (int row = i + 1 + tid; row < n; row += NT) S.vh[row] = P[(size_t)i * ldp + row];
        __syncthreads();
        for (int c = g8; c < keep; c += ngr) {
          double w = 0.0;
          for (int row = i + gl; row < n; row += 8)
            w = fma(row == i ? 1.0 : S.vh[row], Y[(size_t)row * ldy + c], w);
          w = grp_sum(w, gm);
          const double t = -tau * w;
          for (int row = i + gl; row < n; row += 8)
            Y[(size_t)row * ldy + c] = fma(t, row == i ? 1.0 : S.vh[row], Y[(size_t)row * ldy + c]);
        }
        __syncthreads();
      }
      if (ysm) {
        for (int e = tid; e < n * keep; e += NT) Yg[e] = Y[(e / keep) * ldy + e % keep];
        __syncthreads();
      }
    }
    if (dbg) {
      tsv[5] = clock64();
      long long* o = A.dbg + blockIdx.x * 8;
      for (int q = 0; q < 5; ++q) o[q] = tsv[q + 1] - tsv[q];
      o[5] = kp; o[6] = keep + 1000 * sweeps_done; o[7] = n * 1000 + nn;
    }
    ++dbg_n;
  }
}

// Jacobi sweeps of a chunk of nodes on the L factors a mode-3 launch left in the per-node
// workspace: one CTA per node at a time, L (up to 64 x 64) in 36 KB of shared memory, four
// CTAs per SM -- twice the nodes in flight of the fused kernel, whose 96 KB work area the
// sweeps do not need.  Larger L are rotated in place in the workspace.
constexpr int JAC_KP = 64;
constexpr int JAC_SMEM_DOUBLES = JAC_KP * JAC_KP + SVD_SLACK + 256 + 8;

struct JacArgs {
  int lb, le, ws_lb;
  double* gws;
  int64_t gws_stride;
  const int* kp_g;
  const int64_t* joff_g;
};


// The launches of one level (hss_level_svd's plan), per kernel kind and dimension.  The k_svd
// instantiations are compiled in one translation unit per kernel kind (svd_<kernel>.cu) so
// they build in parallel.
struct SvdLaunch {
  SvdArgs A;
  int run_lb, run_le, chunk, nsm, grid, big2;
  bool split, jsplit, hyb;
  size_t smem, smem2;
  cudaStream_t s;
};

void svd_launch_jacobi(const JacArgs& a, int grid, cudaStream_t s);  // svd.cu

template <int KER, int D>
void svd_launch_dim(const SvdLaunch& L) {
  const SvdArgs& A = L.A;
  const int run_lb = L.run_lb, run_le = L.run_le, chunk = L.chunk, nsm = L.nsm, grid = L.grid, big2 = L.big2;
  const bool split = L.split, jsplit = L.jsplit, hyb = L.hyb;
  const size_t smem = L.smem, smem2 = L.smem2;
  cudaStream_t s = L.s;
    SvdArgs Ar = A;
    Ar.lb = run_lb;
    Ar.le = run_le;
    if (run_le <= run_lb) return;
    if (chunk) {
      if (split)
        SMASH_CUDA(cudaFuncSetAttribute(k_svd<KER, D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
      SMASH_CUDA(cudaFuncSetAttribute(k_svd<KER, D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem2));
      for (int c0 = run_lb; c0 < run_le; c0 += chunk) {
        Ar.lb = c0;
        Ar.le = std::min(run_le, c0 + chunk);
        Ar.ws_lb = c0;
        const int cn = Ar.le - Ar.lb;
        if (split) {
          Ar.mode = 1;
          Ar.big = A.big;
          k_svd<KER, D, true><<<std::min(nsm, cn), SVD_THREADS, smem, s>>>(Ar);
        }
        Ar.big = big2;
        Ar.prefac = split ? 1 : 0;
        if (jsplit) {
          Ar.mode = 3;
          k_svd<KER, D, false><<<std::min(2 * nsm, cn), SVD_THREADS, smem2, s>>>(Ar);
          JacArgs Ja{Ar.lb, Ar.le, Ar.ws_lb, A.gws, A.gws_stride, A.kp_g, A.joff_g};
          svd_launch_jacobi(Ja, std::min(4 * nsm, cn), s);
          Ar.mode = 4;
          k_svd<KER, D, false><<<std::min(2 * nsm, cn), SVD_THREADS, smem2, s>>>(Ar);
        } else {
          Ar.mode = 2;
          k_svd<KER, D, false><<<std::min(2 * nsm, cn), SVD_THREADS, smem2, s>>>(Ar);
        }
      }
    } else if (hyb) {
      SMASH_CUDA(cudaFuncSetAttribute(k_svd<KER, D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
      k_svd<KER, D, true><<<std::min(grid, run_le - run_lb), SVD_THREADS, smem, s>>>(Ar);
    } else {
      SMASH_CUDA(cudaFuncSetAttribute(k_svd<KER, D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
      k_svd<KER, D, false><<<std::min(grid, run_le - run_lb), SVD_THREADS, smem, s>>>(Ar);
    }
}

template <int KER>
void svd_launch(int dim, const SvdLaunch& L) {
  if constexpr (KER == SMASH_KERNEL_CAUCHY) {
    if (dim != 1) throw Error(SMASH_ERR_INVALID, "unsupported kernel / dimension combination");
    svd_launch_dim<KER, 1>(L);
  } else {
    switch (dim) {
      case 1: svd_launch_dim<KER, 1>(L); break;
      case 2: svd_launch_dim<KER, 2>(L); break;
      case 3: svd_launch_dim<KER, 3>(L); break;
      default: throw Error(SMASH_ERR_INVALID, "unsupported kernel / dimension combination");
    }
  }
}

}  // namespace svdk
}  // namespace smash
