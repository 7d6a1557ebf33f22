// K7 / K9 point-to-point kernels: coupling and nearfield blocks generated on the
// fly in registers (never stored) -- smash/apply.py:55-58 (coupling, with the
// B(i, j) accessor smash/hss.py:138-148) and smash/apply.py:74-76 (nearfield,
// NF(i, j) smash/hss.py:150-162).
//
// One CTA per target node (coupling: skeleton points; nearfield: leaf points).
//  * RC = 8 / 16 right-hand-side columns: the block product is a real dense
//    contraction, so each K tile is produced directly in the A-fragment layout of
//    mma.sync.m8n8k4.f64 (DMMA) and multiplied by the weights' B fragments.  The
//    source points of all partner nodes form one stream (segments = partner
//    nodes), consumed by the 4 warps in 32-point chunks (lane = source) with a
//    register prefetch of the next chunk; the number of 8-row target tiles is a
//    compile-time constant per CTA (runtime switch), so the kernel evaluations
//    of all tiles are straight-line code.
//  * RC < 8: DFMA path, lane = target, warps split the partner list.
// The four warps' partial sums are added in a fixed order (deterministic).
#pragma once

#include <cstdlib>

#include "matvec_impl.cuh"

namespace smash {
namespace mv {

// ---------------------------------------------------------------------------
// DFMA path
// ---------------------------------------------------------------------------
template <int KER, int D, int RC>
__device__ __forceinline__ void p2p_sources(const double* xt, const double* ys, int64_t ystride,
                                            const double* w, int ns, double dx, double* acc,
                                            double* stage, int lane, const double2* ktab) {
  for (int s0 = 0; s0 < ns; s0 += 32) {
    const int cnt = min(32, ns - s0);
    double vc[D], vw[RC];
#pragma unroll
    for (int a = 0; a < D; ++a) vc[a] = lane < cnt ? ys[(int64_t)a * ystride + s0 + lane] : 0.0;
#pragma unroll
    for (int r = 0; r < RC; ++r) vw[r] = lane < cnt ? w[(int64_t)(s0 + lane) * RC + r] : 0.0;
    __syncwarp();
#pragma unroll
    for (int a = 0; a < D; ++a) stage[a * 32 + lane] = vc[a];
#pragma unroll
    for (int r = 0; r < RC; ++r) stage[(D + r) * 32 + lane] = vw[r];
    __syncwarp();
#pragma unroll 4  // independent evaluations in flight (the lane's chain is ~25 dependent FP64 ops)
    for (int s = 0; s < cnt; ++s) {
      double y[D];
#pragma unroll
      for (int a = 0; a < D; ++a) y[a] = stage[a * 32 + s];
      const double kv = kval_mv<KER, D>(xt, y, dx, ktab, lane);
#pragma unroll
      for (int r = 0; r < RC; ++r) acc[r] = fma(kv, stage[(D + r) * 32 + s], acc[r]);
    }
  }
}

// Block: lane = target (chunks of 32), warps split [p0, p1); sums into red[warp][r][32]
// and hands (target, r, sum) to `out`.
template <int KER, int D, int RC, typename SegF, typename OutF>
__device__ __forceinline__ void dfma_block(const double* tx, int64_t tstride, int nt, int p0,
                                           int p1, SegF seg, const double* spts, int64_t sstride,
                                           const double* wts, double dx, OutF out) {
  __shared__ double stage[P2P_WARPS][32 * (D + RC)];
  __shared__ double red[P2P_WARPS][32 * RC];
  __shared__ double2 ktab[kertab_used<KER>() ? KERTAB_BYTES / 16 : 1];  // log / exp table (kernels.cuh)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if constexpr (kertab_used<KER>()) {
    kertab_fill<KER>(ktab);
    __syncthreads();
  }
  for (int t0 = 0; t0 < nt; t0 += 32) {
    const int t = t0 + lane;
    double xt[D];
#pragma unroll
    for (int a = 0; a < D; ++a) xt[a] = t < nt ? tx[(int64_t)a * tstride + t] : 0.0;
    double acc[RC];
#pragma unroll
    for (int r = 0; r < RC; ++r) acc[r] = 0.0;
    for (int e = p0 + wid; e < p1; e += P2P_WARPS) {
      const int2 oc = seg(e);
      p2p_sources<KER, D, RC>(xt, spts + oc.x, sstride, wts + (int64_t)oc.x * RC, oc.y, dx, acc,
                              stage[wid], lane, ktab);
    }
#pragma unroll
    for (int r = 0; r < RC; ++r) red[wid][r * 32 + lane] = acc[r];
    __syncthreads();
    if (wid == 0 && t < nt) {
#pragma unroll
      for (int r = 0; r < RC; ++r) {
        double sm = red[0][r * 32 + lane];
        for (int w = 1; w < P2P_WARPS; ++w) sm += red[w][r * 32 + lane];
        out(t, r, sm);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// DMMA path
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

constexpr int MMA_MTMAX = 8;      // target tiles (8 rows) per pass: 64 targets
// staged weights are row-major (source x RC) with row stride RC + 4 = 4 (mod 8)
// doubles: the B-fragment reads (4 rows x 8 consecutive) are conflict-free
template <int RC>
constexpr int mma_wstride() { return RC + 4; }
constexpr int MMA_SEG_CAP = 512;  // source segments per table fill

template <int D, int RC>
constexpr int mma_stage_doubles() { return 2 * (32 * D + 32 * mma_wstride<RC>()); }  // 2 buffers

template <int D, int RC>
constexpr int mma_smem_doubles() {
  return P2P_WARPS * MMA_MTMAX * 8 * RC > P2P_WARPS * mma_stage_doubles<D, RC>()
             ? P2P_WARPS * MMA_MTMAX * 8 * RC
             : P2P_WARPS * mma_stage_doubles<D, RC>();
}

struct SegTable {
  int pre[MMA_SEG_CAP + 1];  // prefix of segment lengths
  int off[MMA_SEG_CAP];      // segment start row in the source arrays
  int n;
};

// the segment table's footprint in doubles, rounded to 16 bytes (the log table follows it)
constexpr int p2p_segtable_doubles() { return (int)((sizeof(SegTable) + 15) / 16 * 2); }

__device__ __forceinline__ void cp_async16z(void* dst, const void* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src),
               "r"(valid ? 16 : 0) : "memory");
}

__device__ __forceinline__ void cp_async8z(void* dst, const void* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src),
               "r"(valid ? 8 : 0) : "memory");
}

// Stage source p (this lane's slot of one 32-source chunk) asynchronously:
// coordinates SoA sc[a][lane], weights row-major sw[lane][RC]; slots past the
// end are zero-filled (their kernel values are selected to 0, and 0 * stale
// NaN would not be).
template <int D, int RC>
__device__ __forceinline__ void mma_issue(const SegTable& T, int p, int total, const double* spts,
                                          int64_t sstride, const double* wts, double* sc,
                                          double* sw) {
  const int lane = threadIdx.x & 31;
  const bool ok = p < total;
  int row = 0;
  if (ok) {
    int lo = 0, hi = T.n - 1;  // last segment with pre <= p
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (T.pre[mid] <= p) lo = mid; else hi = mid - 1;
    }
    row = T.off[lo] + (p - T.pre[lo]);
    SMASH_DASSERT(row >= 0 && p - T.pre[lo] < T.pre[lo + 1] - T.pre[lo]);
  }
#pragma unroll
  for (int a = 0; a < D; ++a) cp_async8z(sc + a * 32 + lane, spts + (int64_t)a * sstride + row, ok);
  double* dw = sw + lane * mma_wstride<RC>();
  const double* w = wts + (int64_t)row * RC;
#pragma unroll
  for (int u = 0; u < RC / 2; ++u) cp_async16z(dw + 2 * u, w + 2 * u, ok);
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int KER, int D, int RC, int MTX>
__device__ __forceinline__ void mma_warp_stream(const SegTable& T, const double* spts,
                                                int64_t sstride, const double* wts,
                                                const double (&xt)[MTX][D], const bool (&tv)[MTX],
                                                double dx, double* stage,
                                                double (&c)[MTX][RC / 8][2], const double2* ltab) {
  constexpr int NT = RC / 8;
  constexpr int WS = mma_wstride<RC>();
  constexpr int BUF = 32 * D + 32 * WS;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int total = T.pre[T.n];
  const int nch = (total + 31) >> 5;
  const int per = (nch + P2P_WARPS - 1) / P2P_WARPS;
  const int c0 = wid * per, c1 = min(nch, c0 + per);
  if (c0 < c1) mma_issue<D, RC>(T, c0 * 32 + lane, total, spts, sstride, wts, stage, stage + 32 * D);
  for (int ch = c0; ch < c1; ++ch) {
    double* sc = stage + ((ch - c0) & 1) * BUF;
    double* sw = sc + 32 * D;
    if (ch + 1 < c1) {  // double buffering: the next chunk streams in during this one
      double* nc = stage + ((ch + 1 - c0) & 1) * BUF;
      mma_issue<D, RC>(T, (ch + 1) * 32 + lane, total, spts, sstride, wts, nc, nc + 32 * D);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    const int cnt = min(32, total - ch * 32);
    for (int kk = 0; kk < cnt; kk += 4) {
      const int si = kk + q;
      const bool sv = si < cnt;
      double ys[D];
#pragma unroll
      for (int a = 0; a < D; ++a) ys[a] = sc[a * 32 + si];
      double b[NT];
#pragma unroll
      for (int n = 0; n < NT; ++n) b[n] = sw[si * WS + n * 8 + g];
      double av[MTX];
#pragma unroll
      for (int m = 0; m < MTX; ++m) {  // straight-line: padded entries selected to 0
        const double kv = kval_mv<KER, D>(xt[m], ys, dx, ltab, lane);
        av[m] = (sv && tv[m]) ? kv : 0.0;
      }
#pragma unroll
      for (int m = 0; m < MTX; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) dmma_8x8x4(c[m][n][0], c[m][n][1], av[m], b[n]);
    }
    __syncwarp();  // this buffer is refilled two chunks later
  }
}

// Targets [0, nt) (nt <= 64) against the CSR source list [p0, p1); seg(e) ->
// (row offset, count) of source set e.  Leaves per-warp partial sums in
// buf[warp][t][r].
template <int KER, int D, int RC, int MTX, typename SegF>
__device__ __forceinline__ void mma_block(const double* tx, int64_t tstride, int nt, int p0,
                                          int p1, SegF seg, const double* spts, int64_t sstride,
                                          const double* wts, double dx, SegTable& T,
                                          double* buf, const double2* ltab) {
  constexpr int NT = RC / 8;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  double xt[MTX][D];
  bool tv[MTX];
#pragma unroll
  for (int m = 0; m < MTX; ++m) {
    const int t = m * 8 + g;
    tv[m] = t < nt;
#pragma unroll
    for (int a = 0; a < D; ++a) xt[m][a] = tv[m] ? tx[(int64_t)a * tstride + t] : 0.0;
  }
  double c[MTX][NT][2];
#pragma unroll
  for (int m = 0; m < MTX; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) c[m][n][0] = c[m][n][1] = 0.0;
  for (int e0 = p0; e0 < p1; e0 += MMA_SEG_CAP) {
    const int ns = min(MMA_SEG_CAP, p1 - e0);
    __syncthreads();
    if (threadIdx.x == 0) T.n = ns;
    for (int e = threadIdx.x; e < ns; e += blockDim.x) {
      const int2 oc = seg(e0 + e);
      T.off[e] = oc.x;
      T.pre[e + 1] = oc.y;
    }
    __syncthreads();
    if (wid == 0) {  // prefix sum of the segment lengths
      int carry = 0;
      for (int b0 = 0; b0 < ns; b0 += 32) {
        int x = b0 + lane < ns ? T.pre[b0 + lane + 1] : 0;
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (b0 + lane < ns) T.pre[b0 + lane + 1] = x + carry;
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) T.pre[0] = 0;
    }
    __syncthreads();
    mma_warp_stream<KER, D, RC, MTX>(T, spts, sstride, wts, xt, tv, dx,
                                     buf + wid * mma_stage_doubles<D, RC>(), c, ltab);
  }
  __syncthreads();  // the sums alias the staging buffers
  double* rw = buf + wid * (MMA_MTMAX * 8 * RC);
#pragma unroll
  for (int m = 0; m < MTX; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int t = m * 8 + g, r = n * 8 + 2 * q;
      rw[t * RC + r] = c[m][n][0];
      rw[t * RC + r + 1] = c[m][n][1];
    }
}

template <int KER, int D, int RC, int MT, typename... Args>
__device__ __forceinline__ void mma_block_dispatch(int mt, Args&&... args) {
  switch (mt) {
    case 1: mma_block<KER, D, RC, 1>(args...); break;
    case 2: mma_block<KER, D, RC, 2>(args...); break;
    case 3: mma_block<KER, D, RC, 3>(args...); break;
    case 4: mma_block<KER, D, RC, 4>(args...); break;
    case 5: mma_block<KER, D, RC, (MT < 5 ? MT : 5)>(args...); break;
    case 6: mma_block<KER, D, RC, (MT < 6 ? MT : 6)>(args...); break;
    case 7: mma_block<KER, D, RC, (MT < 7 ? MT : 7)>(args...); break;
    default: mma_block<KER, D, RC, MT>(args...); break;
  }
}

// Targets [0, nt) in MT * 8-row passes; out(t, r, value).  MT (<= MMA_MTMAX)
// bounds the register footprint: MT = 5 (40-row passes) fits 4 CTAs per SM.
template <int KER, int D, int RC, int MT, typename SegF, typename OutF>
__device__ __forceinline__ void p2p_block(const double* tx, int64_t tstride, int nt, int p0, int p1,
                                          SegF seg, const double* spts, int64_t sstride,
                                          const double* wts, double dx, OutF out) {
  if constexpr (RC == 8 || RC == 16) {
    extern __shared__ __align__(16) double p2p_dyn[];  // see p2p_smem_bytes
    double* buf = p2p_dyn;
    SegTable& T = *reinterpret_cast<SegTable*>(p2p_dyn + mma_smem_doubles<D, RC>());
    // the log / exp kernel's table (kernels.cuh) behind the segment table, 16-byte aligned
    double2* ltab = reinterpret_cast<double2*>(p2p_dyn + mma_smem_doubles<D, RC>() + p2p_segtable_doubles());
    if constexpr (kertab_used<KER>()) kertab_fill<KER>(ltab);  // (the loop's first barrier orders it)
    for (int t0 = 0; t0 < nt; t0 += MT * 8) {
      const int n = min(MT * 8, nt - t0);
      __syncthreads();
      mma_block_dispatch<KER, D, RC, MT>((n + 7) >> 3, tx + t0, tstride, n, p0, p1, seg, spts, sstride,
                                     wts, dx, T, buf, ltab);
      __syncthreads();
      for (int e = threadIdx.x; e < n * RC; e += blockDim.x) {
        double sm = 0.0;
        if (p1 > p0) {
          sm = buf[e];
          for (int w = 1; w < P2P_WARPS; ++w) sm += buf[w * (MMA_MTMAX * 8 * RC) + e];
        }
        out(t0 + e / RC, e % RC, sm);
      }
    }
  } else {
    dfma_block<KER, D, RC>(tx, tstride, nt, p0, p1, seg, spts, sstride, wts, dx, out);
  }
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
template <int MT>
constexpr int p2p_min_blocks() { return MT <= 5 ? 4 : 3; }

template <int KER, int D, int RC, int MT>
__global__ void __launch_bounds__(P2P_THREADS, p2p_min_blocks<MT>()) k_coupling(CouplingArgs A) {
  if ((int)blockIdx.x >= A.n_nodes) return;
  const int v = A.list ? A.list[blockIdx.x] : (int)blockIdx.x;
  if (v == 0) return;  // the root has no factor and no coupling
  const int k = A.rs.rank[v];
  if (k == 0) return;
  const int to = A.rs.skel_off[v];
  SMASH_DASSERT(k <= A.max_targets && to >= 0);
  const Side cs = A.cs;
  const int* Lsrc = A.Lsrc;
  auto seg = [&](int e) {
    const int j = Lsrc[e];
    return make_int2(cs.skel_off[j], cs.rank[j]);
  };
  double* zo = A.zhat + (int64_t)to * RC;
  p2p_block<KER, D, RC, MT>(A.rs.skel_pts + to, A.rs.skel_stride, k, A.Lptr[v], A.Lptr[v + 1], seg,
                        cs.skel_pts, cs.skel_stride, A.qhat, A.dx,
                        [&](int t, int r, double val) { zo[(int64_t)t * RC + r] = val; });
}

template <int KER, int D, int RC, int MT>
__global__ void __launch_bounds__(P2P_THREADS, p2p_min_blocks<MT>()) k_near(NearArgs A) {
  const int li = blockIdx.x;
  if (li >= A.n_leaves) return;
  const int v = A.leaves[li];
  const int ra = A.row_a[v], nr = A.row_b[v] - ra;
  SMASH_DASSERT(nr >= 0 && nr <= A.max_targets && ra + nr <= A.nrow);
  const int* col_a = A.col_a;
  const int* col_b = A.col_b;
  const int* Lmsrc = A.Lmsrc;
  auto seg = [&](int e) {
    const int j = Lmsrc[e];
    return make_int2(col_a[j], col_b[j] - col_a[j]);
  };
  const int* slot = A.slot_of + ra;
  double* zn = A.zn;
  p2p_block<KER, D, RC, MT>(A.pts_row + ra, A.nrow, nr, A.Lmptr[v], A.Lmptr[v + 1], seg, A.pts_col,
                        A.ncol, A.qt, A.dx,
                        [&](int t, int r, double val) { zn[(int64_t)slot[t] * RC + r] = val; });
}

// ---------------------------------------------------------------------------
// symmetric coupling (SymCoupling, matvec_impl.cuh): each block K(S_v, S_j), j > v, is
// generated once and contracted both ways.  Per 8-source block (two 4-source DMMA
// steps) the lanes hold A[t][s] for target t = 8m + g, source s = 4h + q; the transposed
// fragment A^T (8 sources x 4 targets) is gathered with two shuffles per K chunk and
// contracted with the target's own coefficients (B operand), giving B_vj^T qhat_v for the
// 8 sources, which go to the pair buffer rows (added over the target passes).
// ---------------------------------------------------------------------------
struct SegTableSym {
  int pre[MMA_SEG_CAP + 1];
  int off[MMA_SEG_CAP];
  int64_t boff[MMA_SEG_CAP];  // pair buffer row of the segment's first source
  int n;
};

template <int D, int RC>
constexpr int mma_stage_doubles_sym() { return 2 * (32 * D + 32 * mma_wstride<RC>() + 32); }

template <int D, int RC>
constexpr int mma_smem_doubles_sym() {
  return P2P_WARPS * MMA_MTMAX * 8 * RC > P2P_WARPS * mma_stage_doubles_sym<D, RC>()
             ? P2P_WARPS * MMA_MTMAX * 8 * RC
             : P2P_WARPS * mma_stage_doubles_sym<D, RC>();
}

template <int D, int RC>
__device__ __forceinline__ void mma_issue_sym(const SegTableSym& T, int p, int total,
                                              const double* spts, int64_t sstride,
                                              const double* wts, double* sc, double* sw,
                                              long long* sb) {
  const int lane = threadIdx.x & 31;
  const bool ok = p < total;
  int row = 0;
  long long brow = -1;
  if (ok) {
    int lo = 0, hi = T.n - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (T.pre[mid] <= p) lo = mid; else hi = mid - 1;
    }
    row = T.off[lo] + (p - T.pre[lo]);
    brow = T.boff[lo] + (p - T.pre[lo]);
  }
  sb[lane] = brow;  // plain store: read after this chunk's wait + __syncwarp
#pragma unroll
  for (int a = 0; a < D; ++a) cp_async8z(sc + a * 32 + lane, spts + (int64_t)a * sstride + row, ok);
  double* dw = sw + lane * mma_wstride<RC>();
  const double* w = wts + (int64_t)row * RC;
#pragma unroll
  for (int u = 0; u < RC / 2; ++u) cp_async16z(dw + 2 * u, w + 2 * u, ok);
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int KER, int D, int RC, int MTX>
__device__ __forceinline__ void mma_warp_stream_sym(const SegTableSym& T, const double* spts,
                                                    int64_t sstride, const double* wts,
                                                    const double (&xt)[MTX][D],
                                                    const bool (&tv)[MTX],
                                                    const double (&bq)[MTX][2][RC / 8], double dx,
                                                    double* stage, double* buf, bool first_pass,
                                                    double (&c)[MTX][RC / 8][2]) {
  constexpr int NT = RC / 8;
  constexpr int WS = mma_wstride<RC>();
  constexpr int BUF = 32 * D + 32 * WS + 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int total = T.pre[T.n];
  const int nch = (total + 31) >> 5;
  const int per = (nch + P2P_WARPS - 1) / P2P_WARPS;
  const int c0 = wid * per, c1 = min(nch, c0 + per);
  auto bufs = [&](int k) { return stage + (k & 1) * BUF; };
  if (c0 < c1) {
    double* sc = bufs(0);
    mma_issue_sym<D, RC>(T, c0 * 32 + lane, total, spts, sstride, wts, sc, sc + 32 * D,
                         reinterpret_cast<long long*>(sc + 32 * D + 32 * WS));
  }
  for (int ch = c0; ch < c1; ++ch) {
    double* sc = bufs(ch - c0);
    double* sw = sc + 32 * D;
    const long long* sb = reinterpret_cast<const long long*>(sw + 32 * WS);
    if (ch + 1 < c1) {
      double* nc = bufs(ch + 1 - c0);
      mma_issue_sym<D, RC>(T, (ch + 1) * 32 + lane, total, spts, sstride, wts, nc, nc + 32 * D,
                           reinterpret_cast<long long*>(nc + 32 * D + 32 * WS));
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    const int cnt = min(32, total - ch * 32);
    for (int kk = 0; kk < cnt; kk += 8) {
      double av[2][MTX];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int si = kk + 4 * h + q;
        const bool sv = si < cnt;
        double ys[D];
#pragma unroll
        for (int a = 0; a < D; ++a) ys[a] = sc[a * 32 + (si & 31)];
        double b[NT];
#pragma unroll
        for (int n = 0; n < NT; ++n) b[n] = sw[(si & 31) * WS + n * 8 + g];
#pragma unroll
        for (int m = 0; m < MTX; ++m) {
          const double kv = kval<KER, D>(xt[m], ys, dx);
          av[h][m] = (sv && tv[m]) ? kv : 0.0;
        }
#pragma unroll
        for (int m = 0; m < MTX; ++m)
#pragma unroll
          for (int n = 0; n < NT; ++n) dmma_8x8x4(c[m][n][0], c[m][n][1], av[h][m], b[n]);
      }
      // transposed: D[s][r] = sum_t A[t][s] qhat_v[t][r] for the 8 sources kk..kk+7
      double dacc[NT][2];
#pragma unroll
      for (int n = 0; n < NT; ++n) dacc[n][0] = dacc[n][1] = 0.0;
#pragma unroll
      for (int m = 0; m < MTX; ++m)
#pragma unroll
        for (int ck = 0; ck < 2; ++ck) {
          const int src = (4 * ck + q) * 4 + (g & 3);  // lane holding A[4ck + q][g]
          const double x0 = __shfl_sync(0xffffffffu, av[0][m], src);
          const double x1 = __shfl_sync(0xffffffffu, av[1][m], src);
          const double at = g < 4 ? x0 : x1;
#pragma unroll
          for (int n = 0; n < NT; ++n) dmma_8x8x4(dacc[n][0], dacc[n][1], at, bq[m][ck][n]);
        }
      const int si = kk + g;  // this lane's source row of D
      if (si < cnt) {
        const long long br = sb[si];
        double* o = buf + br * RC;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const int r = n * 8 + 2 * q;
          if (first_pass) {
            o[r] = dacc[n][0];
            o[r + 1] = dacc[n][1];
          } else {
            o[r] += dacc[n][0];
            o[r + 1] += dacc[n][1];
          }
        }
      }
    }
    __syncwarp();
  }
}

template <int KER, int D, int RC, int MTX, typename SegF>
__device__ __forceinline__ void mma_block_sym(const double* tx, int64_t tstride, int nt, int p0,
                                              int p1, SegF seg, const double* spts,
                                              int64_t sstride, const double* wts,
                                              const double* qv, double* pbuf_base,
                                              const int64_t* pbuf, double dx, bool first_pass,
                                              SegTableSym& T, double* buf) {
  constexpr int NT = RC / 8;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  double xt[MTX][D];
  bool tv[MTX];
  double bq[MTX][2][NT];
#pragma unroll
  for (int m = 0; m < MTX; ++m) {
    const int t = m * 8 + g;
    tv[m] = t < nt;
#pragma unroll
    for (int a = 0; a < D; ++a) xt[m][a] = tv[m] ? tx[(int64_t)a * tstride + t] : 0.0;
#pragma unroll
    for (int ck = 0; ck < 2; ++ck) {
      const int tk = m * 8 + 4 * ck + q;  // B operand row k = target, column n = rhs
#pragma unroll
      for (int n = 0; n < NT; ++n) bq[m][ck][n] = tk < nt ? qv[(int64_t)tk * RC + n * 8 + g] : 0.0;
    }
  }
  double c[MTX][NT][2];
#pragma unroll
  for (int m = 0; m < MTX; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) c[m][n][0] = c[m][n][1] = 0.0;
  for (int e0 = p0; e0 < p1; e0 += MMA_SEG_CAP) {
    const int ns = min(MMA_SEG_CAP, p1 - e0);
    __syncthreads();
    if (threadIdx.x == 0) T.n = ns;
    for (int e = threadIdx.x; e < ns; e += blockDim.x) {
      const int2 oc = seg(e0 + e);
      T.off[e] = oc.x;
      T.pre[e + 1] = oc.y;
      T.boff[e] = pbuf[e0 + e];
    }
    __syncthreads();
    if (wid == 0) {
      int carry = 0;
      for (int b0 = 0; b0 < ns; b0 += 32) {
        int x = b0 + lane < ns ? T.pre[b0 + lane + 1] : 0;
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (b0 + lane < ns) T.pre[b0 + lane + 1] = x + carry;
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) T.pre[0] = 0;
    }
    __syncthreads();
    mma_warp_stream_sym<KER, D, RC, MTX>(T, spts, sstride, wts, xt, tv, bq, dx,
                                         buf + wid * mma_stage_doubles_sym<D, RC>(), pbuf_base,
                                         first_pass, c);
  }
  __syncthreads();
  double* rw = buf + wid * (MMA_MTMAX * 8 * RC);
#pragma unroll
  for (int m = 0; m < MTX; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int t = m * 8 + g, r = n * 8 + 2 * q;
      rw[t * RC + r] = c[m][n][0];
      rw[t * RC + r + 1] = c[m][n][1];
    }
}

template <int KER, int D, int RC, int MT>
__global__ void __launch_bounds__(P2P_THREADS, 2) k_coupling_sym(CouplingArgs A, SymCoupling Y) {
  if ((int)blockIdx.x >= A.n_nodes) return;
  const int v = (int)blockIdx.x;
  if (v == 0) return;
  const int k = A.rs.rank[v];
  if (k == 0) return;
  const int to = A.rs.skel_off[v];
  SMASH_DASSERT(k <= A.max_targets && to >= 0);
  const Side cs = A.cs;
  const int* Usrc = Y.Usrc;
  auto seg = [&](int e) {
    const int j = Usrc[e];
    return make_int2(cs.skel_off[j], cs.rank[j]);
  };
  double* zo = A.zhat + (int64_t)to * RC;
  const double* qv = A.qhat + (int64_t)cs.skel_off[v] * RC;
  extern __shared__ __align__(16) double p2p_dyn[];
  double* buf = p2p_dyn;
  SegTableSym& T = *reinterpret_cast<SegTableSym*>(p2p_dyn + mma_smem_doubles_sym<D, RC>());
  const int p0 = Y.Uptr[v], p1 = Y.Uptr[v + 1];
  for (int t0 = 0; t0 < k; t0 += MT * 8) {
    const int n = min(MT * 8, k - t0);
    __syncthreads();
    const double* tx = A.rs.skel_pts + to + t0;
    const int64_t ts = A.rs.skel_stride;
    const bool first = t0 == 0;
    switch ((n + 7) >> 3) {
      case 1: mma_block_sym<KER, D, RC, 1>(tx, ts, n, p0, p1, seg, cs.skel_pts, cs.skel_stride, A.qhat, qv + (int64_t)t0 * RC, Y.buf, Y.pbuf, A.dx, first, T, buf); break;
      case 2: mma_block_sym<KER, D, RC, 2>(tx, ts, n, p0, p1, seg, cs.skel_pts, cs.skel_stride, A.qhat, qv + (int64_t)t0 * RC, Y.buf, Y.pbuf, A.dx, first, T, buf); break;
      case 3: mma_block_sym<KER, D, RC, 3>(tx, ts, n, p0, p1, seg, cs.skel_pts, cs.skel_stride, A.qhat, qv + (int64_t)t0 * RC, Y.buf, Y.pbuf, A.dx, first, T, buf); break;
      default: mma_block_sym<KER, D, RC, MT>(tx, ts, n, p0, p1, seg, cs.skel_pts, cs.skel_stride, A.qhat, qv + (int64_t)t0 * RC, Y.buf, Y.pbuf, A.dx, first, T, buf); break;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * RC; e += blockDim.x) {
      double sm = 0.0;
      if (p1 > p0) {
        sm = buf[e];
        for (int w = 1; w < P2P_WARPS; ++w) sm += buf[w * (MMA_MTMAX * 8 * RC) + e];
      }
      zo[(int64_t)t0 * RC + e] = sm;
    }
  }
}

// pass 2: zhat[j] += sum over the upper pairs (i, j), i < j (ascending i), of their rows
template <int RC>
__global__ void __launch_bounds__(128) k_coupling_tsum(CouplingArgs A, SymCoupling Y) {
  const int j = (int)blockIdx.x;
  if (j == 0 || j >= A.n_nodes) return;
  const int k = A.cs.rank[j];
  const int e0 = Y.tptr[j], e1 = Y.tptr[j + 1];
  if (k == 0 || e0 == e1) return;
  double* zo = A.zhat + (int64_t)A.rs.skel_off[j] * RC;
  for (int x = threadIdx.x; x < k * RC; x += blockDim.x) {
    double acc = zo[x];
    for (int e = e0; e < e1; ++e) acc += Y.buf[Y.pbuf[Y.te[e]] * RC + x];
    zo[x] = acc;
  }
}

template <int KER, int D>
__global__ void k_block(const double* X, int64_t nx, const double* Y, int64_t ny, double dx,
                        double* out) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= nx * ny) return;
  int64_t i = e / ny, j = e % ny;
  double x[D], y[D];
#pragma unroll
  for (int a = 0; a < D; ++a) { x[a] = X[i * D + a]; y[a] = Y[j * D + a]; }
  out[e] = kval<KER, D>(x, y, dx);
}

// ---------------------------------------------------------------------------
// launchers (explicitly instantiated per kernel in p2p_<kernel>.cu)
// ---------------------------------------------------------------------------
template <int KER, int D, int RC>
constexpr size_t p2p_smem_bytes() {
  return RC >= 8 ? (mma_smem_doubles<D, RC>() + p2p_segtable_doubles()) * sizeof(double) +
                       (kertab_used<KER>() ? KERTAB_BYTES : 0)
                 : 0;
}

template <typename K>
void p2p_attrs(K kern, size_t smem) {
  SMASH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SMASH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
}

// 8-row target tiles per pass: 5 (<= 40 targets, 4 CTAs/SM) or 8
inline bool p2p_small(int max_targets) {
  static const int mode = getenv("SMASH_P2P_MT") ? atoi(getenv("SMASH_P2P_MT")) : 0;
  if (mode == 8) return false;
  if (mode == 5) return true;
  return max_targets <= 64;  // 40-row passes; 120 registers -> 4 CTAs per SM
}

template <int KER, int D, int RC>
void launch_coupling(const CouplingArgs& a, cudaStream_t s) {
  constexpr size_t smem = p2p_smem_bytes<KER, D, RC>();
  static const bool attr = [] {
    p2p_attrs(k_coupling<KER, D, RC, 5>, smem);
    p2p_attrs(k_coupling<KER, D, RC, 8>, smem);
    return true;
  }();
  (void)attr;
  if (a.n_nodes <= 0) return;
  if (p2p_small(a.max_targets)) k_coupling<KER, D, RC, 5><<<a.n_nodes, P2P_THREADS, smem, s>>>(a);
  else k_coupling<KER, D, RC, 8><<<a.n_nodes, P2P_THREADS, smem, s>>>(a);
}

template <int KER, int D, int RC>
void launch_coupling_sym(const CouplingArgs& a, const SymCoupling& y, cudaStream_t s) {
  if constexpr (RC == 8 || RC == 16) {
    constexpr size_t smem = mma_smem_doubles_sym<D, RC>() * sizeof(double) + sizeof(SegTableSym);
    static const bool attr = [] {
      p2p_attrs(k_coupling_sym<KER, D, RC, 4>, smem);
      return true;
    }();
    (void)attr;
    if (a.n_nodes <= 0) return;
    k_coupling_sym<KER, D, RC, 4><<<a.n_nodes, P2P_THREADS, smem, s>>>(a, y);
    k_coupling_tsum<RC><<<a.n_nodes, 128, 0, s>>>(a, y);
  } else {
    throw Error(SMASH_ERR_INVALID, "symmetric coupling needs 8 or 16 right-hand-side columns");
  }
}

template <int KER, int D, int RC>
void launch_near(const NearArgs& a, cudaStream_t s) {
  constexpr size_t smem = p2p_smem_bytes<KER, D, RC>();
  static const bool attr = [] {
    p2p_attrs(k_near<KER, D, RC, 5>, smem);
    p2p_attrs(k_near<KER, D, RC, 8>, smem);
    return true;
  }();
  (void)attr;
  if (a.n_leaves <= 0) return;
  if (p2p_small(a.max_targets)) k_near<KER, D, RC, 5><<<a.n_leaves, P2P_THREADS, smem, s>>>(a);
  else k_near<KER, D, RC, 8><<<a.n_leaves, P2P_THREADS, smem, s>>>(a);
}

template <int KER, int D>
void launch_block(const double* X, int64_t nx, const double* Y, int64_t ny, double dx, double* out,
                  cudaStream_t s) {
  if (nx * ny > 0) k_block<KER, D><<<cdiv(nx * ny, 256), 256, 0, s>>>(X, nx, Y, ny, dx, out);
}

#define SMASH_P2P_INSTANTIATE(KER, D)                                                 \
  template void launch_coupling<KER, D, 1>(const CouplingArgs&, cudaStream_t);        \
  template void launch_coupling<KER, D, 2>(const CouplingArgs&, cudaStream_t);        \
  template void launch_coupling<KER, D, 4>(const CouplingArgs&, cudaStream_t);        \
  template void launch_coupling<KER, D, 8>(const CouplingArgs&, cudaStream_t);        \
  template void launch_coupling<KER, D, 16>(const CouplingArgs&, cudaStream_t);       \
  template void launch_near<KER, D, 1>(const NearArgs&, cudaStream_t);                \
  template void launch_near<KER, D, 2>(const NearArgs&, cudaStream_t);                \
  template void launch_near<KER, D, 4>(const NearArgs&, cudaStream_t);                \
  template void launch_near<KER, D, 8>(const NearArgs&, cudaStream_t);                \
  template void launch_near<KER, D, 16>(const NearArgs&, cudaStream_t);               \
  template void launch_coupling_sym<KER, D, 8>(const CouplingArgs&, const SymCoupling&, cudaStream_t); \
  template void launch_coupling_sym<KER, D, 16>(const CouplingArgs&, const SymCoupling&, cudaStream_t); \
  template void launch_block<KER, D>(const double*, int64_t, const double*, int64_t,  \
                                     double, double*, cudaStream_t);

}  // namespace mv
}  // namespace smash
