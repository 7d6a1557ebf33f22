// K6-K10: the H^2 / HSS matvec -- replaces smash.apply.matvec_nodewise
// (smash/apply.py:34-80).
//
// Phases (all coefficient vectors are (count, nrhs) row-major, nrhs processed
// in chunks of RC <= 16 columns kept in registers):
//   K10 gather   qt = q[perm_col]                               (apply.py:39)
//   K6  upward   qhat_v = X_v^T ibar-vector, level L..2         (apply.py:42-53)
//   K7  coupling zhat_i = sum_{j in L(i)} K(S_i, S_j) qhat_j     (apply.py:55-58)
//   K8  downward zhat_children += X_v zhat_v, level 2..L-1      (apply.py:60-72)
//   K9  leaves   z[perm_row] = X_v zhat_v + sum_{j in Lm(v)} K(P_v, P_j) qt_j
//                                                              (apply.py:66-80)
// X_v = P [I; G] is applied implicitly from (perm, G) (lowrank.py:224-229).
// The coupling and nearfield blocks are generated on the fly in registers
// (never stored): one CTA per target node, lanes = target points, warps split
// the source list, sources staged per warp in shared memory; the four warps'
// partial sums are reduced in a fixed order (deterministic).
#include "kernels.cuh"
#include "smash_impl.cuh"

namespace smash {

namespace {

constexpr int P2P_WARPS = 4;
constexpr int P2P_THREADS = 32 * P2P_WARPS;

__global__ void k_gather_rows(const double* q, int64_t ldq, const int* perm, int64_t n, int rc,
                              int64_t c0, double* qt, int64_t ldt) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * rc) return;
  int64_t p = e / rc;
  int r = (int)(e % rc);
  qt[p * ldt + r] = q[(int64_t)perm[p] * ldq + c0 + r];
}

struct Side {
  const int* nib;
  const int* rank;
  const int64_t* ib_off;
  const int64_t* g_off;
  const int* skel_off;
  const int* perm;
  const double* G;
  const double* skel_pts;
  int64_t skel_stride;
};

// Block-wide staging copy dst[e] = f(e), e < n: each thread issues U independent
// global loads before its shared-memory stores so a whole tile is one memory
// round trip instead of n / blockDim dependent ones.
template <int U, typename F, typename S>
__device__ __forceinline__ void stage_block(int n, F load, S store) {
  for (int e0 = threadIdx.x; e0 < n; e0 += U * blockDim.x) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * blockDim.x;
      v[u] = e < n ? load(e) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < n) store(e, v[u]);
    }
  }
}

// Tile of G rows staged in shared memory (TB rows, <= 4096 doubles).
__device__ __forceinline__ int g_tile_rows(int ks) { return max(1, min(64, 4096 / ks)); }

constexpr int XFER_THREADS = 256;
constexpr int XFER_MAXO = 8;  // outputs per thread in the upward kernel (k * RC <= 2048)

// ---- K6 upward: qhat[v] = ivec[perm[:k]] + G^T ivec[perm[k:]]
// One CTA per node: the permuted ibar-vector and row tiles of G are staged in
// shared memory with coalesced loads; each thread owns <= 8 (a, r) outputs.
template <int RC>
__global__ void __launch_bounds__(XFER_THREADS) k_upward(int lb, int le, Side cs, const int* nchild,
                                                         const int* child_first, const int* col_a,
                                                         const double* qt, double* qhat) {
  extern __shared__ double sh[];
  const int v = lb + blockIdx.x;
  if (v >= le) return;
  const int n = cs.nib[v], k = cs.rank[v];
  if (k == 0) return;
  const double* ivec = nchild[v] == 0 ? qt + (int64_t)col_a[v] * RC
                                      : qhat + (int64_t)cs.skel_off[child_first[v]] * RC;
  const int* perm = cs.perm + cs.ib_off[v];
  double* iv = sh;               // n * RC: iv[c] = ivec[perm[c]]
  double* gs = sh + n * RC;      // TB * k
  stage_block<8>(n * RC, [&](int e) { return ivec[(int64_t)perm[e / RC] * RC + e % RC]; },
                 [&](int e, double x) { iv[e] = x; });
  __syncthreads();
  const int nout = k * RC;
  double acc[XFER_MAXO];
#pragma unroll
  for (int j = 0; j < XFER_MAXO; ++j) {
    int e = threadIdx.x + j * blockDim.x;
    acc[j] = e < nout ? iv[e] : 0.0;
  }
  const double* G = cs.G + cs.g_off[v];
  const int nk = n - k;
  const int TB = g_tile_rows(k);
  for (int b0 = 0; b0 < nk; b0 += TB) {
    const int tb = min(TB, nk - b0);
    const double* src = G + (int64_t)b0 * k;
    stage_block<16>(tb * k, [&](int e) { return src[e]; }, [&](int e, double x) { gs[e] = x; });
    __syncthreads();
#pragma unroll
    for (int j = 0; j < XFER_MAXO; ++j) {
      int e = threadIdx.x + j * blockDim.x;
      if (e < nout) {
        int a = e / RC, r = e % RC;
        double t = acc[j];
        const double* ivb = iv + (k + b0) * RC + r;
        for (int bb = 0; bb < tb; ++bb) t = fma(gs[bb * k + a], ivb[bb * RC], t);
        acc[j] = t;
      }
    }
    __syncthreads();
  }
  double* out = qhat + (int64_t)cs.skel_off[v] * RC;
#pragma unroll
  for (int j = 0; j < XFER_MAXO; ++j) {
    int e = threadIdx.x + j * blockDim.x;
    if (e < nout) out[e] = acc[j];
  }
}

// ---- K8 downward: zhat[children] += X_v zhat[v]
// Skeleton rows add zhat directly; the other rows are dot products of staged G
// rows (odd row stride -> conflict-free) with zhat_v.
template <int RC>
__global__ void __launch_bounds__(XFER_THREADS) k_downward(int lb, int le, Side rs, const int* nchild,
                                                           const int* child_first, double* zhat) {
  extern __shared__ double sh[];
  const int v = lb + blockIdx.x;
  if (v >= le || nchild[v] == 0) return;
  const int n = rs.nib[v], k = rs.rank[v];
  if (k == 0 || n == 0) return;
  const int ks = k | 1;
  double* zv = sh;           // k * RC
  double* gs = sh + k * RC;  // TB * ks
  const int* perm = rs.perm + rs.ib_off[v];
  const double* zsrc = zhat + (int64_t)rs.skel_off[v] * RC;
  double* dst = zhat + (int64_t)rs.skel_off[child_first[v]] * RC;
  for (int e = threadIdx.x; e < k * RC; e += blockDim.x) {
    double x = zsrc[e];
    zv[e] = x;
    int a = e / RC, r = e % RC;
    dst[(int64_t)perm[a] * RC + r] += x;
  }
  const double* G = rs.G + rs.g_off[v];
  const int nk = n - k;
  const int TB = g_tile_rows(ks);
  for (int b0 = 0; b0 < nk; b0 += TB) {
    const int tb = min(TB, nk - b0);
    const double* src = G + (int64_t)b0 * k;
    __syncthreads();
    stage_block<16>(tb * k, [&](int e) { return src[e]; },
                    [&](int e, double x) { gs[(e / k) * ks + e % k] = x; });
    __syncthreads();
    for (int e = threadIdx.x; e < tb * RC; e += blockDim.x) {
      int bb = e / RC, r = e % RC;
      const double* g = gs + bb * ks;
      double y = 0.0;
      for (int a = 0; a < k; ++a) y = fma(g[a], zv[a * RC + r], y);
      dst[(int64_t)perm[k + b0 + bb] * RC + r] += y;
    }
  }
}

// ---- P2P core: accumulate sum_s K(x_t, y_s) w_s over one source set into acc
template <int KER, int D, int RC>
__device__ __forceinline__ void p2p_sources(const double* xt, const double* ys, int64_t ystride,
                                            const double* w, int ns, double dx, double* acc,
                                            double* stage, int lane) {
  // stage: per-warp buffer of 32 * (D + RC) doubles
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
    for (int s = 0; s < cnt; ++s) {
      double y[D];
#pragma unroll
      for (int a = 0; a < D; ++a) y[a] = stage[a * 32 + s];
      double kv = kval<KER, D>(xt, y, dx);
#pragma unroll
      for (int r = 0; r < RC; ++r) acc[r] = fma(kv, stage[(D + r) * 32 + s], acc[r]);
    }
  }
}

struct P2PArgs {
  // targets
  const double* tpts;  // SoA
  int64_t tstride;
  // sources
  const double* spts;
  int64_t sstride;
  const double* w;  // source weights (count, RC)
  // CSR
  const int* ptr;
  const int* src;
  double dx;
};

// ---- K7 coupling: zhat[v] = sum_{j in L(v)} K(S_v, S_j) qhat_j (one CTA per target node)
template <int KER, int D, int RC>
__global__ void __launch_bounds__(P2P_THREADS) k_coupling(int n_nodes, Side rs, Side cs,
                                                          const int* Lptr, const int* Lsrc,
                                                          const double* qhat, double* zhat,
                                                          double dx) {
  __shared__ double stage[P2P_WARPS][32 * (D + RC)];
  __shared__ double red[P2P_WARPS][32 * RC];
  const int v = blockIdx.x;
  if (v >= n_nodes || v == 0) return;  // root has no factor / no coupling
  const int k = rs.rank[v];
  if (k == 0) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int p0 = Lptr[v], p1 = Lptr[v + 1];
  const int to = rs.skel_off[v];
  for (int t0 = 0; t0 < k; t0 += 32) {
    const int t = t0 + lane;
    double xt[D];
#pragma unroll
    for (int a = 0; a < D; ++a) xt[a] = t < k ? rs.skel_pts[(int64_t)a * rs.skel_stride + to + t] : 0.0;
    double acc[RC];
#pragma unroll
    for (int r = 0; r < RC; ++r) acc[r] = 0.0;
    for (int e = p0 + wid; e < p1; e += P2P_WARPS) {
      const int j = Lsrc[e];
      const int so = cs.skel_off[j];
      p2p_sources<KER, D, RC>(xt, cs.skel_pts + so, cs.skel_stride, qhat + (int64_t)so * RC,
                              cs.rank[j], dx, acc, stage[wid], lane);
    }
#pragma unroll
    for (int r = 0; r < RC; ++r) red[wid][r * 32 + lane] = acc[r];
    __syncthreads();
    if (wid == 0 && t < k) {
#pragma unroll
      for (int r = 0; r < RC; ++r) {
        double s = red[0][r * 32 + lane];
        for (int w = 1; w < P2P_WARPS; ++w) s += red[w][r * 32 + lane];
        zhat[(int64_t)(to + t) * RC + r] = s;
      }
    }
    __syncthreads();
  }
}

// ---- K9 leaves: z[perm_row[p]] = (X_v zhat_v)[p] + sum_{j in Lm(v)} K(x_p, y_s) qt_s
template <int KER, int D, int RC>
__global__ void __launch_bounds__(P2P_THREADS) k_leaf(
    int lb_unused, const int* leaves, int n_leaves, Side rs, const int* row_a, const int* row_b,
    const int* col_a, const int* col_b, const double* pts_row, int64_t nrow, const double* pts_col,
    int64_t ncol, const int* Lmptr, const int* Lmsrc, const double* qt, const double* zhat,
    const int* perm_row, double* z, int64_t ldz, int64_t c0, double dx) {
  extern __shared__ int inv[];  // leaf row count (<= nu0)
  __shared__ double stage[P2P_WARPS][32 * (D + RC)];
  __shared__ double red[P2P_WARPS][32 * RC];
  (void)lb_unused;
  const int li = blockIdx.x;
  if (li >= n_leaves) return;
  const int v = leaves[li];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int ra = row_a[v], nr = row_b[v] - ra;
  const bool has = v != 0;
  const int k = has ? rs.rank[v] : 0;
  const int* perm = has ? rs.perm + rs.ib_off[v] : nullptr;
  if (has)
    for (int c = threadIdx.x; c < nr; c += blockDim.x) inv[perm[c]] = c;
  __syncthreads();
  const int p0 = Lmptr[v], p1 = Lmptr[v + 1];
  for (int t0 = 0; t0 < nr; t0 += 32) {
    const int t = t0 + lane;
    double xt[D];
#pragma unroll
    for (int a = 0; a < D; ++a) xt[a] = t < nr ? pts_row[(int64_t)a * nrow + ra + t] : 0.0;
    double acc[RC];
#pragma unroll
    for (int r = 0; r < RC; ++r) acc[r] = 0.0;
    for (int e = p0 + wid; e < p1; e += P2P_WARPS) {
      const int j = Lmsrc[e];
      const int ca = col_a[j];
      p2p_sources<KER, D, RC>(xt, pts_col + ca, ncol, qt + (int64_t)ca * RC, col_b[j] - ca, dx,
                              acc, stage[wid], lane);
    }
#pragma unroll
    for (int r = 0; r < RC; ++r) red[wid][r * 32 + lane] = acc[r];
    __syncthreads();
    if (wid == 0 && t < nr) {
      double y[RC];
#pragma unroll
      for (int r = 0; r < RC; ++r) y[r] = 0.0;
      if (k > 0) {
        const double* zv = zhat + (int64_t)rs.skel_off[v] * RC;
        const int pos = inv[t];
        if (pos < k) {
#pragma unroll
          for (int r = 0; r < RC; ++r) y[r] = zv[pos * RC + r];
        } else {
          const double* g = rs.G + rs.g_off[v] + (int64_t)(pos - k) * k;
          for (int a = 0; a < k; ++a) {
            double ga = g[a];
#pragma unroll
            for (int r = 0; r < RC; ++r) y[r] = fma(ga, zv[a * RC + r], y[r]);
          }
        }
      }
      double* zo = z + (int64_t)perm_row[ra + t] * ldz + c0;
#pragma unroll
      for (int r = 0; r < RC; ++r) {
        double s = red[0][r * 32 + lane];
        for (int w = 1; w < P2P_WARPS; ++w) s += red[w][r * 32 + lane];
        zo[r] = y[r] + s;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// DMMA path (nrhs chunk RC = 8 or 16): the coupling / nearfield block is a real
// dense contraction Z(t, r) += sum_s K(x_t, y_s) W(s, r), so the K tile is
// generated in registers directly in the A-fragment layout of
// mma.sync.m8n8k4.f64 (DMMA) and multiplied by the weights' B fragments.
// Per warp: all target tiles (8 rows each) x a quarter of the source list;
// the four warps' C fragments are summed in shared memory in a fixed order.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

constexpr int MMA_MTMAX = 8;      // target tiles (8 rows) per pass: 64 targets
constexpr int MMA_WSTRIDE = 36;   // staged weight row stride (doubles): 4 (mod 16)
constexpr int MMA_SEG_CAP = 512;  // source segments per table fill

template <int D, int RC>
constexpr int mma_stage_doubles() { return 32 * D + MMA_WSTRIDE * RC; }

template <int D, int RC>
constexpr int mma_smem_doubles() {
  return P2P_WARPS * MMA_MTMAX * 8 * RC > P2P_WARPS * mma_stage_doubles<D, RC>()
             ? P2P_WARPS * MMA_MTMAX * 8 * RC
             : P2P_WARPS * mma_stage_doubles<D, RC>();
}

struct SegTable {
  int pre[MMA_SEG_CAP + 1];  // prefix of segment lengths
  int off[MMA_SEG_CAP];      // segment start (row index into the source arrays)
  int n;
};

// Source chunk (32 consecutive stream positions) -> registers of this lane.
template <int D, int RC>
__device__ __forceinline__ void mma_fetch(const SegTable& T, int p, int total, const double* spts,
                                          int64_t sstride, const double* wts, double* vc,
                                          double* vw) {
  if (p < total) {
    int lo = 0, hi = T.n - 1;  // last segment with pre <= p
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (T.pre[mid] <= p) lo = mid; else hi = mid - 1;
    }
    const int row = T.off[lo] + (p - T.pre[lo]);
#pragma unroll
    for (int a = 0; a < D; ++a) vc[a] = spts[(int64_t)a * sstride + row];
    const double2* wp = reinterpret_cast<const double2*>(wts + (int64_t)row * RC);
#pragma unroll
    for (int u = 0; u < RC / 2; ++u) {
      const double2 t = wp[u];
      vw[2 * u] = t.x;
      vw[2 * u + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int a = 0; a < D; ++a) vc[a] = 0.0;
#pragma unroll
    for (int u = 0; u < RC; ++u) vw[u] = 0.0;
  }
}

// One warp: accumulate sum over its share of the source stream for MTX target
// tiles into the C fragments c.  Sources stream in chunks of 32 (lane = source)
// across segment boundaries; the next chunk is fetched into registers while
// the current one is consumed from shared memory.
template <int KER, int D, int RC, int MTX>
__device__ __forceinline__ void mma_warp_stream(const SegTable& T, const double* spts,
                                                int64_t sstride, const double* wts,
                                                const double (&xt)[MTX][D], const bool (&tv)[MTX],
                                                double dx, double* stage,
                                                double (&c)[MTX][RC / 8][2]) {
  constexpr int NT = RC / 8;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int total = T.pre[T.n];
  const int nch = (total + 31) >> 5;
  const int per = (nch + P2P_WARPS - 1) / P2P_WARPS;
  const int c0 = wid * per, c1 = min(nch, c0 + per);
  double* sc = stage;
  double* sw = stage + D * 32;
  double vc[D], vw[RC];
  if (c0 < c1) mma_fetch<D, RC>(T, c0 * 32 + lane, total, spts, sstride, wts, vc, vw);
  for (int ch = c0; ch < c1; ++ch) {
    const int cnt = min(32, total - ch * 32);
    __syncwarp();
#pragma unroll
    for (int a = 0; a < D; ++a) sc[a * 32 + lane] = vc[a];
#pragma unroll
    for (int u = 0; u < RC; ++u) sw[u * MMA_WSTRIDE + lane] = vw[u];
    __syncwarp();
    if (ch + 1 < c1) mma_fetch<D, RC>(T, (ch + 1) * 32 + lane, total, spts, sstride, wts, vc, vw);
    for (int kk = 0; kk < cnt; kk += 4) {
      const int si = kk + q;
      const bool sv = si < cnt;
      double ys[D];
#pragma unroll
      for (int a = 0; a < D; ++a) ys[a] = sc[a * 32 + si];
      double b[NT];
#pragma unroll
      for (int n = 0; n < NT; ++n) b[n] = sw[(n * 8 + g) * MMA_WSTRIDE + si];
      double av[MTX];
#pragma unroll
      for (int m = 0; m < MTX; ++m) {  // straight-line: padded entries selected to 0
        const double kv = kval<KER, D>(xt[m], ys, dx);
        av[m] = (sv && tv[m]) ? kv : 0.0;
      }
#pragma unroll
      for (int m = 0; m < MTX; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) dmma_8x8x4(c[m][n][0], c[m][n][1], av[m], b[n]);
    }
  }
}

// Block: targets [0, nt) (nt <= 64) against the CSR source list [p0, p1);
// seg(e) -> (row offset, count) of source set e.  Leaves the per-warp partial
// sums in red[warp][t][r].
template <int KER, int D, int RC, int MTX, typename SegF>
__device__ __forceinline__ void mma_block(const double* tx, int64_t tstride, int nt, int p0,
                                          int p1, SegF seg, const double* spts, int64_t sstride,
                                          const double* wts, double dx, SegTable& T,
                                          double* buf) {
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
      int2 oc = seg(e0 + e);
      T.off[e] = oc.x;
      T.pre[e + 1] = oc.y;  // lengths, prefix-summed below
    }
    __syncthreads();
    if (wid == 0) {  // warp prefix sum of the lengths
      int carry = 0;
      for (int b0 = 0; b0 < ns; b0 += 32) {
        int x = b0 + lane < ns ? T.pre[b0 + lane + 1] : 0;
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (b0 + lane < ns) T.pre[b0 + lane + 1] = x + carry;
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) T.pre[0] = 0;
    }
    __syncthreads();
    mma_warp_stream<KER, D, RC, MTX>(T, spts, sstride, wts, xt, tv, dx,
                                     buf + wid * mma_stage_doubles<D, RC>(), c);
  }
  __syncthreads();  // red aliases the staging buffers
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

// runtime tile count -> compile-time MTX
template <int KER, int D, int RC, typename... Args>
__device__ __forceinline__ void mma_block_dispatch(int mt, Args&&... args) {
  switch (mt) {
    case 1: mma_block<KER, D, RC, 1>(args...); break;
    case 2: mma_block<KER, D, RC, 2>(args...); break;
    case 3: mma_block<KER, D, RC, 3>(args...); break;
    case 4: mma_block<KER, D, RC, 4>(args...); break;
    case 5: mma_block<KER, D, RC, 5>(args...); break;
    case 6: mma_block<KER, D, RC, 6>(args...); break;
    case 7: mma_block<KER, D, RC, 7>(args...); break;
    default: mma_block<KER, D, RC, 8>(args...); break;
  }
}

template <int KER, int D, int RC>
__global__ void __launch_bounds__(P2P_THREADS) k_coupling_mma(int n_nodes, Side rs, Side cs,
                                                              const int* Lptr, const int* Lsrc,
                                                              const double* qhat, double* zhat,
                                                              double dx) {
  __shared__ double buf[mma_smem_doubles<D, RC>()];  // per-warp staging, then the warp sums
  __shared__ SegTable T;
  const int v = blockIdx.x;
  if (v >= n_nodes || v == 0) return;
  const int k = rs.rank[v];
  if (k == 0) return;
  const int p0 = Lptr[v], p1 = Lptr[v + 1];
  const int to = rs.skel_off[v];
  auto seg = [&](int e) {
    const int j = Lsrc[e];
    return make_int2(cs.skel_off[j], cs.rank[j]);
  };
  for (int t0 = 0; t0 < k; t0 += MMA_MTMAX * 8) {
    const int nt = min(MMA_MTMAX * 8, k - t0);
    __syncthreads();
    mma_block_dispatch<KER, D, RC>((nt + 7) >> 3, rs.skel_pts + to + t0, rs.skel_stride, nt, p0,
                                   p1, seg, cs.skel_pts, cs.skel_stride, qhat, dx, T, buf);
    __syncthreads();
    for (int e = threadIdx.x; e < nt * RC; e += blockDim.x) {
      double sum = 0.0;
      if (p1 > p0) {
        sum = buf[e];
        for (int w = 1; w < P2P_WARPS; ++w) sum += buf[w * (MMA_MTMAX * 8 * RC) + e];
      }
      zhat[(int64_t)(to + t0) * RC + e] = sum;
    }
  }
}

template <int KER, int D, int RC>
__global__ void __launch_bounds__(P2P_THREADS) k_leaf_mma(
    const int* leaves, int n_leaves, Side rs, const int* row_a, const int* row_b, const int* col_a,
    const int* col_b, const double* pts_row, int64_t nrow, const double* pts_col, int64_t ncol,
    const int* Lmptr, const int* Lmsrc, const double* qt, const double* zhat, const int* perm_row,
    double* z, int64_t ldz, int64_t c0, double dx) {
  __shared__ double buf[mma_smem_doubles<D, RC>()];
  __shared__ SegTable T;
  extern __shared__ double dyn[];  // zhat_v (k * RC) then inv (nr ints)
  const int li = blockIdx.x;
  if (li >= n_leaves) return;
  const int v = leaves[li];
  const int ra = row_a[v], nr = row_b[v] - ra;
  const bool has = v != 0;
  const int k = has ? rs.rank[v] : 0;
  double* zv = dyn;
  int* inv = reinterpret_cast<int*>(dyn + k * RC);
  if (has) {
    const int* perm = rs.perm + rs.ib_off[v];
    for (int c = threadIdx.x; c < nr; c += blockDim.x) inv[perm[c]] = c;
    const double* zsrc = zhat + (int64_t)rs.skel_off[v] * RC;
    for (int e = threadIdx.x; e < k * RC; e += blockDim.x) zv[e] = zsrc[e];
  }
  const int p0 = Lmptr[v], p1 = Lmptr[v + 1];
  auto seg = [&](int e) {
    const int j = Lmsrc[e];
    return make_int2(col_a[j], col_b[j] - col_a[j]);
  };
  const double* G = has ? rs.G + rs.g_off[v] : nullptr;
  for (int t0 = 0; t0 < nr; t0 += MMA_MTMAX * 8) {
    const int nt = min(MMA_MTMAX * 8, nr - t0);
    __syncthreads();
    mma_block_dispatch<KER, D, RC>((nt + 7) >> 3, pts_row + ra + t0, nrow, nt, p0, p1, seg,
                                   pts_col, ncol, qt, dx, T, buf);
    __syncthreads();
    for (int e = threadIdx.x; e < nt * RC; e += blockDim.x) {
      const int tl = e / RC, r = e % RC, t = t0 + tl;
      double sum = 0.0;
      if (p1 > p0) {
        sum = buf[e];
        for (int w = 1; w < P2P_WARPS; ++w) sum += buf[w * (MMA_MTMAX * 8 * RC) + e];
      }
      double y = 0.0;
      if (k > 0) {
        const int pos = inv[t];
        if (pos < k) {
          y = zv[pos * RC + r];
        } else {
          const double* gr = G + (int64_t)(pos - k) * k;
          double y0 = 0.0, y1 = 0.0, y2 = 0.0, y3 = 0.0;
          int a = 0;
          for (; a + 3 < k; a += 4) {
            y0 = fma(gr[a], zv[a * RC + r], y0);
            y1 = fma(gr[a + 1], zv[(a + 1) * RC + r], y1);
            y2 = fma(gr[a + 2], zv[(a + 2) * RC + r], y2);
            y3 = fma(gr[a + 3], zv[(a + 3) * RC + r], y3);
          }
          for (; a < k; ++a) y0 = fma(gr[a], zv[a * RC + r], y0);
          y = (y0 + y1) + (y2 + y3);
        }
      }
      z[(int64_t)perm_row[ra + t] * ldz + c0 + r] = y + sum;
    }
  }
}

__global__ void k_list_leaves(int n, const int* nchild, int* out, int* cnt) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n && nchild[v] == 0) out[atomicAdd(cnt, 1)] = v;
}

// exact block evaluation (kernel_block API)
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

Side side_of(const SideFactors& F) {
  return Side{F.nib.p, F.rank.p, F.ib_off.p, F.g_off.p, F.skel_off.p, F.perm.p, F.G.p,
              F.skel_pts.p, F.skel_stride};
}

template <int KER, int D, int RC>
void run_chunk(MatrixImpl* m, const double* q, double* z, int64_t nrhs, int64_t c0,
               cudaStream_t s, const int* leaves, int n_leaves, int max_nib, int max_rank) {
  TreeImpl* t = m->tree;
  const SideFactors& R = m->rowf;
  const SideFactors& C = *m->colf;
  Side rs = side_of(R), cs = side_of(C);
  const int* perm_col = t->shared ? t->perm_row.p : t->perm_col.p;
  const double* pts_col = t->shared ? t->pts_row.p : t->pts_col.p;
  const int* col_a = t->shared ? t->row_a.p : t->col_a.p;
  const int* col_b = t->shared ? t->row_b.p : t->col_b.p;
  auto mark = [&](int i) {
    if (m->profile) SMASH_CUDA(cudaEventRecord(m->ev[i], s));
  };
  mark(0);
  // K10 gather
  k_gather_rows<<<cdiv(t->ny * RC, 256), 256, 0, s>>>(q, nrhs, perm_col, t->ny, RC, c0, m->qt.p, RC);
  mark(1);
  // K6 upward
  const size_t sm_up = ((size_t)max_nib * RC + 4096) * sizeof(double);
  for (int l = t->n_levels; l >= 2; --l) {
    int lb = t->level_begin(l), le = t->level_end(l);
    k_upward<RC><<<le - lb, XFER_THREADS, sm_up, s>>>(lb, le, cs, t->nchild.p, t->child_first.p,
                                                      col_a, m->qt.p, m->qhat.p);
  }
  mark(2);
  // K7 coupling
  if constexpr (RC == 8 || RC == 16) {
    k_coupling_mma<KER, D, RC><<<t->n_nodes, P2P_THREADS, 0, s>>>(
        t->n_nodes, rs, cs, m->pl->L_ptr.p, m->pl->L_j.p, m->qhat.p, m->zhat.p, m->p.dx);
  } else {
    k_coupling<KER, D, RC><<<t->n_nodes, P2P_THREADS, 0, s>>>(t->n_nodes, rs, cs, m->pl->L_ptr.p,
                                                              m->pl->L_j.p, m->qhat.p, m->zhat.p,
                                                              m->p.dx);
  }
  mark(3);
  // K8 downward
  const size_t sm_down = ((size_t)max_nib * RC + 4096 + 64) * sizeof(double);
  for (int l = 2; l < t->n_levels; ++l) {
    int lb = t->level_begin(l), le = t->level_end(l);
    k_downward<RC><<<le - lb, XFER_THREADS, sm_down, s>>>(lb, le, rs, t->nchild.p,
                                                          t->child_first.p, m->zhat.p);
  }
  mark(4);
  // K9 leaves (+ K10 scatter)
  if constexpr (RC == 8 || RC == 16) {
    size_t smd = (size_t)max_rank * RC * sizeof(double) + (size_t)(t->nu0 + 1) * sizeof(int);
    k_leaf_mma<KER, D, RC><<<n_leaves, P2P_THREADS, smd, s>>>(
        leaves, n_leaves, rs, t->row_a.p, t->row_b.p, col_a, col_b, t->pts_row.p, t->nx, pts_col,
        t->ny, m->pl->Lm_ptr.p, m->pl->Lm_j.p, m->qt.p, m->zhat.p, t->perm_row.p, z, nrhs, c0,
        m->p.dx);
  } else {
    size_t sm = (size_t)(t->nu0 + 1) * sizeof(int);
    k_leaf<KER, D, RC><<<n_leaves, P2P_THREADS, sm, s>>>(
        0, leaves, n_leaves, rs, t->row_a.p, t->row_b.p, col_a, col_b, t->pts_row.p, t->nx,
        pts_col, t->ny, m->pl->Lm_ptr.p, m->pl->Lm_j.p, m->qt.p, m->zhat.p, t->perm_row.p, z, nrhs,
        c0, m->p.dx);
  }
  mark(5);
  m->launches += 3 + (t->n_levels - 1) + std::max(0, t->n_levels - 2);
  if (m->profile) {
    SMASH_CUDA(cudaEventSynchronize(m->ev[5]));
    for (int i = 0; i < 5; ++i) {
      float ms = 0;
      SMASH_CUDA(cudaEventElapsedTime(&ms, m->ev[i], m->ev[i + 1]));
      m->phase_ms[i] += ms;
    }
  }
}

template <int KER, int D>
void run_all(MatrixImpl* m, const double* q, double* z, int64_t nrhs, cudaStream_t s,
             const int* leaves, int n_leaves, int max_nib, int max_rank, int rc_cap) {
  int64_t c0 = 0;
  while (c0 < nrhs) {
    int64_t left = std::min<int64_t>(nrhs - c0, rc_cap);
    if (left >= 16) { run_chunk<KER, D, 16>(m, q, z, nrhs, c0, s, leaves, n_leaves, max_nib, max_rank); c0 += 16; }
    else if (left >= 8) { run_chunk<KER, D, 8>(m, q, z, nrhs, c0, s, leaves, n_leaves, max_nib, max_rank); c0 += 8; }
    else if (left >= 4) { run_chunk<KER, D, 4>(m, q, z, nrhs, c0, s, leaves, n_leaves, max_nib, max_rank); c0 += 4; }
    else if (left >= 2) { run_chunk<KER, D, 2>(m, q, z, nrhs, c0, s, leaves, n_leaves, max_nib, max_rank); c0 += 2; }
    else { run_chunk<KER, D, 1>(m, q, z, nrhs, c0, s, leaves, n_leaves, max_nib, max_rank); c0 += 1; }
  }
}

}  // namespace

struct MatvecPlan {
  DBuf<int> leaves;
  int n_leaves = 0;
  int max_nib = 0;
  int max_rank = 0;
};

static std::map<const MatrixImpl*, std::unique_ptr<MatvecPlan>> g_plans;

static MatvecPlan* plan_of(MatrixImpl* m, cudaStream_t s) {
  auto it = g_plans.find(m);
  if (it != g_plans.end()) return it->second.get();
  std::unique_ptr<MatvecPlan> P(new MatvecPlan());
  TreeImpl* t = m->tree;
  DBuf<int> cnt;
  cnt.alloc(1, s);
  cnt.zero(s);
  P->leaves.alloc(t->n_nodes, s);
  k_list_leaves<<<cdiv(t->n_nodes, 128), 128, 0, s>>>(t->n_nodes, t->nchild.p, P->leaves.p, cnt.p);
  d2h(&P->n_leaves, cnt.p, 1, s);
  // max |ibar| over both sides (host copy of nib)
  std::vector<int> nib(t->n_nodes);
  d2h(nib.data(), m->rowf.nib.p, t->n_nodes, s);
  sync(s);
  int mx = 1;
  for (int x : nib) mx = std::max(mx, x);
  std::vector<int> rk(t->n_nodes);
  d2h(rk.data(), m->rowf.rank.p, t->n_nodes, s);
  sync(s);
  int mr = 1;
  for (int x : rk) mr = std::max(mr, x);
  if (m->colf != &m->rowf) {
    d2h(nib.data(), m->colf->nib.p, t->n_nodes, s);
    d2h(rk.data(), m->colf->rank.p, t->n_nodes, s);
    sync(s);
    for (int x : nib) mx = std::max(mx, x);
    for (int x : rk) mr = std::max(mr, x);
  }
  P->max_nib = mx;
  P->max_rank = mr;
  MatvecPlan* out = P.get();
  g_plans[m] = std::move(P);
  return out;
}

void matvec_release_plan(const MatrixImpl* m) { g_plans.erase(m); }

void matvec(MatrixImpl* m, const double* q, double* z, int64_t nrhs, cudaStream_t s) {
  SMASH_CHECK(nrhs >= 1, SMASH_ERR_INVALID, "nrhs must be positive");
  TreeImpl* t = m->tree;
  MatvecPlan* P = plan_of(m, s);
  const int rc_max = (int)std::min<int64_t>(nrhs, 16);
  if (m->ws_nrhs < rc_max) {
    m->qt.alloc((size_t)t->ny * 16, s);
    m->qhat.alloc((size_t)std::max<int64_t>(m->colf->skel_total, 1) * 16, s);
    m->zhat.alloc((size_t)std::max<int64_t>(m->rowf.skel_total, 1) * 16, s);
    m->ws_nrhs = 16;
  }
  // shared-memory needs of the upward/downward kernels
  // largest nrhs chunk whose transfer-kernel shared memory and registers fit
  int rc_cap = 16;
  while (rc_cap > 1 && (((size_t)P->max_nib * rc_cap + 4096 + 64) * sizeof(double) > 200 * 1024 ||
                        P->max_rank * rc_cap > XFER_THREADS * XFER_MAXO))
    rc_cap /= 2;
  size_t need = ((size_t)P->max_nib * rc_cap + 4096 + 64) * sizeof(double);
  SMASH_CHECK(need <= 227 * 1024 && P->max_rank <= XFER_THREADS * XFER_MAXO, SMASH_ERR_INVALID,
              "intermediate sets too large for the matvec");
  static bool attr_set = false;
  (void)attr_set;
  dispatch_kernel_dim(m->p.kernel, t->dim, [&]<int KER, int D>() {
    auto setattr = [&](auto kern) {
      SMASH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need));
    };
    setattr(k_upward<1>); setattr(k_upward<2>); setattr(k_upward<4>); setattr(k_upward<8>);
    setattr(k_upward<16>);
    setattr(k_downward<1>); setattr(k_downward<2>); setattr(k_downward<4>); setattr(k_downward<8>);
    setattr(k_downward<16>);
    run_all<KER, D>(m, q, z, nrhs, s, P->leaves.p, P->n_leaves, P->max_nib, P->max_rank, rc_cap);
  });
  SMASH_CUDA(cudaGetLastError());
}

void matvec_profile(MatrixImpl* m, int enable, double* phase_ms, int64_t* launches) {
  if (phase_ms)
    for (int i = 0; i < 5; ++i) phase_ms[i] = m->phase_ms[i];
  if (launches) *launches = m->launches;
  if (enable >= 0) {
    if (enable && !m->ev[0])
      for (auto& e : m->ev) SMASH_CUDA(cudaEventCreate(&e));
    m->profile = enable != 0;
    for (double& x : m->phase_ms) x = 0;
    m->launches = 0;
  }
}

void kernel_block(int kernel, double dx, int dim, const double* X, int64_t nx, const double* Y,
                  int64_t ny, double* out, cudaStream_t s) {
  if (nx * ny == 0) return;
  dispatch_kernel_dim(kernel, dim, [&]<int KER, int D>() {
    k_block<KER, D><<<cdiv(nx * ny, 256), 256, 0, s>>>(X, nx, Y, ny, dx, out);
  });
  SMASH_CUDA(cudaGetLastError());
}

}  // namespace smash
