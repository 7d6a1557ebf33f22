// K6 / K8 / K10: permutation gather, upward and downward transfer passes and
// the final far + near combine of the matvec (smash/apply.py:39-53, 60-72, 78-80).
//
// The transfer passes are level-ordered dataflow: a node's upward projection
// needs its children's, its downward step needs its parent's.  Each pass is ONE
// persistent launch over all its nodes (leaves included): CTAs take node
// tickets from an atomic counter in level order (deepest first upward,
// shallowest first downward) and spin on the producers' done flags, which were
// necessarily handed out earlier to CTAs that are already running -- so the
// wait cannot deadlock.  Cross-CTA data is published with a CTA barrier + a
// gpu-scope release flag and read through L2 (cp.async.cg / ld.cg) after an
// acquire.
//
// Leaves are handled by warp-per-leaf launches on either side of the
// persistent passes (no producers upward; downward the far field is fused
// with the final z = near + far combine).
//
// Per node the work is a small GEMM with the interpolative factor
// X_v = P [I; G] (G: (|ibar| - k) x k row-major):
//   upward    qhat_v          = in[perm[:k]] + G^T in[perm[k:]]    (in: children's
//                                coefficients, or the leaf's qt rows)
//   downward  out[perm[:k]]  += zhat_v,  out[perm[k:]] += G zhat_v (out: children's
//                                zhat, or the leaf's far-field rows)
// G and the permutation are read-only, so their cp.async staging is issued
// before the producer wait; the producer rows follow in one more asynchronous
// batch.  The GEMM runs on the FP64 tensor cores (mma.sync m8n8k4 DMMA) with
// operands read from shared memory at bank-conflict-free strides (row strides
// = 4 mod 8 doubles), one 8x8 output tile per warp and item.
#include <cstdlib>

#include "matvec_impl.cuh"

namespace smash {
namespace mv {

#ifdef SMASH_XFER_TRACE
// instrumented build only: per item (kernel << 32 | node, smid, t_start,
// t_producers_done, t_staged, t_end) in globaltimer ns
__device__ unsigned long long g_trace[1 << 20];
__device__ unsigned g_trace_n;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
#define TRACE_DECL unsigned long long t0 = gtimer(), t1 = t0, t2 = t0, t3 = t0
#define TRACE_SET(var) var = gtimer()
#define TRACE_EMIT(kid, v, t0, t1, t2)                                                      \
  if (threadIdx.x == 0) {                                                                   \
    const unsigned long long te = gtimer();                                                 \
    const unsigned i = atomicAdd(&g_trace_n, 1u);                                           \
    if (i < (1u << 20) / 8) {                                                               \
      unsigned long long* o = g_trace + 8 * i;                                              \
      o[0] = ((unsigned long long)(kid) << 32) | (unsigned)(v);                             \
      o[1] = smid(); o[2] = t0; o[3] = t1; o[4] = t2; o[5] = t3; o[6] = te; o[7] = 0;      \
    }                                                                                       \
  }
#else
#define TRACE_DECL
#define TRACE_SET(var)
#define TRACE_EMIT(kid, v, t0, t1, t2)
#endif

namespace {

template <int RC>
__global__ void k_gather(const double* q, int64_t ldq, const int* perm, int64_t n, int64_t c0,
                         double* qt) {
  const int64_t p = blockIdx.x * (int64_t)(blockDim.x / RC) + threadIdx.x / RC;
  const int r = threadIdx.x % RC;
  if (p < n) qt[p * RC + r] = q[(int64_t)perm[p] * ldq + c0 + r];
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void cp_async16_cg(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}

__device__ __forceinline__ void cp_commit_wait() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// RC doubles of a coherent (written by other CTAs of this launch) row -> shared
template <int RC>
__device__ __forceinline__ void row_l2(double* dst, const double* src) {
  if constexpr (RC % 2 == 0) {
#pragma unroll
    for (int u = 0; u < RC / 2; ++u) cp_async16_cg(dst + 2 * u, src + 2 * u);
  } else {
#pragma unroll
    for (int u = 0; u < RC; ++u) dst[u] = __ldcg(src + u);
  }
}

// named barriers of the persistent passes: 1 = the XFER_THREADS compute
// threads, 2 = compute threads + the descriptor-prefetch warp
__device__ __forceinline__ void bar_compute() {
  asm volatile("bar.sync 1, %0;" ::"n"(XFER_THREADS) : "memory");
}
__device__ __forceinline__ void bar_handover() {
  asm volatile("bar.sync 2, %0;" ::"n"(XFER_THREADS + 32) : "memory");
}

// Read-only G rows [r0, r0 + nr) (row length k) -> shared rows of stride ks
// (compute threads): flat element loop, the (row, col) of element e advanced
// incrementally (no division per element).
__device__ __forceinline__ void stage_g(const double* G, int k, int r0, int nr, double* gs, int ks) {
  const int n = nr * k;
  int e = threadIdx.x;
  int row = e / k, col = e - row * k;
  const int drow = XFER_THREADS / k, dcol = XFER_THREADS - drow * k;
  const double* src = G + (int64_t)r0 * k;
  for (; e < n; e += XFER_THREADS) {
    cp_async8(gs + row * ks + col, src + e);
    row += drow;
    col += dcol;
    if (col >= k) {
      col -= k;
      ++row;
    }
  }
}

// Release of a node's rows: the CTA barrier orders every compute thread's
// stores before thread 0's gpu-scope release (cumulative), as in CUTLASS's
// semaphore; consumers acquire the flag and then barrier.
__device__ __forceinline__ void publish(unsigned* done, int v) {
  bar_compute();
  if (threadIdx.x == 0) st_release(&done[v], 1u);
}

// Node descriptor of one ticket.  A ninth warp takes the next ticket and loads
// its descriptor while the eight compute warps process the current node
// (double-buffered in shared memory, handed over at named barrier 2), so the
// ticket -> node -> descriptor latency chain is off the critical path.
struct NodeDesc {
  int v, ni, k, nc, cf, parent, skel, base;  // base: skel_off of the children block
  int64_t g_off, ib_off;
  unsigned wait;  // upward: bit c = child c is produced by this launch; downward: bit 0 = parent
};

// Warp-cooperative descriptor fetch of the next ticket (the whole prefetch warp).
__device__ __forceinline__ void fetch_desc(NodeDesc* d, const XferArgs& A, const int* order, int n,
                                           unsigned* counter, const unsigned char* inset,
                                           bool upward) {
  const int lane = threadIdx.x & 31;
  int t = 0;
  if (lane == 0) t = (int)atomicAdd(counter, 1u);
  t = __shfl_sync(0xffffffffu, t, 0);
  NodeDesc x;
  x.v = t < n ? order[t] : -1;
  x.wait = 0;
  if (x.v >= 0) {
    const Side& S = A.side;
    const int v = x.v;
    x.ni = S.nib[v];
    x.k = S.rank[v];
    x.nc = A.nchild[v];
    x.cf = A.child_first[v];
    x.parent = A.parent[v];
    x.skel = S.skel_off[v];
    x.g_off = S.g_off[v];
    x.ib_off = S.ib_off[v];
    x.base = x.nc > 0 ? S.skel_off[x.cf] : 0;
    if (upward) {
      x.wait = __ballot_sync(0xffffffffu, lane < x.nc && inset[x.cf + lane] != 0);
    } else {
      x.wait = (x.parent > 0 && inset[x.parent] != 0) ? 1u : 0u;
    }
  }
  if (lane == 0) *d = x;
}

// The prefetch warp's loop (returns when the order is exhausted).
__device__ __forceinline__ void desc_producer(NodeDesc* s_desc, const XferArgs& A, const int* order,
                                              int n, unsigned* counter, const unsigned char* inset,
                                              bool upward) {
  for (int i = 0;; ++i) {
    fetch_desc(&s_desc[i & 1], A, order, n, counter, inset, upward);
    __syncwarp();
    const int v = s_desc[i & 1].v;
    bar_handover();
    if (v < 0) return;
  }
}

// Branch-free DMMA inner loops over shared-memory fragments: all fragment
// loads of a step pair are issued before its MMAs, and every accumulator
// chain is independent (the DMMA latency is ~26 cycles, its issue interval 16).
// Upward: MT tiles x 2 partial chains (even / odd K steps).
template <int MT>
__device__ __forceinline__ void mma_up(const double* const* ga, const double* const* bb, int ks4,
                                       int rs4, int steps, double (&c)[2][2][2]) {
  int s = 0;
#pragma unroll 2
  for (; s + 1 < steps; s += 2) {
    double a[MT][2], b[MT][2];
#pragma unroll
    for (int t = 0; t < MT; ++t)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        a[t][h] = ga[t][(s + h) * ks4];
        b[t][h] = bb[t][(s + h) * rs4];
      }
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int t = 0; t < MT; ++t) dmma(c[t][h][0], c[t][h][1], a[t][h], b[t][h]);
  }
  if (s < steps) {
#pragma unroll
    for (int t = 0; t < MT; ++t) dmma(c[t][0][0], c[t][0][1], ga[t][s * ks4], bb[t][s * rs4]);
  }
}

// Downward: NT independent tiles, one chain each.
template <int NT>
__device__ __forceinline__ void mma_down(const double* const* ga, const double* const* zb, int rs4,
                                         int steps, double (&c)[4][2]) {
#pragma unroll 2
  for (int s = 0; s < steps; ++s) {
    double a[NT], b[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      a[t] = ga[t][4 * s];
      b[t] = zb[t][s * rs4];
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) dmma(c[t][0], c[t][1], a[t], b[t]);
  }
}

// qhat_v = ivp[:k] + G^T ivp[k:] for every internal node of `order`, where
// ivp = the children's coefficients already in v's ibar order (qp, scattered
// there by the children's epilogues); the result is also scattered into the
// parent's ibar order (qp[up_pos]).  Each warp owns up to two 8x8 output
// tiles, each accumulated in two partial chains (even / odd K steps).
template <int RC>
__global__ void __launch_bounds__(XFER_THREADS + 32) k_upward(XferArgs A, XferGeom Gm,
                                                              const int* order, int n,
                                                              const unsigned char* inset,
                                                              unsigned* counter, unsigned* done) {
  extern __shared__ __align__(16) double sh[];
  __shared__ NodeDesc s_desc[2];
  const int ks = Gm.ks, rcs = Gm.rcs;
  double* gs = sh;                        // tb x ks   (G chunk)
  double* ivp = sh + Gm.tb * ks;          // (max_nib + 16) x rcs (ibar rows + fragment over-read)
  const Side cs = A.side;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  constexpr int NR = (RC + 7) / 8;
  if (wid == XFER_THREADS / 32) {
    desc_producer(s_desc, A, order, n, counter, inset, true);
    return;
  }
  bar_handover();
  for (int cur = 0;; cur ^= 1) {
    const NodeDesc d = s_desc[cur];
    if (d.v < 0) break;
    TRACE_DECL;
    const int ni = d.ni, k = d.k;
    const int nk = ni - k, nk4 = (nk + 3) & ~3;
    if (k > 0) {
      const double* G = cs.G + d.g_off;
      const int tb0 = min(Gm.tb, nk);
      stage_g(G, k, 0, tb0, gs, ks);  // read-only: in flight during the producer wait
      if (nk4 <= Gm.tb)
        for (int e = tid; e < (nk4 - nk) * k; e += XFER_THREADS) gs[(nk + e / k) * ks + e % k] = 0.0;
      for (int e = tid; e < (nk4 - nk) * rcs; e += XFER_THREADS) ivp[ni * rcs + e] = 0.0;
      SMASH_DASSERT(ni <= Gm.max_nib && k <= Gm.max_rank && d.nc <= 32);
      if (tid < 32 && ((d.wait >> tid) & 1u)) {
#ifdef SMASH_CHECKED
        long long spins = 0;
        while (ld_acquire(&done[d.cf + tid]) == 0u) { __nanosleep(32); SMASH_DASSERT(++spins < (1ll << 26)); }
#else
        while (ld_acquire(&done[d.cf + tid]) == 0u) __nanosleep(32);
#endif
      }
      bar_compute();
      TRACE_SET(t1);
      const double* in = A.qp + (int64_t)d.base * RC;
      for (int j = tid; j < ni; j += XFER_THREADS) row_l2<RC>(ivp + j * rcs, in + (int64_t)j * RC);
      const int NA = (k + 7) >> 3, T = NA * NR;
      const int mt = T > wid ? (T - wid + 7) >> 3 : 0;  // tiles of this warp (<= C)
      int pos[2];  // parent-order rows of this lane's output rows (prefetched)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int t = wid + 8 * i, a = (t / NR) * 8 + g;
        pos[i] = (i < mt && a < k) ? A.up_pos[d.skel + a] : -1;
      }
      cp_commit_wait();
      bar_compute();
      TRACE_SET(t2);
      // this warp's tiles wid, wid + 8 (<= 2; larger T is rejected by the planner)
      double c[2][2][2];
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int h = 0; h < 2; ++h) c[t][h][0] = c[t][h][1] = 0.0;
      const double* ga[2];
      const double* bb[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int tt = min(wid + 8 * t, T - 1);
        ga[t] = gs + q * ks + (tt / NR) * 8 + g;
        bb[t] = ivp + (k + q) * rcs + (tt % NR) * 8 + g;
      }
      for (int cb = 0;;) {
        const int tbc = min(Gm.tb, nk - cb);
        const int steps = (tbc + 3) >> 2;
        const double* bbc[2] = {bb[0] + cb * rcs, bb[1] + cb * rcs};
        if (mt == 2) mma_up<2>(ga, bbc, 4 * ks, 4 * rcs, steps, c);
        else if (mt == 1) mma_up<1>(ga, bbc, 4 * ks, 4 * rcs, steps, c);
        cb += tbc;
        if (cb >= nk) break;
        bar_compute();
        const int tbn = min(Gm.tb, nk - cb);
        stage_g(G, k, cb, tbn, gs, ks);
        if (cb + tbn == nk)
          for (int e = tid; e < (nk4 - nk) * k; e += XFER_THREADS) gs[(tbn + e / k) * ks + e % k] = 0.0;
        cp_commit_wait();
        bar_compute();
      }
      TRACE_SET(t3);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        c[t][0][0] += c[t][1][0];
        c[t][0][1] += c[t][1][1];
      }
      double* out = A.qhat + (int64_t)d.skel * RC;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int t = wid + 8 * i;
        if (i < mt) {
          const int a = (t / NR) * 8 + g, r = (t % NR) * 8 + 2 * q;
          if (a < k) {
            double* o2 = A.qp + (int64_t)pos[i] * RC;
            if (r < RC) {
              const double y = c[i][0][0] + ivp[a * rcs + r];
              out[(int64_t)a * RC + r] = y;
              if (pos[i] >= 0) o2[r] = y;
            }
            if (r + 1 < RC) {
              const double y = c[i][0][1] + ivp[a * rcs + r + 1];
              out[(int64_t)a * RC + r + 1] = y;
              if (pos[i] >= 0) o2[r + 1] = y;
            }
          }
        }
      }
    }
    publish(done, d.v);
    TRACE_EMIT(1, d.v, t0, t1, t2);
    bar_handover();  // the next descriptor is ready
  }
}

// Downward over internal nodes: z_v = zhat_v (coupling) + zd_v (from the
// parent); the children's contributions are written (plain stores, each row
// once) into zd at the children's rows: zd[perm[a]] = z_v[a],
// zd[perm[k + b]] = (G z_v)[b].  Output tiles (b, r) are processed four per
// warp pass (independent DMMA chains).
template <int RC>
__global__ void __launch_bounds__(XFER_THREADS + 32) k_downward(XferArgs A, XferGeom Gm,
                                                                const int* order, int n,
                                                                const unsigned char* inset,
                                                                unsigned* counter, unsigned* done) {
  extern __shared__ __align__(16) double sh[];
  __shared__ NodeDesc s_desc[2];
  const int ks = Gm.ks, rcs = Gm.rcs;
  double* gs = sh;                             // tb x ks
  double* zv = sh + Gm.tb * ks;                 // (max_rank + 16) x rcs
  double* zv2 = zv + (Gm.max_rank + 16) * rcs;  // (max_rank + 16) x rcs  (zd part)
  int* pm = reinterpret_cast<int*>(zv2 + (Gm.max_rank + 16) * rcs);  // max_nib
  const Side rs = A.side;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  constexpr int NR = (RC + 7) / 8;
  if (wid == XFER_THREADS / 32) {
    desc_producer(s_desc, A, order, n, counter, inset, false);
    return;
  }
  bar_handover();
  for (int cur = 0;; cur ^= 1) {
    const NodeDesc d = s_desc[cur];
    if (d.v < 0) break;
    TRACE_DECL;
    const int ni = d.ni, k = d.k;
    const int nk = ni - k, k4 = (k + 3) & ~3;
    if (k > 0) {
      const double* G = rs.G + d.g_off;
      const int* perm = rs.perm + d.ib_off;
      const int tb0 = min(Gm.tb, nk);
      stage_g(G, k, 0, tb0, gs, ks);
      for (int e = tid; e < tb0 * (k4 - k); e += XFER_THREADS) {  // K padding columns
        const int dd = k4 - k;
        gs[(e / dd) * ks + k + e % dd] = 0.0;
      }
      for (int j = tid; j < ni; j += XFER_THREADS) pm[j] = perm[j];
      for (int e = tid; e < (k4 - k) * rcs; e += XFER_THREADS) zv[k * rcs + e] = 0.0;
      const bool from_parent = d.parent > 0;
      SMASH_DASSERT(ni <= Gm.max_nib && k <= Gm.max_rank);
      if (tid == 0 && d.wait)
      {
#ifdef SMASH_CHECKED
        long long spins = 0;
        while (ld_acquire(&done[d.parent]) == 0u) { __nanosleep(32); SMASH_DASSERT(++spins < (1ll << 26)); }
#else
        while (ld_acquire(&done[d.parent]) == 0u) __nanosleep(32);
#endif
      }
      bar_compute();
      TRACE_SET(t1);
      const double* zsrc = A.zhat + (int64_t)d.skel * RC;
      const double* dsrc = A.zd + (int64_t)d.skel * RC;
      for (int a = tid; a < k; a += XFER_THREADS) {
        row_l2<RC>(zv + a * rcs, zsrc + (int64_t)a * RC);
        if (from_parent) row_l2<RC>(zv2 + a * rcs, dsrc + (int64_t)a * RC);
      }
      cp_commit_wait();
      bar_compute();
      if (from_parent) {
        for (int e = tid; e < k * rcs; e += XFER_THREADS) zv[e] += zv2[e];
        bar_compute();
      }
      TRACE_SET(t2);
      double* dst = A.zd + (int64_t)d.base * RC;
      for (int e = tid; e < k * RC; e += XFER_THREADS) {  // identity rows
        const int a = e / RC, r = e - a * RC;
        dst[(int64_t)pm[a] * RC + r] = zv[a * rcs + r];
      }
      const int ksteps = k4 >> 2;
      for (int cb = 0; cb < nk;) {
        const int tbc = min(Gm.tb, nk - cb);
        const int T = ((tbc + 7) >> 3) * NR;
        for (int t0 = wid; t0 < T; t0 += 32) {  // up to four independent tiles per warp pass
          double c[4][2];
          const double* ga[4];
          const double* zb[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            c[i][0] = c[i][1] = 0.0;
            const int t = min(t0 + 8 * i, T - 1);
            ga[i] = gs + ((t / NR) * 8 + g) * ks + q;
            zb[i] = zv + q * rcs + (t % NR) * 8 + g;
          }
          const int nt = min(4, (T - t0 + 7) >> 3);
          switch (nt) {
            case 4: mma_down<4>(ga, zb, 4 * rcs, ksteps, c); break;
            case 3: mma_down<3>(ga, zb, 4 * rcs, ksteps, c); break;
            case 2: mma_down<2>(ga, zb, 4 * rcs, ksteps, c); break;
            default: mma_down<1>(ga, zb, 4 * rcs, ksteps, c); break;
          }
          TRACE_SET(t3);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int t = t0 + 8 * i;
            if (i >= nt) break;
            const int b = (t / NR) * 8 + g, r = (t % NR) * 8 + 2 * q;
            if (b < tbc) {
              double* o = dst + (int64_t)pm[k + cb + b] * RC + r;
              if (r < RC) o[0] = c[i][0];
              if (r + 1 < RC) o[1] = c[i][1];
            }
          }
        }
        cb += tbc;
        if (cb >= nk) break;
        bar_compute();
        const int tbn = min(Gm.tb, nk - cb);
        stage_g(G, k, cb, tbn, gs, ks);
        for (int e = tid; e < tbn * (k4 - k); e += XFER_THREADS) {
          const int dd = k4 - k;
          gs[(e / dd) * ks + k + e % dd] = 0.0;
        }
        cp_commit_wait();
        bar_compute();
      }
    }
    publish(done, d.v);
    TRACE_EMIT(2, d.v, t0, t1, t2);
    bar_handover();
  }
}

// ---------------------------------------------------------------------------
// Leaves: one warp per leaf, every operand loaded straight from global memory
// with no dependent loads (the DMMA A fragments from the read-only G).
// ---------------------------------------------------------------------------

// Leaf upward (leaves have no producers): qhat_v = qt[perm[:k]] + G^T qt[perm[k:]],
// also scattered into the parent's ibar order (qp[up_pos]).
template <int RC>
__global__ void __launch_bounds__(256) k_up_leaves(XferArgs A, const int* leaves, int n) {
  const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (w >= n) return;
  const int v = leaves[w];
  const Side cs = A.side;
  const int k = v == 0 ? 0 : cs.rank[v];  // a root leaf carries no factor
  if (k == 0) return;
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  constexpr int NR = (RC + 7) / 8;
  const int ni = cs.nib[v], nk = ni - k;
  const int* __restrict__ perm = cs.perm + cs.ib_off[v];
  const double* __restrict__ G = cs.G + cs.g_off[v];
  const double* __restrict__ in = A.qt + (int64_t)A.pt_a[v] * RC;
  const int skel = cs.skel_off[v];
  double* __restrict__ out = A.qhat + (int64_t)skel * RC;
  const int* __restrict__ pos = A.up_pos + skel;
  for (int ag = 0; ag < k; ag += 8 * XFER_MAXT) {
    double c[XFER_MAXT][NR][2];
#pragma unroll
    for (int i = 0; i < XFER_MAXT; ++i)
#pragma unroll
      for (int m = 0; m < NR; ++m) c[i][m][0] = c[i][m][1] = 0.0;
#pragma unroll 2
    for (int b0 = 0; b0 < nk; b0 += 4) {
      const int b = b0 + q;
      const bool bv = b < nk;
      const int row = bv ? perm[k + b] : 0;
      double bf[NR];
#pragma unroll
      for (int m = 0; m < NR; ++m)
        bf[m] = (bv && m * 8 + g < RC) ? in[(int64_t)row * RC + m * 8 + g] : 0.0;
#pragma unroll
      for (int i = 0; i < XFER_MAXT; ++i) {
        const int a = ag + i * 8 + g;
        const double af = (bv && a < k) ? __ldg(G + (int64_t)b * k + a) : 0.0;
#pragma unroll
        for (int m = 0; m < NR; ++m) dmma(c[i][m][0], c[i][m][1], af, bf[m]);
      }
    }
    // epilogue: all loads first (identity rows, parent positions), then the stores
    double x[XFER_MAXT][NR][2];
    int pp[XFER_MAXT];
#pragma unroll
    for (int i = 0; i < XFER_MAXT; ++i) {
      const int a = ag + i * 8 + g;
      const int64_t src = a < k ? (int64_t)perm[a] * RC : 0;
      pp[i] = a < k ? pos[a] : -1;
#pragma unroll
      for (int m = 0; m < NR; ++m) {
        const int r = m * 8 + 2 * q;
        x[i][m][0] = (a < k && r < RC) ? in[src + r] : 0.0;
        x[i][m][1] = (a < k && r + 1 < RC) ? in[src + r + 1] : 0.0;
      }
    }
#pragma unroll
    for (int i = 0; i < XFER_MAXT; ++i) {
      const int a = ag + i * 8 + g;
      if (a < k) {
        double* __restrict__ o2 = A.qp + (int64_t)pp[i] * RC;  // -1: the parent is the root
#pragma unroll
        for (int m = 0; m < NR; ++m) {
          const int r = m * 8 + 2 * q;
          const double y0 = c[i][m][0] + x[i][m][0], y1 = c[i][m][1] + x[i][m][1];
          if (r < RC) out[(int64_t)a * RC + r] = y0;
          if (r + 1 < RC) out[(int64_t)a * RC + r + 1] = y1;
          if (pp[i] >= 0) {
            if (r < RC) o2[r] = y0;
            if (r + 1 < RC) o2[r + 1] = y1;
          }
        }
      }
    }
  }
}

// Leaf far field fused with the final combine (after the downward pass and
// the nearfield).  Rows are addressed in the leaf's ibar order a (slot
// ra + a): the nearfield wrote zn in that order and zrow[ra + a] =
// perm_row[ra + perm[a]] is precomputed, so every load is independent:
//   z[zrow[ra + a], c0 + r] = zn[ra + a, r] + (a < k ? z_v[a, r] : (G z_v)[a - k, r]),
// z_v = zhat_v + zd_v.
template <int RC>
__global__ void __launch_bounds__(256) k_down_leaves(XferArgs A, const int* leaves, int n,
                                                     const int* zrow, const double* zn, double* z,
                                                     int64_t ldz, int64_t c0) {
  const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (w >= n) return;
  const int v = leaves[w];
  const Side rs = A.side;
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  constexpr int NR = (RC + 7) / 8;
  const int ra = A.pt_a[v], nr = A.pt_b[v] - ra;
  const int k = v == 0 ? 0 : rs.rank[v];
  const int* __restrict__ zr = zrow + ra;
  const double* __restrict__ zn_v = zn + (int64_t)ra * RC;
  double* __restrict__ zo = z + c0;
  const int skel = k > 0 ? rs.skel_off[v] : 0;
  const bool from_parent = k > 0 && A.parent[v] > 0;
  const double* __restrict__ zh = A.zhat + (int64_t)skel * RC;
  const double* __restrict__ zdv = A.zd + (int64_t)skel * RC;
  // identity rows a < k (or every row without a factor)
#pragma unroll 4
  for (int e = lane; e < (k > 0 ? k : nr) * RC; e += 32) {
    const int a = e / RC, r = e - a * RC;
    double x = zn_v[e];
    if (k > 0) x += from_parent ? zh[e] + zdv[e] : zh[e];
    zo[(int64_t)zr[a] * ldz + r] = x;
  }
  const int nk = nr - k;
  if (k == 0 || nk <= 0) return;
  const double* __restrict__ G = rs.G + rs.g_off[v];
  for (int b0 = 0; b0 < nk; b0 += 16) {  // (G z_v): M = b (two 8-row tiles), N = r, K = a
    double c[2][NR][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int m = 0; m < NR; ++m) c[i][m][0] = c[i][m][1] = 0.0;
#pragma unroll 4
    for (int a0 = 0; a0 < k; a0 += 4) {
      const int a = a0 + q;
      const bool av = a < k;
      double bf[NR];
#pragma unroll
      for (int m = 0; m < NR; ++m) {
        const int64_t e = (int64_t)a * RC + m * 8 + g;
        bf[m] = (av && m * 8 + g < RC) ? (from_parent ? zh[e] + zdv[e] : zh[e]) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int b = b0 + i * 8 + g;
        const double af = (av && b < nk) ? __ldg(G + (int64_t)b * k + a) : 0.0;
#pragma unroll
        for (int m = 0; m < NR; ++m) dmma(c[i][m][0], c[i][m][1], af, bf[m]);
      }
    }
    int64_t zrr[2];
    double x[2][NR][2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int b = b0 + i * 8 + g;
      zrr[i] = b < nk ? (int64_t)zr[k + b] * ldz : -1;
#pragma unroll
      for (int m = 0; m < NR; ++m) {
        const int r = m * 8 + 2 * q;
        x[i][m][0] = (b < nk && r < RC) ? zn_v[(int64_t)(k + b) * RC + r] : 0.0;
        x[i][m][1] = (b < nk && r + 1 < RC) ? zn_v[(int64_t)(k + b) * RC + r + 1] : 0.0;
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      if (zrr[i] < 0) continue;
#pragma unroll
      for (int m = 0; m < NR; ++m) {
        const int r = m * 8 + 2 * q;
        if (r < RC) zo[zrr[i] + r] = x[i][m][0] + c[i][m][0];
        if (r + 1 < RC) zo[zrr[i] + r + 1] = x[i][m][1] + c[i][m][1];
      }
    }
  }
}

int xfer_grid(size_t smem) {
  int dev = 0, nsm = 0;
  SMASH_CUDA(cudaGetDevice(&dev));
  SMASH_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  int per = (int)std::max<size_t>(1, std::min<size_t>(8, (220 * 1024) / (smem + 1024)));
  return nsm * per;
}

}  // namespace

XferGeom xfer_geom(int max_nib, int max_rank, int max_nk, int rc) {
  XferGeom G;
  G.ks = (max_rank + 3) & ~3;
  if (G.ks % 8 == 0) G.ks += 4;  // row stride = 4 (mod 8) doubles: conflict-free fragments
  G.rcs = rc < 8 ? rc : rc + 4;
  static const int kb = getenv("SMASH_XFER_GKB") ? atoi(getenv("SMASH_XFER_GKB")) : 64;
  const int cap = std::max(8, ((kb * 1024) / (G.ks * 8)) & ~7);
  G.tb = std::min(cap, std::max(8, (max_nk + 7) & ~7));
  G.max_nib = max_nib;
  G.max_rank = max_rank;
  return G;
}

// The B-fragment reads of the padded K / N ranges run up to 3 rows + 7 columns
// past the staged rows (their products are zero or discarded): 16 rows of slack.
size_t xfer_smem_up(const XferGeom& G) {
  return ((size_t)G.tb * G.ks + (size_t)(G.max_nib + 16) * G.rcs + 16) * sizeof(double);
}

size_t xfer_smem_down(const XferGeom& G) {
  return ((size_t)G.tb * G.ks + 2 * (size_t)(G.max_rank + 16) * G.rcs + 16) * sizeof(double) +
         (size_t)G.max_nib * sizeof(int);
}

namespace {
__global__ void k_up_pos(Side cs, const int* nchild, const int* child_first, int n, int* up_pos) {
  const int v = blockIdx.x;
  if (v == 0 || v >= n || nchild[v] == 0 || cs.rank[v] == 0) return;
  const int base = cs.skel_off[child_first[v]];
  const int* perm = cs.perm + cs.ib_off[v];
  for (int j = threadIdx.x; j < cs.nib[v]; j += blockDim.x) up_pos[base + perm[j]] = base + j;
}
}  // namespace

void launch_up_pos(const Side& cs, const int* nchild, const int* child_first, int n, int* up_pos,
                   int64_t rows, cudaStream_t s) {
  SMASH_CUDA(cudaMemsetAsync(up_pos, 0xff, std::max<int64_t>(rows, 1) * sizeof(int), s));
  if (n > 1) k_up_pos<<<n, 128, 0, s>>>(cs, nchild, child_first, n, up_pos);
}

template <int RC>
void launch_gather(const double* q, int64_t ldq, const int* perm, int64_t n, int64_t c0,
                   double* qt, cudaStream_t s) {
  const int per = 256 / RC;
  if (n) k_gather<RC><<<cdiv(n, per), per * RC, 0, s>>>(q, ldq, perm, n, c0, qt);
}

template <int RC>
void launch_upward(const XferArgs& a, XferPlan& P, const int* order, int n,
                   const unsigned char* inset, cudaStream_t s) {
  if (!n) return;
  const XferGeom G = xfer_geom(P.max_nib, P.max_rank, P.max_nk, RC);
  const size_t smem = xfer_smem_up(G);
  SMASH_CUDA(cudaFuncSetAttribute(k_upward<RC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SMASH_CUDA(cudaFuncSetAttribute(k_upward<RC>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
  // flags and ticket counter are reset on the stream (graph-replay safe)
  SMASH_CUDA(cudaMemsetAsync(P.counters.p, 0, sizeof(unsigned), s));
  SMASH_CUDA(cudaMemsetAsync(P.done.p, 0, P.done.n * sizeof(unsigned), s));
  const int grid = std::min(n, xfer_grid(smem));
  k_upward<RC><<<grid, XFER_THREADS + 32, smem, s>>>(a, G, order, n, inset, P.counters.p, P.done.p);
}

template <int RC>
void launch_downward(const XferArgs& a, XferPlan& P, const int* order, int n,
                     const unsigned char* inset, cudaStream_t s) {
  if (!n) return;
  const XferGeom G = xfer_geom(P.max_nib, P.max_rank, P.max_nk, RC);
  const size_t smem = xfer_smem_down(G);
  SMASH_CUDA(cudaFuncSetAttribute(k_downward<RC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SMASH_CUDA(cudaFuncSetAttribute(k_downward<RC>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
  SMASH_CUDA(cudaMemsetAsync(P.counters.p + 1, 0, sizeof(unsigned), s));
  SMASH_CUDA(cudaMemsetAsync(P.done.p, 0, P.done.n * sizeof(unsigned), s));
  const int grid = std::min(n, xfer_grid(smem));
  k_downward<RC><<<grid, XFER_THREADS + 32, smem, s>>>(a, G, order, n, inset, P.counters.p + 1,
                                                  P.done.p);
}

template <int RC>
void launch_up_leaves(const XferArgs& a, const int* leaves, int n, cudaStream_t s) {
  if (n) k_up_leaves<RC><<<cdiv((int64_t)n * 32, 256), 256, 0, s>>>(a, leaves, n);
}

template <int RC>
void launch_down_leaves(const XferArgs& a, const int* leaves, int n, const int* zrow,
                        const double* zn, double* z, int64_t ldz, int64_t c0, cudaStream_t s) {
  if (n)
    k_down_leaves<RC><<<cdiv((int64_t)n * 32, 256), 256, 0, s>>>(a, leaves, n, zrow, zn, z, ldz,
                                                                 c0);
}

namespace {
// Within-leaf ibar order of the row side: slot_of[ra + perm[a]] = ra + a and
// zrow[ra + a] = perm_row[ra + perm[a]] (identity for a leaf without factor).
__global__ void k_leaf_slots(Side rs, const int* leaves, int n, const int* row_a, const int* row_b,
                             const int* perm_row, int* slot_of, int* zrow) {
  const int li = blockIdx.x;
  if (li >= n) return;
  const int v = leaves[li];
  const int ra = row_a[v], nr = row_b[v] - ra;
  const bool fac = v != 0 && rs.rank[v] > 0;
  const int* perm = rs.perm + rs.ib_off[v];
  for (int a = threadIdx.x; a < nr; a += blockDim.x) {
    const int p = ra + (fac ? perm[a] : a);
    slot_of[p] = ra + a;
    zrow[ra + a] = perm_row[p];
  }
}
}  // namespace

void launch_leaf_slots(const Side& rs, const int* leaves, int n, const int* row_a, const int* row_b,
                       const int* perm_row, int* slot_of, int* zrow, cudaStream_t s) {
  if (n) k_leaf_slots<<<n, 64, 0, s>>>(rs, leaves, n, row_a, row_b, perm_row, slot_of, zrow);
}

#define SMASH_XFER_INSTANTIATE(RC)                                                              \
  template void launch_gather<RC>(const double*, int64_t, const int*, int64_t, int64_t, double*, \
                                  cudaStream_t);                                               \
  template void launch_upward<RC>(const XferArgs&, XferPlan&, const int*, int,                  \
                                  const unsigned char*, cudaStream_t);                          \
  template void launch_downward<RC>(const XferArgs&, XferPlan&, const int*, int,                \
                                    const unsigned char*, cudaStream_t);                        \
  template void launch_up_leaves<RC>(const XferArgs&, const int*, int, cudaStream_t);           \
  template void launch_down_leaves<RC>(const XferArgs&, const int*, int, const int*,            \
                                       const double*, double*, int64_t, int64_t, cudaStream_t);
SMASH_XFER_INSTANTIATE(1)
SMASH_XFER_INSTANTIATE(2)
SMASH_XFER_INSTANTIATE(4)
SMASH_XFER_INSTANTIATE(8)
SMASH_XFER_INSTANTIATE(16)

}  // namespace mv
}  // namespace smash

#ifdef SMASH_XFER_TRACE
extern "C" int smash_debug_xfer_trace(unsigned long long* out, int max_items, int reset) {
  unsigned n = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&n, smash::mv::g_trace_n, sizeof(unsigned));
  n = std::min<unsigned>(n, std::min<unsigned>((unsigned)max_items, (1u << 20) / 8));
  if (n) cudaMemcpyFromSymbol(out, smash::mv::g_trace, n * 8 * sizeof(unsigned long long));
  if (reset) {
    unsigned z = 0;
    cudaMemcpyToSymbol(smash::mv::g_trace_n, &z, sizeof(unsigned));
  }
  return (int)n;
}
#endif
