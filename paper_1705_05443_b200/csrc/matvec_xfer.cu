// K6 / K8 / K10: permutation gather, upward and downward transfer passes and
// the final far + near combine of the matvec (smash/apply.py:39-53, 60-72, 78-80).
//
// The transfer passes are level-ordered dataflow: a node's upward projection
// needs its children's, its downward step needs its parent's.  Each pass is ONE
// persistent launch over all its nodes (leaves included): CTAs take node
// tickets from an atomic counter in level order (deepest first upward,
// shallowest first downward) and spin on the producers' done flags, which were
// necessarily handed out earlier to CTAs that are already running -- so the
// wait cannot deadlock.  Cross-CTA data is published with __threadfence() + a
// release flag and read through L2 (cp.async.cg / ld.cg).
//
// Per node the work is a small GEMM with the interpolative factor
// X_v = P [I; G] (G: (|ibar| - k) x k row-major):
//   upward    qhat_v          = in[perm[:k]] + G^T in[perm[k:]]    (in: children's
//                                coefficients, or the leaf's qt rows)
//   downward  out[perm[:k]]  += zhat_v,  out[perm[k:]] += G zhat_v (out: children's
//                                zhat, or the leaf's far-field rows zf)
// G and the permutation are read-only, so their cp.async staging is issued
// before the producer wait; the producer rows follow in one more asynchronous
// batch.  The GEMM runs on the FP64 tensor cores (mma.sync m8n8k4 DMMA) with
// operands read from shared memory at bank-conflict-free strides (row strides
// = 4 mod 8 doubles), one 8x8 output tile per warp and item.
#include "matvec_impl.cuh"

namespace smash {
namespace mv {

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

// Read-only G rows [r0, r0 + nr) (row length k) -> shared rows of stride ks.
__device__ __forceinline__ void stage_g(const double* G, int k, int r0, int nr, double* gs, int ks) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int row = wid; row < nr; row += nw) {
    const double* src = G + (int64_t)(r0 + row) * k;
    for (int c = lane; c < k; c += 32) cp_async8(gs + row * ks + c, src + c);
  }
}

__device__ __forceinline__ void publish(unsigned* done, int v) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) st_release(&done[v], 1u);
}

// qhat_v = in[perm[:k]] + G^T in[perm[k:]] for every node of `order`.
template <int RC>
__global__ void __launch_bounds__(XFER_THREADS) k_upward(XferArgs A, XferGeom Gm, const int* order,
                                                         int n, const unsigned char* inset,
                                                         unsigned* counter, unsigned* done) {
  extern __shared__ __align__(16) double sh[];
  __shared__ int s_tk;
  const int ks = Gm.ks, rcs = Gm.rcs;
  double* gs = sh;                        // tb x ks   (G chunk)
  double* ivp = sh + Gm.tb * ks;          // (max_nib + 8) x rcs (permuted ibar rows)
  const Side cs = A.side;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  constexpr int NR = (RC + 7) / 8;
  if (tid == 0) s_tk = (int)atomicAdd(counter, 1u);
  __syncthreads();
  int tk = s_tk;
  while (tk < n) {
    const int v = order[tk];
    __syncthreads();  // s_tk consumed; the previous node's shared memory is free
    if (tid == 0) s_tk = (int)atomicAdd(counter, 1u);  // prefetch the next ticket
    const int ni = cs.nib[v], k = cs.rank[v], nc = A.nchild[v];
    const int nk = ni - k, nk4 = (nk + 3) & ~3;
    if (k > 0) {
      const double* G = cs.G + cs.g_off[v];
      const int* perm = cs.perm + cs.ib_off[v];
      const double* in = nc == 0 ? A.qt + (int64_t)A.pt_a[v] * RC
                                 : A.qhat + (int64_t)cs.skel_off[A.child_first[v]] * RC;
      const int tb0 = min(Gm.tb, nk);
      stage_g(G, k, 0, tb0, gs, ks);  // read-only: in flight during the producer wait
      for (int e = tid; e < (nk4 - nk) * k; e += blockDim.x) {  // K padding rows (nk <= tb)
        if (nk4 <= Gm.tb) gs[(nk + e / k) * ks + e % k] = 0.0;
      }
      for (int e = tid; e < (nk4 - nk) * rcs; e += blockDim.x) ivp[ni * rcs + e] = 0.0;
      if (tid < nc) {
        const int c = A.child_first[v] + tid;
        if (inset[c])  // producers outside this launch are final already
          while (ld_acquire(&done[c]) == 0u) __nanosleep(32);
      }
      __syncthreads();
      for (int j = tid; j < ni; j += blockDim.x) row_l2<RC>(ivp + j * rcs, in + (int64_t)perm[j] * RC);
      cp_commit_wait();
      __syncthreads();
      const int NA = (k + 7) >> 3, T = NA * NR;
      double c[XFER_MAXT][2];
#pragma unroll
      for (int i = 0; i < XFER_MAXT; ++i) c[i][0] = c[i][1] = 0.0;
      for (int cb = 0;;) {
        const int tbc = min(Gm.tb, nk - cb);
        const int steps = (tbc + 3) >> 2;
#pragma unroll
        for (int i = 0; i < XFER_MAXT; ++i) {
          const int t = wid + 8 * i;
          if (t < T) {
            const int a0 = (t / NR) * 8, r0 = (t % NR) * 8;
            const double* ga = gs + q * ks + a0 + g;
            const double* bb = ivp + (k + cb + q) * rcs + r0 + g;
#pragma unroll 4
            for (int s = 0; s < steps; ++s) dmma(c[i][0], c[i][1], ga[s * 4 * ks], bb[s * 4 * rcs]);
          }
        }
        cb += tbc;
        if (cb >= nk) break;
        __syncthreads();
        const int tbn = min(Gm.tb, nk - cb);
        stage_g(G, k, cb, tbn, gs, ks);
        for (int e = tid; e < (nk4 - nk) * k; e += blockDim.x)
          if (cb + tbn == nk && tbn + (nk4 - nk) <= Gm.tb) gs[(tbn + e / k) * ks + e % k] = 0.0;
        cp_commit_wait();
        __syncthreads();
      }
      double* out = A.qhat + (int64_t)cs.skel_off[v] * RC;
#pragma unroll
      for (int i = 0; i < XFER_MAXT; ++i) {
        const int t = wid + 8 * i;
        if (t < T) {
          const int a = (t / NR) * 8 + g, r = (t % NR) * 8 + 2 * q;
          if (a < k) {
            if (r < RC) out[(int64_t)a * RC + r] = c[i][0] + ivp[a * rcs + r];
            if (r + 1 < RC) out[(int64_t)a * RC + r + 1] = c[i][1] + ivp[a * rcs + r + 1];
          }
        }
      }
    }
    publish(done, v);
    tk = s_tk;
  }
}

// Downward: for internal nodes out = the children's zhat block (read-modify-
// write), for leaves out = the leaf's rows of the far-field buffer zf (store).
template <int RC>
__global__ void __launch_bounds__(XFER_THREADS) k_downward(XferArgs A, XferGeom Gm,
                                                           const int* order, int n,
                                                           const unsigned char* inset,
                                                           unsigned* counter, unsigned* done,
                                                           double* zf) {
  extern __shared__ __align__(16) double sh[];
  __shared__ int s_tk;
  const int ks = Gm.ks, rcs = Gm.rcs;
  double* gs = sh;                             // tb x ks
  double* zv = sh + Gm.tb * ks;                // (max_rank + 8) x rcs
  int* pm = reinterpret_cast<int*>(zv + (Gm.max_rank + 8) * rcs);  // max_nib
  const Side rs = A.side;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  constexpr int NR = (RC + 7) / 8;
  if (tid == 0) s_tk = (int)atomicAdd(counter, 1u);
  __syncthreads();
  int tk = s_tk;
  while (tk < n) {
    const int v = order[tk];
    __syncthreads();
    if (tid == 0) s_tk = (int)atomicAdd(counter, 1u);
    const int ni = rs.nib[v], k = rs.rank[v], nc = A.nchild[v];
    const bool leaf = nc == 0;
    const int nk = ni - k, k4 = (k + 3) & ~3;
    if (k == 0) {
      if (leaf) {  // no factor (a root leaf): the far field is zero
        const int ra = A.pt_a[v], nr = A.pt_b[v] - ra;
        for (int e = tid; e < nr * RC; e += blockDim.x) zf[(int64_t)ra * RC + e] = 0.0;
      }
    } else {
      const double* G = rs.G + rs.g_off[v];
      const int* perm = rs.perm + rs.ib_off[v];
      const int tb0 = min(Gm.tb, nk);
      stage_g(G, k, 0, tb0, gs, ks);
      for (int e = tid; e < tb0 * (k4 - k); e += blockDim.x) {  // K padding columns
        const int d = k4 - k;
        gs[(e / d) * ks + k + e % d] = 0.0;
      }
      for (int j = tid; j < ni; j += blockDim.x) pm[j] = perm[j];
      for (int e = tid; e < (k4 - k) * rcs; e += blockDim.x) zv[k * rcs + e] = 0.0;
      const int p = A.parent[v];
      if (tid == 0 && p > 0 && inset[p])
        while (ld_acquire(&done[p]) == 0u) __nanosleep(32);
      __syncthreads();
      const double* zsrc = A.zhat + (int64_t)rs.skel_off[v] * RC;
      for (int a = tid; a < k; a += blockDim.x) row_l2<RC>(zv + a * rcs, zsrc + (int64_t)a * RC);
      cp_commit_wait();
      __syncthreads();
      double* dst = leaf ? zf + (int64_t)A.pt_a[v] * RC
                         : A.zhat + (int64_t)rs.skel_off[A.child_first[v]] * RC;
      // identity rows: out[perm[a]] (+)= zhat_v[a]
      for (int e = tid; e < k * RC; e += blockDim.x) {
        const int a = e / RC, r = e - a * RC;
        double* d = dst + (int64_t)pm[a] * RC + r;
        const double x = zv[a * rcs + r];
        *d = leaf ? x : __ldcg(d) + x;
      }
      const int ksteps = k4 >> 2;
      for (int cb = 0; cb < nk;) {
        const int tbc = min(Gm.tb, nk - cb);
        const int T = ((tbc + 7) >> 3) * NR;
        for (int t0 = wid; t0 < T; t0 += 16) {  // two independent tiles per warp pass
          double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
          const int t1 = t0 + 8;
          const int b00 = (t0 / NR) * 8, r00 = (t0 % NR) * 8;
          const int b01 = (t1 / NR) * 8, r01 = (t1 % NR) * 8;
          const double* ga0 = gs + (b00 + g) * ks + q;
          const double* ga1 = gs + (b01 + g) * ks + q;
          const double* zb0 = zv + q * rcs + r00 + g;
          const double* zb1 = zv + q * rcs + r01 + g;
          if (t1 < T) {
#pragma unroll 4
            for (int s = 0; s < ksteps; ++s) {
              dmma(c[0][0], c[0][1], ga0[4 * s], zb0[4 * s * rcs]);
              dmma(c[1][0], c[1][1], ga1[4 * s], zb1[4 * s * rcs]);
            }
          } else {
#pragma unroll 4
            for (int s = 0; s < ksteps; ++s) dmma(c[0][0], c[0][1], ga0[4 * s], zb0[4 * s * rcs]);
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int t = i ? t1 : t0;
            if (t >= T) break;
            const int b = (t / NR) * 8 + g, r = (t % NR) * 8 + 2 * q;
            if (b < tbc) {
              double* d = dst + (int64_t)pm[k + cb + b] * RC + r;
              if (leaf) {
                if (r < RC) d[0] = c[i][0];
                if (r + 1 < RC) d[1] = c[i][1];
              } else {
                if (r < RC) d[0] = __ldcg(d) + c[i][0];
                if (r + 1 < RC) d[1] = __ldcg(d + 1) + c[i][1];
              }
            }
          }
        }
        cb += tbc;
        if (cb >= nk) break;
        __syncthreads();
        const int tbn = min(Gm.tb, nk - cb);
        stage_g(G, k, cb, tbn, gs, ks);
        for (int e = tid; e < tbn * (k4 - k); e += blockDim.x) {
          const int d = k4 - k;
          gs[(e / d) * ks + k + e % d] = 0.0;
        }
        cp_commit_wait();
        __syncthreads();
      }
    }
    if (!leaf) publish(done, v);  // (no consumer waits on a leaf)
    else __syncthreads();          // s_tk written by thread 0 above
    tk = s_tk;
  }
}

// z[perm_row[p], c0 + r] = zn[p, r] + zf[p, r] for the rows of the listed leaves
// (one warp per leaf).
template <int RC>
__global__ void k_combine(const int* leaves, int n_leaves, const int* row_a, const int* row_b,
                          const int* perm_row, const double* zn, const double* zf, double* z,
                          int64_t ldz, int64_t c0) {
  const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= n_leaves) return;
  const int v = leaves[w];
  const int ra = row_a[v], nr = row_b[v] - ra;
  for (int e = lane; e < nr * RC; e += 32) {
    const int t = e / RC, r = e - t * RC;
    const int64_t p = ra + t;
    z[(int64_t)perm_row[p] * ldz + c0 + r] = zn[p * RC + r] + zf[p * RC + r];
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
  const int cap = std::max(8, ((64 * 1024) / (G.ks * 8)) & ~7);
  G.tb = std::min(cap, std::max(8, (max_nk + 7) & ~7));
  G.max_nib = max_nib;
  G.max_rank = max_rank;
  return G;
}

size_t xfer_smem_up(const XferGeom& G) {
  return ((size_t)G.tb * G.ks + (size_t)(G.max_nib + 8) * G.rcs) * sizeof(double);
}

size_t xfer_smem_down(const XferGeom& G) {
  return ((size_t)G.tb * G.ks + (size_t)(G.max_rank + 8) * G.rcs) * sizeof(double) +
         (size_t)G.max_nib * sizeof(int);
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
  // flags and ticket counter are reset on the stream (graph-replay safe)
  SMASH_CUDA(cudaMemsetAsync(P.counters.p, 0, sizeof(unsigned), s));
  SMASH_CUDA(cudaMemsetAsync(P.done.p, 0, P.done.n * sizeof(unsigned), s));
  const int grid = std::min(n, xfer_grid(smem));
  k_upward<RC><<<grid, XFER_THREADS, smem, s>>>(a, G, order, n, inset, P.counters.p, P.done.p);
}

template <int RC>
void launch_downward(const XferArgs& a, XferPlan& P, const int* order, int n,
                     const unsigned char* inset, double* zf, cudaStream_t s) {
  if (!n) return;
  const XferGeom G = xfer_geom(P.max_nib, P.max_rank, P.max_nk, RC);
  const size_t smem = xfer_smem_down(G);
  SMASH_CUDA(cudaFuncSetAttribute(k_downward<RC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SMASH_CUDA(cudaMemsetAsync(P.counters.p + 1, 0, sizeof(unsigned), s));
  SMASH_CUDA(cudaMemsetAsync(P.done.p, 0, P.done.n * sizeof(unsigned), s));
  const int grid = std::min(n, xfer_grid(smem));
  k_downward<RC><<<grid, XFER_THREADS, smem, s>>>(a, G, order, n, inset, P.counters.p + 1,
                                                  P.done.p, zf);
}

template <int RC>
void launch_combine(const int* leaves, int n_leaves, const int* row_a, const int* row_b,
                    const int* perm_row, const double* zn, const double* zf, double* z,
                    int64_t ldz, int64_t c0, cudaStream_t s) {
  if (!n_leaves) return;
  k_combine<RC><<<cdiv((int64_t)n_leaves * 32, 256), 256, 0, s>>>(leaves, n_leaves, row_a, row_b,
                                                                  perm_row, zn, zf, z, ldz, c0);
}

#define SMASH_XFER_INSTANTIATE(RC)                                                              \
  template void launch_gather<RC>(const double*, int64_t, const int*, int64_t, int64_t, double*, \
                                  cudaStream_t);                                               \
  template void launch_upward<RC>(const XferArgs&, XferPlan&, const int*, int,                  \
                                  const unsigned char*, cudaStream_t);                          \
  template void launch_downward<RC>(const XferArgs&, XferPlan&, const int*, int,                \
                                    const unsigned char*, double*, cudaStream_t);               \
  template void launch_combine<RC>(const int*, int, const int*, const int*, const int*,         \
                                   const double*, const double*, double*, int64_t, int64_t,     \
                                   cudaStream_t);
SMASH_XFER_INSTANTIATE(1)
SMASH_XFER_INSTANTIATE(2)
SMASH_XFER_INSTANTIATE(4)
SMASH_XFER_INSTANTIATE(8)
SMASH_XFER_INSTANTIATE(16)

}  // namespace mv
}  // namespace smash
