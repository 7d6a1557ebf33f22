// K6 / K8 / K10: permutation gather, upward and downward transfer passes and
// the leaf far-field epilogue of the matvec (smash/apply.py:39-53, 60-72, 78-80).
//
// The transfer passes are level-ordered dataflow: a node's upward projection
// needs its children's, its downward step needs its parent's.  Instead of one
// launch per level (the small top levels are pure latency), each pass is ONE
// persistent launch: CTAs take node tickets from an atomic counter in level
// order (deepest first upward, shallowest first downward) and spin on the
// producers' epoch flags, which were necessarily handed out earlier to CTAs
// that are already running -- so the wait cannot deadlock.  Cross-CTA data is
// published with __threadfence() + a release flag and read with __ldcg (L2).
// X_v = P [I; G] is applied implicitly; G row tiles are staged in shared memory
// with batched loads.
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

__device__ __forceinline__ int g_tile_rows(int ks) { return max(1, min(64, 4096 / ks)); }

__device__ __forceinline__ int next_ticket(unsigned* counter) {
  __shared__ int s_t;
  __syncthreads();
  if (threadIdx.x == 0) s_t = (int)atomicAdd(counter, 1u);
  __syncthreads();
  return s_t;
}

__device__ __forceinline__ void publish(unsigned* done, int v, unsigned epoch) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) st_release(&done[v], epoch);
}

// qhat[v] = ivec[perm[:k]] + G^T ivec[perm[k:]]
template <int RC>
__global__ void __launch_bounds__(XFER_THREADS) k_upward(XferArgs A, const int* order, int n,
                                                         const unsigned char* inset,
                                                         unsigned* counter, unsigned* done,
                                                         unsigned epoch) {
  extern __shared__ double sh[];
  const Side cs = A.side;
  for (;;) {
    const int tk = next_ticket(counter);
    if (tk >= n) break;
    const int v = order[tk];
    const int nc = A.nchild[v];
    if (threadIdx.x < nc) {
      const int c = A.child_first[v] + threadIdx.x;
      if (inset[c])  // producers outside this launch are final already (sharded stages)
        while (ld_acquire(&done[c]) != epoch) __nanosleep(40);
    }
    __syncthreads();
    const int ni = cs.nib[v], k = cs.rank[v];
    if (k > 0) {
      const bool leaf = nc == 0;
      const double* ivec = leaf ? A.qt + (int64_t)A.pt_a[v] * RC
                                : A.qhat + (int64_t)cs.skel_off[A.child_first[v]] * RC;
      const int* perm = cs.perm + cs.ib_off[v];
      double* iv = sh;           // ni * RC
      double* gs = sh + ni * RC;  // TB * k
      stage_block<8>(ni * RC,
                     [&](int e) { return __ldcg(ivec + (int64_t)perm[e / RC] * RC + e % RC); },
                     [&](int e, double x) { iv[e] = x; });
      __syncthreads();
      const int nout = k * RC;
      double acc[XFER_MAXO];
#pragma unroll
      for (int j = 0; j < XFER_MAXO; ++j) {
        const int e = threadIdx.x + j * blockDim.x;
        acc[j] = e < nout ? iv[e] : 0.0;
      }
      const double* G = cs.G + cs.g_off[v];
      const int nk = ni - k;
      const int TB = g_tile_rows(k);
      for (int b0 = 0; b0 < nk; b0 += TB) {
        const int tb = min(TB, nk - b0);
        const double* src = G + (int64_t)b0 * k;
        stage_block<16>(tb * k, [&](int e) { return src[e]; }, [&](int e, double x) { gs[e] = x; });
        __syncthreads();
#pragma unroll
        for (int j = 0; j < XFER_MAXO; ++j) {
          const int e = threadIdx.x + j * blockDim.x;
          if (e < nout) {
            const int a = e / RC, r = e % RC;
            double t = acc[j];
            const double* ivb = iv + (k + b0) * RC + r;
            for (int bb = 0; bb < tb; ++bb) t = fma(gs[bb * k + a], ivb[bb * RC], t);
            acc[j] = t;
          }
        }
        __syncthreads();
      }
      double* out = A.qhat + (int64_t)cs.skel_off[v] * RC;
#pragma unroll
      for (int j = 0; j < XFER_MAXO; ++j) {
        const int e = threadIdx.x + j * blockDim.x;
        if (e < nout) out[e] = acc[j];
      }
    }
    publish(done, v, epoch);
  }
}

// zhat[children] += X_v zhat[v] (internal non-root nodes, after the coupling)
template <int RC>
__global__ void __launch_bounds__(XFER_THREADS) k_downward(XferArgs A, const int* order, int n,
                                                           const unsigned char* inset,
                                                           unsigned* counter, unsigned* done,
                                                           unsigned epoch, int root) {
  extern __shared__ double sh[];
  const Side rs = A.side;
  for (;;) {
    const int tk = next_ticket(counter);
    if (tk >= n) break;
    const int v = order[tk];
    const int p = A.parent[v];
    if (threadIdx.x == 0 && p != root && inset[p])
      while (ld_acquire(&done[p]) != epoch) __nanosleep(40);
    __syncthreads();
    const int ni = rs.nib[v], k = rs.rank[v];
    if (k > 0 && ni > 0) {
      const int ks = k | 1;
      double* zv = sh;           // k * RC
      double* gs = sh + k * RC;  // TB * ks
      const int* perm = rs.perm + rs.ib_off[v];
      const double* zsrc = A.zhat + (int64_t)rs.skel_off[v] * RC;
      double* dst = A.zhat + (int64_t)rs.skel_off[A.child_first[v]] * RC;
      for (int e = threadIdx.x; e < k * RC; e += blockDim.x) {
        const double x = __ldcg(zsrc + e);
        zv[e] = x;
        const int a = e / RC, r = e % RC;
        double* d = dst + (int64_t)perm[a] * RC + r;
        *d = __ldcg(d) + x;
      }
      const double* G = rs.G + rs.g_off[v];
      const int nk = ni - k;
      const int TB = g_tile_rows(ks);
      for (int b0 = 0; b0 < nk; b0 += TB) {
        const int tb = min(TB, nk - b0);
        const double* src = G + (int64_t)b0 * k;
        __syncthreads();
        stage_block<16>(tb * k, [&](int e) { return src[e]; },
                        [&](int e, double x) { gs[(e / k) * ks + e % k] = x; });
        __syncthreads();
        for (int e = threadIdx.x; e < tb * RC; e += blockDim.x) {
          const int bb = e / RC, r = e % RC;
          const double* g = gs + bb * ks;
          double y0 = 0.0, y1 = 0.0;
          int a = 0;
          for (; a + 1 < k; a += 2) {
            y0 = fma(g[a], zv[a * RC + r], y0);
            y1 = fma(g[a + 1], zv[(a + 1) * RC + r], y1);
          }
          if (a < k) y0 = fma(g[a], zv[a * RC + r], y0);
          double* d = dst + (int64_t)perm[k + b0 + bb] * RC + r;
          *d = __ldcg(d) + (y0 + y1);
        }
      }
    }
    publish(done, v, epoch);
  }
}

// z[perm_row[p]] += (X_v zhat_v)[p] for the rows of every non-root leaf
template <int RC>
__global__ void __launch_bounds__(XFER_THREADS) k_leaf_add(XferArgs A, const int* leaves,
                                                           int n_leaves, const int* row_a,
                                                           const int* row_b, const int* perm_row,
                                                           double* z, int64_t ldz, int64_t c0,
                                                           int root) {
  extern __shared__ double sh[];
  const int li = blockIdx.x;
  if (li >= n_leaves) return;
  const int v = leaves[li];
  if (v == root) return;
  const Side rs = A.side;
  const int k = rs.rank[v];
  if (k == 0) return;
  const int ra = row_a[v], nr = row_b[v] - ra;
  double* zv = sh;
  int* inv = reinterpret_cast<int*>(sh + k * RC);
  const int* perm = rs.perm + rs.ib_off[v];
  const double* zsrc = A.zhat + (int64_t)rs.skel_off[v] * RC;
  for (int c = threadIdx.x; c < nr; c += blockDim.x) inv[perm[c]] = c;
  for (int e = threadIdx.x; e < k * RC; e += blockDim.x) zv[e] = zsrc[e];
  __syncthreads();
  const double* G = rs.G + rs.g_off[v];
  for (int e = threadIdx.x; e < nr * RC; e += blockDim.x) {
    const int t = e / RC, r = e % RC;
    const int pos = inv[t];
    double y;
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
    double* zo = z + (int64_t)perm_row[ra + t] * ldz + c0 + r;
    *zo += y;
  }
}

int xfer_grid(size_t smem) {
  int dev = 0, nsm = 0;
  SMASH_CUDA(cudaGetDevice(&dev));
  SMASH_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  int per = (int)std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / (smem + 2048)));
  return nsm * per;
}

}  // namespace

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
  const size_t smem = ((size_t)P.max_nib * RC + 4096) * sizeof(double);
  SMASH_CUDA(cudaFuncSetAttribute(k_upward<RC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SMASH_CUDA(cudaMemsetAsync(P.counters.p, 0, sizeof(unsigned), s));
  const int grid = std::min(n, xfer_grid(smem));
  k_upward<RC><<<grid, XFER_THREADS, smem, s>>>(a, order, n, inset, P.counters.p, P.done.p,
                                                P.epoch);
}

template <int RC>
void launch_downward(const XferArgs& a, XferPlan& P, const int* order, int n,
                     const unsigned char* inset, cudaStream_t s) {
  if (!n) return;
  const size_t smem = ((size_t)P.max_rank * RC + 4096 + 64) * sizeof(double);
  SMASH_CUDA(cudaFuncSetAttribute(k_downward<RC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SMASH_CUDA(cudaMemsetAsync(P.counters.p + 1, 0, sizeof(unsigned), s));
  const int grid = std::min(n, xfer_grid(smem));
  k_downward<RC><<<grid, XFER_THREADS, smem, s>>>(a, order, n, inset, P.counters.p + 1, P.done.p,
                                                  P.epoch, 0);
}

template <int RC>
void launch_leaf_add(const XferArgs& a, const XferPlan& P, const int* leaves, int n_leaves,
                     const int* row_a, const int* row_b, const int* perm_row, double* z,
                     int64_t ldz, int64_t c0, int nu0, cudaStream_t s) {
  if (!n_leaves) return;
  const size_t smem = (size_t)P.max_rank * RC * sizeof(double) + (size_t)(nu0 + 1) * sizeof(int);
  SMASH_CUDA(cudaFuncSetAttribute(k_leaf_add<RC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_leaf_add<RC><<<n_leaves, XFER_THREADS, smem, s>>>(a, leaves, n_leaves, row_a, row_b, perm_row,
                                                      z, ldz, c0, 0);
}

#define SMASH_XFER_INSTANTIATE(RC)                                                              \
  template void launch_gather<RC>(const double*, int64_t, const int*, int64_t, int64_t, double*, \
                                  cudaStream_t);                                               \
  template void launch_upward<RC>(const XferArgs&, XferPlan&, const int*, int,                  \
                                  const unsigned char*, cudaStream_t);                          \
  template void launch_downward<RC>(const XferArgs&, XferPlan&, const int*, int,                \
                                    const unsigned char*, cudaStream_t);                        \
  template void launch_leaf_add<RC>(const XferArgs&, const XferPlan&, const int*, int,          \
                                    const int*, const int*, const int*, double*, int64_t,       \
                                    int64_t, int, cudaStream_t);
SMASH_XFER_INSTANTIATE(1)
SMASH_XFER_INSTANTIATE(2)
SMASH_XFER_INSTANTIATE(4)
SMASH_XFER_INSTANTIATE(8)
SMASH_XFER_INSTANTIATE(16)

}  // namespace mv
}  // namespace smash
