// K6 / K8 / K10: permutation gather, upward and downward transfer passes and
// the leaf far-field epilogue of the matvec (smash/apply.py:39-53, 60-72, 78-80).
//
// The transfer passes are level-ordered dataflow: a node's upward projection
// needs its children's, its downward step needs its parent's.  Instead of one
// launch per level (the small top levels are pure latency), each pass is ONE
// persistent launch: CTAs take node tickets from an atomic counter in level
// order (deepest first upward, shallowest first downward) and spin on the
// producers' done flags, which were necessarily handed out earlier to CTAs
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
// The node's ibar-vector is ONE contiguous block (leaf: its qt rows; internal:
// its children's coefficient rows), so it is staged in the same batched load as
// the permutation and the first G tile: one memory round trip per node.
template <int RC>
__device__ __forceinline__ void up_node(const XferArgs& A, int v, double* sh) {
  const Side& cs = A.side;
  const int nc = A.nchild[v];
    const int ni = cs.nib[v], k = cs.rank[v];
    if (k > 0) {
      const bool leaf = nc == 0;
      const double* ivec = leaf ? A.qt + (int64_t)A.pt_a[v] * RC
                                : A.qhat + (int64_t)cs.skel_off[A.child_first[v]] * RC;
      const int* perm = cs.perm + cs.ib_off[v];
      const double* G = cs.G + cs.g_off[v];
      const int nk = ni - k;
      const int TB = g_tile_rows(k);
      double* iv = sh;                 // ni * RC, unpermuted
      double* pm = iv + ni * RC;       // ni permutation entries (as doubles)
      double* gs = pm + ni;            // TB * k
      const int n_iv = ni * RC, n_g0 = min(TB, nk) * k;
      stage_block<16>(n_iv + ni + n_g0,
                      [&](int e) {
                        return e < n_iv ? __ldcg(ivec + e)
                                        : e < n_iv + ni ? (double)perm[e - n_iv]
                                                        : G[e - n_iv - ni];
                      },
                      [&](int e, double x) { iv[e] = x; });
      __syncthreads();
      // gather the permuted ibar rows once: ivp[c] = iv[perm[c]] (after gs, reusing pm's slot
      // would alias; ivp lives after the G tile)
      double* ivp = gs + TB * k;
      for (int e = threadIdx.x; e < ni * RC; e += blockDim.x)
        ivp[e] = iv[(int)pm[e / RC] * RC + e % RC];
      __syncthreads();
      // register tile: TA rows (a) x TR columns (r) per thread
      constexpr int TR = RC < 4 ? RC : 4;
      constexpr int TA = 2;
      const int na = (k + TA - 1) / TA, nrq = RC / TR;
      const int items = na * nrq;
      for (int it0 = 0; it0 < items; it0 += blockDim.x) {
        const int it = it0 + threadIdx.x;
        const bool ok = it < items;
        const int a0 = ok ? (it / nrq) * TA : 0, r0 = ok ? (it % nrq) * TR : 0;
        double acc[TA][TR];
#pragma unroll
        for (int i = 0; i < TA; ++i)
#pragma unroll
          for (int j = 0; j < TR; ++j)
            acc[i][j] = (ok && a0 + i < k) ? ivp[(a0 + i) * RC + r0 + j] : 0.0;
        for (int b0 = 0; b0 < nk; b0 += TB) {
          const int tb = min(TB, nk - b0);
          if (b0 > 0) {
            __syncthreads();
            const double* src = G + (int64_t)b0 * k;
            stage_block<16>(tb * k, [&](int e) { return src[e]; }, [&](int e, double x) { gs[e] = x; });
            __syncthreads();
          }
          if (ok) {
            const double* wb = ivp + (k + b0) * RC + r0;
            for (int bb = 0; bb < tb; ++bb) {
              double g[TA], w[TR];
#pragma unroll
              for (int i = 0; i < TA; ++i) g[i] = a0 + i < k ? gs[bb * k + a0 + i] : 0.0;
#pragma unroll
              for (int j = 0; j < TR; ++j) w[j] = wb[bb * RC + j];
#pragma unroll
              for (int i = 0; i < TA; ++i)
#pragma unroll
                for (int j = 0; j < TR; ++j) acc[i][j] = fma(g[i], w[j], acc[i][j]);
            }
          }
        }
        if (ok) {
          double* out = A.qhat + (int64_t)cs.skel_off[v] * RC;
#pragma unroll
          for (int i = 0; i < TA; ++i)
            if (a0 + i < k)
#pragma unroll
              for (int j = 0; j < TR; ++j) out[(int64_t)(a0 + i) * RC + r0 + j] = acc[i][j];
        }
        if (it0 + blockDim.x < items && nk > TB) {  // the G tiles must be restaged
          __syncthreads();
          const int tb0 = min(TB, nk);
          stage_block<16>(tb0 * k, [&](int e) { return G[e]; }, [&](int e, double x) { gs[e] = x; });
          __syncthreads();
        }
      }
    }
}

template <int RC>
__global__ void __launch_bounds__(XFER_THREADS) k_upward(XferArgs A, const int* order, int n,
                                                         const unsigned char* inset,
                                                         unsigned* counter, unsigned* done,
                                                         unsigned epoch) {
  extern __shared__ double sh[];
  for (;;) {
    const int tk = next_ticket(counter);
    if (tk >= n) break;
    const int v = order[tk];
    const int nc = A.nchild[v];
    if (threadIdx.x < nc) {
      const int c = A.child_first[v] + threadIdx.x;
      if (inset[c])  // producers outside this launch are final already
        while (ld_acquire(&done[c]) != epoch) __nanosleep(40);
    }
    __syncthreads();
    up_node<RC>(A, v, sh);
    publish(done, v, epoch);
  }
}

// Leaves have no producers: one CTA per leaf, no tickets, no flags.
template <int RC>
__global__ void __launch_bounds__(64) k_upward_leaves(XferArgs A, const int* leaves, int n) {
  extern __shared__ double sh[];
  if ((int)blockIdx.x >= n) return;
  const int v = leaves[blockIdx.x];
  if (v == 0) return;  // a leaf root has no factor
  up_node<RC>(A, v, sh);
}

// zhat[children] += X_v zhat[v] (internal non-root nodes, after the coupling).
// zhat_v, the children's contiguous coefficient block, the permutation and the
// first G tile are staged in one batched load; the block is updated in shared
// memory and written back coalesced.
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
      const int* perm = rs.perm + rs.ib_off[v];
      const double* zsrc = A.zhat + (int64_t)rs.skel_off[v] * RC;
      double* dst = A.zhat + (int64_t)rs.skel_off[A.child_first[v]] * RC;
      const double* G = rs.G + rs.g_off[v];
      const int nk = ni - k;
      const int TB = g_tile_rows(ks);
      double* zv = sh;             // k * RC
      double* db = zv + k * RC;    // ni * RC: the children's block
      double* pm = db + ni * RC;   // ni
      double* gs = pm + ni;        // TB * ks
      const int n_z = k * RC, n_d = ni * RC, tb0 = min(TB, nk);
      stage_block<16>(n_z + n_d + ni + tb0 * k,
                      [&](int e) {
                        return e < n_z ? __ldcg(zsrc + e)
                               : e < n_z + n_d ? __ldcg(dst + (e - n_z))
                               : e < n_z + n_d + ni ? (double)perm[e - n_z - n_d]
                                                    : G[e - n_z - n_d - ni];
                      },
                      [&](int e, double x) {
                        if (e < n_z + n_d + ni) {
                          zv[e] = x;
                        } else {
                          const int g = e - n_z - n_d - ni;
                          gs[(g / k) * ks + g % k] = x;
                        }
                      });
      __syncthreads();
      for (int e = threadIdx.x; e < k * RC; e += blockDim.x) {
        const int a = e / RC, r = e % RC;
        db[(int)pm[a] * RC + r] += zv[e];
      }
      constexpr int TR = RC < 4 ? RC : 4;
      constexpr int TB2 = 2;
      for (int b0 = 0; b0 < nk; b0 += TB) {
        const int tb = min(TB, nk - b0);
        if (b0 > 0) {
          const double* src = G + (int64_t)b0 * k;
          __syncthreads();
          stage_block<16>(tb * k, [&](int e) { return src[e]; },
                          [&](int e, double x) { gs[(e / k) * ks + e % k] = x; });
          __syncthreads();
        }
        const int nb = (tb + TB2 - 1) / TB2, nrq = RC / TR;
        for (int it = threadIdx.x; it < nb * nrq; it += blockDim.x) {
          const int bl = (it / nrq) * TB2, r0 = (it % nrq) * TR;
          double y[TB2][TR];
#pragma unroll
          for (int i = 0; i < TB2; ++i)
#pragma unroll
            for (int j = 0; j < TR; ++j) y[i][j] = 0.0;
          const double* g0 = gs + bl * ks;
          const bool two = bl + 1 < tb;
          for (int a = 0; a < k; ++a) {
            double w[TR];
#pragma unroll
            for (int j = 0; j < TR; ++j) w[j] = zv[a * RC + r0 + j];
            const double ga = g0[a], gb = two ? g0[ks + a] : 0.0;
#pragma unroll
            for (int j = 0; j < TR; ++j) {
              y[0][j] = fma(ga, w[j], y[0][j]);
              y[1][j] = fma(gb, w[j], y[1][j]);
            }
          }
#pragma unroll
          for (int i = 0; i < TB2; ++i)
            if (bl + i < tb) {
              double* d = db + (int)pm[k + b0 + bl + i] * RC + r0;
#pragma unroll
              for (int j = 0; j < TR; ++j) d[j] += y[i][j];
            }
        }
      }
      __syncthreads();
      for (int e = threadIdx.x; e < ni * RC; e += blockDim.x) dst[e] = db[e];
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
  const size_t smem = ((size_t)P.max_nib * (2 * RC + 1) + 4096) * sizeof(double);
  SMASH_CUDA(cudaFuncSetAttribute(k_upward<RC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // flags and ticket counter are reset on the stream (graph-replay safe)
  SMASH_CUDA(cudaMemsetAsync(P.counters.p, 0, sizeof(unsigned), s));
  SMASH_CUDA(cudaMemsetAsync(P.done.p, 0, P.done.n * sizeof(unsigned), s));
  const int grid = std::min(n, xfer_grid(smem));
  k_upward<RC><<<grid, XFER_THREADS, smem, s>>>(a, order, n, inset, P.counters.p, P.done.p, 1u);
}

template <int RC>
void launch_upward_leaves(const XferArgs& a, const XferPlan& P, const int* leaves, int n,
                          cudaStream_t s) {
  if (!n) return;
  const size_t smem = ((size_t)P.max_leaf_nib * (2 * RC + 1) + 4096) * sizeof(double);
  SMASH_CUDA(cudaFuncSetAttribute(k_upward_leaves<RC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  k_upward_leaves<RC><<<n, 64, smem, s>>>(a, leaves, n);
}

template <int RC>
void launch_downward(const XferArgs& a, XferPlan& P, const int* order, int n,
                     const unsigned char* inset, cudaStream_t s) {
  if (!n) return;
  const size_t smem = ((size_t)P.max_rank * RC + (size_t)P.max_nib * (RC + 1) + 4096 + 64) *
                       sizeof(double);
  SMASH_CUDA(cudaFuncSetAttribute(k_downward<RC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SMASH_CUDA(cudaMemsetAsync(P.counters.p + 1, 0, sizeof(unsigned), s));
  SMASH_CUDA(cudaMemsetAsync(P.done.p, 0, P.done.n * sizeof(unsigned), s));
  const int grid = std::min(n, xfer_grid(smem));
  k_downward<RC><<<grid, XFER_THREADS, smem, s>>>(a, order, n, inset, P.counters.p + 1, P.done.p,
                                                  1u, 0);
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
  template void launch_upward_leaves<RC>(const XferArgs&, const XferPlan&, const int*, int,      \
                                         cudaStream_t);                                         \
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
