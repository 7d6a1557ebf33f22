// Level-synchronous transfer passes of matvec_levelwise (smash/apply.py:98-165,
// SURVEY.md 8(f) item 2) for perfect trees.
//
// The node-wise device matvec (matvec_xfer.cu) runs each transfer pass as ONE
// persistent dataflow launch whose CTAs spin on their producers' done flags.
// The level-wise path is the reference's other schedule: one launch per tree
// level, the level's coefficient block (level-major, so level l's nodes are one
// contiguous slice of qhat / zhat -- the reference's per-level buffers qbuf[l] /
// zbuf[l]) produced completely before the next level starts, and the upward
// sum taken child by child as the reference writes it:
//   upward    qbuf[l][v] = sum_{c in children(v)} W(c)^T qbuf[l+1][c]
//             W(c) = rows of X_v = P_v [I; G_v] at child c's slice of ibar_v,
//             each child's product accumulated on its own, then added in child order
//   downward  zbuf[l+1][c] += R(c) zbuf[l][v]   (written to zd, the parent part,
//             which the shared leaf kernel adds to the coupling part)
// One CTA per node, one thread per (output row, right-hand side column).
#include "matvec_impl.cuh"

namespace smash {
namespace mv {

namespace {

constexpr int LVL_THREADS = 256;
constexpr int LVL_MAX_NIB = 4096;  // ibar rows whose inverse permutation fits shared memory

// inverse of the node's local permutation: pos_of[x] = position of ibar row x in perm
__device__ __forceinline__ void load_inverse_perm(const int* perm, int nib, int* pos_of) {
  for (int p = threadIdx.x; p < nib; p += blockDim.x) pos_of[perm[p]] = p;
  __syncthreads();
}

// X_v[x, a] for ibar row x: identity rows for the skeleton, G rows for the rest
__device__ __forceinline__ double xval(const int* pos_of, const double* G, int k, int x, int a) {
  const int p = pos_of[x];
  return p < k ? (p == a ? 1.0 : 0.0) : __ldg(G + (int64_t)(p - k) * k + a);
}

// Internal nodes [lb, le) of one level: qhat_v = sum_c W(c)^T qhat_c.
__global__ void __launch_bounds__(LVL_THREADS) k_level_up(Side cs, const int* nchild,
                                                          const int* child_first, int lb, int le,
                                                          double* qhat, int RC) {
  __shared__ int pos_of[LVL_MAX_NIB];
  const int v = lb + blockIdx.x;
  if (v >= le || nchild[v] == 0) return;
  const int nib = cs.nib[v], k = cs.rank[v];
  if (k == 0) return;
  load_inverse_perm(cs.perm + cs.ib_off[v], nib, pos_of);
  const double* G = cs.G + cs.g_off[v];
  const int base = cs.skel_off[child_first[v]];  // children's coefficients, in ibar order
  double* out = qhat + (int64_t)cs.skel_off[v] * RC;
  const int nc = nchild[v], cf = child_first[v];
  for (int e = threadIdx.x; e < k * RC; e += blockDim.x) {
    const int a = e / RC, r = e - a * RC;
    double acc = 0.0;
    int x = 0;
    for (int c = 0; c < nc; ++c) {
      const int kc = cs.rank[cf + c];
      double part = 0.0;
      for (int t = 0; t < kc; ++t, ++x)
        part = fma(xval(pos_of, G, k, x, a), qhat[(int64_t)(base + x) * RC + r], part);
      acc += part;
    }
    out[e] = acc;
  }
}

// Internal nodes [lb, le) of one level: zd[children's rows] = X_v (zhat_v + zd_v).
__global__ void __launch_bounds__(LVL_THREADS) k_level_down(Side rs, const int* nchild,
                                                            const int* child_first,
                                                            const int* parent, int lb, int le,
                                                            const double* zhat, double* zd,
                                                            int RC) {
  __shared__ int pos_of[LVL_MAX_NIB];
  extern __shared__ double zv[];  // k x RC
  const int v = lb + blockIdx.x;
  if (v >= le || nchild[v] == 0) return;
  const int nib = rs.nib[v], k = rs.rank[v];
  const int base = rs.skel_off[child_first[v]];
  double* out = zd + (int64_t)base * RC;
  if (k == 0) {  // no skeleton: the children receive nothing from above
    for (int e = threadIdx.x; e < nib * RC; e += blockDim.x) out[e] = 0.0;
    return;
  }
  load_inverse_perm(rs.perm + rs.ib_off[v], nib, pos_of);
  const double* G = rs.G + rs.g_off[v];
  const int64_t so = (int64_t)rs.skel_off[v] * RC;
  const bool from_parent = parent[v] > 0;  // level-2 nodes have no parent contribution
  for (int e = threadIdx.x; e < k * RC; e += blockDim.x)
    zv[e] = from_parent ? zhat[so + e] + zd[so + e] : zhat[so + e];
  __syncthreads();
  for (int e = threadIdx.x; e < nib * RC; e += blockDim.x) {
    const int x = e / RC, r = e - x * RC;
    const int p = pos_of[x];
    double y;
    if (p < k) {
      y = zv[p * RC + r];
    } else {
      const double* g = G + (int64_t)(p - k) * k;
      y = 0.0;
      for (int a = 0; a < k; ++a) y = fma(__ldg(g + a), zv[a * RC + r], y);
    }
    out[e] = y;
  }
}

}  // namespace

void launch_level_up(const Side& cs, const int* nchild, const int* child_first, int lb, int le,
                     double* qhat, int rc, cudaStream_t s) {
  if (le > lb) k_level_up<<<le - lb, LVL_THREADS, 0, s>>>(cs, nchild, child_first, lb, le, qhat, rc);
}

void launch_level_down(const Side& rs, const int* nchild, const int* child_first, const int* parent,
                       int lb, int le, const double* zhat, double* zd, int rc, int max_rank,
                       cudaStream_t s) {
  if (le > lb)
    k_level_down<<<le - lb, LVL_THREADS, (size_t)max_rank * rc * 8, s>>>(
        rs, nchild, child_first, parent, lb, le, zhat, zd, rc);
}

int level_max_nib() { return LVL_MAX_NIB; }

}  // namespace mv
}  // namespace smash
