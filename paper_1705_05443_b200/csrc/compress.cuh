// K3 + K4: batched Chebyshev/Lagrange basis + strong rank-revealing QR
// (see compress.cu).
#pragma once

#include "smash_impl.cuh"

namespace smash {

constexpr int COMPRESS_THREADS = 256;
constexpr int MAX_M_AXIS_1D = 128;  // 1-D: r <= 128 (numpy pairwise block, one level)
constexpr int MAX_M_AXIS_ND = 16;   // 2-D/3-D: nodes per axis

struct BasisTables {
  // Chebyshev cos((2k+1)pi/2m) and barycentric weights (-1)^k sin(...) for the
  // per-axis node count m, computed on the host with libm (== numpy's values).
  const double* cosv = nullptr;
  const double* wv = nullptr;
  const int* order = nullptr;  // [r][3] tensor indices in (degree, i, j, k) order
  int m = 0;                   // nodes per axis
};

struct CompressArgs {
  int lb = 0, le = 0;  // BFS node range of the level
  int dim = 1, r = 0;
  int side = 0;
  // tree
  const int* nchild = nullptr;
  const int* child_first = nullptr;
  const int* pt_a = nullptr;   // leaf point range start (tree order) for this side
  const double* lo = nullptr;  // node boxes [n][dim]
  const double* hi = nullptr;
  double half_pad = 0;         // pad / 2 (hss.py:39-45, 221-222)
  double pad = 0;
  // ibar sources
  const double* P = nullptr;   // tree-ordered points, SoA, stride P_stride
  int64_t P_stride = 0;
  const double* Sk = nullptr;  // compact skeleton points of the previous level, SoA
  int64_t S_stride = 0;
  const int* Slab = nullptr;   // compact skeleton labels
  const int* skel_off = nullptr;  // compact offset per BFS node
  const int* nib = nullptr;       // |ibar| per node
  const int64_t* ib_off = nullptr;
  const int64_t* g_off = nullptr;
  int64_t ib_level_base = 0;      // ib_off of the level's first node
  // HSS: extra panel rows from the truncated SVD (hss.py:286-287)
  const int* keep = nullptr;
  const int64_t* sv_off = nullptr;
  const double* sv = nullptr;     // S: (nib x keep) row-major per node
  BasisTables tab;
  double s_bound = 2.0, rtol = 1e-14;
  // outputs
  int* rank = nullptr;
  int* perm = nullptr;
  double* G = nullptr;
  int* tmp_lab = nullptr;     // level-local, at ib_off - ib_level_base
  double* tmp_pts = nullptr;  // SoA [dim][level ib total]
  int64_t tmp_stride = 0;
  int* err = nullptr;
  unsigned long long* swaps = nullptr;
  // panel storage
  int nmax = 0, mmax = 0;
  int64_t panel_cap = 0;   // nodes with |ibar| * rows <= panel_cap keep the panel in shared memory
  double* gws = nullptr;   // global workspace, per block mmax * nmax (the other nodes)
  // single-call mode: C given explicitly (nrows x ncols row-major) instead of a basis
  const double* Cexp = nullptr;
  int C_cols = 0;
  unsigned long long* prof = nullptr;
  int* next = nullptr;  // dynamic node counter (launch_compress)
  int threads = COMPRESS_THREADS;  // CTA size (plan_compress_launch)
  int n_lo = -1, n_hi = 0x7fffffff;  // size class of this launch: n_lo < |ibar| <= n_hi
  bool chains4 = true;  // four-chain dot products (qr_device.cuh); SMASH_QR_CHAINS=1: sequential
};

size_t compress_smem_bytes(int nmax, int mmax, bool panel_in_smem);
// Launch plan of a level: sets A.panel_cap, returns the dynamic shared memory
// per CTA and the grid (persistent CTAs over the level's cnt nodes).
size_t plan_compress_launch(CompressArgs& A, int cnt, int smem_limit, int nsm, int* grid);
// slot: the node counter of this launch (launches of one level may run concurrently)
void launch_compress(const CompressArgs& a, int grid, size_t smem, cudaStream_t s, int slot = 0);
// Register-column kernel (compress_rc.cuh): CTA size = maximum columns, rows kept in
// registers, R11 of the back substitution in shared memory or in a global/L2 slice.
struct RcVariant {
  int nt = 0;  // 0: k_compress
  int rr = 0;
  bool r11g = false;  // R11 of the back substitution streamed four rows at a time (else resident)
  int cs = 1;         // thread-block cluster size: a node's columns spread over cs CTAs
};
__host__ __device__ inline int rc_round4(int x) { return (x + 3) & ~3; }
__host__ __device__ inline int rc_vhn(int mmax, int rr) { return rc_round4(mmax) + rr + 4; }
__host__ __device__ inline int rc_kcap(int mmax, int nt) { return rc_round4(mmax < nt ? mmax : nt); }
// row length of R11: >= rbase + rr of every node
__host__ __device__ inline int rc_kld(int mmax, int rr) { return rc_round4(mmax) > rr ? rc_round4(mmax) : rr; }
__host__ __device__ inline int rc_srows(int mmax, int rr) { return mmax > rr ? rc_round4(mmax - rr) : 0; }
inline size_t rc_r11_doubles(const RcVariant& v, int mmax) {  // resident, or four streamed rows
  return (size_t)(v.r11g ? 4 : rc_kcap(mmax, v.nt)) * rc_kld(mmax, v.rr);
}
// Chebyshev nodes per axis: up to 128 in 1-D, 16 per axis in 2-D / 3-D
__host__ __device__ constexpr int rc_nodes_stride(int dim) { return dim == 1 ? MAX_M_AXIS_1D : MAX_M_AXIS_ND; }
inline size_t compress_rc_smem_bytes(const RcVariant& v, int mmax, int dim) {
  const size_t d = 3 * (size_t)rc_vhn(mmax, v.rr) + rc_round4(mmax) + dim * rc_nodes_stride(dim) + 32 + 8 +
                   rc_r11_doubles(v, mmax) + (size_t)rc_srows(mmax, v.rr) * v.nt;
  const size_t i = 32 + 8 + (size_t)v.nt;
  return 8 * d + 4 * i + 16;
}
// global workspace (doubles) of a register-column launch: the clusters' position tables
inline size_t compress_rc_gws_doubles(const RcVariant& v, int grid) {
  return v.cs > 1 ? (size_t)grid * v.nt / 2 + 1 : 0;
}
void launch_compress_rc(const CompressArgs& a, const RcVariant& v, int grid, size_t smem, cudaStream_t s, int slot = 0);
template <int D>
void launch_compress_rc_dim(const CompressArgs& a, const RcVariant& v, int grid, size_t smem, cudaStream_t s);

constexpr int MAX_COMPRESS_PASSES = 7;
struct CompressPass {
  CompressArgs a;
  int grid = 0;
  size_t smem = 0;
  RcVariant rc;  // rc.nt > 0: register-column kernel (launch_compress_rc)
};
// The size-class launches of a level (see compress.cu); returns their count (<= MAX_COMPRESS_PASSES).
int plan_compress_passes(const CompressArgs& A, int cnt, int smem_limit, int nsm, CompressPass* out);
void launch_basis_single(int dim, const double* plo, const double* phi, const BasisTables& tab,
                         int r, const double* pts_soa, int64_t n, double* out, int* err,
                         cudaStream_t s);

}  // namespace smash
