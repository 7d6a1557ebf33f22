// Internal data structures of the SMASH B200 library.
//
// Node storage is level-major ("BFS") order: level l's nodes are the contiguous
// range [level_ptr[l-1], level_ptr[l]) in left-to-right (= reference postorder
// index) order, and every node's children are consecutive.  That makes every
// per-level batch a contiguous slice and makes a parent's intermediate set ibar
// (the concatenation of its children's skeletons, smash/hss.py:241-244) one
// contiguous range of the next level's skeleton buffer.  The reference's
// postorder TreeNode.index is kept as `post` for the exports.
#pragma once

#include <map>
#include <memory>
#include <utility>

#include "common.cuh"

namespace smash {

struct PairLists {
  // sorted by (target, source), BFS ids
  DBuf<int> L_i, L_j, Lm_i, Lm_j;
  DBuf<int> L_ptr, Lm_ptr;  // CSR by target BFS id, size n_nodes + 1
  int64_t nL = 0, nLm = 0;
  // buffers built on an auxiliary stream are released on the owner's stream
  void rehome(cudaStream_t s) {
    L_i.st = s; L_j.st = s; Lm_i.st = s; Lm_j.st = s; L_ptr.st = s; Lm_ptr.st = s;
  }
};

struct NearSets {
  DBuf<int> ptr;  // BFS-indexed CSR, size n_nodes + 1
  DBuf<int> idx;  // BFS ids, reference candidate order
  int64_t total = 0;
};

struct TreeImpl {
  int dim = 0, mode = 0, nu0 = 0;
  bool shared = false;  // points_col is points_row
  int64_t nx = 0, ny = 0;
  int n_nodes = 0, n_levels = 0;
  std::vector<int> level_ptr;  // host: level l (1-based) = [level_ptr[l-1], level_ptr[l])
  double root_lo[3] = {0, 0, 0}, root_hi[3] = {0, 0, 0};

  // device, BFS order
  DBuf<int> lev, parent, child_first, nchild, post, bfs_of_post;
  DBuf<int> row_a, row_b, col_a, col_b;  // tree-order point ranges
  DBuf<double> lo, hi;                   // [n][dim] node boxes (reference Box)
  DBuf<double> ctr, rad;                 // [n][dim] centres, [n] radii

  DBuf<int> perm_row, perm_col;  // tree position -> original index
  DBuf<double> pts_row, pts_col; // SoA [dim][n] tree-ordered coordinates

  std::map<std::pair<double, int>, std::unique_ptr<PairLists>> pairs;
  std::map<double, std::unique_ptr<NearSets>> near;
  cudaStream_t stream = 0;

  int level_begin(int l) const { return level_ptr[l - 1]; }
  int level_end(int l) const { return level_ptr[l]; }
};

TreeImpl* tree_build(const double* X, int64_t nx, const double* Y, int64_t ny, int dim, int nu0,
                     int mode, cudaStream_t s);
void tree_export(TreeImpl* t, int64_t* level, int64_t* parent, int64_t* child_ptr,
                 int64_t* child_idx, double* lo, double* hi, int64_t* row_start, int64_t* row_stop,
                 int64_t* col_start, int64_t* col_stop, int64_t* perm_row, int64_t* perm_col,
                 double* points_row, double* points_col, cudaStream_t s);

PairLists* get_pairs(TreeImpl* t, double tau, int structure, cudaStream_t s);
NearSets* get_near(TreeImpl* t, double tau, cudaStream_t s);
void pairs_export(TreeImpl* t, PairLists* P, int64_t* L, int64_t* Lm, cudaStream_t s);
void near_export(TreeImpl* t, NearSets* N, int64_t* ptr, int64_t* idx, cudaStream_t s);

// BFS-indexed int array -> postorder-indexed int64 export
void export_bfs_to_post_i64(const TreeImpl* t, const int* src_bfs, int64_t* dst, bool map_value,
                            cudaStream_t s);

// ---------------------------------------------------------------------------
// compressed matrix
// ---------------------------------------------------------------------------
struct SideFactors {
  // per node (BFS): ibar size, rank, offsets
  DBuf<int> nib, rank;           // |ibar|, k
  DBuf<int64_t> ib_off, g_off;   // perm offset (|ibar| prefix), G offset
  DBuf<int> skel_off;            // compact skeleton offset (coef layout)
  DBuf<int> perm;                // local permutations, concatenated
  DBuf<double> G;                // (|ibar|-k) x k row-major per node
  DBuf<int> skel;                // compact skeleton labels (tree-order point ids)
  DBuf<double> skel_pts;         // SoA [dim][skel_total] skeleton coordinates
  int64_t ib_total = 0, g_total = 0, skel_total = 0;
  int64_t skel_stride = 0;       // SoA row stride of skel_pts
  int64_t swaps = 0;
  std::vector<int64_t> level_skel_begin;  // host: compact offset of each level's skeletons
};

struct MatrixImpl {
  std::shared_ptr<void> pending;  // state of a sharded build between its phases
  TreeImpl* tree = nullptr;
  smash_build_params p{};
  PairLists* pl = nullptr;
  SideFactors rowf, colf_own;
  SideFactors* colf = nullptr;  // == &rowf when the points are shared
  // matvec workspaces
  DBuf<double> qt, qhat, zhat, zd;
  DBuf<double> zn;  // tree-ordered nearfield rows of one chunk
  int64_t ws_nrhs = 0;
  // optional per-phase timing of the matvec (CUDA events on the launch streams)
  bool profile = false;
  bool serial_phases = false;  // profiling mode 2: nearfield on the main stream
  cudaEvent_t ev[9] = {};
  double phase_ms[7] = {0, 0, 0, 0, 0, 0, 0};  // gather, up, coupling, down, near, leaf-add, total
  int64_t launches = 0;
  // nearfield stream (runs concurrently with the far-field chain) + fork/join events
  cudaStream_t s2 = nullptr;
  cudaStream_t sc = nullptr;  // graph capture origin (the caller's stream may be the legacy one)
  cudaEvent_t fork = nullptr, join = nullptr;
  // Stream ordering of the shared scratch (qt, qhat, zhat, zd, zn): every product waits
  // for the previous one, whatever stream it ran on, and the matrix is freed only after
  // its last product completes.
  cudaEvent_t last_use = nullptr;
  // sharded build: owning rank of every node (BFS), -1 above the cut level; empty otherwise
  std::vector<int> shard_owner;
  void order_after_last_use(cudaStream_t s) {
    if (!last_use) SMASH_CUDA(cudaEventCreateWithFlags(&last_use, cudaEventDisableTiming));
    SMASH_CUDA(cudaStreamWaitEvent(s, last_use, 0));
  }
  void mark_use(cudaStream_t s) { SMASH_CUDA(cudaEventRecord(last_use, s)); }
  ~MatrixImpl() {
    if (last_use) {
      cudaEventSynchronize(last_use);
      cudaEventDestroy(last_use);
    }
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    if (s2) cudaStreamDestroy(s2);
    if (sc) cudaStreamDestroy(sc);
  }
};

MatrixImpl* matrix_build(TreeImpl* t, const smash_build_params& p, cudaStream_t s);
// level-distributed construction: every level's nodes are split over the ranks, the
// level's outputs summed over them through the caller's exchange (smash_exchange_fn)
MatrixImpl* matrix_build_sharded(TreeImpl* t, const smash_build_params& p, int rank, int world,
                                 smash_exchange_fn fn, void* ctx, cudaStream_t s);
void dense_matvec(int kernel, double dx, int dim, const double* X, int64_t nx, const double* Y,
                  int64_t ny, const double* q, int64_t nrhs, double* z, cudaStream_t s);
// sharded construction (build.cu): local levels, buffers to sum over ranks, finish
struct ExchangeBuf {
  void* ptr;
  int64_t count;
  int dtype;  // 0 int32, 1 float64, 2 int64
};
MatrixImpl* matrix_build_local(TreeImpl* t, const smash_build_params& p, int rank, int world,
                               int cut_level, const double* cut_weight, int replicate,
                               cudaStream_t s);
void matvec_coeff_layout(MatrixImpl* m, int64_t* row_off_post, int64_t* up_pos, int64_t* half_rows,
                         cudaStream_t s);
// saved factors of one side, postorder-indexed host arrays (smash_matrix_import)
struct ImportSide {
  const int64_t* rank;
  const int64_t* perm_ptr;
  const int64_t* perm;
  const int64_t* skel_ptr;
  const int64_t* skel;
  const int64_t* g_ptr;
  const double* G;
};
MatrixImpl* matrix_import(TreeImpl* t, const smash_build_params& p, const ImportSide* sides,
                          int nsides, cudaStream_t s);
void matrix_exchange_buffers(MatrixImpl* m, std::vector<ExchangeBuf>& out);
void matrix_build_finish(MatrixImpl* m, cudaStream_t s);
void matrix_export(MatrixImpl* m, int side, int64_t* has, int64_t* rank, int64_t* perm_ptr,
                   int64_t* perm, int64_t* skel_ptr, int64_t* skel, int64_t* g_ptr, double* G,
                   cudaStream_t s);
void matvec(MatrixImpl* m, const double* q, double* z, int64_t nrhs, cudaStream_t s);
void matvec_levelwise(MatrixImpl* m, const double* q, double* z, int64_t nrhs, cudaStream_t s);
void sum_matvec(int T, MatrixImpl* const* bases, const double* dl, const double* dr,
                const double* q, double* z, int64_t nrhs, int levelwise, cudaStream_t s);
void matvec_profile(MatrixImpl* m, int enable, double* phase_ms, int64_t* launches);
void matvec_set_partition(MatrixImpl* m, const int64_t* own_post, int64_t n_own,
                          const int64_t* top_post, int64_t n_top, cudaStream_t s);
void matvec_stage(MatrixImpl* m, int stage, const double* q, double* z, int64_t nrhs,
                  cudaStream_t s);
void matvec_coeffs(MatrixImpl* m, double** qhat, int64_t* rows);

// HSS ULV factorisation / solve (ulv.cu)
struct UlvImpl;
UlvImpl* ulv_factor(MatrixImpl* m, cudaStream_t s);
void ulv_solve(UlvImpl* f, const double* b, double* x, int64_t nrhs, cudaStream_t s);
void ulv_free(UlvImpl* f);

void kernel_block(int kernel, double dx, int dim, const double* X, int64_t nx, const double* Y,
                  int64_t ny, double* out, cudaStream_t s);
void interp_basis_single(int dim, const double* lo, const double* hi, const double* pts, int64_t n,
                         int r, double* out, cudaStream_t s);
void compr_single(const double* C, int64_t nrows, int64_t ncols, double s_bound, double rtol,
                  int64_t* perm, double* G, int64_t* rank, int64_t* swaps, cudaStream_t s);

}  // namespace smash
