/*
 * smash_b200.h -- C ABI of the B200-native SMASH hot path (arXiv 1705.05443).
 *
 * Drop-in boundary for the reference Python package's tree / construct / matvec
 * path (/root/reference/pkg/src/smash, "smash/" below).  The reference has no
 * FFI layer of its own; each entry point replaces the Python function cited next
 * to it, and the Python package paper_1705_05443_b200 binds these symbols with
 * ctypes exactly as INTEGRATION.md shows for the reference side.
 *
 * Conventions
 *  - Every pointer argument named X, Y, q, z, out, or an export destination is a
 *    DEVICE pointer (CUDA global memory) unless documented as host.  Point arrays
 *    are row-major (n, dim) float64, like smash.PointSet.coords.
 *  - `stream` is a cudaStream_t passed as void*; all work is stream ordered.  Calls
 *    that must return sizes synchronise that stream before returning.
 *  - Node indices in exports are the reference's postorder TreeNode.index (root last).
 *  - Status codes mirror the reference CLI's exit codes (smash/cli.py:266-278):
 *      0 ok, 2 invalid argument (Python ValueError), 3 numerical failure
 *      (Python RuntimeError: sRRQR swap cap smash/lowrank.py:196-197, unsplittable
 *      cluster smash/cluster.py:340-341, degenerate interpolation box
 *      smash/lowrank.py:131-134), 4 CUDA / internal error.
 *    smash_last_error() returns the message of the last failure on this thread.
 *  - The library never frees caller memory.  Opaque handles own device memory
 *    (stream-ordered allocations) and are released by their *_free function.
 */
#ifndef SMASH_B200_H
#define SMASH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMASH_OK 0
#define SMASH_ERR_INVALID 2
#define SMASH_ERR_NUMERICAL 3
#define SMASH_ERR_CUDA 4

/* tree modes (smash/cluster.py:263 `mode`) */
#define SMASH_MODE_BINARY 0
#define SMASH_MODE_2D 1 /* "2d" / "2^d" */

/* block structures (smash/cluster.py:402 `structure`) */
#define SMASH_STRUCT_H2 0
#define SMASH_STRUCT_HSS 1

/* kernels: BASELINE kernels (log, 1/r, exp(-r)) extend smash/kernel.py:200-233;
 * cauchy is the reference's real 1-D Cauchy 1/(x-y) (smash/kernel.py:286-298). */
#define SMASH_KERNEL_LOG 0    /* log|x-y|, coincident -> dx (0)       */
#define SMASH_KERNEL_INV_R 1  /* 1/|x-y|, coincident -> dx (0)        */
#define SMASH_KERNEL_EXP 2    /* exp(-|x-y|), coincident -> 1         */
#define SMASH_KERNEL_CAUCHY 3 /* 1/(x-y), d = 1, coincident -> dx     */

typedef struct smash_tree_s* smash_tree_t;
typedef struct smash_matrix_s* smash_matrix_t;

int smash_abi_version(void);
const char* smash_last_error(void);

/* ---- cluster tree: replaces smash.cluster.build_tree (smash/cluster.py:263-353) ----
 * X: (nx, dim) device, Y: (ny, dim) device or NULL (= X, shared points as in the
 * reference's points_col=None).  mode: SMASH_MODE_*.  */
int smash_tree_build(const double* X, int64_t nx, const double* Y, int64_t ny, int32_t dim,
                     int32_t nu0, int32_t mode, void* stream, smash_tree_t* out);
/* sizes of the finished tree (host outputs) */
int smash_tree_sizes(smash_tree_t t, int64_t* n_nodes, int32_t* n_levels, int64_t* n_row,
                     int64_t* n_col, int32_t* dim, int32_t* shared_points);
/* Copy the tree into caller device buffers, postorder node indexing:
 *   level/parent/row_start/row_stop/col_start/col_stop: int64[n_nodes]
 *   child_ptr: int64[n_nodes+1], child_idx: int64[n_nodes-1] (children in order)
 *   lo/hi: float64[n_nodes, dim]; perm_row: int64[n_row]; perm_col: int64[n_col]
 *   points_row: float64[n_row, dim]; points_col: float64[n_col, dim]
 * Any destination may be NULL (skipped).  Mirrors ClusterTree (cluster.py:118-135). */
int smash_tree_export(smash_tree_t t, int64_t* level, int64_t* parent, int64_t* child_ptr,
                      int64_t* child_idx, double* lo, double* hi, int64_t* row_start,
                      int64_t* row_stop, int64_t* col_start, int64_t* col_stop,
                      int64_t* perm_row, int64_t* perm_col, double* points_row,
                      double* points_col, void* stream);
int smash_tree_free(smash_tree_t t);

/* ---- block partition: replaces smash.cluster.leaf_sets (smash/cluster.py:402-447) ----
 * Computes (and caches on the tree) L and Lm; returns their sizes (host). */
int smash_leaf_sets(smash_tree_t t, double tau, int32_t structure, void* stream, int64_t* n_L,
                    int64_t* n_Lm);
/* L: int64[n_L, 2], Lm: int64[n_Lm, 2] device, lexicographically sorted (i, j). */
int smash_leaf_sets_export(smash_tree_t t, double tau, int32_t structure, int64_t* L, int64_t* Lm,
                           void* stream);

/* ---- nearfield sets: replaces smash.cluster.nearfield_set (smash/cluster.py:374-399) ----
 * N_i for every node, in the reference's candidate order; total entries (host). */
int smash_nearfield(smash_tree_t t, double tau, void* stream, int64_t* total);
/* ptr: int64[n_nodes+1], idx: int64[total] device (postorder indexing) */
int smash_nearfield_export(smash_tree_t t, double tau, int64_t* ptr, int64_t* idx, void* stream);

/* ---- construction: replaces smash.h2.build_h2 (smash/h2.py:25-54) and
 *      smash.hss.build_hss (smash/hss.py:247-303) with BuildParams (hss.py:23-32)
 *      plus the sRRQR rank tolerance rtol (smash/lowrank.py:19,163-167). ---- */
typedef struct {
  int32_t structure; /* SMASH_STRUCT_* */
  int32_t kernel;    /* SMASH_KERNEL_* */
  double dx;         /* value at coincident points (KernelSpec.dx) */
  int32_t r;         /* interpolation nodes (BuildParams.r) */
  double tau;        /* admissibility (BuildParams.tau) */
  double s;          /* swap bound (BuildParams.s) */
  double rtol;       /* sRRQR rank tolerance */
  double eps_svd;    /* HSS nearfield SVD cutoff (BuildParams.eps_svd) */
} smash_build_params;

int smash_matrix_build(smash_tree_t t, const smash_build_params* p, void* stream,
                       smash_matrix_t* out);
/* Sharded H2 construction (replaces the level loop of smash/h2.py:44-53
 * when one process per GPU builds its share).  Phase 1 compresses rank's contiguous node
 * ranges of the levels at and below the cut level (cut_level < 2: the shallowest level with
 * >= 8 nodes per rank); the caller then sums every buffer listed by
 * smash_matrix_exchange_buffers over the ranks (all-reduce, in place; dtype 0 int32,
 * 1 float64, 2 int64), and phase 2 compacts the cut levels and compresses the top levels
 * on every rank.  The result equals smash_matrix_build's bit for bit. */
int smash_matrix_build_local(smash_tree_t t, const smash_build_params* p, int32_t rank,
                             int32_t world, int32_t cut_level, void* stream, smash_matrix_t* out);
/* Level-distributed HSS construction (SURVEY.md 8(e) for configs 1 and 4; replaces the level
 * loop of smash/hss.py:271-299 when one process per GPU builds): at every level each rank
 * runs the nearfield SVDs and compressions of its contiguous share of the level's nodes, then
 * calls fn(ctx, n, ptrs, counts, dtypes) -- the caller must sum each listed device buffer over
 * the ranks in place (dtype 0 int32, 1 float64 summed as int64 bit patterns, 2 int64, 3 int32
 * maximum; the shares are disjoint and zero elsewhere) and return 0 -- and compacts the level's
 * skeletons.  Every rank ends with the full matrix, identical to smash_matrix_build's. */
typedef int32_t (*smash_exchange_fn)(void* ctx, int64_t n, void** ptrs, const int64_t* counts,
                                     const int32_t* dtypes);
int smash_matrix_build_sharded(smash_tree_t t, const smash_build_params* p, int32_t rank,
                               int32_t world, smash_exchange_fn fn, void* ctx, void* stream,
                               smash_matrix_t* out);
/* As smash_matrix_build_local, with cut_weight (HOST float64[number of cut-level nodes],
 * left to right; NULL = subtree point counts) balancing the contiguous cut-level ranges,
 * and replicate = 0 to keep the factors sharded: perm and G are then NOT in the exchange list,
 * so every rank ends with the factors of its own subtrees and of the levels above the cut
 * only (enough for the sharded matvec over the same partition, smash_matrix_shard_owner). */
int smash_matrix_build_local_w(smash_tree_t t, const smash_build_params* p, int32_t rank,
                               int32_t world, int32_t cut_level, const double* cut_weight,
                               int32_t replicate, void* stream, smash_matrix_t* out);
/* cut level a sharded build over world ranks uses (cut_level < 2: the default rule); host out */
int smash_matrix_shard_cut(smash_tree_t t, int32_t world, int32_t cut_level, int32_t* cut);
/* owning rank of every node of a sharded build (HOST int64[n_nodes], postorder; -1 above the
 * cut: replicated on every rank) */
int smash_matrix_shard_owner(smash_matrix_t m, int64_t* owner_post);
int smash_matrix_exchange_buffers(smash_matrix_t m, int64_t capacity, int64_t* n, void** ptrs,
                                  int64_t* counts, int32_t* dtypes);
int smash_matrix_build_finish(smash_matrix_t m, void* stream);
/* Matrix from saved factors (container load; replaces the factor part of
 * smash/container.py:load_matrix, container.py:135-211).  HOST arrays per side k < nsides,
 * postorder-indexed exactly as smash_matrix_export writes them (rank[n_nodes],
 * perm_ptr/skel_ptr/g_ptr[n_nodes+1], perm, skel, G); nsides = 1 when the points are shared
 * and colfac == rowfac.  Sizes are validated against the tree (|ibar| of a leaf = its points,
 * of an internal node = the sum of its children's ranks); pair lists are rebuilt from the
 * tree and tau.  The matrix is then used exactly like a built one. */
int smash_matrix_import(smash_tree_t t, const smash_build_params* p, int32_t nsides,
                        const int64_t* const* rank, const int64_t* const* perm_ptr,
                        const int64_t* const* perm, const int64_t* const* skel_ptr,
                        const int64_t* const* skel, const int64_t* const* g_ptr,
                        const double* const* G, void* stream, smash_matrix_t* out);
/* side: 0 = row factors (rowfac), 1 = column factors (colfac).  Host outputs:
 * n_factors (nodes with a factor = non-root), total |ibar|, total skeleton, total G entries. */
int smash_matrix_sizes(smash_matrix_t m, int32_t side, int64_t* has_total, int64_t* ibar_total,
                       int64_t* skel_total, int64_t* g_total);
/* Per-node interpolative factors (InterpolativeFactor, smash/lowrank.py:206-229), postorder:
 *   has: int64[n_nodes] (1 if the node has a factor), rank: int64[n_nodes]
 *   perm_ptr: int64[n_nodes+1], perm: int64[ibar_total]      (local row permutation)
 *   skel_ptr: int64[n_nodes+1], skel: int64[skel_total]      (tree-order labels, ordered)
 *   g_ptr: int64[n_nodes+1], G: float64[g_total]             ((|ibar|-k) x k row-major) */
int smash_matrix_export(smash_matrix_t m, int32_t side, int64_t* has, int64_t* rank,
                        int64_t* perm_ptr, int64_t* perm, int64_t* skel_ptr, int64_t* skel,
                        int64_t* g_ptr, double* G, void* stream);
/* number of sRRQR swap-loop iterations per side (host output) */
int smash_matrix_stats(smash_matrix_t m, int64_t* swaps_row, int64_t* swaps_col);

/* ---- HSS ULV factorisation / solve: replaces smash.apply.ulv_factor / ulv_solve
 * (smash/apply.py:168-354).  The factorisation keeps a pointer
 * to m, which must outlive it.  b: (n_row, nrhs) row-major device, x: (n_col, nrhs)
 * row-major device, caller order.  Status 2 for a non-HSS matrix, 3 for a singular
 * local block or root system (message names the postorder node id, apply.py:218-223). */
typedef struct smash_ulv_s* smash_ulv_t;
int smash_ulv_factor(smash_matrix_t m, void* stream, smash_ulv_t* out);
int smash_ulv_solve(smash_ulv_t f, const double* b, double* x, int64_t nrhs, void* stream);
int smash_ulv_free(smash_ulv_t f);

/* ---- matvec: replaces smash.apply.matvec_nodewise (smash/apply.py:34-80) ----
 * q: (n_col, nrhs) row-major device, z: (n_row, nrhs) row-major device; caller order. */
int smash_matvec(smash_matrix_t m, const double* q, double* z, int64_t nrhs, void* stream);
/* ---- level-synchronous matvec: replaces smash.apply.matvec_levelwise (smash/apply.py:98-165)
 * on perfect trees (status 2 otherwise, apply.py:83-95).  One launch per tree level for the
 * transfer passes, per-level coefficient blocks, the upward sum taken child by child. */
int smash_matvec_levelwise(smash_matrix_t m, const double* q, double* z, int64_t nrhs, void* stream);
/* ---- HSS algebra: the product of diag_scale / hss_add / cauchy_like_hss results
 * (smash/hss.py:317-400), S = sum_t diag(dl_t) A_t diag(dr_t) on one cluster tree.
 * bases: HOST array of n_terms built matrices (repeats allowed: terms sharing a base are
 * applied in one multi-column product); dl: (n_terms, n_row), dr: (n_terms, n_col) row-major
 * device scalings in caller order; q (n_col, nrhs) -> z (n_row, nrhs).  levelwise = 1 applies
 * the bases with smash_matvec_levelwise (perfect trees), 0 with smash_matvec. */
int smash_sum_matvec(int32_t n_terms, const smash_matrix_t* bases, const double* dl,
                     const double* dr, const double* q, double* z, int64_t nrhs, int32_t levelwise,
                     void* stream);
/* Matvec phase timing (CUDA events on the launch streams; synchronises each matvec while on).
 * Returns the accumulated per-phase milliseconds since the last reset into phase_ms[7] =
 * [gather, upward, coupling, downward, nearfield (concurrent stream), leaf far-field, whole
 * matvec] and the number of kernel launches; then
 * enable = 1 turns profiling on and resets, 2 likewise with the nearfield serialised on the main
 * stream (isolated per-phase kernel times), 0 turns it off and resets, -1 leaves it as is. */
int smash_matvec_profile(smash_matrix_t m, int32_t enable, double* phase_ms, int64_t* launches);
/* ---- sharded matvec (one rank of a multi-GPU job; NCCL is driven by the caller) ----
 * Partition: own_nodes = the postorder ids of this rank's subtrees (frontier nodes and all
 * their descendants), top_nodes = the ancestors of all frontier nodes (replicated work).
 * Both are HOST arrays.  Stage 1: gather q and compute the coefficients qhat of the owned
 * subtrees (other rows of the coefficient buffer untouched); the caller then brings in the
 * coefficient rows stage 2 reads from other ranks (shard.halo_rows: the cut-level skeleton
 * coefficients and the coupling sources of its targets).  Stage 2: top-level
 * upward pass, coupling / downward / nearfield for the owned targets; writes only the owned
 * rows of z.  Stage 3 + stage 4 split stage 2 so the nearfield can overlap the exchange:
 * stage 3 (after stage 1, on any stream) runs the owned leaves' nearfield alone, stage 4 is
 * stage 2 without it (ordered after stage 3 by the caller).  nrhs: a power of two <= 16. */
int smash_matvec_set_partition(smash_matrix_t m, const int64_t* own_nodes, int64_t n_own,
                               const int64_t* top_nodes, int64_t n_top, void* stream);
int smash_matvec_stage(smash_matrix_t m, int32_t stage, const double* q, double* z, int64_t nrhs,
                       void* stream);
/* layout of that buffer (HOST outputs): row_off_post[n_nodes] = first row of each node's
 * skeleton coefficients (postorder; -1 for the root / rank-0 nodes), up_pos[half_rows] = row in
 * the second half (coefficients in the parent's ibar order, minus half_rows) of every
 * coefficient row (-1 below the root) or NULL, half_rows = rows of each half */
int smash_matvec_coeff_layout(smash_matrix_t m, int64_t* row_off_post, int64_t* up_pos,
                              int64_t* half_rows, void* stream);
/* device pointer of the coefficient buffer exchanged between stages: rows x nrhs doubles */
int smash_matvec_coeffs(smash_matrix_t m, double** qhat, int64_t* rows);
int smash_matrix_free(smash_matrix_t m);

/* ---- exact kernel entries: replaces smash.kernel.kernel_block (smash/kernel.py:278-310)
 *      and the block accessors B / NF (smash/hss.py:138-162) ----
 * X: (nx, dim), Y: (ny, dim) device; out: (nx, ny) row-major device. */
int smash_kernel_block(int32_t kernel, double dx, int32_t dim, const double* X, int64_t nx,
                       const double* Y, int64_t ny, double* out, void* stream);

/* ---- single-call primitives (smash/lowrank.py) ----
 * interp_basis (lowrank.py:123-144): lo/hi HOST float64[dim]; pts (n, dim) device;
 * out (n, r) row-major device.  dim 3 is this library's tensor extension. */
/* Exact product z = K(X, Y) q on the GPU, never storing K (the dense oracle of
 * smash/bench.py:284-296, dense_matvec): X (nx x dim), Y (ny x dim) row-major device
 * arrays in caller order, q (ny x nrhs) and z (nx x nrhs) row-major device float64. */
int smash_dense_matvec(int32_t kernel, double dx, int32_t dim, const double* X, int64_t nx,
                       const double* Y, int64_t ny, const double* q, int64_t nrhs, double* z,
                       void* stream);
int smash_interp_basis(int32_t dim, const double* lo, const double* hi, const double* pts,
                       int64_t n, int32_t r, double* out, void* stream);
/* compr (lowrank.py:232-255) on C (nrows, ncols) row-major device:
 * perm int64[nrows] device, G float64[nrows*min(nrows,ncols)] device (first (nrows-k)*k
 * entries valid, row-major), rank/swaps host. */
int smash_compr(const double* C, int64_t nrows, int64_t ncols, double s, double rtol, int64_t* perm,
                double* G, int64_t* rank, int64_t* swaps, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SMASH_B200_H */
