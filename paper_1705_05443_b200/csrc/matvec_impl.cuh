// Shared device code and launch interfaces of the matvec (K6-K10), split over
// several translation units so the per-kernel P2P instantiations compile in
// parallel (p2p_<kernel>.cu), see matvec.cu for the phase structure.
#pragma once

#include "kernels.cuh"
#include "smash_impl.cuh"

namespace smash {
namespace mv {

constexpr int P2P_WARPS = 4;
constexpr int P2P_THREADS = 32 * P2P_WARPS;
constexpr int XFER_THREADS = 256;
constexpr int XFER_MAXT = 4;  // leaf upward: a-tiles per warp pass

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

inline Side side_of(const SideFactors& F) {
  return Side{F.nib.p, F.rank.p, F.ib_off.p, F.g_off.p, F.skel_off.p, F.perm.p, F.G.p,
              F.skel_pts.p, F.skel_stride};
}

// coupling: zhat[v] = sum_{j in L(v)} K(S_v, S_j) qhat_j, for every non-root node
struct CouplingArgs {
  int n_nodes;        // number of targets (list length, or all nodes when list == nullptr)
  const int* list;    // optional target node list (BFS ids)
  Side rs, cs;
  const int* Lptr;
  const int* Lsrc;
  const double* qhat;
  double* zhat;
  double dx;
  int max_targets;  // largest target set (skeleton rank) -> CTA size of the DMMA path
};

// symmetric coupling (X = Y, K(x, y) = K(y, x)): every coupling block is evaluated once.
// Pass 1 runs over the upper pair list U(v) = {j in L(v) : j > v}: zhat[v] = sum_{j in U(v)}
// B_vj qhat_j, and for each pair its transposed product B_vj^T qhat_v goes to the pair's
// rows of `buf` (pbuf[e] = first row of upper pair e).  Pass 2 adds, per target j, the rows
// of the pairs (i, j), i < j, listed by the source-major index (tptr / te), in order.
struct SymCoupling {
  const int* Uptr;   // CSR by target over the upper pairs
  const int* Usrc;
  const int64_t* pbuf;
  double* buf;
  const int* tptr;   // per target j: upper pairs (i, j) with i < j, sorted by i
  const int* te;
};

// nearfield: zn[p] = sum_{j in Lm(v)} K(x_p, y_s) qt_s for the rows p of every listed leaf v
struct NearArgs {
  const int* leaves;
  int n_leaves;
  const int* row_a;
  const int* row_b;
  const int* col_a;
  const int* col_b;
  const double* pts_row;
  int64_t nrow;
  const double* pts_col;
  int64_t ncol;
  const int* Lmptr;
  const int* Lmsrc;
  const double* qt;
  const int* slot_of;  // tree row -> its slot in the leaf's ibar order
  double* zn;          // nearfield rows in leaf ibar order (RC per row)
  double dx;
  int max_targets;  // largest leaf row count
};

template <int KER, int D, int RC>
void launch_coupling(const CouplingArgs& a, cudaStream_t s);
template <int KER, int D, int RC>
void launch_near(const NearArgs& a, cudaStream_t s);
// symmetric coupling (RC = 8 / 16): pass 1 + pass 2
template <int KER, int D, int RC>
void launch_coupling_sym(const CouplingArgs& a, const SymCoupling& y, cudaStream_t s);
template <int KER, int D>
void launch_block(const double* X, int64_t nx, const double* Y, int64_t ny, double dx, double* out,
                  cudaStream_t s);

// transfer passes (matvec_xfer.cu)
struct XferPlan {
  DBuf<int> up_order;    // internal non-root nodes, deepest level first (BFS ids descending)
  DBuf<int> down_order;  // internal non-root nodes, shallowest level first (BFS ids ascending)
  DBuf<int> leaves;
  DBuf<unsigned char> inset_int;  // membership of the whole-tree internal passes
  DBuf<unsigned> done;   // per node flags (reset before each pass)
  DBuf<unsigned> counters;  // [0] upward tickets, [1] downward tickets
  int n_up = 0, n_down = 0, n_leaves = 0;
  int max_nib = 0, max_rank = 0, max_nk = 0;
  DBuf<int> up_pos;
  DBuf<int> slot_of, zrow;  // row side, see launch_leaf_slots  // column side, see launch_up_pos
};

struct XferArgs {
  const int* nchild;
  const int* child_first;
  const int* parent;
  const int* pt_a;  // leaf point range [pt_a, pt_b) (column side upward, row side downward)
  const int* pt_b;
  const double* qt;
  double* qhat;
  double* qp;          // coefficient rows in their parent's ibar order (upward input)
  const int* up_pos;   // per skeleton row: its row in qp (-1 below the root)
  double* zhat;        // coupling result
  double* zd;          // contributions of the parent (downward)
  Side side;
};

// shared-memory geometry of the transfer kernels (from the plan maxima)
struct XferGeom {
  int ks;   // G row stride in shared memory (>= max rank, = 4 mod 8)
  int rcs;  // row stride of staged coefficient rows
  int tb;   // G rows per staged chunk
  int max_nib, max_rank;
};
XferGeom xfer_geom(int max_nib, int max_rank, int max_nk, int rc);
size_t xfer_smem_up(const XferGeom& G);
size_t xfer_smem_down(const XferGeom& G);

// up_pos[x] = row of skeleton row x in its parent's ibar order (-1 below the root)
void launch_up_pos(const Side& cs, const int* nchild, const int* child_first, int n, int* up_pos,
                   int64_t rows, cudaStream_t s);
template <int RC>
void launch_gather(const double* q, int64_t ldq, const int* perm, int64_t n, int64_t c0,
                   double* qt, cudaStream_t s);
// inset[v] != 0: v is processed by this launch (its flag must be waited for)
template <int RC>
void launch_upward(const XferArgs& a, XferPlan& P, const int* order, int n,
                   const unsigned char* inset, cudaStream_t s);
template <int RC>
void launch_downward(const XferArgs& a, XferPlan& P, const int* order, int n,
                     const unsigned char* inset, cudaStream_t s);
template <int RC>
void launch_up_leaves(const XferArgs& a, const int* leaves, int n, cudaStream_t s);
template <int RC>
void launch_down_leaves(const XferArgs& a, const int* leaves, int n, const int* zrow,
                        const double* zn, double* z, int64_t ldz, int64_t c0, cudaStream_t s);
// level-synchronous transfer passes (matvec_level.cu): one launch per level
void launch_level_up(const Side& cs, const int* nchild, const int* child_first, int lb, int le,
                     double* qhat, int rc, cudaStream_t s);
void launch_level_down(const Side& rs, const int* nchild, const int* child_first, const int* parent,
                       int lb, int le, const double* zhat, double* zd, int rc, int max_rank,
                       cudaStream_t s);
int level_max_nib();
void launch_leaf_slots(const Side& rs, const int* leaves, int n, const int* row_a, const int* row_b,
                       const int* perm_row, int* slot_of, int* zrow, cudaStream_t s);

}  // namespace mv
}  // namespace smash
