// K1: adaptive cluster tree on the GPU -- replaces smash.cluster.build_tree
// (smash/cluster.py:247-353).
//
// The reference recursion bisects a node's box at its midpoint (points with
// p[a] <= mid go low), discards empty cells, and when only one cell is occupied
// shrinks the box to it and retries (axis advancing in binary mode).  Because a
// shrink is itself a bisection, the box at every attempt is a cell of the plain
// recursive bisection of the root box, so each point's path is a digit string:
//   binary: one bit per attempt on axis (t mod d)
//   2d    : one d-bit digit per attempt, axis 0 most significant (cluster.py:325-331)
// computed per point with the reference's exact fp64 midpoints.  After a stable
// radix sort by key, a node is a contiguous key range: it is a leaf iff
// max(#row, #col) <= nu0; otherwise it splits at the first digit where its keys
// differ (every earlier digit is a shrink) into the occupied digit groups, and
// its box is the cell at that depth (a leaf keeps the cell it was created in).
// Levels are expanded breadth-first, one launch per level; postorder indices,
// point ranges and the per-leaf original-index order of the perms follow.
#include <cub/cub.cuh>

#include "smash_impl.cuh"

namespace smash {

namespace {

constexpr int KEY_BITS = 128;
constexpr int MAX_KIDS = 8;

__device__ __forceinline__ unsigned long long ord_of(double x) {
  unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ULL);
}
inline double dbl_of_ord(unsigned long long u) {
  u = (u >> 63) ? (u & 0x7fffffffffffffffULL) : ~u;
  double d;
  memcpy(&d, &u, 8);
  return d;
}

__global__ void k_bbox(const double* P, int64_t n, int dim, unsigned long long* mn,
                       unsigned long long* mx) {
  unsigned long long lmn[3] = {~0ULL, ~0ULL, ~0ULL}, lmx[3] = {0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int a = 0; a < dim; ++a) {
      unsigned long long o = ord_of(P[i * dim + a]);
      lmn[a] = o < lmn[a] ? o : lmn[a];
      lmx[a] = o > lmx[a] ? o : lmx[a];
    }
  }
  for (int a = 0; a < dim; ++a) {
    for (int off = 16; off; off >>= 1) {
      unsigned long long t1 = __shfl_xor_sync(0xffffffffu, lmn[a], off);
      unsigned long long t2 = __shfl_xor_sync(0xffffffffu, lmx[a], off);
      lmn[a] = t1 < lmn[a] ? t1 : lmn[a];
      lmx[a] = t2 > lmx[a] ? t2 : lmx[a];
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&mn[a], lmn[a]);
      atomicMax(&mx[a], lmx[a]);
    }
  }
}

struct RootBox {
  double lo[3], hi[3];
};

__device__ __forceinline__ void put_bit(uint64_t& khi, uint64_t& klo, int pos, uint64_t bit) {
  if (pos < 64)
    khi |= bit << (63 - pos);
  else
    klo |= bit << (127 - pos);
}
__device__ __forceinline__ uint64_t get_bits(uint64_t khi, uint64_t klo, int pos, int w) {
  uint64_t v = 0;
  for (int b = 0; b < w; ++b) {
    int p = pos + b;
    uint64_t bit = p < 64 ? (khi >> (63 - p)) & 1ULL : (klo >> (127 - p)) & 1ULL;
    v = (v << 1) | bit;
  }
  return v;
}

// Per-point bisection path keys (exact midpoints, cluster.py:253-255).
template <int D>
__global__ void k_keys(const double* P, int64_t n, int mode, int ndig, RootBox rb,
                       uint64_t* khi, uint64_t* klo) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[D], lo[D], hi[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    p[a] = P[i * D + a];
    lo[a] = rb.lo[a];
    hi[a] = rb.hi[a];
  }
  uint64_t h = 0, l = 0;
  int pos = 0;
  if (mode == SMASH_MODE_BINARY) {
    for (int t = 0; t < ndig; ++t) {
      int a = t % D;
      double mid = __dmul_rn(0.5, __dadd_rn(lo[a], hi[a]));
      uint64_t bit = p[a] <= mid ? 0ULL : 1ULL;
      if (bit) lo[a] = mid; else hi[a] = mid;
      put_bit(h, l, pos++, bit);
    }
  } else {
    for (int t = 0; t < ndig; ++t) {
#pragma unroll
      for (int a = 0; a < D; ++a) {
        double mid = __dmul_rn(0.5, __dadd_rn(lo[a], hi[a]));
        uint64_t bit = p[a] <= mid ? 0ULL : 1ULL;
        if (bit) lo[a] = mid; else hi[a] = mid;
        put_bit(h, l, pos++, bit);
      }
    }
  }
  khi[i] = h;
  klo[i] = l;
}

// Box of the cell reached after `depth` digits of a key (same arithmetic as k_keys).
__device__ void cell_of(uint64_t khi, uint64_t klo, int depth, int mode, int dim,
                        const RootBox& rb, double* lo, double* hi) {
  for (int a = 0; a < dim; ++a) { lo[a] = rb.lo[a]; hi[a] = rb.hi[a]; }
  int pos = 0;
  for (int t = 0; t < depth; ++t) {
    int na = mode == SMASH_MODE_BINARY ? 1 : dim;
    for (int q = 0; q < na; ++q) {
      int a = mode == SMASH_MODE_BINARY ? t % dim : q;
      double mid = __dmul_rn(0.5, __dadd_rn(lo[a], hi[a]));
      uint64_t bit = pos < 64 ? (khi >> (63 - pos)) & 1ULL : (klo >> (127 - pos)) & 1ULL;
      ++pos;
      if (bit) lo[a] = mid; else hi[a] = mid;
    }
  }
}

__device__ __forceinline__ int clz128(uint64_t h, uint64_t l) {
  return h ? __clzll(h) : 64 + __clzll(l);
}

struct ExpandArgs {
  const uint64_t* khi;
  const uint64_t* klo;
  const int* xpref;  // x items before sorted position i, size ntot + 1
  int shared, nu0, mode, dim, w, ndig;
  RootBox rb;
  int* item_a;
  int* item_b;
  int* tdep;
  int* tsplit;
  double* lo;
  double* hi;
  int* nkids;
  int* bounds;  // [node][MAX_KIDS + 1]
  int* err;
};

// Level bounds come from the device (dlev[l] = first node of level l+1 in 0-based
// level index), so several levels are enqueued between host round trips; threads
// past the level's end clear their nkids slot (the scan runs over a fixed size).
__global__ void k_expand(const int* dlev, int l, int nk_size, ExpandArgs A) {
  const int lb = dlev[l], le = dlev[l + 1];
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
  if (t0 >= le - lb) {
    if (t0 < nk_size) A.nkids[t0] = 0;
    return;
  }
  int v = lb + t0;
  int a = A.item_a[v], b = A.item_b[v], t = A.tdep[v];
  int cx = A.xpref[b] - A.xpref[a];
  int cy = A.shared ? cx : (b - a) - cx;
  int nk = 0;
  double lo[3], hi[3];
  int depth = t;
  if (max(cx, cy) > A.nu0) {
    uint64_t xh = A.khi[a] ^ A.khi[b - 1], xl = A.klo[a] ^ A.klo[b - 1];
    int bitpos = (xh | xl) ? clz128(xh, xl) : KEY_BITS;
    int tp = bitpos / A.w;
    if (tp >= A.ndig || tp - t >= 200) {
      atomicOr(A.err, DEV_UNSPLITTABLE);
    } else {
      depth = tp;
      A.tsplit[v] = tp;
      int ng = 1 << A.w;
      int* bd = A.bounds + (size_t)v * (MAX_KIDS + 1);
      int prev = a;
      for (int g = 1; g <= ng; ++g) {
        int pos;
        if (g == ng) {
          pos = b;
        } else {
          int lo_i = prev, hi_i = b;  // first index with digit >= g
          while (lo_i < hi_i) {
            int mid = (lo_i + hi_i) >> 1;
            if ((int)get_bits(A.khi[mid], A.klo[mid], tp * A.w, A.w) >= g)
              hi_i = mid;
            else
              lo_i = mid + 1;
          }
          pos = lo_i;
        }
        if (pos > prev) bd[nk++] = prev;
        prev = pos;
      }
      bd[nk] = b;
    }
  }
  cell_of(A.khi[a], A.klo[a], depth, A.mode, A.dim, A.rb, lo, hi);
  for (int k = 0; k < A.dim; ++k) {
    A.lo[(size_t)v * A.dim + k] = lo[k];
    A.hi[(size_t)v * A.dim + k] = hi[k];
  }
  A.nkids[v - lb] = nk;
}

__global__ void k_link(int* dlev, int l, int cap, const int* nkids, const int* off,
                       const int* bounds, const int* tsplit, int* child_first, int* nchild,
                       int* item_a, int* item_b, int* tdep, int* lev, int* parent, int* err) {
  const int lb = dlev[l], le = dlev[l + 1];
  const int cnt = le - lb;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
  if (t0 == 0) {  // end of the next level
    const int total = cnt > 0 ? off[cnt - 1] + nkids[cnt - 1] : 0;
    if (le + total > cap) atomicOr(err, DEV_CAPACITY);
    dlev[l + 2] = le + (le + total > cap ? 0 : total);
  }
  if (t0 >= cnt || le + off[cnt - 1] + nkids[cnt - 1] > cap) return;
  int v = lb + t0;
  int nk = nkids[v - lb];
  int base = le + off[v - lb];
  child_first[v] = nk ? base : -1;
  nchild[v] = nk;
  const int* bd = bounds + (size_t)v * (MAX_KIDS + 1);
  for (int c = 0; c < nk; ++c) {
    int u = base + c;
    item_a[u] = bd[c];
    item_b[u] = bd[c + 1];
    tdep[u] = tsplit[v] + 1;
    lev[u] = lev[v] + 1;
    parent[u] = v;
  }
}

__global__ void k_subtree_size(int lb, int le, const int* child_first, const int* nchild,
                               int* size) {
  int v = lb + blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= le) return;
  int s = 1;
  for (int c = 0; c < nchild[v]; ++c) s += size[child_first[v] + c];
  size[v] = s;
}

__global__ void k_postorder(int lb, int le, const int* child_first, const int* nchild,
                            const int* size, int* left, int* post, int* bfs_of_post) {
  int v = lb + blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= le) return;
  int cur = left[v];
  for (int c = 0; c < nchild[v]; ++c) {
    int u = child_first[v] + c;
    left[u] = cur;
    cur += size[u];
  }
  int p = left[v] + size[v] - 1;
  post[v] = p;
  bfs_of_post[p] = v;
}

__global__ void k_ranges_geom(int n, int dim, int shared, const int* item_a, const int* item_b,
                              const int* xpref, const double* lo, const double* hi, int* row_a,
                              int* row_b, int* col_a, int* col_b, double* ctr, double* rad) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  int a = item_a[v], b = item_b[v];
  row_a[v] = xpref[a];
  row_b[v] = xpref[b];
  col_a[v] = shared ? xpref[a] : a - xpref[a];
  col_b[v] = shared ? xpref[b] : b - xpref[b];
  double c[3], r;
  box_center_radius(lo + (size_t)v * dim, hi + (size_t)v * dim, dim, c, &r);
  for (int k = 0; k < dim; ++k) ctr[(size_t)v * dim + k] = c[k];
  rad[v] = r;
}

__global__ void k_item_is_x(const int* sorted_item, int64_t ntot, int64_t nx, int* flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < ntot) flag[i] = sorted_item[i] < nx ? 1 : 0;
}

__global__ void k_leaf_starts(int n, const int* nchild, const int* item_a, int* flag) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n && nchild[v] == 0) flag[item_a[v]] = 1;
}

__global__ void k_perm_keys(int64_t ntot, int64_t nx, const int* sorted_item, const int* xpref,
                            const int* lord, int ibits, uint64_t* kx, uint64_t* ky) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= ntot) return;
  int it = sorted_item[i];
  uint64_t hi = (uint64_t)lord[i] << ibits;
  if (it < nx)
    kx[xpref[i]] = hi | (uint64_t)it;
  else
    ky[i - xpref[i]] = hi | (uint64_t)(it - nx);
}

__global__ void k_perm_gather(int64_t n, int dim, const uint64_t* k, int ibits, const double* P,
                              int* perm, double* pts_soa) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  int idx = (int)(k[p] & ((1ULL << ibits) - 1ULL));
  perm[p] = idx;
  for (int a = 0; a < dim; ++a) pts_soa[(size_t)a * n + p] = P[(size_t)idx * dim + a];
}

__global__ void k_iota(int* x, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[i] = (int)i;
}

// any neighbours (in high-word order) with equal high but different low words?
__global__ void k_hi_ties(const uint64_t* hi_sorted, const int* item, const uint64_t* lo, int64_t n,
                          int* flag) {
  for (int64_t i = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (hi_sorted[i] == hi_sorted[i - 1] && lo[item[i]] != lo[item[i - 1]]) *flag = 1;
}

__global__ void k_gather_u64(const uint64_t* src, const int* idx, uint64_t* dst, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

template <typename F>
void cub_call(F f, DBuf<char>& tmp, cudaStream_t s) {
  size_t bytes = 0;
  SMASH_CUDA(f((void*)nullptr, bytes));
  if (bytes > tmp.n) tmp.alloc(bytes, s);
  SMASH_CUDA(f((void*)tmp.p, bytes));
}

}  // namespace

TreeImpl* tree_build(const double* X, int64_t nx, const double* Y, int64_t ny, int dim, int nu0,
                     int mode, cudaStream_t s) {
  SMASH_CHECK(nx > 0, SMASH_ERR_INVALID, "row point set is empty");
  SMASH_CHECK(nu0 >= 1, SMASH_ERR_INVALID, "nu0 must be positive");
  SMASH_CHECK(dim >= 1 && dim <= 3, SMASH_ERR_INVALID, "points must have 1..3 coordinates");
  SMASH_CHECK(mode == SMASH_MODE_BINARY || mode == SMASH_MODE_2D, SMASH_ERR_INVALID,
              "mode must be 'binary' or '2d'");
  bool shared = (Y == nullptr) || (Y == X && ny == nx);
  if (shared) ny = nx;
  int64_t ntot = shared ? nx : nx + ny;
  SMASH_CHECK(ntot < (1LL << 30), SMASH_ERR_INVALID, "too many points for int32 indexing");

  init_pool();
  std::unique_ptr<TreeImpl> T(new TreeImpl());
  T->dim = dim; T->mode = mode; T->nu0 = nu0; T->shared = shared;
  T->nx = nx; T->ny = ny; T->stream = s;

  // ---- root box: componentwise min/max of vstack(X, Y) (cluster.py:290-291)
  DBuf<unsigned long long> bb;
  bb.alloc(6, s);
  {
    unsigned long long init[6] = {~0ULL, ~0ULL, ~0ULL, 0, 0, 0};
    h2d(bb.p, init, 6, s);
    k_bbox<<<296, 256, 0, s>>>(X, nx, dim, bb.p, bb.p + 3);
    if (!shared && ny) k_bbox<<<296, 256, 0, s>>>(Y, ny, dim, bb.p, bb.p + 3);
    unsigned long long hb[6];
    d2h(hb, bb.p, 6, s);
    sync(s);
    for (int a = 0; a < dim; ++a) {
      T->root_lo[a] = dbl_of_ord(hb[a]);
      T->root_hi[a] = dbl_of_ord(hb[3 + a]);
    }
  }
  RootBox rb;
  for (int a = 0; a < 3; ++a) { rb.lo[a] = T->root_lo[a]; rb.hi[a] = T->root_hi[a]; }
  const int w = mode == SMASH_MODE_BINARY ? 1 : dim;
  const int ndig = KEY_BITS / w;

  // ---- keys + stable sort (LSD over the two 64-bit words)
  DBuf<uint64_t> khi, klo, khi2, klo2;
  DBuf<int> item, item2;
  khi.alloc(ntot, s); klo.alloc(ntot, s); khi2.alloc(ntot, s); klo2.alloc(ntot, s);
  item.alloc(ntot, s); item2.alloc(ntot, s);
  SMASH_CUDA(cudaMemsetAsync(khi.p, 0, ntot * 8, s));
  {
    auto launch = [&](const double* P, int64_t n, int64_t base) {
      if (!n) return;
      unsigned g = cdiv(n, 256);
      if (dim == 1) k_keys<1><<<g, 256, 0, s>>>(P, n, mode, ndig, rb, khi.p + base, klo.p + base);
      if (dim == 2) k_keys<2><<<g, 256, 0, s>>>(P, n, mode, ndig, rb, khi.p + base, klo.p + base);
      if (dim == 3) k_keys<3><<<g, 256, 0, s>>>(P, n, mode, ndig, rb, khi.p + base, klo.p + base);
    };
    launch(X, nx, 0);
    if (!shared) launch(Y, ny, nx);
  }
  k_iota<<<cdiv(ntot, 256), 256, 0, s>>>(item.p, ntot);
  DBuf<char> tmp;
  // Stable sort by the 128-bit key.  First by the high word alone: unless two
  // points agree on the whole high word (the first 64 bisection bits) but not on
  // the low word, that order is already the full-key order (ties keep the
  // original index order either way), and half the radix passes are saved.
  bool need_low = false;
  {
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, khi.p, khi2.p, item.p, item2.p, (int)ntot, 0, 64, s);
    }, tmp, s);
    DBuf<int> tie;
    tie.alloc(1, s);
    tie.zero(s);
    k_hi_ties<<<std::min<int64_t>(cdiv(ntot, 256), 4096), 256, 0, s>>>(khi2.p, item2.p, klo.p, ntot,
                                                                       tie.p);
    int h = 0;
    d2h(&h, tie.p, 1, s);
    sync(s);
    need_low = h != 0;
  }
  if (!need_low) {
    std::swap(khi, khi2);
    std::swap(item, item2);
    k_gather_u64<<<cdiv(ntot, 256), 256, 0, s>>>(klo.p, item.p, klo2.p, ntot);
    std::swap(klo, klo2);
  } else {
    // LSD over the two words: low word, then high word (stable)
    k_iota<<<cdiv(ntot, 256), 256, 0, s>>>(item.p, ntot);
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, klo.p, klo2.p, item.p, item2.p, (int)ntot, 0, 64, s);
    }, tmp, s);
    k_gather_u64<<<cdiv(ntot, 256), 256, 0, s>>>(khi.p, item2.p, khi2.p, ntot);
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, khi2.p, khi.p, item2.p, item.p, (int)ntot, 0, 64, s);
    }, tmp, s);
    // (SortPairs leaves its inputs intact: klo still holds the original low words)
    k_gather_u64<<<cdiv(ntot, 256), 256, 0, s>>>(klo.p, item.p, klo2.p, ntot);
    std::swap(klo, klo2);
  }
  khi2.release(); klo2.release(); item2.release();

  // ---- x-item prefix counts over sorted positions
  DBuf<int> flag, xpref;
  flag.alloc(ntot + 1, s);
  xpref.alloc(ntot + 1, s);
  SMASH_CUDA(cudaMemsetAsync(flag.p, 0, (ntot + 1) * 4, s));
  k_item_is_x<<<cdiv(ntot, 256), 256, 0, s>>>(item.p, ntot, nx, flag.p);
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, flag.p, xpref.p, (int)(ntot + 1), s);
  }, tmp, s);

  // ---- breadth-first expansion
  const int cap = (int)(2 * ntot + 2);
  T->lev.alloc(cap, s); T->parent.alloc(cap, s); T->child_first.alloc(cap, s);
  T->nchild.alloc(cap, s); T->lo.alloc((size_t)cap * dim, s); T->hi.alloc((size_t)cap * dim, s);
  DBuf<int> item_a, item_b, tdep, tsplit, nk, off, bounds, err;
  item_a.alloc(cap, s); item_b.alloc(cap, s); tdep.alloc(cap, s); tsplit.alloc(cap, s);
  nk.alloc(cap, s); off.alloc(cap, s); bounds.alloc((size_t)cap * (MAX_KIDS + 1), s);
  err.alloc(1, s);
  {
    int h_root[5] = {0, (int)ntot, 0, 1, -1};
    h2d(item_a.p, &h_root[0], 1, s);
    h2d(item_b.p, &h_root[1], 1, s);
    h2d(tdep.p, &h_root[2], 1, s);
    h2d(T->lev.p, &h_root[3], 1, s);
    h2d(T->parent.p, &h_root[4], 1, s);
    err.zero(s);
  }
  ExpandArgs A{khi.p, klo.p, xpref.p, shared ? 1 : 0, nu0, mode, dim, w, ndig, rb,
               item_a.p, item_b.p, tdep.p, tsplit.p, T->lo.p, T->hi.p, nk.p, bounds.p, err.p};
  // Breadth-first expansion, LEVELS_PER_SYNC levels enqueued per host round trip
  // (level bounds live on the device; a finished tree leaves empty levels that
  // the kernels skip).  Node count per level <= points, so grids and the scan
  // are sized by ntot.
  constexpr int LEVELS_PER_SYNC = 4;
  constexpr int MAX_LEVELS = 4 * KEY_BITS + 8;
  DBuf<int> dlev;
  dlev.alloc(MAX_LEVELS + 2, s);
  {
    int h01[2] = {0, 1};
    h2d(dlev.p, h01, 2, s);
  }
  const int nk_size = (int)std::min<int64_t>(ntot, cap);
  const unsigned lgrid = cdiv(nk_size, 128);
  T->level_ptr = {0, 1};
  int l = 0;
  std::vector<int> hl(MAX_LEVELS + 2, 0);
  while (true) {
    SMASH_CHECK(l + LEVELS_PER_SYNC <= MAX_LEVELS, SMASH_ERR_NUMERICAL,
                "box subdivision failed to separate points (tree too deep)");
    for (int q = 0; q < LEVELS_PER_SYNC; ++q, ++l) {
      k_expand<<<lgrid, 128, 0, s>>>(dlev.p, l, nk_size, A);
      cub_call([&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(t, b, nk.p, off.p, nk_size, s);
      }, tmp, s);
      k_link<<<lgrid, 128, 0, s>>>(dlev.p, l, cap, nk.p, off.p, bounds.p, tsplit.p,
                                   T->child_first.p, T->nchild.p, item_a.p, item_b.p, tdep.p,
                                   T->lev.p, T->parent.p, err.p);
    }
    int herr = 0;
    d2h(hl.data(), dlev.p, l + 2, s);
    d2h(&herr, err.p, 1, s);
    sync(s);
    SMASH_CHECK((herr & DEV_CAPACITY) == 0, SMASH_ERR_CUDA, "node capacity exceeded");
    SMASH_CHECK(herr == 0, SMASH_ERR_NUMERICAL,
                "box subdivision failed to separate points (coincident points)");
    if (hl[l + 1] == hl[l]) break;  // the last enqueued level produced no children
  }
  // level_ptr = the distinct, increasing prefix of hl
  for (int q = 2; q <= l + 1 && hl[q] > hl[q - 1]; ++q) T->level_ptr.push_back(hl[q]);
  const int le = T->level_ptr.back();
  T->n_nodes = le;
  T->n_levels = (int)T->level_ptr.size() - 1;
  const int n = T->n_nodes;

  // ---- postorder numbering
  DBuf<int> size, left;
  size.alloc(n, s); left.alloc(n, s);
  T->post.alloc(n, s); T->bfs_of_post.alloc(n, s);
  for (int l = T->n_levels; l >= 1; --l) {
    int b0 = T->level_begin(l), b1 = T->level_end(l);
    k_subtree_size<<<cdiv(b1 - b0, 128), 128, 0, s>>>(b0, b1, T->child_first.p, T->nchild.p, size.p);
  }
  SMASH_CUDA(cudaMemsetAsync(left.p, 0, 4, s));
  for (int l = 1; l <= T->n_levels; ++l) {
    int b0 = T->level_begin(l), b1 = T->level_end(l);
    k_postorder<<<cdiv(b1 - b0, 128), 128, 0, s>>>(b0, b1, T->child_first.p, T->nchild.p, size.p,
                                                   left.p, T->post.p, T->bfs_of_post.p);
  }

  // ---- point ranges, centres, radii
  T->row_a.alloc(n, s); T->row_b.alloc(n, s); T->col_a.alloc(n, s); T->col_b.alloc(n, s);
  T->ctr.alloc((size_t)n * dim, s); T->rad.alloc(n, s);
  k_ranges_geom<<<cdiv(n, 128), 128, 0, s>>>(n, dim, shared ? 1 : 0, item_a.p, item_b.p, xpref.p,
                                              T->lo.p, T->hi.p, T->row_a.p, T->row_b.p,
                                              T->col_a.p, T->col_b.p, T->ctr.p, T->rad.p);

  // ---- perms: leaves in key order, original index order inside each leaf (cluster.py:307-311)
  DBuf<int> lord;
  lord.alloc(ntot, s);
  SMASH_CUDA(cudaMemsetAsync(flag.p, 0, (ntot + 1) * 4, s));
  k_leaf_starts<<<cdiv(n, 128), 128, 0, s>>>(n, T->nchild.p, item_a.p, flag.p);
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceScan::InclusiveSum(t, b, flag.p, lord.p, (int)ntot, s);
  }, tmp, s);
  int64_t nyy = shared ? 0 : ny;
  DBuf<uint64_t> kx, ky, kx2, ky2;
  kx.alloc(nx, s); kx2.alloc(nx, s);
  if (nyy) { ky.alloc(nyy, s); ky2.alloc(nyy, s); }
  // (leaf order, original index) keys with only the bits they need: leaf ranks
  // are < n_nodes, indices < max(nx, ny)
  auto nbits = [](int64_t v) { int b = 1; while ((1LL << b) <= v) ++b; return b; };
  const int ibits = nbits(std::max<int64_t>(nx, ny));
  const int end_bit = std::min(64, ibits + nbits(n + 1));
  k_perm_keys<<<cdiv(ntot, 256), 256, 0, s>>>(ntot, nx, item.p, xpref.p, lord.p, ibits, kx.p, ky.p);
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, kx.p, kx2.p, (int)nx, 0, end_bit, s);
  }, tmp, s);
  T->perm_row.alloc(nx, s);
  T->pts_row.alloc((size_t)nx * dim, s);
  k_perm_gather<<<cdiv(nx, 256), 256, 0, s>>>(nx, dim, kx2.p, ibits, X, T->perm_row.p, T->pts_row.p);
  if (nyy) {
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortKeys(t, b, ky.p, ky2.p, (int)nyy, 0, end_bit, s);
    }, tmp, s);
    T->perm_col.alloc(nyy, s);
    T->pts_col.alloc((size_t)nyy * dim, s);
    k_perm_gather<<<cdiv(nyy, 256), 256, 0, s>>>(nyy, dim, ky2.p, ibits, Y, T->perm_col.p, T->pts_col.p);
  }
  // (no trailing host round trip: everything after the tree is stream-ordered)
  SMASH_CUDA(cudaGetLastError());
  return T.release();
}

// ---------------------------------------------------------------------------
// exports (postorder indexing, int64)
// ---------------------------------------------------------------------------
namespace {

__global__ void k_exp_int(int n, const int* post, const int* src, const int* map_post,
                          int64_t* dst) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  int x = src[v];
  if (map_post) x = x >= 0 ? map_post[x] : -1;
  dst[post[v]] = x;
}

__global__ void k_exp_box(int n, int dim, const int* post, const double* src, double* dst) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  for (int k = 0; k < dim; ++k) dst[(size_t)post[v] * dim + k] = src[(size_t)v * dim + k];
}

__global__ void k_nchild_post(int n, const int* post, const int* nchild, int64_t* cnt) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) cnt[post[v]] = nchild[v];
}

__global__ void k_children_post(int n, const int* post, const int* child_first, const int* nchild,
                                const int64_t* child_ptr, int64_t* child_idx) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  int64_t o = child_ptr[post[v]];
  for (int c = 0; c < nchild[v]; ++c) child_idx[o + c] = post[child_first[v] + c];
}

__global__ void k_i32_to_i64(const int* a, int64_t* b, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

__global__ void k_soa_to_aos(const double* soa, int64_t n, int dim, double* aos) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int k = 0; k < dim; ++k) aos[i * dim + k] = soa[(size_t)k * n + i];
}

}  // namespace

void export_bfs_to_post_i64(const TreeImpl* t, const int* src_bfs, int64_t* dst, bool map_value,
                            cudaStream_t s) {
  int n = t->n_nodes;
  k_exp_int<<<cdiv(n, 128), 128, 0, s>>>(n, t->post.p, src_bfs, map_value ? t->post.p : nullptr,
                                         dst);
}

void tree_export(TreeImpl* t, int64_t* level, int64_t* parent, int64_t* child_ptr,
                 int64_t* child_idx, double* lo, double* hi, int64_t* row_start, int64_t* row_stop,
                 int64_t* col_start, int64_t* col_stop, int64_t* perm_row, int64_t* perm_col,
                 double* points_row, double* points_col, cudaStream_t s) {
  int n = t->n_nodes;
  unsigned g = cdiv(n, 128);
  if (level) k_exp_int<<<g, 128, 0, s>>>(n, t->post.p, t->lev.p, nullptr, level);
  if (parent) k_exp_int<<<g, 128, 0, s>>>(n, t->post.p, t->parent.p, t->post.p, parent);
  if (row_start) k_exp_int<<<g, 128, 0, s>>>(n, t->post.p, t->row_a.p, nullptr, row_start);
  if (row_stop) k_exp_int<<<g, 128, 0, s>>>(n, t->post.p, t->row_b.p, nullptr, row_stop);
  if (col_start) k_exp_int<<<g, 128, 0, s>>>(n, t->post.p, t->col_a.p, nullptr, col_start);
  if (col_stop) k_exp_int<<<g, 128, 0, s>>>(n, t->post.p, t->col_b.p, nullptr, col_stop);
  if (lo) k_exp_box<<<g, 128, 0, s>>>(n, t->dim, t->post.p, t->lo.p, lo);
  if (hi) k_exp_box<<<g, 128, 0, s>>>(n, t->dim, t->post.p, t->hi.p, hi);
  if (child_ptr) {
    DBuf<int64_t> cnt;
    cnt.alloc(n + 1, s);
    cnt.zero(s);
    k_nchild_post<<<g, 128, 0, s>>>(n, t->post.p, t->nchild.p, cnt.p);
    DBuf<char> tmp;
    cub_call([&](void* tp, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(tp, b, cnt.p, child_ptr, n + 1, s);
    }, tmp, s);
    if (child_idx)
      k_children_post<<<g, 128, 0, s>>>(n, t->post.p, t->child_first.p, t->nchild.p, child_ptr,
                                        child_idx);
    sync(s);
  }
  const int* pc = t->shared ? t->perm_row.p : t->perm_col.p;
  const double* xc = t->shared ? t->pts_row.p : t->pts_col.p;
  if (perm_row) k_i32_to_i64<<<cdiv(t->nx, 256), 256, 0, s>>>(t->perm_row.p, perm_row, t->nx);
  if (perm_col) k_i32_to_i64<<<cdiv(t->ny, 256), 256, 0, s>>>(pc, perm_col, t->ny);
  if (points_row) k_soa_to_aos<<<cdiv(t->nx, 256), 256, 0, s>>>(t->pts_row.p, t->nx, t->dim, points_row);
  if (points_col) k_soa_to_aos<<<cdiv(t->ny, 256), 256, 0, s>>>(xc, t->ny, t->dim, points_col);
  SMASH_CUDA(cudaGetLastError());
}

}  // namespace smash
