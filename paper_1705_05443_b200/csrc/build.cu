// Construction driver: replaces smash.h2.build_h2 (smash/h2.py:25-54) and
// smash.hss.build_hss (smash/hss.py:247-303).
//
// Host orchestration of the level-synchronous bottom-up sweep: for each level
// L..2 and each side, (1) |ibar| per node, (2) capacity offsets, (3) [HSS] the
// nearfield SVD, (4) the batched basis + sRRQR kernel, (5) compaction of the
// level's ordered skeletons (labels + coordinates) so the next level's ibar
// sets are contiguous slices.  When row and column points are shared the
// column factors alias the row factors (bitwise identical in the reference,
// SURVEY.md 7 / probe p12).
#include <thread>
#include <functional>
#include <condition_variable>
#include <mutex>
#include <chrono>
#include <cstdio>
#include <exception>
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "compress.cuh"
#include "svd.cuh"

namespace smash {

namespace {

template <typename F>
void cub_call(F f, DBuf<char>& tmp, cudaStream_t s) {
  size_t bytes = 0;
  SMASH_CUDA(f((void*)nullptr, bytes));
  if (bytes > tmp.n) tmp.alloc(bytes, s);
  SMASH_CUDA(f((void*)tmp.p, bytes));
}

template <typename T>
void grow(DBuf<T>& b, size_t used, size_t need, cudaStream_t s) {
  if (need <= b.n) return;
  size_t nc = std::max(need, b.n * 2 + 1024);
  DBuf<T> nb;
  nb.alloc(nc, s);
  d2d(nb.p, b.p, used, s);
  b = std::move(nb);
}

// G capacity per node: |ibar| x min(|ibar|, bound) with bound = r (H2) or, for HSS,
// r + keep_v (the compression panel's row count, known after the nearfield SVD)
__global__ void k_level_sizes(int lb, int le, const int* nchild, const int* child_first,
                              const int* pt_a, const int* pt_b, const int* rank, int* nib,
                              int64_t* ibcnt, int64_t* gcnt, int mrows_bound,
                              const int* keep = nullptr) {
  int v = lb + blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= le) return;
  int n;
  if (nchild[v] == 0) {
    n = pt_b[v] - pt_a[v];
  } else {
    n = 0;
    for (int c = 0; c < nchild[v]; ++c) n += rank[child_first[v] + c];
  }
  nib[v] = n;
  ibcnt[v - lb] = n;
  gcnt[v - lb] = (int64_t)n * min(n, keep ? mrows_bound + keep[v] : mrows_bound);
}

__global__ void k_level_nib(int lb, int le, const int* nchild, const int* child_first,
                            const int* pt_a, const int* pt_b, const int* rank, int* nib) {
  int v = lb + blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= le) return;
  int n;
  if (nchild[v] == 0) {
    n = pt_b[v] - pt_a[v];
  } else {
    n = 0;
    for (int c = 0; c < nchild[v]; ++c) n += rank[child_first[v] + c];
  }
  nib[v] = n;
}

// device-resident running skeleton count: compaction base of the next level
__global__ void k_skel_bump(int* used, const int* level_off, int cnt) { *used += level_off[cnt]; }

__global__ void k_add_base(int lb, int le, const int64_t* loc, int64_t base, int64_t* glob) {
  int v = lb + blockIdx.x * blockDim.x + threadIdx.x;
  if (v < le) glob[v] = base + loc[v - lb];
}

__global__ void k_rank_cnt(int lb, int le, const int* rank, int* cnt) {
  int v = lb + blockIdx.x * blockDim.x + threadIdx.x;
  if (v < le) cnt[v - lb] = rank[v];
}

__global__ void k_skel_compact(int lb, int le, const int* rank, const int* loc_off, int base,
                               const int* base_dev, const int64_t* ib_off, int64_t ib_level_base,
                               const int* tmp_lab, const double* tmp_pts, int64_t tmp_stride, int dim,
                               int* skel_off, int* skel, double* skel_pts, int64_t skel_stride) {
  int v = lb + blockIdx.x;
  if (v >= le) return;
  int o = (base_dev ? *base_dev : base) + loc_off[v - lb];
  if (threadIdx.x == 0) skel_off[v] = o;
  int k = rank[v];
  int64_t src = ib_off[v] - ib_level_base;
  for (int a = threadIdx.x; a < k; a += blockDim.x) {
    skel[o + a] = tmp_lab[src + a];
    for (int d = 0; d < dim; ++d)
      skel_pts[(size_t)d * skel_stride + o + a] = tmp_pts[(size_t)d * tmp_stride + src + a];
  }
}

__global__ void k_skel_bound(int n, int root, const int* pt_a, const int* pt_b, int kb,
                             int64_t* out) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  out[v] = v == root ? 0 : (int64_t)min(pt_b[v] - pt_a[v], kb);
}

__global__ void k_max_int(const int* x, int n, int* out) {
  int m = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    m = max(m, x[i]);
  for (int off = 16; off; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// host tables: cos/sin exactly as numpy evaluates them (lowrank.py:103-111)
struct HostTables {
  std::vector<double> cosv, wv;
  std::vector<int> order;
  int m = 0;
};

HostTables make_tables(int r, int dim) {
  HostTables H;
  int m;
  if (dim == 1) {
    m = r;
  } else if (dim == 2) {
    m = (int)std::ceil(std::sqrt((double)r));
  } else {
    m = 1;
    while (m * m * m < r) ++m;
  }
  H.m = m;
  for (int k = 0; k < m; ++k) {
    double arg = ((double)(2 * k + 1) * M_PI) / (double)(2 * m);
    H.cosv.push_back(std::cos(arg));
    H.wv.push_back(((k & 1) ? -1.0 : 1.0) * std::sin(arg));
  }
  // tensor order: sorted by (degree, i, j[, k]), first r (lowrank.py:143; 3-D extension)
  std::vector<std::array<int, 4>> idx;
  if (dim == 1) {
    for (int i = 0; i < r; ++i) idx.push_back({i, i, 0, 0});
  } else if (dim == 2) {
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) idx.push_back({i + j, i, j, 0});
  } else {
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j)
        for (int k = 0; k < m; ++k) idx.push_back({i + j + k, i, j, k});
  }
  std::sort(idx.begin(), idx.end());
  for (int q = 0; q < r; ++q) {
    H.order.push_back(idx[q][1]);
    H.order.push_back(idx[q][2]);
    H.order.push_back(idx[q][3]);
  }
  return H;
}

struct DevTables {
  DBuf<double> cosv, wv;
  DBuf<int> order;
  BasisTables view;
  void upload(const HostTables& H, cudaStream_t s) {
    cosv.alloc(H.cosv.size(), s); wv.alloc(H.wv.size(), s); order.alloc(H.order.size(), s);
    h2d(cosv.p, H.cosv.data(), H.cosv.size(), s);
    h2d(wv.p, H.wv.data(), H.wv.size(), s);
    h2d(order.p, H.order.data(), H.order.size(), s);
    view.cosv = cosv.p; view.wv = wv.p; view.order = order.p; view.m = H.m;
  }
};

void check_basis_params(int r, int dim) {
  SMASH_CHECK(r >= 1, SMASH_ERR_INVALID, "r must be positive");
  if (dim == 1)
    SMASH_CHECK(r <= MAX_M_AXIS_1D, SMASH_ERR_INVALID, "1-D interpolation supports r <= 128");
  HostTables H = make_tables(r, dim);
  if (dim > 1)
    SMASH_CHECK(H.m <= MAX_M_AXIS_ND, SMASH_ERR_INVALID, "interpolation grid too large (m > 16 per axis)");
  SMASH_CHECK((int)H.order.size() == 3 * r, SMASH_ERR_INVALID, "r exceeds the tensor grid");
}

double host_norm_fma(const double* v, int d) {
  double s = v[0] * v[0];
  for (int k = 1; k < d; ++k) s = std::fma(v[k], v[k], s);
  return std::sqrt(s);
}

void raise_dev_err(int e) {
  if (e & DEV_SWAP_CAP)
    throw Error(SMASH_ERR_NUMERICAL, "srrqr swap loop exceeded 200 iterations");
  if (e & DEV_DEGENERATE_BOX)
    throw Error(SMASH_ERR_NUMERICAL,
                "degenerate box dimension; interpolation nodes would coincide");
  if (e & DEV_CAPACITY) throw Error(SMASH_ERR_CUDA, "internal capacity exceeded");
  if (e) throw Error(SMASH_ERR_NUMERICAL, "numerical failure in construction");
}

int max_sm_smem() {
  int dev = 0, v = 0;
  SMASH_CUDA(cudaGetDevice(&dev));
  SMASH_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  return v;
}

int num_sms() {
  int dev = 0, v = 0;
  SMASH_CUDA(cudaGetDevice(&dev));
  SMASH_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
  return v;
}

}  // namespace

// Level-synchronous compression state of one side (row or column factors).
// Streams and events for the concurrent size-class launches of a level, pooled per device
// and handed to one SideBuild at a time.
struct PassResources {
  int dev = 0;
  cudaStream_t st[MAX_COMPRESS_PASSES] = {};
  cudaEvent_t ev[MAX_COMPRESS_PASSES + 1] = {};  // completion events, [MAX_COMPRESS_PASSES]: the fork
  static std::mutex& mu() { static std::mutex m; return m; }
  static std::vector<PassResources*>& pool() { static std::vector<PassResources*> p; return p; }
  static PassResources* acquire() {
    int dev = 0;
    SMASH_CUDA(cudaGetDevice(&dev));
    {
      std::lock_guard<std::mutex> g(mu());
      auto& p = pool();
      for (size_t i = 0; i < p.size(); ++i)
        if (p[i]->dev == dev) {
          PassResources* r = p[i];
          p.erase(p.begin() + i);
          return r;
        }
    }
    PassResources* r = new PassResources();
    r->dev = dev;
    for (cudaStream_t& x : r->st) SMASH_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    for (cudaEvent_t& e : r->ev) SMASH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return r;
  }
  static void release(PassResources* r) {  // (its work was joined into the build's stream)
    std::lock_guard<std::mutex> g(mu());
    pool().push_back(r);
  }
};

struct SideBuild {
  MatrixImpl* M;
  int side;
  SideFactors* F;
  const DevTables* tabs;
  double pad;
  cudaStream_t s;
  const int* pt_a;
  const int* pt_b;
  const double* P;
  int64_t Pn;
  int64_t skel_cap = 0, skel_used = 0;
  DBuf<char> tmp;
  DBuf<int> err, dmax;
  DBuf<unsigned long long> swaps;
  DBuf<double> gws;
  SvdWorkspace svdws;
  int smem_limit = 0, nsm = 0;
  // H2: every size of the level loop comes from host-side bounds computed once
  // from the tree (|ibar_v| <= sum_c min(r, |ibar_c|), leaves: their points), so
  // the whole sweep is enqueued without a host round trip; the device keeps the
  // running skeleton count.  HSS needs the SVD keep counts on the host.
  bool async = false;
  // level-distributed build (matrix_build_sharded): this rank's share of every level
  int shard_rank = 0, shard_world = 1;
  smash_exchange_fn xfn = nullptr;
  void* xctx = nullptr;
  std::vector<int64_t> lvl_ib_b, lvl_g_b, lvl_ib_base;
  std::vector<int> lvl_nmax_b;
  DBuf<int> d_used;
  PassResources* pres = nullptr;  // streams / events of a level's size-class launches
  ~SideBuild() {
    if (pres) PassResources::release(pres);
  }

  void init() {
    TreeImpl* t = M->tree;
    const int n = t->n_nodes, dim = t->dim, r = M->p.r;
    const bool hss = M->p.structure == SMASH_STRUCT_HSS;
    const bool col = side == 1 && !t->shared;
    pt_a = col ? t->col_a.p : t->row_a.p;
    pt_b = col ? t->col_b.p : t->row_b.p;
    P = col ? t->pts_col.p : t->pts_row.p;
    Pn = col ? t->ny : t->nx;
    F->nib.alloc(n, s); F->rank.alloc(n, s); F->ib_off.alloc(n, s); F->g_off.alloc(n, s);
    F->skel_off.alloc(n, s);
    F->rank.zero(s); F->nib.zero(s); F->ib_off.zero(s); F->g_off.zero(s); F->skel_off.zero(s);
    async = !hss && getenv("SMASH_BUILD_SYNC") == nullptr;
    if (async) {
      plan_bounds();  // host-side capacities (one round trip), skeleton capacity included
    } else {
      // skeleton capacity: k_v <= min(rows, |points below v|); HSS rows r + keep are bounded by |ibar|
      DBuf<int64_t> kb, kbs;
      kb.alloc(n + 1, s);
      kb.zero(s);
      kbs.alloc(1, s);
      k_skel_bound<<<cdiv(n, 128), 128, 0, s>>>(n, 0, pt_a, pt_b, hss ? (1 << 30) : r, kb.p);
      cub_call([&](void* tp, size_t& b) { return cub::DeviceReduce::Sum(tp, b, kb.p, kbs.p, n, s); },
               tmp, s);
      d2h(&skel_cap, kbs.p, 1, s);
      sync(s);
      F->perm.alloc(std::max<int64_t>(Pn * 2, 1024), s);
      // HSS (level-synchronous path): room for ~ (n_leaf - k) k G entries per leaf point
      // up front, so the leaf level does not reallocate + copy (grow() stays the fallback)
      F->G.alloc(std::max<int64_t>(Pn * (hss ? 32 : 8), 1024), s);
    }
    skel_cap = std::max<int64_t>(skel_cap, 1);
    F->skel_stride = skel_cap;
    F->skel.alloc(skel_cap, s);
    F->skel_pts.alloc((size_t)skel_cap * dim, s);
    F->level_skel_begin.assign(t->n_levels + 2, 0);
    err.alloc(1, s); err.zero(s);
    swaps.alloc(1, s); swaps.zero(s);
    dmax.alloc(1, s);
    smem_limit = max_sm_smem();
    nsm = num_sms();
  }

  void plan_bounds() {
    TreeImpl* t = M->tree;
    const int n = t->n_nodes, r = M->p.r, L = t->n_levels;
    std::vector<int> nch(n), cf(n), a(n), b(n);
    d2h(nch.data(), t->nchild.p, n, s);
    d2h(cf.data(), t->child_first.p, n, s);
    d2h(a.data(), pt_a, n, s);
    d2h(b.data(), pt_b, n, s);
    sync(s);
    // skeleton capacity (k_skel_bound): sum over non-root nodes of min(r, |points below|)
    skel_cap = 0;
    for (int v = 1; v < n; ++v) skel_cap += std::min<int64_t>(b[v] - a[v], r);
    std::vector<int64_t> bib(n, 0), bk(n, 0);
    for (int v = n - 1; v >= 0; --v) {  // BFS ids: children after their parent
      int64_t ib = 0;
      if (nch[v] == 0) ib = b[v] - a[v];
      else for (int c = 0; c < nch[v]; ++c) ib += bk[cf[v] + c];
      bib[v] = ib;
      bk[v] = std::min<int64_t>(ib, r);
    }
    std::vector<int64_t> ibo(n, 0), go(n, 0);
    lvl_ib_b.assign(L + 2, 0); lvl_g_b.assign(L + 2, 0); lvl_ib_base.assign(L + 2, 0);
    lvl_nmax_b.assign(L + 2, 1);
    int64_t ib_acc = 0, g_acc = 0;
    for (int l = L; l >= 2; --l) {
      lvl_ib_base[l] = ib_acc;
      for (int v = t->level_begin(l); v < t->level_end(l); ++v) {
        ibo[v] = ib_acc;
        go[v] = g_acc;
        ib_acc += bib[v];
        // (|ibar| - k) k with k <= min(r, |ibar|)
        const int64_t nb = bib[v];
        g_acc += 2 * std::min<int64_t>(nb, r) >= nb ? (nb / 2) * (nb - nb / 2) : (nb - r) * r;
        lvl_nmax_b[l] = std::max<int>(lvl_nmax_b[l], (int)bib[v]);
      }
      lvl_ib_b[l] = ib_acc - lvl_ib_base[l];
    }
    F->perm.alloc(std::max<int64_t>(ib_acc, 1), s);
    F->G.alloc(std::max<int64_t>(g_acc, 1), s);
    h2d(F->ib_off.p, ibo.data(), n, s);
    h2d(F->g_off.p, go.data(), n, s);
    F->ib_total = ib_acc;
    F->g_total = g_acc;
    d_used.alloc(1, s);
    d_used.zero(s);
  }

  // compress nodes [lb, le) of level l (a rank's owned range, or the whole
  // level); tmp_lab / tmp_pts receive the ordered skeleton labels / coordinates
  // at ib_off - lvl_ib_base[l] (row stride tmp_stride)
  void compress_range(int l, int lb, int le, int* tmp_lab, double* tmp_pts, int64_t tmp_stride) {
    TreeImpl* t = M->tree;
    const int dim = t->dim, r = M->p.r;
    const int cnt = le - lb;
    if (cnt <= 0) return;
    k_level_nib<<<cdiv(cnt, 128), 128, 0, s>>>(lb, le, t->nchild.p, t->child_first.p, pt_a, pt_b,
                                               F->rank.p, F->nib.p);
    CompressArgs A;
    A.lb = lb; A.le = le; A.dim = dim; A.r = r; A.side = side;
    A.nchild = t->nchild.p; A.child_first = t->child_first.p; A.pt_a = pt_a;
    A.lo = t->lo.p; A.hi = t->hi.p; A.pad = pad; A.half_pad = pad / 2;
    A.P = P; A.P_stride = Pn;
    A.Sk = F->skel_pts.p; A.S_stride = skel_cap; A.Slab = F->skel.p; A.skel_off = F->skel_off.p;
    A.nib = F->nib.p; A.ib_off = F->ib_off.p; A.g_off = F->g_off.p; A.ib_level_base = lvl_ib_base[l];
    A.tab = tabs->view;
    A.s_bound = M->p.s; A.rtol = M->p.rtol;
    A.rank = F->rank.p; A.perm = F->perm.p; A.G = F->G.p;
    A.tmp_lab = tmp_lab; A.tmp_pts = tmp_pts; A.tmp_stride = tmp_stride;
    A.err = err.p; A.swaps = swaps.p;
    A.nmax = std::max(lvl_nmax_b[l], 1);
    A.mmax = r;
    launch_level(A, cnt);
  }

  // compact level l's ordered skeletons (offsets stay on the device)
  void compact_level(int l, const int* tmp_lab, const double* tmp_pts, int64_t tmp_stride) {
    TreeImpl* t = M->tree;
    compact_range(l, t->level_begin(l), t->level_end(l), tmp_lab, tmp_pts, tmp_stride, d_used.p);
  }

  // compaction of nodes [lb, le) of level l at the device-resident base *used
  void compact_range(int l, int lb, int le, const int* tmp_lab, const double* tmp_pts,
                     int64_t tmp_stride, int* used) {
    TreeImpl* t = M->tree;
    const int cnt = le - lb;
    if (cnt <= 0) return;
    DBuf<int> rc, ro;
    rc.alloc(cnt + 1, s); ro.alloc(cnt + 1, s);
    SMASH_CUDA(cudaMemsetAsync(rc.p + cnt, 0, 4, s));
    k_rank_cnt<<<cdiv(cnt, 128), 128, 0, s>>>(lb, le, F->rank.p, rc.p);
    cub_call([&](void* tp, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(tp, b, rc.p, ro.p, cnt + 1, s);
    }, tmp, s);
    k_skel_compact<<<cnt, 128, 0, s>>>(lb, le, F->rank.p, ro.p, 0, used, F->ib_off.p,
                                       lvl_ib_base[l], tmp_lab, tmp_pts, tmp_stride, t->dim,
                                       F->skel_off.p, F->skel.p, F->skel_pts.p, skel_cap);
    k_skel_bump<<<1, 1, 0, s>>>(used, ro.p, cnt);
  }

  void level_async(int l) {
    TreeImpl* t = M->tree;
    const int64_t lvl_ib = std::max<int64_t>(lvl_ib_b[l], 1);
    DBuf<int> tmp_lab;
    DBuf<double> tmp_pts;
    tmp_lab.alloc(lvl_ib, s);
    tmp_pts.alloc((size_t)lvl_ib * t->dim, s);
    compress_range(l, t->level_begin(l), t->level_end(l), tmp_lab.p, tmp_pts.p, lvl_ib);
    compact_level(l, tmp_lab.p, tmp_pts.p, lvl_ib);
  }

  // The size-class launches of a level are independent: each runs on its own stream
  // (forked from s, joined back into s), so their tails overlap.  The streams and events
  // come from a per-device pool (creating them costs more than a small level's sweep).
  cudaStream_t pass_stream(int k) {
    if (!pres) pres = PassResources::acquire();
    return pres->st[k];
  }
  cudaEvent_t pass_event(int k) {
    if (!pres) pres = PassResources::acquire();
    return pres->ev[k];
  }

  void launch_level(CompressArgs& A, int cnt) {
    CompressPass ps[MAX_COMPRESS_PASSES];
    const int np = plan_compress_passes(A, cnt, smem_limit, nsm, ps);
    static const bool dbg = getenv("SMASH_COMPRESS_DBG") != nullptr;
#ifdef SMASH_COMPRESS_PROF
    const bool conc = false;
#else
    // (small levels: the fork / join costs more than the overlapping tails save)
    static const bool serial = getenv("SMASH_COMPRESS_SERIAL") != nullptr;
    static const int conc_min = getenv("SMASH_COMPRESS_CONC_MIN") ? atoi(getenv("SMASH_COMPRESS_CONC_MIN")) : 0;
    const bool conc = np > 1 && !dbg && !serial && cnt >= conc_min;
#endif
    // global workspace: one slice per launch (clusters' position tables, global/L2 panels)
    size_t need[MAX_COMPRESS_PASSES], tot = 0;
    for (int k = 0; k < np; ++k) {
      const CompressArgs& a = ps[k].a;
      need[k] = ps[k].rc.nt ? compress_rc_gws_doubles(ps[k].rc, ps[k].grid)
                            : a.panel_cap < (int64_t)a.nmax * a.mmax ? (size_t)ps[k].grid * a.mmax * a.nmax : 0;
      tot += need[k];
    }
    if (tot && gws.n < tot) gws.alloc(tot, s);
    if (conc) SMASH_CUDA(cudaEventRecord(pass_event(MAX_COMPRESS_PASSES), s));
    size_t goff = 0;
    for (int k = 0; k < np; ++k) {
      CompressArgs& a = ps[k].a;
      if (need[k]) { a.gws = gws.p + goff; goff += need[k]; }
      if (conc) {
        cudaStream_t sk = pass_stream(k);
        SMASH_CUDA(cudaStreamWaitEvent(sk, pass_event(MAX_COMPRESS_PASSES), 0));
        if (ps[k].rc.nt) launch_compress_rc(a, ps[k].rc, ps[k].grid, ps[k].smem, sk, k);
        else launch_compress(a, ps[k].grid, ps[k].smem, sk, k);
        SMASH_CUDA(cudaEventRecord(pass_event(k), sk));
        SMASH_CUDA(cudaStreamWaitEvent(s, pass_event(k), 0));
        continue;
      }
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      if (dbg) {
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
      }
      if (ps[k].rc.nt) launch_compress_rc(a, ps[k].rc, ps[k].grid, ps[k].smem, s);
      else launch_compress(a, ps[k].grid, ps[k].smem, s);
      if (dbg) {
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        {  // nodes and columns of this size class
          std::vector<int> hn(a.le - a.lb);
          cudaMemcpy(hn.data(), a.nib + a.lb, sizeof(int) * hn.size(), cudaMemcpyDeviceToHost);
          long long nn = 0, cols = 0;
          for (int x : hn) if (x > a.n_lo && x <= a.n_hi) { ++nn; cols += x; }
          fprintf(stderr, "  class holds %lld nodes, %lld columns (%.1f per node): %.2f us per node x CTA slot\n", nn, cols,
                  nn ? (double)cols / nn : 0.0, nn ? ms * 1e3 * ps[k].grid / nn : 0.0);
        }
        fprintf(stderr, "compress launch: %s nodes %d class (%d, %d] nmax %d mmax %d threads %d grid %d smem %zu cap %lld: %.3f ms\n",
                ps[k].rc.nt ? (ps[k].rc.cs > 1 ? "rcc" : ps[k].rc.rr > 32 ? "rc48" : "rc") : "sm", cnt, a.n_lo, a.n_hi, a.nmax, a.mmax, a.threads, ps[k].grid, ps[k].smem, (long long)a.panel_cap, ms);
        cudaEventDestroy(e0); cudaEventDestroy(e1);
      }
    }
  }

  void level(int l, NearSets* near) {
    if (async) {
      level_async(l);
      return;
    }
    TreeImpl* t = M->tree;
    const int dim = t->dim, r = M->p.r;
    const bool hss = M->p.structure == SMASH_STRUCT_HSS;
    const int lb = t->level_begin(l), le = t->level_end(l), cnt = le - lb;
    static const bool timing = getenv("SMASH_BUILD_TIMING") != nullptr;
    auto now = [&] {
      if (timing) sync(s);
      return std::chrono::steady_clock::now();
    };
    auto t0 = now();
    // level-distributed build: this rank's contiguous share of the level's nodes; the
    // level's outputs are zero elsewhere and summed over the ranks below
    const bool sharded = shard_world > 1;
    const int sub_lb = sharded ? lb + (int)((int64_t)cnt * shard_rank / shard_world) : lb;
    const int sub_le = sharded ? lb + (int)((int64_t)cnt * (shard_rank + 1) / shard_world) : le;

    // ---- HSS nearfield SVD (hss.py:279-299) first: the kept count bounds the rank
    // (the compression panel has r + keep rows) and so the G capacity
    int max_keep = 0;
    auto t1 = t0;
    if (hss) {
      k_level_nib<<<cdiv(cnt, 128), 128, 0, s>>>(lb, le, t->nchild.p, t->child_first.p, pt_a, pt_b,
                                                  F->rank.p, F->nib.p);
      dmax.zero(s);
      k_max_int<<<std::min<unsigned>(cdiv(cnt, 256), 64), 256, 0, s>>>(F->nib.p + lb, cnt, dmax.p);
      int nmax0 = 0;
      d2h(&nmax0, dmax.p, 1, s);
      sync(s);
      t1 = now();
      max_keep = hss_level_svd(M, side, l, near, nmax0, svdws, s, sub_lb, sub_le);
      if (sharded) {  // every rank sizes the level identically
        sync(s);
        void* ptrs[1] = {svdws.keep.p + lb};
        int64_t counts[1] = {cnt};
        int32_t dts[1] = {0};
        SMASH_CHECK(xfn(xctx, 1, ptrs, counts, dts) == 0, SMASH_ERR_CUDA, "sharded build exchange failed");
      }
    }
    auto t2 = now();

    DBuf<int64_t> ibc, gc, ibo, go;
    ibc.alloc(cnt + 1, s); gc.alloc(cnt + 1, s); ibo.alloc(cnt + 1, s); go.alloc(cnt + 1, s);
    SMASH_CUDA(cudaMemsetAsync(ibc.p + cnt, 0, 8, s));
    SMASH_CUDA(cudaMemsetAsync(gc.p + cnt, 0, 8, s));
    k_level_sizes<<<cdiv(cnt, 128), 128, 0, s>>>(lb, le, t->nchild.p, t->child_first.p, pt_a,
                                                 pt_b, F->rank.p, F->nib.p, ibc.p, gc.p, r,
                                                 hss ? svdws.keep.p : nullptr);
    cub_call([&](void* tp, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(tp, b, ibc.p, ibo.p, cnt + 1, s);
    }, tmp, s);
    cub_call([&](void* tp, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(tp, b, gc.p, go.p, cnt + 1, s);
    }, tmp, s);
    dmax.zero(s);
    k_max_int<<<std::min<unsigned>(cdiv(cnt, 256), 64), 256, 0, s>>>(F->nib.p + lb, cnt, dmax.p);
    int64_t tot[2];
    int nmax = 0;
    d2h(&tot[0], ibo.p + cnt, 1, s);
    d2h(&tot[1], go.p + cnt, 1, s);
    d2h(&nmax, dmax.p, 1, s);
    sync(s);
    const int64_t lvl_ib = tot[0], lvl_g = tot[1];
    grow(F->perm, F->ib_total, F->ib_total + lvl_ib, s);
    grow(F->G, F->g_total, F->g_total + lvl_g, s);
    k_add_base<<<cdiv(cnt, 128), 128, 0, s>>>(lb, le, ibo.p, F->ib_total, F->ib_off.p);
    k_add_base<<<cdiv(cnt, 128), 128, 0, s>>>(lb, le, go.p, F->g_total, F->g_off.p);

    DBuf<int> tmp_lab;
    DBuf<double> tmp_pts;
    tmp_lab.alloc(std::max<int64_t>(lvl_ib, 1), s);
    tmp_pts.alloc((size_t)std::max<int64_t>(lvl_ib, 1) * dim, s);
    if (sharded) {
      SMASH_CUDA(cudaMemsetAsync(F->rank.p + lb, 0, 4 * (size_t)cnt, s));
      SMASH_CUDA(cudaMemsetAsync(F->perm.p + F->ib_total, 0, 4 * (size_t)lvl_ib, s));
      SMASH_CUDA(cudaMemsetAsync(F->G.p + F->g_total, 0, 8 * (size_t)lvl_g, s));
      tmp_lab.zero(s);
      tmp_pts.zero(s);
    }

    CompressArgs A;
    A.lb = lb; A.le = le; A.dim = dim; A.r = r; A.side = side;
    A.nchild = t->nchild.p; A.child_first = t->child_first.p; A.pt_a = pt_a;
    A.lo = t->lo.p; A.hi = t->hi.p; A.pad = pad; A.half_pad = pad / 2;
    A.P = P; A.P_stride = Pn;
    A.Sk = F->skel_pts.p; A.S_stride = skel_cap; A.Slab = F->skel.p; A.skel_off = F->skel_off.p;
    A.nib = F->nib.p; A.ib_off = F->ib_off.p; A.g_off = F->g_off.p; A.ib_level_base = F->ib_total;
    if (hss) { A.keep = svdws.keep.p; A.sv_off = svdws.sv_off.p; A.sv = svdws.sv.p; }
    A.tab = tabs->view;
    A.s_bound = M->p.s; A.rtol = M->p.rtol;
    A.rank = F->rank.p; A.perm = F->perm.p; A.G = F->G.p;
    A.tmp_lab = tmp_lab.p; A.tmp_pts = tmp_pts.p; A.tmp_stride = std::max<int64_t>(lvl_ib, 1);
    A.err = err.p; A.swaps = swaps.p;
    A.nmax = std::max(nmax, 1);
    A.mmax = r + max_keep;
    if (sharded) {
      A.lb = sub_lb;
      A.le = sub_le;
      if (sub_le > sub_lb) launch_level(A, sub_le - sub_lb);
      // the cut-level exchange of this level: ranks, perm, G, ordered skeleton labels and
      // coordinates (disjoint shares summed), error flags (maximum)
      sync(s);
      void* ptrs[6] = {F->rank.p + lb, F->perm.p + F->ib_total, F->G.p + F->g_total, tmp_lab.p,
                       tmp_pts.p, err.p};
      int64_t counts[6] = {cnt, lvl_ib, lvl_g, lvl_ib, lvl_ib * dim, 1};
      int32_t dts[6] = {0, 0, 1, 0, 1, 3};
      SMASH_CHECK(xfn(xctx, 6, ptrs, counts, dts) == 0, SMASH_ERR_CUDA, "sharded build exchange failed");
    } else {
      launch_level(A, cnt);
    }
    auto t3 = now();
    if (timing)
      fprintf(stderr, "level %d side %d cnt %d: nib %.3f ms svd %.3f ms sizes+compress %.3f ms\n", l, side,
              cnt, std::chrono::duration<double, std::milli>(t1 - t0).count(),
              std::chrono::duration<double, std::milli>(t2 - t1).count(),
              std::chrono::duration<double, std::milli>(t3 - t2).count());

    // ---- compact this level's skeletons
    DBuf<int> rc, ro;
    rc.alloc(cnt + 1, s); ro.alloc(cnt + 1, s);
    SMASH_CUDA(cudaMemsetAsync(rc.p + cnt, 0, 4, s));
    k_rank_cnt<<<cdiv(cnt, 128), 128, 0, s>>>(lb, le, F->rank.p, rc.p);
    cub_call([&](void* tp, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(tp, b, rc.p, ro.p, cnt + 1, s);
    }, tmp, s);
    int lvl_k = 0, herr = 0;
    d2h(&lvl_k, ro.p + cnt, 1, s);
    d2h(&herr, err.p, 1, s);
    sync(s);
    raise_dev_err(herr);
    SMASH_CHECK(skel_used + lvl_k <= skel_cap, SMASH_ERR_CUDA, "skeleton capacity exceeded");
    F->level_skel_begin[l] = skel_used;
    k_skel_compact<<<cnt, 128, 0, s>>>(lb, le, F->rank.p, ro.p, (int)skel_used, nullptr, F->ib_off.p,
                                       F->ib_total, tmp_lab.p, tmp_pts.p, A.tmp_stride, dim,
                                       F->skel_off.p, F->skel.p, F->skel_pts.p, skel_cap);
    skel_used += lvl_k;
    F->ib_total += lvl_ib;
    F->g_total += lvl_g;
  }

  void finish() {
    if (shard_world > 1) {  // the rank's pivot-swap count -> the job's
      sync(s);
      void* ptrs[1] = {swaps.p};
      int64_t counts[1] = {1};
      int32_t dts[1] = {2};
      SMASH_CHECK(xfn(xctx, 1, ptrs, counts, dts) == 0, SMASH_ERR_CUDA, "sharded build exchange failed");
    }
    unsigned long long hs = 0;
    int used = 0, herr = 0;
    d2h(&hs, swaps.p, 1, s);
    d2h(&herr, err.p, 1, s);
    if (async) d2h(&used, d_used.p, 1, s);
    sync(s);
    raise_dev_err(herr);
    if (async) skel_used = used;
    SMASH_CHECK(skel_used <= skel_cap, SMASH_ERR_CUDA, "skeleton capacity exceeded");
    F->level_skel_begin[1] = skel_used;
    F->skel_total = skel_used;
    F->swaps = (int64_t)hs;
    SMASH_CUDA(cudaGetLastError());
  }
};

// get_pairs on its own host thread and stream (see matrix_build)
// A persistent helper thread per device with its own high-priority stream: runs
// get_pairs while the calling thread enqueues the compression sweep (matrix_build).
// Created on first use and kept for the life of the process (no per-build thread
// or stream creation on the build's critical path).
struct PairsWorker {
  std::mutex job_mu;  // one job at a time per device
  std::mutex mu;
  std::condition_variable cv;
  std::function<void()> task;
  bool has = false, done = true;
  cudaStream_t s2 = nullptr;
  cudaEvent_t ev = nullptr;
  explicit PairsWorker(int dev) {
    int lo = 0, hi = 0;
    SMASH_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    SMASH_CUDA(cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, hi));
    SMASH_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    std::thread([this, dev] {
      cudaSetDevice(dev);
      std::unique_lock<std::mutex> lk(mu);
      for (;;) {
        cv.wait(lk, [this] { return has; });
        has = false;
        auto f = std::move(task);
        lk.unlock();
        f();
        lk.lock();
        done = true;
        cv.notify_all();
      }
    }).detach();
  }
  static PairsWorker& get(int dev) {
    static std::mutex reg_mu;
    static PairsWorker* w[64] = {};
    std::lock_guard<std::mutex> g(reg_mu);
    SMASH_CHECK(dev >= 0 && dev < 64, SMASH_ERR_INVALID, "device index out of range");
    if (!w[dev]) w[dev] = new PairsWorker(dev);
    return *w[dev];
  }
  void submit(std::function<void()> f) {
    std::lock_guard<std::mutex> lk(mu);
    task = std::move(f);
    has = true;
    done = false;
    cv.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [this] { return done; });
  }
};

// get_pairs on the device's helper thread and stream (see matrix_build)
struct PairsJob {
  PairsWorker* w = nullptr;
  std::unique_lock<std::mutex> hold;
  PairLists* out = nullptr;
  std::exception_ptr err;
  bool pending = false;
  void start(TreeImpl* t, double tau, int structure, cudaStream_t s) {
    int dev = 0;
    SMASH_CUDA(cudaGetDevice(&dev));
    w = &PairsWorker::get(dev);
    hold = std::unique_lock<std::mutex>(w->job_mu);
    SMASH_CUDA(cudaEventRecord(w->ev, s));  // the tree is complete on s
    SMASH_CUDA(cudaStreamWaitEvent(w->s2, w->ev, 0));
    cudaStream_t s2 = w->s2;
    w->submit([this, t, tau, structure, s2] {
      try {
        out = get_pairs(t, tau, structure, s2);
      } catch (...) {
        err = std::current_exception();
      }
    });
    pending = true;
  }
  PairLists* join(cudaStream_t s) {
    w->wait();
    pending = false;
    if (!err) {
      out->rehome(s);  // released on the owner's stream later
      SMASH_CUDA(cudaEventRecord(w->ev, w->s2));
      SMASH_CUDA(cudaStreamWaitEvent(s, w->ev, 0));
    }
    if (err) std::rethrow_exception(err);
    return out;
  }
  ~PairsJob() {
    if (pending && w) w->wait();
  }
};

// The level sweep of matrix_build; with world > 1 (HSS only) every level is split over
// the ranks and summed through fn (matrix_build_sharded).
static MatrixImpl* build_levels(TreeImpl* t, const smash_build_params& p, cudaStream_t s, int rank,
                                int world, smash_exchange_fn fn, void* ctx) {
  SMASH_CHECK(p.kernel >= SMASH_KERNEL_LOG && p.kernel <= SMASH_KERNEL_CAUCHY, SMASH_ERR_INVALID,
              "unknown kernel kind");
  SMASH_CHECK(p.structure == SMASH_STRUCT_H2 || p.structure == SMASH_STRUCT_HSS,
              SMASH_ERR_INVALID, "structure must be 'hss' or 'h2'");
  if (p.kernel == SMASH_KERNEL_CAUCHY)
    SMASH_CHECK(t->dim == 1, SMASH_ERR_INVALID, "the real Cauchy kernel needs 1-D points");
  if (p.structure == SMASH_STRUCT_H2)
    SMASH_CHECK(t->mode == SMASH_MODE_2D || t->dim == 1, SMASH_ERR_INVALID,
                "H2 construction expects a 2^d-mode tree");
  check_basis_params(p.r, t->dim);
  init_pool();
  std::unique_ptr<MatrixImpl> M(new MatrixImpl());
  M->tree = t;
  M->p = p;
  const bool hss_build = p.structure == SMASH_STRUCT_HSS;
  // H2: the pair lists (a host-synchronising frontier sweep, independent of the
  // compression) are built by a second host thread on a high-priority stream
  // while this thread enqueues the compression sweep; HSS needs them first (N_i).
  PairsJob pj;
  if (hss_build) M->pl = get_pairs(t, p.tau, p.structure, s);
  else pj.start(t, p.tau, p.structure, s);
  HostTables H = make_tables(p.r, t->dim);
  DevTables D;
  D.upload(H, s);
  // pad = max(1e-9 * diam, 1e-300), diam = 2 * root radius (hss.py:221-222)
  double w[3];
  for (int a = 0; a < t->dim; ++a) w[a] = t->root_hi[a] - t->root_lo[a];
  double diam = 2 * (0.5 * host_norm_fma(w, t->dim));
  double pad = std::max(1e-9 * diam, 1e-300);
  const bool hss = p.structure == SMASH_STRUCT_HSS;
  // Shared points: H2 skeletons are kernel independent and HSS ones depend on the
  // kernel only through the nearfield block, so the column factors equal the row
  // factors whenever the kernel is symmetric (all but the Cauchy kernel).
  const bool alias = t->shared && (!hss || p.kernel != SMASH_KERNEL_CAUCHY);
  M->colf = alias ? &M->rowf : &M->colf_own;
  NearSets* near = hss ? get_near(t, p.tau, s) : nullptr;
  SideBuild rowb{M.get(), 0, &M->rowf, &D, pad, s};
  rowb.init();
  std::unique_ptr<SideBuild> colb;
  if (!alias) {
    colb.reset(new SideBuild{M.get(), 1, &M->colf_own, &D, pad, s});
    colb->init();
  }
  for (SideBuild* b : {&rowb, colb.get()})
    if (b) { b->shard_rank = rank; b->shard_world = world; b->xfn = fn; b->xctx = ctx; }
  // row and column passes interleave per level: the HSS row pass at level l
  // reads the column side's level-(l+1) skeletons and vice versa (hss.py:274-299)
  for (int l = t->n_levels; l >= 2; --l) {
    rowb.level(l, near);
    if (colb) colb->level(l, near);
  }
  static const bool jdbg = getenv("SMASH_JOIN_DBG") != nullptr;
  auto tj0 = std::chrono::steady_clock::now();
  if (!hss_build) M->pl = pj.join(s);
  auto tj1 = std::chrono::steady_clock::now();
  rowb.finish();
  if (jdbg)
    fprintf(stderr, "build: waited %.3f ms for the pair lists after enqueueing the sweep, %.3f ms more for the sweep\n",
            std::chrono::duration<double, std::milli>(tj1 - tj0).count(),
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tj1).count());
  if (colb) colb->finish();
  sync(s);
  return M.release();
}

MatrixImpl* matrix_build(TreeImpl* t, const smash_build_params& p, cudaStream_t s) {
  return build_levels(t, p, s, 0, 1, nullptr, nullptr);
}

MatrixImpl* matrix_build_sharded(TreeImpl* t, const smash_build_params& p, int rank, int world,
                                 smash_exchange_fn fn, void* ctx, cudaStream_t s) {
  SMASH_CHECK(p.structure == SMASH_STRUCT_HSS, SMASH_ERR_INVALID,
              "level-distributed construction builds HSS matrices (H2: smash_matrix_build_local)");
  SMASH_CHECK(world >= 1 && rank >= 0 && rank < world && fn, SMASH_ERR_INVALID,
              "bad rank / world size / exchange function");
  return build_levels(t, p, s, rank, world, fn, ctx);
}

// ---------------------------------------------------------------------------
// Sharded construction: levels are stored level-major, so the
// subtrees under a contiguous range of cut-level nodes occupy one contiguous
// node range at every deeper level.  Rank r compresses its ranges of levels
// L..cut with no data movement (the host-side capacity layout gives every node
// a fixed slot in perm / G / the skeleton temporaries), the caller sums the
// disjoint, zero-initialised buffers over the ranks (one all-reduce each), and
// finish() compacts the cut levels and compresses the few top levels
// redundantly on every rank.
// ---------------------------------------------------------------------------
struct ShardState {
  DevTables D;
  std::unique_ptr<SideBuild> rowb;
  int cut = 0, rank = 0, world = 1;
  bool replicate = true;            // exchange perm and G too (every rank holds the full matrix)
  std::vector<int> own_lb, own_le;  // per level l (>= cut): owned BFS range
  DBuf<int> tmp_lab;                // ordered skeleton labels of levels L..cut (perm layout)
  DBuf<double> tmp_pts;             // [dim][tmp_len]
  int64_t tmp_len = 1, perm_len = 1, g_len = 1;
  DBuf<long long> swaps64;          // exchanged counters
  DBuf<int> err32;
};

MatrixImpl* matrix_build_local(TreeImpl* t, const smash_build_params& p, int rank, int world,
                               int cut_level, const double* cut_weight, int replicate,
                               cudaStream_t s) {
  SMASH_CHECK(p.structure == SMASH_STRUCT_H2, SMASH_ERR_INVALID,
              "sharded construction supports the H2 structure");
  SMASH_CHECK(world >= 1 && rank >= 0 && rank < world, SMASH_ERR_INVALID, "bad rank / world size");
  SMASH_CHECK(t->mode == SMASH_MODE_2D || t->dim == 1, SMASH_ERR_INVALID,
              "H2 construction expects a 2^d-mode tree");
  SMASH_CHECK(p.kernel >= SMASH_KERNEL_LOG && p.kernel <= SMASH_KERNEL_CAUCHY, SMASH_ERR_INVALID,
              "unknown kernel kind");
  check_basis_params(p.r, t->dim);
  init_pool();
  std::unique_ptr<MatrixImpl> M(new MatrixImpl());
  M->tree = t;
  M->p = p;
  M->pl = get_pairs(t, p.tau, p.structure, s);
  std::shared_ptr<ShardState> st(new ShardState());
  st->D.upload(make_tables(p.r, t->dim), s);
  double w[3];
  for (int a = 0; a < t->dim; ++a) w[a] = t->root_hi[a] - t->root_lo[a];
  const double pad = std::max(1e-9 * (2 * (0.5 * host_norm_fma(w, t->dim))), 1e-300);
  M->colf = t->shared ? &M->rowf : &M->colf_own;
  SMASH_CHECK(t->shared, SMASH_ERR_INVALID, "sharded construction expects shared row/column points");
  st->rowb.reset(new SideBuild{M.get(), 0, &M->rowf, &st->D, pad, s});
  st->rowb->init();  // H2 -> capacity layout (async path)
  SideBuild& B = *st->rowb;
  SMASH_CHECK(B.async, SMASH_ERR_INVALID, "sharded construction needs the capacity layout");
  const int L = t->n_levels;
  // cut level: the shallowest level with >= 8 nodes per rank (else the leaves' level)
  int cut = L;
  for (int l = 2; l <= L; ++l)
    if (t->level_end(l) - t->level_begin(l) >= 8 * world) { cut = l; break; }
  if (cut_level >= 2 && cut_level <= L) cut = cut_level;
  st->cut = cut;
  st->rank = rank;
  st->world = world;
  st->replicate = replicate != 0;
  // balance contiguous cut-level ranges by the caller's per-node weights (left to right,
  // e.g. the subtrees' coupling + nearfield work), else by subtree point counts
  const int n = t->n_nodes;
  std::vector<int> ra(n), rb(n), par(n);
  d2h(ra.data(), t->row_a.p, n, s);
  d2h(rb.data(), t->row_b.p, n, s);
  d2h(par.data(), t->parent.p, n, s);
  sync(s);
  const int cb = t->level_begin(cut), ce = t->level_end(cut);
  std::vector<int> owner(n, -1);
  auto weight = [&](int v) { return cut_weight ? cut_weight[v - cb] : (double)(rb[v] - ra[v]); };
  double total = 0;
  for (int v = cb; v < ce; ++v) total += weight(v);
  double acc = 0;
  for (int v = cb; v < ce; ++v) {
    const double mid = acc + 0.5 * weight(v);
    owner[v] = std::min(world - 1, (int)(mid * world / std::max(total, 1e-300)));
    acc += weight(v);
  }
  st->own_lb.assign(L + 2, 0);
  st->own_le.assign(L + 2, 0);
  for (int l = cut; l <= L; ++l) {
    if (l > cut)  // inherit the owner of the parent (parents at level l - 1)
      for (int v = t->level_begin(l); v < t->level_end(l); ++v) owner[v] = owner[par[v]];
    int lo = -1, hi = -1;
    for (int v = t->level_begin(l); v < t->level_end(l); ++v)
      if (owner[v] == rank) { if (lo < 0) lo = v; hi = v + 1; }
    st->own_lb[l] = lo < 0 ? 0 : lo;
    st->own_le[l] = lo < 0 ? 0 : hi;
  }
  M->shard_owner = owner;  // BFS: rank owning the subtree, -1 above the cut (replicated)
  // exchanged buffers: zero them (owned slots are written, the rest stays 0)
  st->perm_len = std::max<int64_t>(B.lvl_ib_base[cut] + B.lvl_ib_b[cut], 1);
  st->g_len = std::max<int64_t>(M->rowf.g_total, 1);  // whole G (top levels are zero too)
  st->tmp_len = st->perm_len;
  st->tmp_lab.alloc(st->tmp_len, s);
  st->tmp_pts.alloc((size_t)st->tmp_len * t->dim, s);
  st->tmp_lab.zero(s);
  st->tmp_pts.zero(s);
  SMASH_CUDA(cudaMemsetAsync(M->rowf.perm.p, 0, 4 * (size_t)st->perm_len, s));
  SMASH_CUDA(cudaMemsetAsync(M->rowf.G.p, 0, 8 * (size_t)st->g_len, s));
  // local compaction of the owned ranges (parents read their children's skeletons
  // from the compact arrays); finish() rebuilds the global compact layout
  DBuf<int> used_loc;
  used_loc.alloc(1, s);
  used_loc.zero(s);
  for (int l = L; l >= cut; --l) {
    B.compress_range(l, st->own_lb[l], st->own_le[l], st->tmp_lab.p + B.lvl_ib_base[l],
                     st->tmp_pts.p + B.lvl_ib_base[l], st->tmp_len);
    B.compact_range(l, st->own_lb[l], st->own_le[l], st->tmp_lab.p + B.lvl_ib_base[l],
                    st->tmp_pts.p + B.lvl_ib_base[l], st->tmp_len, used_loc.p);
  }
  st->swaps64.alloc(1, s);
  st->err32.alloc(1, s);
  SMASH_CUDA(cudaMemcpyAsync(st->swaps64.p, B.swaps.p, 8, cudaMemcpyDeviceToDevice, s));
  SMASH_CUDA(cudaMemcpyAsync(st->err32.p, B.err.p, 4, cudaMemcpyDeviceToDevice, s));
  sync(s);
  M->pending = st;
  return M.release();
}

void matrix_exchange_buffers(MatrixImpl* m, std::vector<ExchangeBuf>& out) {
  SMASH_CHECK(m->pending, SMASH_ERR_INVALID, "matrix has no pending sharded build");
  ShardState* st = static_cast<ShardState*>(m->pending.get());
  const int n = m->tree->n_nodes;
  out.clear();
  out.push_back({m->rowf.rank.p, (int64_t)n, 0});
  out.push_back({m->rowf.nib.p, (int64_t)n, 0});
  if (st->replicate) out.push_back({m->rowf.perm.p, st->perm_len, 0});
  out.push_back({st->tmp_lab.p, st->tmp_len, 0});
  out.push_back({st->err32.p, 1, 0});
  if (st->replicate) out.push_back({m->rowf.G.p, st->g_len, 1});
  out.push_back({st->tmp_pts.p, st->tmp_len * m->tree->dim, 1});
  out.push_back({st->swaps64.p, 1, 2});
}

void matrix_build_finish(MatrixImpl* m, cudaStream_t s) {
  SMASH_CHECK(m->pending, SMASH_ERR_INVALID, "matrix has no pending sharded build");
  ShardState* st = static_cast<ShardState*>(m->pending.get());
  SideBuild& B = *st->rowb;
  B.s = s;
  SMASH_CUDA(cudaMemcpyAsync(B.swaps.p, st->swaps64.p, 8, cudaMemcpyDeviceToDevice, s));
  SMASH_CUDA(cudaMemcpyAsync(B.err.p, st->err32.p, 4, cudaMemcpyDeviceToDevice, s));
  const int L = m->tree->n_levels;
  for (int l = L; l >= st->cut; --l)
    B.compact_level(l, st->tmp_lab.p + B.lvl_ib_base[l], st->tmp_pts.p + B.lvl_ib_base[l], st->tmp_len);
  for (int l = st->cut - 1; l >= 2; --l) B.level(l, nullptr);
  B.finish();
  sync(s);
  m->pending.reset();
}

// ---------------------------------------------------------------------------
// export (postorder)
// ---------------------------------------------------------------------------
namespace {

__global__ void k_exp_counts(int n, int root, const int* post, const int* nib, const int* rank,
                             const int64_t* g_off_unused, int64_t* has, int64_t* rk, int64_t* cp,
                             int64_t* cs, int64_t* cg) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  int p = post[v];
  bool h = v != root;
  int k = h ? rank[v] : 0, ni = h ? nib[v] : 0;
  if (has) has[p] = h ? 1 : 0;
  if (rk) rk[p] = k;
  cp[p] = ni;
  cs[p] = k;
  cg[p] = (int64_t)(ni - k) * k;
  (void)g_off_unused;
}

__global__ void k_exp_copy(int n, int root, const int* post, const int* nib, const int* rank,
                           const int64_t* ib_off, const int64_t* g_off, const int* skel_off,
                           const int* perm, const double* G, const int* skel, const int64_t* pp,
                           const int64_t* sp, const int64_t* gp, int64_t* operm, int64_t* oskel,
                           double* oG) {
  int v = blockIdx.x;
  if (v >= n || v == root) return;
  int p = post[v];
  int ni = nib[v], k = rank[v];
  if (operm)
    for (int c = threadIdx.x; c < ni; c += blockDim.x) operm[pp[p] + c] = perm[ib_off[v] + c];
  if (oskel)
    for (int a = threadIdx.x; a < k; a += blockDim.x) oskel[sp[p] + a] = skel[skel_off[v] + a];
  if (oG) {
    int64_t ng = (int64_t)(ni - k) * k;
    for (int64_t e = threadIdx.x; e < ng; e += blockDim.x) oG[gp[p] + e] = G[g_off[v] + e];
  }
}

}  // namespace

void matrix_export(MatrixImpl* m, int side, int64_t* has, int64_t* rank, int64_t* perm_ptr,
                   int64_t* perm, int64_t* skel_ptr, int64_t* skel, int64_t* g_ptr, double* G,
                   cudaStream_t s) {
  TreeImpl* t = m->tree;
  SideFactors& F = side == 0 ? m->rowf : *m->colf;
  const int n = t->n_nodes;
  DBuf<int64_t> cp, cs, cg, pp, sp, gp;
  cp.alloc(n + 1, s); cs.alloc(n + 1, s); cg.alloc(n + 1, s);
  cp.zero(s); cs.zero(s); cg.zero(s);
  k_exp_counts<<<cdiv(n, 128), 128, 0, s>>>(n, 0, t->post.p, F.nib.p, F.rank.p, F.g_off.p, has,
                                            rank, cp.p, cs.p, cg.p);
  DBuf<char> tmp;
  auto scan = [&](DBuf<int64_t>& in, int64_t* out, DBuf<int64_t>& own) {
    int64_t* dst = out;
    if (!dst) { own.alloc(n + 1, s); dst = own.p; }
    cub_call([&](void* tp, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(tp, b, in.p, dst, n + 1, s);
    }, tmp, s);
    return dst;
  };
  int64_t* ppp = scan(cp, perm_ptr, pp);
  int64_t* spp = scan(cs, skel_ptr, sp);
  int64_t* gpp = scan(cg, g_ptr, gp);
  k_exp_copy<<<std::max(n, 1), 128, 0, s>>>(n, 0, t->post.p, F.nib.p, F.rank.p, F.ib_off.p,
                                            F.g_off.p, F.skel_off.p, F.perm.p, F.G.p, F.skel.p,
                                            ppp, spp, gpp, perm, skel, G);
  sync(s);
  SMASH_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// Import of saved factors (container load, smash/container.py:135-211): the
// inverse of matrix_export.  Factors arrive postorder-indexed on the host; they
// are laid out like a level-synchronous build (levels L..2, BFS order within a
// level) so a parent's ibar is its children's consecutive compact skeletons.
// ---------------------------------------------------------------------------
namespace {
__global__ void k_gather_skel_pts(int64_t n, int dim, const int* lab, const double* P, int64_t Pn,
                                  double* out, int64_t stride) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int d = 0; d < dim; ++d) out[(size_t)d * stride + i] = P[(size_t)d * Pn + lab[i]];
}

void import_side(TreeImpl* t, int side, const ImportSide& in, SideFactors& F, cudaStream_t s) {
  const int n = t->n_nodes, L = t->n_levels;
  std::vector<int> post(n), nch(n), cf(n), a(n), b(n);
  const bool col = side == 1 && !t->shared;
  d2h(post.data(), t->post.p, n, s);
  d2h(nch.data(), t->nchild.p, n, s);
  d2h(cf.data(), t->child_first.p, n, s);
  d2h(a.data(), col ? t->col_a.p : t->row_a.p, n, s);
  d2h(b.data(), col ? t->col_b.p : t->row_b.p, n, s);
  sync(s);
  std::vector<int> nib(n, 0), rk(n, 0), skoff(n, 0);
  std::vector<int64_t> iboff(n, 0), goff(n, 0);
  std::vector<int> perm, skel;
  std::vector<double> G;
  F.level_skel_begin.assign(L + 2, 0);
  int64_t ib = 0, g = 0, sk = 0;
  for (int l = L; l >= 2; --l) {
    F.level_skel_begin[l] = sk;
    for (int v = t->level_begin(l); v < t->level_end(l); ++v) {
      const int pi = post[v];
      const int64_t p0 = in.perm_ptr[pi], p1 = in.perm_ptr[pi + 1];
      const int64_t s0 = in.skel_ptr[pi], s1 = in.skel_ptr[pi + 1];
      const int64_t g0 = in.g_ptr[pi], g1 = in.g_ptr[pi + 1];
      const int64_t ni = p1 - p0, k = in.rank[pi];
      int64_t want = 0;
      if (nch[v] == 0) want = b[v] - a[v];
      else for (int c = 0; c < nch[v]; ++c) want += rk[cf[v] + c];
      SMASH_CHECK(ni == want, SMASH_ERR_INVALID,
                  "imported factor: |ibar| of node " + std::to_string(pi) + " is " +
                      std::to_string(ni) + ", the tree implies " + std::to_string(want));
      SMASH_CHECK(k >= 0 && k <= ni && s1 - s0 == k && g1 - g0 == (ni - k) * k, SMASH_ERR_INVALID,
                  "imported factor: inconsistent rank / skeleton / G sizes at node " + std::to_string(pi));
      nib[v] = (int)ni; rk[v] = (int)k;
      iboff[v] = ib; goff[v] = g; skoff[v] = (int)sk;
      for (int64_t e = p0; e < p1; ++e) {
        SMASH_CHECK(in.perm[e] >= 0 && in.perm[e] < ni, SMASH_ERR_INVALID,
                    "imported factor: permutation entry out of range at node " + std::to_string(pi));
        perm.push_back((int)in.perm[e]);
      }
      const int64_t npts = col ? t->ny : t->nx;
      for (int64_t e = s0; e < s1; ++e) {
        SMASH_CHECK(in.skel[e] >= 0 && in.skel[e] < npts, SMASH_ERR_INVALID,
                    "imported factor: skeleton label out of range at node " + std::to_string(pi));
        skel.push_back((int)in.skel[e]);
      }
      G.insert(G.end(), in.G + g0, in.G + g1);
      ib += ni; g += (ni - k) * k; sk += k;
    }
  }
  F.level_skel_begin[1] = sk;
  F.nib.alloc(n, s); F.rank.alloc(n, s); F.ib_off.alloc(n, s); F.g_off.alloc(n, s);
  F.skel_off.alloc(n, s);
  h2d(F.nib.p, nib.data(), n, s); h2d(F.rank.p, rk.data(), n, s);
  h2d(F.ib_off.p, iboff.data(), n, s); h2d(F.g_off.p, goff.data(), n, s);
  h2d(F.skel_off.p, skoff.data(), n, s);
  F.perm.alloc(std::max<int64_t>(ib, 1), s);
  F.G.alloc(std::max<int64_t>(g, 1), s);
  F.skel.alloc(std::max<int64_t>(sk, 1), s);
  F.skel_stride = std::max<int64_t>(sk, 1);
  F.skel_pts.alloc((size_t)F.skel_stride * t->dim, s);
  if (ib) h2d(F.perm.p, perm.data(), ib, s);
  if (g) h2d(F.G.p, G.data(), g, s);
  if (sk) {
    h2d(F.skel.p, skel.data(), sk, s);
    k_gather_skel_pts<<<std::min<int64_t>(cdiv(sk, 256), 4096), 256, 0, s>>>(
        sk, t->dim, F.skel.p, col ? t->pts_col.p : t->pts_row.p, col ? t->ny : t->nx,
        F.skel_pts.p, F.skel_stride);
  }
  F.ib_total = ib; F.g_total = g; F.skel_total = sk; F.swaps = 0;
  sync(s);  // the host staging vectors go out of scope
  SMASH_CUDA(cudaGetLastError());
}
}  // namespace

MatrixImpl* matrix_import(TreeImpl* t, const smash_build_params& p, const ImportSide* sides,
                          int nsides, cudaStream_t s) {
  SMASH_CHECK(p.kernel >= SMASH_KERNEL_LOG && p.kernel <= SMASH_KERNEL_CAUCHY, SMASH_ERR_INVALID,
              "unknown kernel kind");
  SMASH_CHECK(p.structure == SMASH_STRUCT_H2 || p.structure == SMASH_STRUCT_HSS,
              SMASH_ERR_INVALID, "structure must be 'hss' or 'h2'");
  SMASH_CHECK(nsides == 1 || nsides == 2, SMASH_ERR_INVALID, "one (shared) or two factor sides");
  SMASH_CHECK(nsides == 2 || t->shared, SMASH_ERR_INVALID,
              "distinct row/column points need both factor sides");
  init_pool();
  std::unique_ptr<MatrixImpl> M(new MatrixImpl());
  M->tree = t;
  M->p = p;
  M->pl = get_pairs(t, p.tau, p.structure, s);
  import_side(t, 0, sides[0], M->rowf, s);
  if (nsides == 2) {
    import_side(t, 1, sides[1], M->colf_own, s);
    M->colf = &M->colf_own;
  } else {
    M->colf = &M->rowf;
  }
  return M.release();
}

// ---------------------------------------------------------------------------
// single-call primitives
// ---------------------------------------------------------------------------
void interp_basis_single(int dim, const double* lo, const double* hi, const double* pts, int64_t n,
                         int r, double* out, cudaStream_t s) {
  SMASH_CHECK(dim >= 1 && dim <= 3, SMASH_ERR_INVALID, "interpolation basis supports d <= 3");
  check_basis_params(r, dim);
  double scale = 1.0;
  for (int a = 0; a < dim; ++a) scale = std::max(scale, hi[a] - lo[a]);
  for (int a = 0; a < dim; ++a)
    SMASH_CHECK(hi[a] - lo[a] > 1e-14 * scale, SMASH_ERR_INVALID,
                "degenerate box dimension; interpolation nodes would coincide");
  HostTables H = make_tables(r, dim);
  DevTables D;
  D.upload(H, s);
  DBuf<double> soa;
  soa.alloc(std::max<int64_t>(n * dim, 1), s);
  // AoS (n, dim) -> SoA
  std::vector<double> dummy;
  (void)dummy;
  if (n) {
    // transpose on device via a strided copy per axis
    for (int a = 0; a < dim; ++a)
      SMASH_CUDA(cudaMemcpy2DAsync(soa.p + (size_t)a * n, sizeof(double), pts + a,
                                   sizeof(double) * dim, sizeof(double), n,
                                   cudaMemcpyDeviceToDevice, s));
    launch_basis_single(dim, lo, hi, D.view, r, soa.p, n, out, nullptr, s);
  }
  sync(s);
}

void compr_single(const double* C, int64_t nrows, int64_t ncols, double s_bound, double rtol,
                  int64_t* perm, double* G, int64_t* rank, int64_t* swaps, cudaStream_t s) {
  SMASH_CHECK(nrows >= 0 && ncols >= 0, SMASH_ERR_INVALID, "bad shape");
  SMASH_CHECK(nrows < (1 << 20), SMASH_ERR_INVALID, "compr: too many rows for one CTA");
  if (nrows == 0 || ncols == 0) {
    *rank = 0;
    *swaps = 0;
    if (nrows) {
      std::vector<int64_t> id(nrows);
      for (int64_t i = 0; i < nrows; ++i) id[i] = i;
      h2d(perm, id.data(), nrows, s);
      sync(s);
    }
    return;
  }
  DBuf<int> nib, rk, pm, err;
  DBuf<int64_t> off;
  DBuf<double> g;
  DBuf<unsigned long long> sw;
  int ni = (int)nrows;
  nib.alloc(1, s); rk.alloc(1, s); pm.alloc(nrows, s); err.alloc(1, s); off.alloc(2, s);
  int64_t kmax = std::min(nrows, ncols);
  g.alloc(std::max<int64_t>(nrows * kmax, 1), s);
  sw.alloc(1, s);
  h2d(nib.p, &ni, 1, s);
  off.zero(s); err.zero(s); sw.zero(s);
  CompressArgs A;
  A.lb = 0; A.le = 1; A.dim = 1; A.r = 0;
  A.nib = nib.p; A.ib_off = off.p; A.g_off = off.p + 1;
  A.Cexp = C; A.C_cols = (int)ncols;
  A.s_bound = s_bound; A.rtol = rtol;
  A.rank = rk.p; A.perm = pm.p; A.G = g.p;
  A.err = err.p; A.swaps = sw.p;
  A.nmax = ni; A.mmax = (int)ncols;
  size_t smem = compress_smem_bytes(A.nmax, A.mmax, true);
  DBuf<double> gws;
  A.panel_cap = (int64_t)A.nmax * A.mmax;
  if ((int)smem > max_sm_smem()) {
    A.panel_cap = 0;
    smem = compress_smem_bytes(A.nmax, A.mmax, false);
    gws.alloc((size_t)A.nmax * A.mmax, s);
    A.gws = gws.p;
  }
  SMASH_CHECK((int)smem <= max_sm_smem(), SMASH_ERR_INVALID, "compr: matrix too large for one CTA");
  launch_compress(A, 1, smem, s);
  int hk = 0, he = 0;
  unsigned long long hs = 0;
  d2h(&hk, rk.p, 1, s);
  d2h(&he, err.p, 1, s);
  d2h(&hs, sw.p, 1, s);
  sync(s);
  raise_dev_err(he);
  *rank = hk;
  *swaps = (int64_t)hs;
  std::vector<int> hp(nrows);
  d2h(hp.data(), pm.p, nrows, s);
  sync(s);
  std::vector<int64_t> hp64(hp.begin(), hp.end());
  h2d(perm, hp64.data(), nrows, s);
  if (hk > 0 && hk < nrows) d2d(G, g.p, (size_t)(nrows - hk) * hk, s);
  sync(s);
}

}  // namespace smash
