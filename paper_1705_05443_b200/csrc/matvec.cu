// K6-K10: the H^2 / HSS matvec -- replaces smash.apply.matvec_nodewise
// (smash/apply.py:34-80).
//
// Phases (coefficient vectors are (count, RC) row-major; nrhs is processed in
// chunks of RC <= 16 columns):
//   main stream:  K10 gather qt = q[perm_col]                     (apply.py:39)
//                 K6  upward  qhat_v = X_v^T ibar-vector, one persistent launch (apply.py:42-53)
//                 K7  coupling zhat_i = sum_{j in L(i)} K(S_i, S_j) qhat_j   (apply.py:55-58)
//                 K8  downward zhat_children += X_v zhat_v, one persistent launch (apply.py:60-72)
//                 --- join ---
//                 K8b leaf far field fused with the combine
//                     z[perm_row] = zn + X_v zhat_v                          (apply.py:66-80)
//   near stream:  K9  nearfield zn = sum_{j in Lm(v)} K(P_v, P_j) qt_j       (apply.py:74-76)
// The nearfield only needs qt, so it overlaps the whole far-field chain.
#include <algorithm>
#include <array>
#include <cstdlib>

#include "matvec_impl.cuh"

namespace smash {

using namespace mv;

namespace {

struct MatvecPlan : XferPlan {
  // symmetric coupling (shared points, symmetric kernel): upper pair list, pair buffer
  bool sym = false;
  DBuf<int> Uptr, Usrc, tptr, te;
  DBuf<int64_t> pbuf;
  DBuf<double> symbuf;  // pair rows x 16
};

// Shared points and a symmetric kernel: the coupling can evaluate each block once
// (SymCoupling, matvec_impl.cuh) -- opt-in with SMASH_COUPLING_SYM=1.  Measured at cfg 5
// (profiles/coupling_sym_r02.txt): 12.1 ms + 1.1 ms pass 2 vs 13.2 ms for the two-sided
// kernel -- half the kernel evaluations, but 218 registers (half the occupancy), a
// 6.2 GB pair buffer written and re-read, and read-modify-write across target passes.
void plan_sym(MatrixImpl* m, MatvecPlan* P, cudaStream_t s) {
  static const bool on = getenv("SMASH_COUPLING_SYM") && getenv("SMASH_COUPLING_SYM")[0] == '1';
  if (!on || m->colf != &m->rowf || m->p.kernel == SMASH_KERNEL_CAUCHY) return;
  TreeImpl* t = m->tree;
  const int n = t->n_nodes;
  std::vector<int> ptr(n + 1), rk(n);
  d2h(ptr.data(), m->pl->L_ptr.p, n + 1, s);
  d2h(rk.data(), m->rowf.rank.p, n, s);
  sync(s);
  std::vector<int> src(ptr[n]);
  d2h(src.data(), m->pl->L_j.p, src.size(), s);
  sync(s);
  std::vector<int> up(n + 1, 0), us;
  std::vector<int64_t> pb;
  int64_t rows = 0;
  us.reserve(src.size() / 2 + 1);
  for (int v = 0; v < n; ++v) {
    up[v] = (int)us.size();
    for (int e = ptr[v]; e < ptr[v + 1]; ++e) {
      const int j = src[e];
      SMASH_CHECK(j != v, SMASH_ERR_CUDA, "coupling pair with itself");
      if (j > v) {
        us.push_back(j);
        pb.push_back(rows);
        rows += rk[j];
      }
    }
  }
  up[n] = (int)us.size();
  // source-major index of the upper pairs: for every j the pairs (i, j), i ascending
  std::vector<int> tp(n + 1, 0), tcount(n, 0);
  for (int j : us) ++tcount[j];
  for (int j = 0; j < n; ++j) tp[j + 1] = tp[j] + tcount[j];
  std::vector<int> te(us.size()), fill(tp.begin(), tp.end() - 1);
  for (int v = 0; v < n; ++v)
    for (int e = up[v]; e < up[v + 1]; ++e) te[fill[us[e]]++] = e;
  auto put = [&](auto& d, const auto& h) {
    d.alloc(std::max<size_t>(h.size(), 1), s);
    h2d(d.p, h.data(), h.size(), s);
  };
  put(P->Uptr, up);
  put(P->Usrc, us);
  put(P->pbuf, pb);
  put(P->tptr, tp);
  put(P->te, te);
  P->symbuf.alloc(std::max<int64_t>(rows, 1) * 16, s);
  sync(s);
  P->sym = true;
}

std::map<const MatrixImpl*, std::unique_ptr<MatvecPlan>> g_plans;

MatvecPlan* plan_of(MatrixImpl* m, cudaStream_t s) {
  auto it = g_plans.find(m);
  if (it != g_plans.end()) return it->second.get();
  std::unique_ptr<MatvecPlan> P(new MatvecPlan());
  TreeImpl* t = m->tree;
  const int n = t->n_nodes;
  std::vector<int> nchild(n), nib(n), rk(n);
  d2h(nchild.data(), t->nchild.p, n, s);
  d2h(nib.data(), m->rowf.nib.p, n, s);
  d2h(rk.data(), m->rowf.rank.p, n, s);
  sync(s);
  int mx = 1, mr = 1;
  for (int v = 0; v < n; ++v) { mx = std::max(mx, nib[v]); mr = std::max(mr, rk[v]); }
  if (m->colf != &m->rowf) {
    d2h(nib.data(), m->colf->nib.p, n, s);
    d2h(rk.data(), m->colf->rank.p, n, s);
    sync(s);
    for (int v = 0; v < n; ++v) { mx = std::max(mx, nib[v]); mr = std::max(mr, rk[v]); }
  }
  P->max_nib = mx;
  P->max_rank = mr;
  {  // largest |ibar| - k over both sides (G rows per node)
    int mk = 0;
    for (SideFactors* F : {&m->rowf, m->colf}) {
      d2h(nib.data(), F->nib.p, n, s);
      d2h(rk.data(), F->rank.p, n, s);
      sync(s);
      for (int v = 0; v < n; ++v) mk = std::max(mk, nib[v] - rk[v]);
    }
    P->max_nk = mk;
  }
  // ticket orders of the internal non-root nodes: BFS ids are level-major, so
  // deepest level first = descending ids (leaves go through the warp-per-leaf
  // launches before / after the persistent passes).
  std::vector<int> up, down, leaves;
  for (int v = n - 1; v >= 1; --v)
    if (nchild[v] > 0) up.push_back(v);
  for (int v = 1; v < n; ++v)
    if (nchild[v] > 0) down.push_back(v);
  for (int v = 0; v < n; ++v)
    if (nchild[v] == 0) leaves.push_back(v);
  P->n_up = (int)up.size();
  P->n_down = (int)down.size();
  P->n_leaves = (int)leaves.size();
  P->up_order.alloc(std::max<size_t>(up.size(), 1), s);
  P->down_order.alloc(std::max<size_t>(down.size(), 1), s);
  P->leaves.alloc(std::max<size_t>(leaves.size(), 1), s);
  h2d(P->up_order.p, up.data(), up.size(), s);
  h2d(P->down_order.p, down.data(), down.size(), s);
  h2d(P->leaves.p, leaves.data(), leaves.size(), s);
  {  // membership of the internal passes (leaf producers are final before them)
    std::vector<unsigned char> in(n, 0);
    for (int v : up) in[v] = 1;
    P->inset_int.alloc(n, s);
    h2d(P->inset_int.p, in.data(), n, s);
  }
  P->up_pos.alloc(std::max<int64_t>(m->colf->skel_total, 1), s);
  launch_up_pos(side_of(*m->colf), t->nchild.p, t->child_first.p, n, P->up_pos.p,
                m->colf->skel_total, s);
  P->slot_of.alloc(std::max<int64_t>(t->nx, 1), s);
  P->zrow.alloc(std::max<int64_t>(t->nx, 1), s);
  launch_leaf_slots(side_of(m->rowf), P->leaves.p, P->n_leaves, t->row_a.p, t->row_b.p,
                    t->perm_row.p, P->slot_of.p, P->zrow.p, s);
  P->done.alloc(n, s);
  P->done.zero(s);
  P->counters.alloc(2, s);
  sync(s);
  plan_sym(m, P.get(), s);
  MatvecPlan* out = P.get();
  g_plans[m] = std::move(P);
  return out;
}

// Node subsets driving one pass (whole tree, or one shard's stage).
struct PhaseSets {
  bool gather = true;
  bool zero_qhat = false;                 // shard: unowned coefficients must be 0 for the all-reduce
  const int* up_leaves = nullptr; int n_up_leaves = 0;  // leaves of the upward pass
  const int* up = nullptr; int n_up = 0;  // internal upward order (deepest level first)
  const unsigned char* up_in = nullptr;   // membership of the upward / downward sets
  const unsigned char* down_in = nullptr;
  bool far = true;                        // run coupling / downward / nearfield / combine
  const int* coup = nullptr; int n_coup = -1;  // coupling targets (nullptr + -1: all nodes)
  const int* down = nullptr; int n_down = 0;   // internal downward order (shallowest first)
  const int* leaves = nullptr; int n_leaves = 0;  // nearfield / far-field + combine rows
  int near_mode = 0;  // 0: nearfield forked here; 1: nearfield only; 2: nearfield done earlier
};

// SMASH_DEBUG_SYNC=1: eager (uncaptured) matvec with a synchronize + error
// check after every launch, naming the failing phase (debug aid).
bool debug_sync() {
  static const bool on = getenv("SMASH_DEBUG_SYNC") != nullptr;
  return on;
}

void check_phase(const char* name, cudaStream_t st) {
  if (!debug_sync()) return;
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess)
    throw Error(SMASH_ERR_CUDA, std::string("matvec phase ") + name + ": " + cudaGetErrorString(e));
}

template <int KER, int D, int RC>
void run_chunk(MatrixImpl* m, MatvecPlan& P, const PhaseSets& S, const double* q, double* z,
               int64_t nrhs, int64_t c0, cudaStream_t s, cudaEvent_t* ev, int* nlaunch) {
  TreeImpl* t = m->tree;
  const SideFactors& R = m->rowf;
  const SideFactors& C = *m->colf;
  const Side rs = side_of(R), cs = side_of(C);
  const int* perm_col = t->shared ? t->perm_row.p : t->perm_col.p;
  const double* pts_col = t->shared ? t->pts_row.p : t->pts_col.p;
  const int* col_a = t->shared ? t->row_a.p : t->col_a.p;
  const int* col_b = t->shared ? t->row_b.p : t->col_b.p;
  static const bool serial_env = getenv("SMASH_MATVEC_SERIAL") != nullptr || debug_sync();
  const bool serial = serial_env || m->serial_phases;
  cudaStream_t sn = serial ? s : m->s2;
  auto mark = [&](int i, cudaStream_t st) {  // external record: a timing node in the graph
    if (ev) SMASH_CUDA(cudaEventRecordWithFlags(ev[i], st, cudaEventRecordExternal));
  };
  int launches = 0;
  if (S.near_mode == 1) {  // sharded stage 3: the owned leaves' nearfield alone (needs only qt)
    NearArgs na{S.leaves, S.n_leaves, t->row_a.p, t->row_b.p, col_a, col_b, t->pts_row.p, t->nx,
                pts_col, t->ny, m->pl->Lm_ptr.p, m->pl->Lm_j.p, m->qt.p, P.slot_of.p, m->zn.p,
                m->p.dx, t->nu0};
    mark(6, s);
    launch_near<KER, D, RC>(na, s);
    mark(7, s);
    mark(5, s);
    *nlaunch += 1;
    return;
  }
  mark(0, s);
  if (S.gather) {
    launch_gather<RC>(q, nrhs, perm_col, t->ny, c0, m->qt.p, s);
    check_phase("gather", s);
    ++launches;
  }
  if (S.zero_qhat) {
    SMASH_CUDA(cudaMemsetAsync(m->qhat.p, 0, 2 * (size_t)std::max<int64_t>(C.skel_total, 1) * RC * 8, s));
    ++launches;
  }
  mark(1, s);
  auto fork_near = [&]() {  // nearfield on the second stream (needs only qt)
    SMASH_CUDA(cudaEventRecord(m->fork, s));
    SMASH_CUDA(cudaStreamWaitEvent(sn, m->fork, 0));
    mark(6, sn);
    NearArgs na{S.leaves, S.n_leaves, t->row_a.p, t->row_b.p, col_a, col_b, t->pts_row.p, t->nx,
                pts_col, t->ny, m->pl->Lm_ptr.p, m->pl->Lm_j.p, m->qt.p, P.slot_of.p, m->zn.p,
                m->p.dx, t->nu0};
    launch_near<KER, D, RC>(na, sn);
    check_phase("near", sn);
    ++launches;
    mark(7, sn);
    SMASH_CUDA(cudaEventRecord(m->join, sn));
  };
  // Fork point: right after the gather, so the nearfield overlaps the latency-bound
  // upward pass and the coupling then runs alone; SMASH_NEAR_LATE=1 forks after the
  // upward pass instead (nearfield overlapping the coupling).  Both orders give the
  // same matvec time on cfg2 (the FP64 work bounds it, profiles/README_r01.md).
  static const bool near_early_env = getenv("SMASH_NEAR_LATE") == nullptr;
  // serialised profiling: the nearfield runs alone after the downward pass
  const bool near_early = near_early_env && !m->serial_phases;
  const bool near_here = S.near_mode == 0;
  if (S.far && near_here && near_early) fork_near();
  double* qp = m->qhat.p + std::max<int64_t>(C.skel_total, 1) * RC;  // second half of qhat
  XferArgs up{t->nchild.p, t->child_first.p, t->parent.p, col_a, col_b, m->qt.p, m->qhat.p,
              qp, P.up_pos.p, m->zhat.p, m->zd.p, cs};
  if (S.n_up_leaves) {
    launch_up_leaves<RC>(up, S.up_leaves, S.n_up_leaves, s);
    check_phase("upward leaves", s);
    ++launches;
  }
  if (S.n_up) {
    launch_upward<RC>(up, P, S.up, S.n_up, S.up_in, s);
    check_phase("upward", s);
    launches += 2;
  }
  mark(2, s);
  if (S.far && near_here && !near_early && !m->serial_phases) fork_near();
  if (S.far) {
    CouplingArgs ca{S.n_coup < 0 ? t->n_nodes : S.n_coup, S.coup, rs, cs, m->pl->L_ptr.p,
                    m->pl->L_j.p, m->qhat.p, m->zhat.p, m->p.dx, P.max_rank};
    if constexpr (RC == 8 || RC == 16) {
      if (P.sym && S.coup == nullptr) {  // whole-tree product: each block evaluated once
        SymCoupling y{P.Uptr.p, P.Usrc.p, P.pbuf.p, P.symbuf.p, P.tptr.p, P.te.p};
        launch_coupling_sym<KER, D, RC>(ca, y, s);
        ++launches;
      } else {
        launch_coupling<KER, D, RC>(ca, s);
      }
    } else {
      launch_coupling<KER, D, RC>(ca, s);
    }
    check_phase("coupling", s);
    ++launches;
    mark(3, s);
    XferArgs down{t->nchild.p, t->child_first.p, t->parent.p, t->row_a.p, t->row_b.p, m->qt.p,
                  m->qhat.p, qp, P.up_pos.p, m->zhat.p, m->zd.p, rs};
    if (S.n_down) {
      launch_downward<RC>(down, P, S.down, S.n_down, S.down_in, s);
      check_phase("downward", s);
      launches += 2;
    }
    mark(4, s);
    if (near_here && m->serial_phases) fork_near();
    if (near_here) SMASH_CUDA(cudaStreamWaitEvent(s, m->join, 0));
    mark(8, s);
    launch_down_leaves<RC>(down, S.leaves, S.n_leaves, P.zrow.p, m->zn.p, z, nrhs, c0, s);
    check_phase("downward leaves", s);
    ++launches;
  }
  mark(5, s);
  *nlaunch += launches;
}

// chunk sizes of an nrhs split (largest power of two <= 16 and <= rc_cap first)
std::vector<int> chunks_of(int64_t nrhs, int rc_cap) {
  std::vector<int> out;
  int64_t left = nrhs;
  while (left > 0) {
    int c = 16;
    while (c > 1 && (c > left || c > rc_cap)) c >>= 1;
    out.push_back(c);
    left -= c;
  }
  return out;
}

template <int KER, int D>
void run_all(MatrixImpl* m, MatvecPlan& P, const PhaseSets& S, const double* q, double* z,
             int64_t nrhs, int rc_cap, cudaStream_t s, std::vector<std::array<cudaEvent_t, 9>>* evs,
             int* nlaunch) {
  int64_t c0 = 0;
  int ci = 0;
  for (int c : chunks_of(nrhs, rc_cap)) {
    cudaEvent_t* ev = evs ? (*evs)[ci].data() : nullptr;
    if (c == 16) run_chunk<KER, D, 16>(m, P, S, q, z, nrhs, c0, s, ev, nlaunch);
    else if (c == 8) run_chunk<KER, D, 8>(m, P, S, q, z, nrhs, c0, s, ev, nlaunch);
    else if (c == 4) run_chunk<KER, D, 4>(m, P, S, q, z, nrhs, c0, s, ev, nlaunch);
    else if (c == 2) run_chunk<KER, D, 2>(m, P, S, q, z, nrhs, c0, s, ev, nlaunch);
    else run_chunk<KER, D, 1>(m, P, S, q, z, nrhs, c0, s, ev, nlaunch);
    c0 += c;
    ++ci;
  }
}

// Captured matvec: one CUDA graph per (q, z, nrhs, stage); replays cost one launch.
struct GraphEntry {
  const double* q = nullptr;
  double* z = nullptr;
  int64_t nrhs = 0;
  int stage = 0;
  bool serial = false;  // captured with the nearfield on the main stream (phase profiling)
  cudaGraphExec_t exec = nullptr;
  std::vector<std::array<cudaEvent_t, 9>> ev;
  bool far = true;
  int launches = 0;
  ~GraphEntry() {
    if (exec) cudaGraphExecDestroy(exec);
    for (auto& a : ev)
      for (auto e : a)
        if (e) cudaEventDestroy(e);
  }
};
std::map<const MatrixImpl*, std::vector<std::unique_ptr<GraphEntry>>> g_graphs;

template <typename F>
GraphEntry* graph_for(MatrixImpl* m, const double* q, double* z, int64_t nrhs, int stage,
                      int n_chunks, bool far, F record) {
  cudaStream_t s = m->sc;  // captured work is recorded on the capture stream
  auto& L = g_graphs[m];
  for (auto& e : L)
    if (e->q == q && e->z == z && e->nrhs == nrhs && e->stage == stage && e->serial == m->serial_phases)
      return e.get();
  std::unique_ptr<GraphEntry> E(new GraphEntry());
  E->q = q; E->z = z; E->nrhs = nrhs; E->stage = stage; E->far = far; E->serial = m->serial_phases;
  E->ev.resize(n_chunks);
  for (auto& a : E->ev)
    for (auto& e : a) SMASH_CUDA(cudaEventCreate(&e));
  cudaGraph_t g = nullptr;
  SMASH_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
  try {
    record(&E->ev, &E->launches);
  } catch (...) {
    cudaStreamEndCapture(s, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  SMASH_CUDA(cudaStreamEndCapture(s, &g));
  SMASH_CUDA(cudaGraphInstantiate(&E->exec, g, 0));
  SMASH_CUDA(cudaGraphDestroy(g));
  if (L.size() >= 8) L.erase(L.begin());
  L.push_back(std::move(E));
  return L.back().get();
}

void replay(MatrixImpl* m, GraphEntry* E, cudaStream_t s) {
  m->order_after_last_use(s);
  SMASH_CUDA(cudaGraphLaunch(E->exec, s));
  m->mark_use(s);
  m->launches += E->launches;
  if (m->profile && E->far) {
    const int pairs[7][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 4}, {6, 7}, {8, 5}, {0, 5}};
    for (auto& ev : E->ev) {
      SMASH_CUDA(cudaEventSynchronize(ev[5]));
      for (int i = 0; i < 7; ++i) {
        // sharded stages: 3 records only the nearfield, 4 everything but it
        if ((E->stage == 4 && i == 4) || (E->stage == 3 && i != 4)) continue;
        float ms = 0;
        SMASH_CUDA(cudaEventElapsedTime(&ms, ev[pairs[i][0]], ev[pairs[i][1]]));
        m->phase_ms[i] += ms;
      }
    }
  }
}

}  // namespace



namespace {

int prepare(MatrixImpl* m, MatvecPlan* P, cudaStream_t s) {
  TreeImpl* t = m->tree;
  if (!m->s2) {
    // the far-field chain (upward -> coupling -> downward) is the critical path:
    // its stream gets the highest priority, the overlapping nearfield the lowest,
    // so freed SMs go to the chain first (captured kernel nodes keep the priority)
    int lo = 0, hi = 0;
    SMASH_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    static const bool flat = getenv("SMASH_FLAT_PRIORITY") != nullptr;
    SMASH_CUDA(cudaStreamCreateWithPriority(&m->s2, cudaStreamNonBlocking, lo));
    SMASH_CUDA(cudaStreamCreateWithPriority(&m->sc, cudaStreamNonBlocking, flat ? lo : hi));
    SMASH_CUDA(cudaEventCreateWithFlags(&m->fork, cudaEventDisableTiming));
    SMASH_CUDA(cudaEventCreateWithFlags(&m->join, cudaEventDisableTiming));
  }
  if (m->ws_nrhs < 16) {
    m->qt.alloc((size_t)t->ny * 16, s);
    m->qhat.alloc(2 * (size_t)std::max<int64_t>(m->colf->skel_total, 1) * 16, s);  // qhat | qp
    m->zhat.alloc((size_t)std::max<int64_t>(m->rowf.skel_total, 1) * 16, s);
    m->zd.alloc((size_t)std::max<int64_t>(m->rowf.skel_total, 1) * 16, s);
    m->zn.alloc((size_t)t->nx * 16, s);
    m->ws_nrhs = 16;
  }
  // largest nrhs chunk whose transfer-kernel tiles and shared memory fit
  auto fits = [&](int rc) {
    const XferGeom G = xfer_geom(P->max_nib, P->max_rank, P->max_nk, rc);
    const int tiles = ((P->max_rank + 7) / 8) * ((rc + 7) / 8);
    return tiles <= 16 && xfer_smem_up(G) <= 200 * 1024 &&  // upward: <= 2 tiles per warp
           xfer_smem_down(G) <= 200 * 1024;
  };
  int rc_cap = 16;
  while (rc_cap > 1 && !fits(rc_cap)) rc_cap /= 2;
  SMASH_CHECK(fits(rc_cap), SMASH_ERR_INVALID, "intermediate sets too large for the matvec");
  return rc_cap;
}

// One shard's node subsets (set by matvec_set_partition).
struct ShardSets {
  DBuf<int> own_up, top_up, coup, down, leaves;
  DBuf<unsigned char> own_in, top_in, down_in;
  int n_own_up = 0, n_top_up = 0, n_coup = 0, n_down = 0, n_leaves = 0;
};
std::map<const MatrixImpl*, std::unique_ptr<ShardSets>> g_shards;

}  // namespace

void matvec(MatrixImpl* m, const double* q, double* z, int64_t nrhs, cudaStream_t s) {
  SMASH_CHECK(nrhs >= 1, SMASH_ERR_INVALID, "nrhs must be positive");
  TreeImpl* t = m->tree;
  MatvecPlan* P = plan_of(m, s);
  const int rc_cap = prepare(m, P, s);
  PhaseSets S;
  S.up_leaves = P->leaves.p; S.n_up_leaves = P->n_leaves;
  S.up = P->up_order.p; S.n_up = P->n_up;
  S.up_in = P->inset_int.p;
  S.down_in = P->inset_int.p;
  S.down = P->down_order.p; S.n_down = P->n_down;
  S.leaves = P->leaves.p; S.n_leaves = P->n_leaves;
  const int nch = (int)chunks_of(nrhs, rc_cap).size();
  if (debug_sync()) {
    int nl = 0;
    m->order_after_last_use(s);
    dispatch_kernel_dim(m->p.kernel, t->dim, [&]<int KER, int D>() {
      run_all<KER, D>(m, *P, S, q, z, nrhs, rc_cap, s, nullptr, &nl);
    });
    m->mark_use(s);
    return;
  }
  GraphEntry* E = graph_for(m, q, z, nrhs, 0, nch, true, [&](auto* evs, int* nl) {
    dispatch_kernel_dim(m->p.kernel, t->dim, [&]<int KER, int D>() {
      run_all<KER, D>(m, *P, S, q, z, nrhs, rc_cap, m->sc, evs, nl);
    });
  });
  replay(m, E, s);
  SMASH_CUDA(cudaGetLastError());
}

// Level-synchronous matvec on perfect trees (smash/apply.py:83-165): gather, the
// leaves' upward projections, one upward launch per level (deepest first), the
// coupling of every node, one downward launch per level (shallowest first), the
// nearfield and the leaf far field + combine.  No dataflow flags, no graph: each
// level's coefficient block is complete before the next level starts.
namespace {
template <int KER, int D, int RC>
void run_chunk_level(MatrixImpl* m, MatvecPlan& P, const double* q, double* z, int64_t nrhs,
                     int64_t c0, cudaStream_t s) {
  TreeImpl* t = m->tree;
  const SideFactors& R = m->rowf;
  const SideFactors& C = *m->colf;
  const Side rs = side_of(R), cs = side_of(C);
  const int* perm_col = t->shared ? t->perm_row.p : t->perm_col.p;
  const double* pts_col = t->shared ? t->pts_row.p : t->pts_col.p;
  const int* col_a = t->shared ? t->row_a.p : t->col_a.p;
  const int* col_b = t->shared ? t->row_b.p : t->col_b.p;
  launch_gather<RC>(q, nrhs, perm_col, t->ny, c0, m->qt.p, s);
  double* qp = m->qhat.p + std::max<int64_t>(C.skel_total, 1) * RC;
  XferArgs up{t->nchild.p, t->child_first.p, t->parent.p, col_a, col_b, m->qt.p, m->qhat.p,
              qp, P.up_pos.p, m->zhat.p, m->zd.p, cs};
  launch_up_leaves<RC>(up, P.leaves.p, P.n_leaves, s);
  for (int l = t->n_levels - 1; l >= 2; --l)
    launch_level_up(cs, t->nchild.p, t->child_first.p, t->level_begin(l), t->level_end(l),
                    m->qhat.p, RC, s);
  CouplingArgs ca{t->n_nodes, nullptr, rs, cs, m->pl->L_ptr.p, m->pl->L_j.p, m->qhat.p,
                  m->zhat.p, m->p.dx, P.max_rank};
  launch_coupling<KER, D, RC>(ca, s);
  for (int l = 2; l <= t->n_levels - 1; ++l)
    launch_level_down(rs, t->nchild.p, t->child_first.p, t->parent.p, t->level_begin(l),
                      t->level_end(l), m->zhat.p, m->zd.p, RC, P.max_rank, s);
  NearArgs na{P.leaves.p, P.n_leaves, t->row_a.p, t->row_b.p, col_a, col_b, t->pts_row.p, t->nx,
              pts_col, t->ny, m->pl->Lm_ptr.p, m->pl->Lm_j.p, m->qt.p, P.slot_of.p, m->zn.p,
              m->p.dx, t->nu0};
  launch_near<KER, D, RC>(na, s);
  XferArgs down{t->nchild.p, t->child_first.p, t->parent.p, t->row_a.p, t->row_b.p, m->qt.p,
                m->qhat.p, qp, P.up_pos.p, m->zhat.p, m->zd.p, rs};
  launch_down_leaves<RC>(down, P.leaves.p, P.n_leaves, P.zrow.p, m->zn.p, z, nrhs, c0, s);
  SMASH_CUDA(cudaGetLastError());
}
}  // namespace

void matvec_levelwise(MatrixImpl* m, const double* q, double* z, int64_t nrhs, cudaStream_t s) {
  SMASH_CHECK(nrhs >= 1, SMASH_ERR_INVALID, "nrhs must be positive");
  TreeImpl* t = m->tree;
  const int n = t->n_nodes;
  {  // apply.py:83-95: all leaves on the deepest level, one child count
    std::vector<int> nchild(n);
    d2h(nchild.data(), t->nchild.p, n, s);
    sync(s);
    int width = -1;
    for (int l = 1; l <= t->n_levels; ++l)
      for (int v = t->level_begin(l); v < t->level_end(l); ++v) {
        if (nchild[v] == 0) {
          SMASH_CHECK(l == t->n_levels, SMASH_ERR_INVALID,
                      "level-synchronous matvec needs all leaves at the deepest level");
        } else {
          SMASH_CHECK(width < 0 || nchild[v] == width, SMASH_ERR_INVALID,
                      "level-synchronous matvec needs a perfect tree");
          width = nchild[v];
        }
      }
  }
  MatvecPlan* P = plan_of(m, s);
  const int rc_cap = prepare(m, P, s);
  SMASH_CHECK(P->max_nib <= level_max_nib(), SMASH_ERR_INVALID,
              "intermediate sets too large for the level-synchronous matvec");
  m->order_after_last_use(s);
  int64_t c0 = 0;
  for (int c : chunks_of(nrhs, rc_cap)) {
    dispatch_kernel_dim(m->p.kernel, t->dim, [&]<int KER, int D>() {
      if (c == 16) run_chunk_level<KER, D, 16>(m, *P, q, z, nrhs, c0, s);
      else if (c == 8) run_chunk_level<KER, D, 8>(m, *P, q, z, nrhs, c0, s);
      else if (c == 4) run_chunk_level<KER, D, 4>(m, *P, q, z, nrhs, c0, s);
      else if (c == 2) run_chunk_level<KER, D, 2>(m, *P, q, z, nrhs, c0, s);
      else run_chunk_level<KER, D, 1>(m, *P, q, z, nrhs, c0, s);
    });
    c0 += c;
  }
  m->mark_use(s);
}

void matvec_set_partition(MatrixImpl* m, const int64_t* own_post, int64_t n_own,
                          const int64_t* top_post, int64_t n_top, cudaStream_t s) {
  TreeImpl* t = m->tree;
  const int n = t->n_nodes;
  std::vector<int> post(n), nchild(n);
  d2h(post.data(), t->post.p, n, s);
  d2h(nchild.data(), t->nchild.p, n, s);
  sync(s);
  std::vector<int> bfs_of_post(n);
  for (int v = 0; v < n; ++v) bfs_of_post[post[v]] = v;
  auto to_bfs = [&](const int64_t* a, int64_t k) {
    std::vector<int> out;
    for (int64_t i = 0; i < k; ++i) {
      SMASH_CHECK(a[i] >= 0 && a[i] < n, SMASH_ERR_INVALID, "partition node out of range");
      const int v = bfs_of_post[a[i]];
      if (v != 0) out.push_back(v);  // the root carries no factor
    }
    return out;
  };
  std::vector<int> own = to_bfs(own_post, n_own), top = to_bfs(top_post, n_top);
  std::vector<int> own_up, top_up = top, coup = own, down, leaves;
  for (int v : own)
    if (nchild[v] > 0) own_up.push_back(v);  // owned leaves go through the leaf launches
  std::sort(own_up.rbegin(), own_up.rend());  // BFS is level-major: descending = deepest first
  std::sort(top_up.rbegin(), top_up.rend());
  coup.insert(coup.end(), top.begin(), top.end());
  std::sort(coup.begin(), coup.end());
  for (int v : coup)
    if (nchild[v] > 0) down.push_back(v);  // ascending = shallowest first
  for (int v : own)
    if (nchild[v] == 0) leaves.push_back(v);
  std::unique_ptr<ShardSets> S(new ShardSets());
  auto up = [&](DBuf<int>& d, const std::vector<int>& h, int& cnt) {
    cnt = (int)h.size();
    d.alloc(std::max<size_t>(h.size(), 1), s);
    h2d(d.p, h.data(), h.size(), s);
  };
  up(S->own_up, own_up, S->n_own_up);
  up(S->top_up, top_up, S->n_top_up);
  up(S->coup, coup, S->n_coup);
  up(S->down, down, S->n_down);
  up(S->leaves, leaves, S->n_leaves);
  auto member = [&](DBuf<unsigned char>& d, const std::vector<int>& h) {
    std::vector<unsigned char> in(n, 0);
    for (int v : h) in[v] = 1;
    d.alloc(n, s);
    h2d(d.p, in.data(), n, s);
  };
  member(S->own_in, own_up);
  member(S->top_in, top_up);
  member(S->down_in, down);
  sync(s);
  g_shards[m] = std::move(S);
  auto& L = g_graphs[m];  // stage graphs captured for an older partition are stale
  L.erase(std::remove_if(L.begin(), L.end(), [](const std::unique_ptr<GraphEntry>& e) {
            return e->stage != 0;
          }), L.end());
}

void matvec_stage(MatrixImpl* m, int stage, const double* q, double* z, int64_t nrhs,
                  cudaStream_t s) {
  auto it = g_shards.find(m);
  SMASH_CHECK(it != g_shards.end(), SMASH_ERR_INVALID, "no partition set (smash_matvec_set_partition)");
  SMASH_CHECK(stage >= 1 && stage <= 4, SMASH_ERR_INVALID, "stage must be 1, 2, 3 or 4");
  TreeImpl* t = m->tree;
  MatvecPlan* P = plan_of(m, s);
  const int rc_cap = prepare(m, P, s);
  SMASH_CHECK(nrhs >= 1 && nrhs <= rc_cap && (nrhs & (nrhs - 1)) == 0, SMASH_ERR_INVALID,
              "sharded matvec takes one nrhs chunk (power of two <= the chunk cap)");
  const ShardSets& H = *it->second;
  PhaseSets S;
  if (stage == 1) {  // local upward of the owned subtrees (other coefficients untouched)
    S.up_leaves = H.leaves.p; S.n_up_leaves = H.n_leaves;
    S.up = H.own_up.p; S.n_up = H.n_own_up; S.up_in = H.own_in.p;
    S.far = false;
  } else if (stage == 3) {  // the owned leaves' nearfield only (overlaps the exchange)
    S.gather = false;
    S.far = false;
    S.leaves = H.leaves.p; S.n_leaves = H.n_leaves;
    S.near_mode = 1;
  } else {  // after the coefficient exchange: top upward, then owned far (+ near) field
    S.gather = false;
    S.up = H.top_up.p; S.n_up = H.n_top_up; S.up_in = H.top_in.p;
    S.coup = H.coup.p; S.n_coup = H.n_coup;
    S.down = H.down.p; S.n_down = H.n_down; S.down_in = H.down_in.p;
    S.leaves = H.leaves.p; S.n_leaves = H.n_leaves;
    S.near_mode = stage == 4 ? 2 : 0;  // 4: the nearfield ran as stage 3
  }
  GraphEntry* E = graph_for(m, q, z, nrhs, stage, 1, stage >= 2, [&](auto* evs, int* nl) {
    dispatch_kernel_dim(m->p.kernel, t->dim, [&]<int KER, int D>() {
      run_all<KER, D>(m, *P, S, q, z, nrhs, rc_cap, m->sc, evs, nl);
    });
  });
  replay(m, E, s);
  SMASH_CUDA(cudaGetLastError());
}

void matvec_coeff_layout(MatrixImpl* m, int64_t* row_off_post, int64_t* up_pos, int64_t* half_rows,
                         cudaStream_t s) {
  TreeImpl* t = m->tree;
  MatvecPlan* P = plan_of(m, s);
  const int n = t->n_nodes;
  const SideFactors& C = *m->colf;
  std::vector<int> post(n), off(n), rk(n);
  d2h(post.data(), t->post.p, n, s);
  d2h(off.data(), C.skel_off.p, n, s);
  d2h(rk.data(), C.rank.p, n, s);
  std::vector<int> up(std::max<int64_t>(C.skel_total, 1));
  d2h(up.data(), P->up_pos.p, up.size(), s);
  sync(s);
  for (int v = 0; v < n; ++v) row_off_post[post[v]] = (v == 0 || rk[v] == 0) ? -1 : off[v];
  if (up_pos)
    for (int64_t x = 0; x < C.skel_total; ++x) up_pos[x] = up[x];
  *half_rows = std::max<int64_t>(C.skel_total, 1);
}

void matvec_coeffs(MatrixImpl* m, double** qhat, int64_t* rows) {
  *qhat = m->qhat.p;  // qhat | qp (both exchanged between the stages)
  *rows = 2 * std::max<int64_t>(m->colf->skel_total, 1);
}

void matvec_release_plan(const MatrixImpl* m) {
  g_graphs.erase(m);
  g_plans.erase(m);
  g_shards.erase(m);
}

void matvec_profile(MatrixImpl* m, int enable, double* phase_ms, int64_t* launches) {
  if (phase_ms)
    for (int i = 0; i < 7; ++i) phase_ms[i] = m->phase_ms[i];
  if (launches) *launches = m->launches;
  if (enable >= 0) {
    if (enable && !m->ev[0])
      for (auto& e : m->ev) SMASH_CUDA(cudaEventCreate(&e));
    m->profile = enable != 0;
    m->serial_phases = enable == 2;  // phases one after another (isolated kernel times)
    for (double& x : m->phase_ms) x = 0;
    m->launches = 0;
  }
}

void kernel_block(int kernel, double dx, int dim, const double* X, int64_t nx, const double* Y,
                  int64_t ny, double* out, cudaStream_t s) {
  if (nx * ny == 0) return;
  dispatch_kernel_dim(kernel, dim, [&]<int KER, int D>() {
    launch_block<KER, D>(X, nx, Y, ny, dx, out, s);
  });
  SMASH_CUDA(cudaGetLastError());
}

}  // namespace smash
