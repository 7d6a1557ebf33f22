// K2: block partitions on the GPU -- replaces smash.cluster.leaf_sets
// (smash/cluster.py:402-447) and smash.cluster.nearfield_set (:374-399).
//
// H2: the reference's dual recursion rec(root, root) is evaluated as a
// level-synchronous frontier of candidate pairs.  Each pair is classified with
// the exact admissibility test (well_separated, cluster.py:81-85): separated ->
// L; leaf x leaf -> Lm; one leaf -> pair it with the other side's children;
// neither -> all child pairs (cluster.py:428-446).  The sets are identical to
// the recursion's; they are returned sorted by (target, source), which is also
// the CSR layout the matvec consumes.
// HSS: L = sibling pairs in both orders, Lm = leaf diagonal (cluster.py:415-424).
// Nearfield sets N_i: top-down by level; candidates are the siblings in child
// order, then per member k of N_parent either k (leaf) or k's children, kept
// when not well separated (cluster.py:383-397).  Candidate order is preserved.
#include <cub/cub.cuh>

#include "smash_impl.cuh"

namespace smash {

namespace {

template <typename F>
void cub_call(F f, DBuf<char>& tmp, cudaStream_t s) {
  size_t bytes = 0;
  SMASH_CUDA(f((void*)nullptr, bytes));
  if (bytes > tmp.n) tmp.alloc(bytes, s);
  SMASH_CUDA(f((void*)tmp.p, bytes));
}

struct Geo {
  const double* ctr;
  const double* rad;
  const int* child_first;
  const int* nchild;
  int dim;
  double tau;
};

__device__ __forceinline__ bool sep(const Geo& g, int i, int j) {
  return well_separated(g.ctr + (size_t)i * g.dim, g.rad[i], g.ctr + (size_t)j * g.dim, g.rad[j],
                        g.dim, g.tau);
}

// classify: 0 -> L, 1 -> Lm, 2 -> refine (emit `nout` child pairs)
__global__ void k_classify(int64_t n, const int* fi, const int* fj, Geo g, int* cls, int64_t* nout) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  int i = fi[t], j = fj[t];
  int c, no = 0;
  if (sep(g, i, j)) {
    c = 0;
  } else {
    int ni = g.nchild[i], nj = g.nchild[j];
    if (!ni && !nj) {
      c = 1;
    } else {
      c = 2;
      no = (ni ? ni : 1) * (nj ? nj : 1);
    }
  }
  cls[t] = c;
  nout[t] = no;
}

__global__ void k_emit(int64_t n, const int* fi, const int* fj, const int* cls,
                       const int64_t* off, Geo g, int* ni_out, int* nj_out, int64_t* cntL,
                       int64_t* cntLm, int* Li, int* Lj, int* Lmi, int* Lmj) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  int i = fi[t], j = fj[t];
  int c = cls[t];
  if (c == 0) {
    unsigned long long p = atomicAdd((unsigned long long*)cntL, 1ULL);
    Li[p] = i;
    Lj[p] = j;
  } else if (c == 1) {
    unsigned long long p = atomicAdd((unsigned long long*)cntLm, 1ULL);
    Lmi[p] = i;
    Lmj[p] = j;
  } else {
    int ci = g.nchild[i], cj = g.nchild[j];
    int64_t o = off[t];
    if (!ci) {
      for (int b = 0; b < cj; ++b) { ni_out[o + b] = i; nj_out[o + b] = g.child_first[j] + b; }
    } else if (!cj) {
      for (int a = 0; a < ci; ++a) { ni_out[o + a] = g.child_first[i] + a; nj_out[o + a] = j; }
    } else {
      for (int a = 0; a < ci; ++a)
        for (int b = 0; b < cj; ++b) {
          ni_out[o + a * cj + b] = g.child_first[i] + a;
          nj_out[o + a * cj + b] = g.child_first[j] + b;
        }
    }
  }
}

// (target, source) keys packed with only the bits node ids need (nb = bits(n_nodes)),
// so the radix sort runs ceil(2 nb / 8) passes instead of 8
__global__ void k_pair_keys(int64_t n, const int* a, const int* b, int nb, uint64_t* k) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) k[t] = ((uint64_t)(uint32_t)a[t] << nb) | (uint32_t)b[t];
}

__global__ void k_pair_split(int64_t n, const uint64_t* k, int nb, int* a, int* b) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) { a[t] = (int)(k[t] >> nb); b[t] = (int)(k[t] & ((1ULL << nb) - 1ULL)); }
}

// CSR pointer by target: ptr[v] = first pair with target >= v
__global__ void k_csr_ptr(int n_nodes, int64_t npairs, const int* tgt, int* ptr) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v > n_nodes) return;
  int64_t lo = 0, hi = npairs;
  while (lo < hi) {
    int64_t m = (lo + hi) >> 1;
    if (tgt[m] >= v) hi = m; else lo = m + 1;
  }
  ptr[v] = (int)lo;
}

__global__ void k_hss_check(int n, const int* nchild, int* err) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n && nchild[v] != 0 && nchild[v] != 2) atomicOr(err, 1);
}

__global__ void k_hss_fill(int n, const int* child_first, const int* nchild, const int64_t* offL,
                           const int64_t* offLm, int* Li, int* Lj, int* Lmi, int* Lmj) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  if (nchild[v] == 2) {
    int c1 = child_first[v], c2 = c1 + 1;
    int64_t o = offL[v];
    Li[o] = c1; Lj[o] = c2;
    Li[o + 1] = c2; Lj[o + 1] = c1;
  } else if (nchild[v] == 0) {
    int64_t o = offLm[v];
    Lmi[o] = v; Lmj[o] = v;
  }
}

__global__ void k_hss_counts(int n, const int* nchild, int64_t* cL, int64_t* cLm) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  cL[v] = nchild[v] == 2 ? 2 : 0;
  cLm[v] = nchild[v] == 0 ? 1 : 0;
}

// sort pairs by (target, source) expressed in POSTORDER ids for the export
// ordering but kept in BFS ids for the matvec.  BFS order within a level equals
// postorder order, but across levels it does not; the CSR is by BFS target and
// the source order inside a row is irrelevant for the sums.
void sort_pairs(int64_t n, int n_nodes, DBuf<int>& a, DBuf<int>& b, DBuf<char>& tmp,
                cudaStream_t s) {
  if (!n) return;
  int nb = 1;
  while ((1LL << nb) <= (int64_t)n_nodes) ++nb;
  DBuf<uint64_t> k, k2;
  k.alloc(n, s); k2.alloc(n, s);
  k_pair_keys<<<cdiv(n, 256), 256, 0, s>>>(n, a.p, b.p, nb, k.p);
  cub_call([&](void* t, size_t& bytes) {
    return cub::DeviceRadixSort::SortKeys(t, bytes, k.p, k2.p, (int)n, 0, 2 * nb, s);
  }, tmp, s);
  k_pair_split<<<cdiv(n, 256), 256, 0, s>>>(n, k2.p, nb, a.p, b.p);
}

}  // namespace

PairLists* get_pairs(TreeImpl* t, double tau, int structure, cudaStream_t s) {
  SMASH_CHECK(structure == SMASH_STRUCT_H2 || structure == SMASH_STRUCT_HSS, SMASH_ERR_INVALID,
              "structure must be 'hss' or 'h2'");
  double key_tau = structure == SMASH_STRUCT_HSS ? 0.0 : tau;
  auto key = std::make_pair(key_tau, structure);
  auto it = t->pairs.find(key);
  if (it != t->pairs.end()) return it->second.get();
  std::unique_ptr<PairLists> P(new PairLists());
  const int n = t->n_nodes;
  DBuf<char> tmp;
  if (structure == SMASH_STRUCT_HSS) {
    DBuf<int> err;
    err.alloc(1, s);
    err.zero(s);
    k_hss_check<<<cdiv(n, 128), 128, 0, s>>>(n, t->nchild.p, err.p);
    DBuf<int64_t> cL, cLm, oL, oLm;
    cL.alloc(n + 1, s); cLm.alloc(n + 1, s); oL.alloc(n + 1, s); oLm.alloc(n + 1, s);
    cL.zero(s); cLm.zero(s);
    k_hss_counts<<<cdiv(n, 128), 128, 0, s>>>(n, t->nchild.p, cL.p, cLm.p);
    cub_call([&](void* tp, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(tp, b, cL.p, oL.p, n + 1, s);
    }, tmp, s);
    cub_call([&](void* tp, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(tp, b, cLm.p, oLm.p, n + 1, s);
    }, tmp, s);
    int64_t h[2];
    int herr = 0;
    d2h(&h[0], oL.p + n, 1, s);
    d2h(&h[1], oLm.p + n, 1, s);
    d2h(&herr, err.p, 1, s);
    sync(s);
    SMASH_CHECK(herr == 0, SMASH_ERR_INVALID, "hss structure needs a binary tree");
    P->nL = h[0];
    P->nLm = h[1];
    P->L_i.alloc(P->nL, s); P->L_j.alloc(P->nL, s);
    P->Lm_i.alloc(P->nLm, s); P->Lm_j.alloc(P->nLm, s);
    k_hss_fill<<<cdiv(n, 128), 128, 0, s>>>(n, t->child_first.p, t->nchild.p, oL.p, oLm.p,
                                            P->L_i.p, P->L_j.p, P->Lm_i.p, P->Lm_j.p);
  } else {
    Geo g{t->ctr.p, t->rad.p, t->child_first.p, t->nchild.p, t->dim, tau};
    // growable outputs
    int64_t capL = 1 << 16, capLm = 1 << 16;
    DBuf<int> Li, Lj, Lmi, Lmj;
    Li.alloc(capL, s); Lj.alloc(capL, s); Lmi.alloc(capLm, s); Lmj.alloc(capLm, s);
    DBuf<int64_t> cnt;  // [0] = |L|, [1] = |Lm|
    cnt.alloc(2, s);
    cnt.zero(s);
    DBuf<int> fi, fj;
    fi.alloc(1, s); fj.alloc(1, s);
    int root = 0;  // BFS id of the root
    h2d(fi.p, &root, 1, s);
    h2d(fj.p, &root, 1, s);
    int64_t nf = 1;
    int64_t hostL = 0, hostLm = 0;
    while (nf > 0) {
      DBuf<int> cls;
      DBuf<int64_t> nout, off;
      cls.alloc(nf, s); nout.alloc(nf + 1, s); off.alloc(nf + 1, s);
      k_classify<<<cdiv(nf, 256), 256, 0, s>>>(nf, fi.p, fj.p, g, cls.p, nout.p);
      // worst case growth of L/Lm this round is nf
      if (hostL + nf > capL || hostLm + nf > capLm) {
        int64_t nl = std::max(capL * 2, hostL + nf), nm = std::max(capLm * 2, hostLm + nf);
        DBuf<int> a, b, c, d;
        a.alloc(nl, s); b.alloc(nl, s); c.alloc(nm, s); d.alloc(nm, s);
        d2d(a.p, Li.p, hostL, s); d2d(b.p, Lj.p, hostL, s);
        d2d(c.p, Lmi.p, hostLm, s); d2d(d.p, Lmj.p, hostLm, s);
        Li = std::move(a); Lj = std::move(b); Lmi = std::move(c); Lmj = std::move(d);
        capL = nl; capLm = nm;
      }
      SMASH_CUDA(cudaMemsetAsync(nout.p + nf, 0, 8, s));
      cub_call([&](void* tp, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(tp, b, nout.p, off.p, (int)(nf + 1), s);
      }, tmp, s);
      int64_t nnext = 0;
      d2h(&nnext, off.p + nf, 1, s);
      sync(s);
      DBuf<int> gi, gj;
      gi.alloc(std::max<int64_t>(nnext, 1), s);
      gj.alloc(std::max<int64_t>(nnext, 1), s);
      k_emit<<<cdiv(nf, 256), 256, 0, s>>>(nf, fi.p, fj.p, cls.p, off.p, g, gi.p, gj.p,
                                           cnt.p, cnt.p + 1, Li.p, Lj.p, Lmi.p, Lmj.p);
      int64_t hc[2];
      d2h(hc, cnt.p, 2, s);
      sync(s);
      hostL = hc[0];
      hostLm = hc[1];
      fi = std::move(gi);
      fj = std::move(gj);
      nf = nnext;
    }
    P->nL = hostL;
    P->nLm = hostLm;
    P->L_i = std::move(Li); P->L_j = std::move(Lj);
    P->Lm_i = std::move(Lmi); P->Lm_j = std::move(Lmj);
  }
  sort_pairs(P->nL, n, P->L_i, P->L_j, tmp, s);
  sort_pairs(P->nLm, n, P->Lm_i, P->Lm_j, tmp, s);
  P->L_ptr.alloc(n + 1, s);
  P->Lm_ptr.alloc(n + 1, s);
  k_csr_ptr<<<cdiv(n + 1, 128), 128, 0, s>>>(n, P->nL, P->L_i.p, P->L_ptr.p);
  k_csr_ptr<<<cdiv(n + 1, 128), 128, 0, s>>>(n, P->nLm, P->Lm_i.p, P->Lm_ptr.p);
  SMASH_CUDA(cudaGetLastError());
  PairLists* out = P.get();
  t->pairs[key] = std::move(P);
  return out;
}

// ---------------------------------------------------------------------------
// nearfield sets
// ---------------------------------------------------------------------------
namespace {

// candidates of node j in reference order; calls f(k) for each
template <typename F>
__device__ void for_candidates(int j, const int* parent, const int* child_first, const int* nchild,
                               const int* nptr, const int* nidx, F f) {
  int p = parent[j];
  for (int c = 0; c < nchild[p]; ++c) {
    int u = child_first[p] + c;
    if (u != j) f(u);
  }
  for (int e = nptr[p]; e < nptr[p + 1]; ++e) {
    int k = nidx[e];
    if (nchild[k] == 0) {
      f(k);
    } else {
      for (int c = 0; c < nchild[k]; ++c) f(child_first[k] + c);
    }
  }
}

__global__ void k_near_count(int lb, int le, Geo g, const int* parent, const int* nptr,
                             const int* nidx, int* cnt) {
  int j = lb + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= le) return;
  int c = 0;
  for_candidates(j, parent, g.child_first, g.nchild, nptr, nidx, [&](int k) {
    if (!sep(g, j, k)) ++c;
  });
  cnt[j - lb] = c;
}

__global__ void k_near_fill(int lb, int le, Geo g, const int* parent, int* nptr, int* nidx,
                            const int* off, int base) {
  int j = lb + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= le) return;
  int o = base + off[j - lb];
  nptr[j] = o;
  int c = 0;
  for_candidates(j, parent, g.child_first, g.nchild, nptr, nidx, [&](int k) {
    if (!sep(g, j, k)) nidx[o + c++] = k;
  });
}

__global__ void k_set_int(int* p, int v) { *p = v; }

}  // namespace

NearSets* get_near(TreeImpl* t, double tau, cudaStream_t s) {
  auto it = t->near.find(tau);
  if (it != t->near.end()) return it->second.get();
  std::unique_ptr<NearSets> N(new NearSets());
  const int n = t->n_nodes;
  Geo g{t->ctr.p, t->rad.p, t->child_first.p, t->nchild.p, t->dim, tau};
  N->ptr.alloc(n + 1, s);
  int64_t cap = std::max<int64_t>(16, 4 * (int64_t)n);
  N->idx.alloc(cap, s);
  DBuf<char> tmp;
  // root: empty set at offset 0
  k_set_int<<<1, 1, 0, s>>>(N->ptr.p, 0);
  k_set_int<<<1, 1, 0, s>>>(N->ptr.p + 1, 0);
  int total = 0;
  for (int l = 2; l <= t->n_levels; ++l) {
    int lb = t->level_begin(l), le = t->level_end(l), cnt = le - lb;
    DBuf<int> c, off;
    c.alloc(cnt + 1, s); off.alloc(cnt + 1, s);
    SMASH_CUDA(cudaMemsetAsync(c.p + cnt, 0, 4, s));
    k_near_count<<<cdiv(cnt, 128), 128, 0, s>>>(lb, le, g, t->parent.p, N->ptr.p, N->idx.p, c.p);
    cub_call([&](void* tp, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(tp, b, c.p, off.p, cnt + 1, s);
    }, tmp, s);
    int add = 0;
    d2h(&add, off.p + cnt, 1, s);
    sync(s);
    if (total + add > cap) {
      int64_t nc = std::max<int64_t>(2 * cap, total + add);
      DBuf<int> bigger;
      bigger.alloc(nc, s);
      d2d(bigger.p, N->idx.p, total, s);
      N->idx = std::move(bigger);
      cap = nc;
    }
    k_near_fill<<<cdiv(cnt, 128), 128, 0, s>>>(lb, le, g, t->parent.p, N->ptr.p, N->idx.p, off.p,
                                               total);
    total += add;
    // the CSR end of this level's last node == start of the next level's first node
    k_set_int<<<1, 1, 0, s>>>(N->ptr.p + le, total);
  }
  N->total = total;
  SMASH_CUDA(cudaGetLastError());
  NearSets* out = N.get();
  t->near[tau] = std::move(N);
  return out;
}

}  // namespace smash

// ---------------------------------------------------------------------------
// exports (postorder ids, lexicographic order)
// ---------------------------------------------------------------------------
namespace smash {
namespace {

__global__ void k_post_pair_keys(int64_t n, const int* a, const int* b, const int* post,
                                 uint64_t* k) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) k[t] = ((uint64_t)(uint32_t)post[a[t]] << 32) | (uint32_t)post[b[t]];
}

__global__ void k_keys_to_pairs(int64_t n, const uint64_t* k, int64_t* out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) {
    out[2 * t] = (int64_t)(k[t] >> 32);
    out[2 * t + 1] = (int64_t)(k[t] & 0xffffffffULL);
  }
}

void export_pairs_one(const TreeImpl* t, int64_t n, const int* a, const int* b, int64_t* out,
                      cudaStream_t s) {
  if (!n || !out) return;
  DBuf<uint64_t> k, k2;
  DBuf<char> tmp;
  k.alloc(n, s); k2.alloc(n, s);
  k_post_pair_keys<<<cdiv(n, 256), 256, 0, s>>>(n, a, b, t->post.p, k.p);
  cub_call([&](void* tp, size_t& bytes) {
    return cub::DeviceRadixSort::SortKeys(tp, bytes, k.p, k2.p, (int)n, 0, 64, s);
  }, tmp, s);
  k_keys_to_pairs<<<cdiv(n, 256), 256, 0, s>>>(n, k2.p, out);
  sync(s);
}

__global__ void k_near_counts_post(int n, const int* post, const int* ptr, int64_t* cnt) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) cnt[post[v]] = ptr[v + 1] - ptr[v];
}

__global__ void k_near_copy_post(int n, const int* post, const int* ptr, const int* idx,
                                 const int64_t* optr, int64_t* oidx) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  int64_t o = optr[post[v]];
  for (int e = ptr[v]; e < ptr[v + 1]; ++e) oidx[o + e - ptr[v]] = post[idx[e]];
}

}  // namespace

void pairs_export(TreeImpl* t, PairLists* P, int64_t* L, int64_t* Lm, cudaStream_t s) {
  export_pairs_one(t, P->nL, P->L_i.p, P->L_j.p, L, s);
  export_pairs_one(t, P->nLm, P->Lm_i.p, P->Lm_j.p, Lm, s);
}

void near_export(TreeImpl* t, NearSets* N, int64_t* ptr, int64_t* idx, cudaStream_t s) {
  const int n = t->n_nodes;
  DBuf<int64_t> cnt, optr_own;
  cnt.alloc(n + 1, s);
  cnt.zero(s);
  k_near_counts_post<<<cdiv(n, 128), 128, 0, s>>>(n, t->post.p, N->ptr.p, cnt.p);
  int64_t* optr = ptr;
  if (!optr) { optr_own.alloc(n + 1, s); optr = optr_own.p; }
  DBuf<char> tmp;
  cub_call([&](void* tp, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(tp, b, cnt.p, optr, n + 1, s);
  }, tmp, s);
  if (idx) k_near_copy_post<<<cdiv(n, 128), 128, 0, s>>>(n, t->post.p, N->ptr.p, N->idx.p, optr, idx);
  sync(s);
}

}  // namespace smash
