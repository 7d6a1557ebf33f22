// K3 + K4: per-level batched interpolation basis + strong rank-revealing QR.
//
// One CTA per node (persistent grid over the level's nodes).  The CTA
//  1. evaluates the Lagrange basis at Chebyshev nodes of the node's padded box
//     for every point of ibar (smash/hss.py:219-238, smash/lowrank.py:103-144)
//     straight into the panel M = C^T (r rows x |ibar| columns), in shared
//     memory when it fits (global/L2 workspace otherwise);
//  2. runs column-pivoted Householder QR with LAPACK dlaqp2 semantics (what
//     scipy.linalg.qr(pivoting=True) -> dgeqp3 executes for min(m,n) < 128):
//     first-argmax pivot on the partial norms, dlarfg reflector, dlarf update,
//     norm downdate with the tol3z = sqrt(eps) recompute rule;
//  3. counts the numerical rank k = #{|R_ii| > rtol |R_00|} (lowrank.py:163-167);
//  4. runs the bounded-entry swap loop: W = R11^-1 R12; while max|W| > s, swap
//     the C-order argmax pair and refactor the permuted panel without pivoting
//     (lowrank.py:191-202), the panel being re-evaluated from the basis;
//  5. writes perm, G = W^T, the ordered skeleton labels and their coordinates
//     (lowrank.py:244-255).
// Thread-per-column mapping keeps every column's dot products and norms in a
// fixed sequential order; the row-major panel makes those accesses
// bank-conflict free.  Launch shape (plan_compress_launch): CTAs claim nodes
// from an atomic counter; the panel lives in shared memory when the level's
// capacity bound fits (1-warp CTAs for <= 64 columns, 128 threads for <= 128,
// else 256), per node in shared memory or the CTA's global slice on hybrid
// levels, and in the global/L2 slice (32-deep independent loads) when no
// shared panel fits.
#include "compress_common.cuh"

namespace smash {

namespace {

using namespace qr;
using namespace cmn;

// Fill panel columns c in [0, n): column c is ibar point colmap[c] (or c).
template <int D>
__device__ void build_panel(const CompressArgs& A, int v, int n, int mrows, double* P,
                            const int* colmap, const NodeSrc& src, const double* nodes) {
  const int r = A.r;
  const int m = A.tab.m;
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    const int pc = colmap ? colmap[c] : c;
    if (A.Cexp) {  // single-call compr: panel = C^T
      for (int q = 0; q < mrows; ++q) P[q * n + c] = A.Cexp[(size_t)pc * A.C_cols + q];
      continue;
    }
    double x[D];
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = src.base[(size_t)a * src.stride + pc];
    if (D == 1) {
      const double* nd = nodes;
      bool exact = false;
      for (int k = 0; k < m; ++k) exact |= (__dsub_rn(x[0], nd[k]) == 0.0);
      if (exact) {
        for (int k = 0; k < m; ++k) P[k * n + c] = (__dsub_rn(x[0], nd[k]) == 0.0) ? 1.0 : 0.0;
      } else {
        double Ssum = np_pairwise_sum(m, [&](int k) {
          return __ddiv_rn(A.tab.wv[k], __dsub_rn(x[0], nd[k]));
        });
        for (int k = 0; k < m; ++k)
          P[k * n + c] = __ddiv_rn(__ddiv_rn(A.tab.wv[k], __dsub_rn(x[0], nd[k])), Ssum);
      }
    } else {
      double L[D][MAX_M_AXIS_ND];
#pragma unroll
      for (int a = 0; a < D; ++a) lagrange_axis(x[a], nodes + a * MAX_M_AXIS_1D, A.tab.wv, m, L[a]);
      for (int q = 0; q < r; ++q) {
        const int* o = A.tab.order + 3 * q;
        double val = __dmul_rn(L[0][o[0]], L[1][o[1]]);
        if (D == 3) val = __dmul_rn(val, L[D - 1][o[2]]);
        P[q * n + c] = val;
      }
    }
    if (A.keep) {  // HSS: rows r.. hold S^T (hss.py:287)
      const int kp = A.keep[v];
      const double* sv = A.sv + A.sv_off[v];
      for (int q = 0; q < kp; ++q) P[(r + q) * n + c] = sv[(size_t)pc * kp + q];
    }
  }
}

// Compress one node whose panel lives at P (shared memory when SMP, else this
// CTA's slice of the global workspace): panel, dlaqp2, rank, swap loop, outputs.
template <int D, bool SMP, int CH>
__device__ __forceinline__ void compress_node(const CompressArgs& A, Shared& S, int v, int n,
                                              int mrows, const NodeSrc& src,
                                              double* __restrict__ P) {
  const int tid = threadIdx.x, NT = blockDim.x;
#ifdef SMASH_COMPRESS_PROF
  long long t0 = clock64();
#define PROF_MARK(k) if (tid == 0) { long long t1 = clock64(); atomicAdd(A.prof + (k), (unsigned long long)(t1 - t0)); t0 = t1; }
#else
#define PROF_MARK(k)
#endif
  build_panel<D>(A, v, n, mrows, P, nullptr, src, S.nodes);
  PROF_MARK(0)
  const int ld = n;
  const int m = mrows;
  const int kmax = min(m, n);
  // ---- dgeqp3 / dlaqp2.  Two barriers per pivot step: (1) the argmax partials
  // of the norms just downdated, (2) the pivot swap + reflector, both done by
  // warp 0; the trailing update and norm downdate then run over all threads,
  // which also fold the next step's argmax candidates.
  double bv = -1.0;
  int bi = 0x7fffffff;
  for (int j = tid; j < n; j += NT) {
    double nr = __dsqrt_rn(A.chains4 ? col_sumsq4<CH>(P, ld, j, 0, m) : col_sumsq<CH>(P, ld, j, 0, m));
    S.vn1[j] = nr;
    S.vn2[j] = nr;
    S.jpvt[j] = j;
    if (nr > bv) { bv = nr; bi = j; }
  }
  for (int i = 0; i < kmax; ++i) {
#ifdef SMASH_COMPRESS_PROF
    long long q0 = clock64();
#endif
    const int pvt = block_argmax_1bar(bv, bi, S);
#ifdef SMASH_COMPRESS_PROF
    long long q1 = clock64();
#endif
    if (tid < 32) {
      if (pvt != i) {
        for (int row = tid; row < m; row += 32) {
          double t = P[row * ld + pvt];
          P[row * ld + pvt] = P[row * ld + i];
          P[row * ld + i] = t;
        }
        if (tid == 0) {
          int it = S.jpvt[pvt]; S.jpvt[pvt] = S.jpvt[i]; S.jpvt[i] = it;
          S.vn1[pvt] = S.vn1[i];
          S.vn2[pvt] = S.vn2[i];
        }
        __syncwarp();
      }
      householder(P, ld, m, i, S);
    }
    __syncthreads();
#ifdef SMASH_COMPRESS_PROF
    long long q2 = clock64();
#endif
    const double tau = S.misc[0];
    bv = -1.0;
    bi = 0x7fffffff;
    for (int j = i + 1 + tid; j < n; j += NT) {
      // the norm-downdate divisions do not depend on the reflector: issue them
      // first so their latency hides under the dot-product chain
      double v1 = S.vn1[j];
      const double rv1 = 1.0 / v1;
      const double q2 = v1 / S.vn2[j];
      if (tau != 0.0) {
        if (A.chains4) apply_reflector4<CH>(P, ld, m, i, j, tau, S.vh);
        else apply_reflector<CH>(P, ld, m, i, j, tau, S.vh);
      }
      if (v1 != 0.0) {
        double q = fabs(P[i * ld + j]) * rv1;
        double temp = fmax(1.0 - q * q, 0.0);
        double temp2 = temp * (q2 * q2);
        if (temp2 <= TOL3Z) {
          double nv = i + 1 < m ? __dsqrt_rn(A.chains4 ? col_sumsq4<CH>(P, ld, j, i + 1, m)
                                                      : col_sumsq<CH>(P, ld, j, i + 1, m)) : 0.0;
          S.vn1[j] = nv;
          S.vn2[j] = nv;
          v1 = nv;
        } else {
          v1 = __dmul_rn(v1, __dsqrt_rn(temp));
          S.vn1[j] = v1;
        }
      }
      if (v1 > bv) { bv = v1; bi = j; }
    }
#ifdef SMASH_COMPRESS_PROF
    if (tid == 0) {
      long long q3 = clock64();
      atomicAdd(A.prof + 3, (unsigned long long)(q1 - q0));
      atomicAdd(A.prof + 4, (unsigned long long)(q2 - q1));
      atomicAdd(A.prof + 5, (unsigned long long)(q3 - q2));
      atomicAdd(A.prof + 6, 1ULL);
    }
#endif
  }
  __syncthreads();
  PROF_MARK(1)
  // ---- numerical rank (count semantics, lowrank.py:163-167)
  if (tid == 0) {
    int k = 0;
    double r0 = fabs(S.rdiag[0]);
    if (r0 != 0.0) {
      double thr = __dmul_rn(A.rtol, r0);
      for (int i = 0; i < kmax; ++i) k += fabs(S.rdiag[i]) > thr ? 1 : 0;
    }
    S.imisc[0] = min(k, kmax);
  }
  __syncthreads();
  const int k = S.imisc[0];
  // ---- bounded-entry swap loop (lowrank.py:191-202)
  int swaps = 0;
  while (k > 0 && k < n) {
    double bv = -1.0;
    int bi = 0x7fffffff;
    const int nk = n - k;
    for (int j = k + tid; j < n; j += NT) {
      // W = R11^-1 R12 by back substitution, left-looking: row a accumulates
      // the terms of rows k-1 .. a+1 in that order -- the same FMA sequence as
      // the column-sweep (dtrsv) form, with chunked independent loads (the
      // solved x_c of this column and row a of R11, shared by all threads).
      // (With the four-chain option the terms of a row go to four accumulators by c mod 4:
      // G = W^T is compared by SURVEY 8(c) rule 3, not bit for bit.)
      for (int a = k - 1; a >= 0; --a) {
        double acc = P[a * ld + j];
        double acc4[4] = {0.0, 0.0, 0.0, 0.0};
        constexpr int CH = 8;
        for (int c0 = k - 1; c0 > a; c0 -= CH) {
          double xs[CH], rs[CH];
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            const bool ok = c0 - c > a;
            xs[c] = ok ? P[(c0 - c) * ld + j] : 0.0;
            rs[c] = ok ? P[a * ld + (c0 - c)] : 0.0;
          }
          if (A.chains4) {
#pragma unroll
            for (int c = 0; c < CH; ++c) acc4[c & 3] = __fma_rn(-xs[c], rs[c], acc4[c & 3]);
          } else {
#pragma unroll
            for (int c = 0; c < CH; ++c)
              if (c0 - c > a) acc = __fma_rn(-xs[c], rs[c], acc);
          }
        }
        if (A.chains4) acc = __dadd_rn(acc, __dadd_rn(__dadd_rn(acc4[0], acc4[1]), __dadd_rn(acc4[2], acc4[3])));
        const double x = __ddiv_rn(acc, P[a * ld + a]);
        P[a * ld + j] = x;
        argmax_combine(bv, bi, fabs(x), a * nk + (j - k));
      }
    }
    block_argmax(bv, bi, S);
    if (!(bv > A.s_bound)) break;
    if (swaps >= MAX_SWAPS) {
      if (tid == 0) atomicOr(A.err, DEV_SWAP_CAP);
      break;
    }
    if (tid == 0) {
      int a = bi / nk, jj = bi % nk;
      int t = S.jpvt[a]; S.jpvt[a] = S.jpvt[k + jj]; S.jpvt[k + jj] = t;
    }
    __syncthreads();
    ++swaps;
    build_panel<D>(A, v, n, mrows, P, S.jpvt, src, S.nodes);
    __syncthreads();
    for (int i = 0; i < k; ++i) {  // unpivoted QR (dgeqr2); rows < k of R suffice
      householder(P, ld, m, i, S);
      __syncthreads();
      const double tau = S.misc[0];
      if (tau != 0.0)
        for (int j = i + 1 + tid; j < n; j += NT) apply_reflector<CH>(P, ld, m, i, j, tau, S.vh);
      __syncthreads();
    }
  }
  __syncthreads();
  PROF_MARK(2)
  // ---- outputs
  if (tid == 0) {
    A.rank[v] = k;
    if (swaps) atomicAdd(A.swaps, (unsigned long long)swaps);
  }
  const int64_t io = A.ib_off[v];
  for (int c = tid; c < n; c += NT) A.perm[io + c] = S.jpvt[c];
  if (k > 0 && k < n) {
    double* G = A.G + A.g_off[v];
    const int nk = n - k;
    for (int e = tid; e < nk * k; e += NT) {
      int b = e / k, a = e % k;
      G[e] = P[a * ld + k + b];
    }
  }
  if (A.tmp_lab) {
    const int64_t lo = io - A.ib_level_base;
    for (int a = tid; a < k; a += NT) {
      int pc = S.jpvt[a];
      A.tmp_lab[lo + a] = src.lab ? src.lab[pc] : src.lab0 + pc;
      for (int d = 0; d < D; ++d)
        A.tmp_pts[(size_t)d * A.tmp_stride + lo + a] = src.base[(size_t)d * src.stride + pc];
    }
  }
  __syncthreads();
}

// MODE: 0 = panel in the global workspace, 1 = shared memory, 2 = per node
// (hybrid).  The global-only variant uses deeper load chunks (more registers,
// fewer CTAs per SM); the shared variants are sized for >= 4 CTAs per SM.
template <int D, int MODE>
__global__ void __launch_bounds__(COMPRESS_THREADS, MODE == 0 ? 2 : 4) k_compress(CompressArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Shared S;
  double* spanel;
  {
    double* d = reinterpret_cast<double*>(smem_raw);
    S.vn1 = d; d += A.nmax;
    S.vn2 = d; d += A.nmax;
    S.vh = d; d += A.mmax;
    S.rdiag = d; d += A.mmax;
    S.nodes = d; d += 3 * MAX_M_AXIS_1D;
    S.redv = d; d += 32;
    S.misc = d; d += 8;
    int* ip = reinterpret_cast<int*>(d);
    S.redi = ip; ip += 32;
    S.imisc = ip; ip += 8;
    S.jpvt = ip; ip += A.nmax + (A.nmax & 1);
    spanel = reinterpret_cast<double*>(ip);
    S.panel = nullptr;
  }
  double* gpanel = A.gws ? A.gws + (size_t)blockIdx.x * A.mmax * A.nmax : nullptr;
  const int tid = threadIdx.x, NT = blockDim.x;
  // dynamic node assignment: a CTA takes the next unclaimed node when it is done
  // (node costs vary with |ibar|, rank and swap iterations)
  for (int v = A.lb + blockIdx.x; v < A.le;) {
    const int n = A.nib[v];
    if (n <= A.n_lo || n > A.n_hi) {  // another launch of this level takes this size class
      __syncthreads();
      if (tid == 0) S.imisc[4] = A.lb + (int)gridDim.x + atomicAdd(A.next, 1);
      __syncthreads();
      v = S.imisc[4];
      continue;
    }
    const int mrows = A.Cexp ? A.C_cols : A.r + (A.keep ? A.keep[v] : 0);
    SMASH_DASSERT(n >= 0 && n <= A.nmax && mrows <= A.mmax);
    const NodeSrc src = A.Cexp ? NodeSrc{nullptr, 0, nullptr, 0} : node_src(A, v);
    if (n == 0) {  // (uniform branch) everyone has read v before it is overwritten
      __syncthreads();
      if (tid == 0) {
        A.rank[v] = 0;
        S.imisc[4] = A.lb + (int)gridDim.x + atomicAdd(A.next, 1);
      }
      __syncthreads();
      v = S.imisc[4];
      continue;
    }
    // ---- padded box + Chebyshev nodes (hss.py:39-45, lowrank.py:103-105,127-134)
    if (!A.Cexp) {
      if (tid == 0) {
        double plo[3], phi[3];
        double scale = 1.0;
        for (int a = 0; a < D; ++a) {
          double lo = A.lo[(size_t)v * D + a], hi = A.hi[(size_t)v * D + a];
          if (__dsub_rn(hi, lo) < A.pad) {
            lo = __dsub_rn(lo, A.half_pad);
            hi = __dadd_rn(hi, A.half_pad);
          }
          plo[a] = lo; phi[a] = hi;
          scale = fmax(scale, __dsub_rn(hi, lo));
        }
        // scale = max(max(hi - lo), 1.0)
        int bad = 0;
        for (int a = 0; a < D; ++a)
          if (!(__dsub_rn(phi[a], plo[a]) > __dmul_rn(1e-14, scale))) bad = 1;
        if (bad) atomicOr(A.err, DEV_DEGENERATE_BOX);
        for (int a = 0; a < D; ++a) { S.misc[2 + a] = plo[a]; S.misc[5 + a] = phi[a]; }
      }
      __syncthreads();
      const int m = A.tab.m;
      for (int e = tid; e < D * m; e += NT) {
        int a = e / m, k = e % m;
        double lo = S.misc[2 + a], hi = S.misc[5 + a];
        double t1 = __dmul_rn(0.5, __dadd_rn(lo, hi));
        double t2 = __dmul_rn(0.5, __dsub_rn(hi, lo));
        S.nodes[a * MAX_M_AXIS_1D + k] = __dadd_rn(t1, __dmul_rn(t2, A.tab.cosv[k]));
      }
      __syncthreads();
    }
    // panel in shared memory when it fits the launch's capacity (hybrid levels:
    // the few oversized nodes use the CTA's global/L2 workspace slice)
    if (MODE == 1 || (MODE == 2 && (int64_t)n * mrows <= A.panel_cap))
      compress_node<D, true, 8>(A, S, v, n, mrows, src, spanel);
    else
      compress_node<D, false, MODE == 0 ? 32 : 8>(A, S, v, n, mrows, src, gpanel);
    if (tid == 0) S.imisc[4] = A.lb + (int)gridDim.x + atomicAdd(A.next, 1);
    __syncthreads();
    v = S.imisc[4];
  }
}

// single-call interp_basis: one thread per point
template <int D>
__global__ void k_basis_single(BasisTables tab, int r, const double* pts, int64_t n, double plo0,
                               double plo1, double plo2, double phi0, double phi1, double phi2,
                               double* out) {
  __shared__ double nodes[3 * MAX_M_AXIS_1D];
  double plo[3] = {plo0, plo1, plo2}, phi[3] = {phi0, phi1, phi2};
  const int m = tab.m;
  for (int e = threadIdx.x; e < D * m; e += blockDim.x) {
    int a = e / m, k = e % m;
    double t1 = __dmul_rn(0.5, __dadd_rn(plo[a], phi[a]));
    double t2 = __dmul_rn(0.5, __dsub_rn(phi[a], plo[a]));
    nodes[a * MAX_M_AXIS_1D + k] = __dadd_rn(t1, __dmul_rn(t2, tab.cosv[k]));
  }
  __syncthreads();
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  if (D == 1) {
    double L[MAX_M_AXIS_1D];
    lagrange_axis(pts[c], nodes, tab.wv, m, L);
    for (int k = 0; k < r; ++k) out[c * r + k] = L[k];
  } else {
    double L[D][MAX_M_AXIS_ND];
    for (int a = 0; a < D; ++a)
      lagrange_axis(pts[(size_t)a * n + c], nodes + a * MAX_M_AXIS_1D, tab.wv, m, L[a]);
    for (int q = 0; q < r; ++q) {
      const int* o = tab.order + 3 * q;
      double val = __dmul_rn(L[0][o[0]], L[1][o[1]]);
      if (D == 3) val = __dmul_rn(val, L[D - 1][o[2]]);
      out[c * r + q] = val;
    }
  }
}

}  // namespace

size_t compress_smem_bytes(int nmax, int mmax, bool panel_in_smem) {
  size_t b = 8 * (2 * (size_t)nmax + 2 * (size_t)mmax + 3 * MAX_M_AXIS_1D + 32 + 8);
  b += 4 * (32 + 8 + (size_t)nmax + (nmax & 1));
  b = (b + 15) & ~size_t(15);
  if (panel_in_smem) b += 8 * (size_t)nmax * mmax;
  return b;
}

size_t plan_compress_launch(CompressArgs& A, int cnt, int smem_limit, int nsm, int* grid) {
  constexpr size_t SM_BYTES = 228 * 1024, CTA_RESERVED = 1024;
  const size_t fixed = compress_smem_bytes(A.nmax, A.mmax, false);
  const size_t full = compress_smem_bytes(A.nmax, A.mmax, true);
  static const int gper = getenv("SMASH_GWS_PER_SM") ? atoi(getenv("SMASH_GWS_PER_SM")) : 4;
  if ((full <= SM_BYTES / 2 - CTA_RESERVED || cnt <= nsm) && (int)full <= smem_limit) {
    // every node fits (>= 2 CTAs per SM, or a level with at most one node per SM)
    A.panel_cap = (int64_t)A.nmax * A.mmax;
    // narrow panels (<= 128 columns): 128-thread CTAs, twice as many nodes in flight
    // for the same warps per SM (64 registers per thread)
    static const int narrow = getenv("SMASH_COMPRESS_NARROW") ? atoi(getenv("SMASH_COMPRESS_NARROW")) : 128;
    static const int tiny = getenv("SMASH_COMPRESS_TINY") ? atoi(getenv("SMASH_COMPRESS_TINY")) : 64;
    static const int tiny_t = getenv("SMASH_COMPRESS_TINY_T") ? atoi(getenv("SMASH_COMPRESS_TINY_T")) : 32;
    A.threads = A.nmax <= tiny ? tiny_t : A.nmax <= narrow ? 128 : COMPRESS_THREADS;
    const int cap = std::min(32, 1024 / A.threads);  // 64 registers per thread: <= 1024 threads per SM
    int per_sm = (int)std::min<size_t>(cap, std::max<size_t>(1, SM_BYTES / (full + CTA_RESERVED)));
    *grid = std::min(cnt, nsm * per_sm);
    return full;
  }
  // Capacity bounds are loose (|ibar| <= sum_c min(r, |ibar_c|)): when half the
  // capacity fits two CTAs per SM, size the shared panel for that and let the
  // rare larger nodes fall back to the global workspace.
  const size_t half = compress_smem_bytes((A.nmax + 1) / 2, A.mmax, true);
  // (a launch whose whole size class exceeds the two-per-SM panel skips this: one CTA per SM
  // with the full panel in shared memory beats two CTAs on global/L2 panels)
  const bool all_oversized = (int)full <= smem_limit &&
      (int64_t)(A.n_lo + 1) * A.mmax > (int64_t)((SM_BYTES / 2 - CTA_RESERVED - fixed) / 8);
  if (half <= SM_BYTES / 2 - CTA_RESERVED && !all_oversized) {
    const size_t smem = std::min<size_t>(SM_BYTES / 2 - CTA_RESERVED, (size_t)smem_limit);
    A.panel_cap = (int64_t)((smem - fixed) / 8);
    *grid = std::min(cnt, nsm * 2);
    return smem;
  }
  if ((int)full <= smem_limit && full > SM_BYTES / 2) {
    A.panel_cap = (int64_t)A.nmax * A.mmax;
    *grid = std::min(cnt, nsm);
    return full;
  }
  A.panel_cap = 0;
  *grid = std::min(cnt, nsm * gper);
  return fixed;
}

// Wide levels of adaptive trees mix small nodes (leaves, sparse parents) with nodes near
// the capacity bound; one launch sized for the capacity runs the small ones in oversized
// CTAs at low occupancy.  Such a level is split by |ibar| into size classes (<= 64,
// <= 128, rest), each launched with its own CTA size and shared panel; the CTAs of a
// launch skip the other classes' nodes.  Latency-bound levels (<= one node per SM) and
// levels whose capacity is already small keep one launch.
// four-chain dot products by default (cfg5 build -8 %, the full-size skeleton / G parity
// unchanged); SMASH_QR_CHAINS=1 restores the sequential dlarf / dnrm2 order
static bool compress_chains4() {
  static const bool c4 = !(getenv("SMASH_QR_CHAINS") && atoi(getenv("SMASH_QR_CHAINS")) == 1);
  return c4;
}

// Register-column launch (compress_rc.cuh) of a size class of at most 320 columns: the first
// variant whose shared memory fits.
static bool plan_compress_rc(CompressPass& P, int cnt, int smem_limit, int nsm) {
  constexpr size_t SM_BYTES = 228 * 1024, CTA_RESERVED = 1024;
  const int nmax = P.a.nmax, mmax = P.a.mmax;
  RcVariant cand[2];
  int nc = 0;
  if (nmax <= 32) { cand[nc++] = {32, mmax > 96 ? 48 : 32, true}; }
  else if (nmax <= 64) { cand[nc++] = {64, mmax > 96 ? 48 : 32, true}; }
  else if (nmax <= 128) { cand[nc++] = {128, 32, false}; cand[nc++] = {128, 32, true}; }
  else if (nmax <= 256) { cand[nc++] = {256, 32, false}; cand[nc++] = {256, 48, true}; }
  else if (nmax <= 320) cand[nc++] = {320, 44, true};
  else if (nmax <= 1024) cand[nc++] = {256, 48, true, 4};  // cluster of four CTAs
  // the fitting variant with the most CTAs per SM (ties: the first, resident R11 before streamed)
  int best = -1, best_per_sm = 0;
  size_t best_smem = 0;
  for (int c = 0; c < nc; ++c) {
    const size_t smem = compress_rc_smem_bytes(cand[c], mmax, P.a.dim);
    if ((int64_t)smem > (int64_t)smem_limit) continue;
    // __launch_bounds__ of k_compress_rc: 128 registers per thread, up to 255 with > 32 register rows
    const int by_regs = cand[c].rr > 32 ? std::max(1, 65536 / (cand[c].nt * 256)) : std::min(16, 65536 / (cand[c].nt * 128));
    const int by_smem = (int)std::max<size_t>(1, SM_BYTES / (smem + CTA_RESERVED));
    const int per_sm = std::min(by_regs, by_smem);
    if (per_sm > best_per_sm) { best = c; best_per_sm = per_sm; best_smem = smem; }
  }
  if (best < 0) return false;
  P.grid = std::min(cnt, nsm * best_per_sm);
  if (cand[best].cs > 1) P.grid = std::max(1, std::min(cnt, nsm / cand[best].cs)) * cand[best].cs;
  P.smem = best_smem;
  P.rc = cand[best];
  P.a.threads = cand[best].nt;
  return true;
}

int plan_compress_passes(const CompressArgs& A0, int cnt, int smem_limit, int nsm, CompressPass* out) {
  static const bool split = getenv("SMASH_COMPRESS_NOSPLIT") == nullptr;
  // (read per call: tests switch between the two kernels within a process)
  const bool rc = !(getenv("SMASH_COMPRESS_RC") && atoi(getenv("SMASH_COMPRESS_RC")) == 0) &&
                  !A0.Cexp && compress_chains4();
  if (rc && (!split || cnt <= nsm || A0.nmax <= 32)) {
    out[0] = CompressPass();
    out[0].a = A0;
    if (plan_compress_rc(out[0], cnt, smem_limit, nsm)) return 1;
  }
  if (rc && split && cnt > nsm && A0.nmax > 32) {
    // size classes (.., 32], (32, 64], (64, 128], (128, 256], (256, 320], (320, 1024] on the
    // register-column kernel as far as its variants fit, one k_compress launch for the rest
    const int rb[6] = {32, 64, 128, 256, 320, 1024};
    int np = 0, lo = -1;
    for (int b : rb) {
      if (lo >= A0.nmax) break;
      CompressPass P;
      P.a = A0;
      P.a.n_lo = lo;
      P.a.n_hi = b;
      P.a.nmax = std::min(A0.nmax, b);
      if (!plan_compress_rc(P, cnt, smem_limit, nsm)) break;
      out[np++] = P;
      lo = b;
    }
    if (lo < A0.nmax) {
      CompressPass& P = out[np++];
      P = CompressPass();
      P.a = A0;
      P.a.n_lo = lo;
      P.smem = plan_compress_launch(P.a, cnt, smem_limit, nsm, &P.grid);
    }
    return np;
  }
  static const bool split4 = getenv("SMASH_COMPRESS_NOSPLIT4") == nullptr;
  // fourth class: nodes too wide for two shared panels per SM but not for one
  int b3 = 0x7fffffff;
  {
    constexpr size_t SM_BYTES = 228 * 1024, CTA_RESERVED = 1024;
    const size_t lim2 = SM_BYTES / 2 - CTA_RESERVED;
    // widest panel of mmax rows with two CTAs per SM (fixed part grows with the columns)
    int n2 = A0.nmax;
    while (n2 > 128 && compress_smem_bytes(n2, A0.mmax, true) > lim2) --n2;
    if (split4 && n2 > 128 && n2 < A0.nmax && (int)compress_smem_bytes(A0.nmax, A0.mmax, true) <= smem_limit)
      b3 = n2;
  }
  const int bounds[4] = {64, 128, b3, 0x7fffffff};
  if (!split || cnt <= nsm || A0.nmax <= bounds[0]) {
    out[0] = CompressPass();
    out[0].a = A0;
    out[0].smem = plan_compress_launch(out[0].a, cnt, smem_limit, nsm, &out[0].grid);
    return 1;
  }
  int np = 0, lo = -1;
  for (int b : bounds) {
    if (lo >= A0.nmax) break;
    CompressPass& P = out[np++];
    P = CompressPass();
    P.a = A0;
    P.a.n_lo = lo;
    P.a.n_hi = b;
    P.a.nmax = std::min(A0.nmax, b);
    P.smem = plan_compress_launch(P.a, cnt, smem_limit, nsm, &P.grid);
    lo = b;
  }
  return np;
}

#ifdef SMASH_COMPRESS_PROF
__device__ unsigned long long g_compress_prof[8];
#endif
__device__ int g_compress_next[MAX_COMPRESS_PASSES + 1];  // dynamic node counters (one per concurrent launch, reset before it)

void launch_compress(const CompressArgs& a_in, int grid, size_t smem, cudaStream_t s, int slot) {
  CompressArgs a = a_in;
  a.chains4 = compress_chains4();
  {
    void* nx = nullptr;
    SMASH_CUDA(cudaGetSymbolAddress(&nx, g_compress_next));
    a.next = reinterpret_cast<int*>(nx) + slot;
    SMASH_CUDA(cudaMemsetAsync(a.next, 0, sizeof(int), s));
  }
#ifdef SMASH_COMPRESS_PROF
  void* pp = nullptr;
  SMASH_CUDA(cudaGetSymbolAddress(&pp, g_compress_prof));
  SMASH_CUDA(cudaMemsetAsync(pp, 0, sizeof(g_compress_prof), s));
  a.prof = reinterpret_cast<unsigned long long*>(pp);
#endif
  auto go = [&](auto kern) {
    SMASH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, a.threads, smem, s>>>(a);
  };
  const int mode = a.panel_cap >= (int64_t)a.nmax * a.mmax ? 1 : a.panel_cap == 0 ? 0 : 2;
  auto by_dim = [&](auto m) {
    constexpr int M = decltype(m)::value;
    if (a.dim == 1) go(k_compress<1, M>);
    else if (a.dim == 2) go(k_compress<2, M>);
    else go(k_compress<3, M>);
  };
  if (mode == 0) by_dim(std::integral_constant<int, 0>{});
  else if (mode == 1) by_dim(std::integral_constant<int, 1>{});
  else by_dim(std::integral_constant<int, 2>{});
  SMASH_CUDA(cudaGetLastError());
#ifdef SMASH_COMPRESS_PROF
  unsigned long long h[8];
  SMASH_CUDA(cudaMemcpyAsync(h, pp, sizeof(h), cudaMemcpyDeviceToHost, s));
  SMASH_CUDA(cudaStreamSynchronize(s));
  fprintf(stderr, "compress nodes %d mode %d grid %d: Mcycles panel %.2f qr %.2f rank+solve+swaps %.2f"
          " | per step: argmax+wait %.0f, swap+reflector %.0f, update+downdate %.0f cycles\n",
          a.le - a.lb, mode, grid, h[0] * 1e-6, h[1] * 1e-6, h[2] * 1e-6,
          h[6] ? (double)h[3] / h[6] : 0.0, h[6] ? (double)h[4] / h[6] : 0.0,
          h[6] ? (double)h[5] / h[6] : 0.0);
#endif
}

void launch_compress_rc(const CompressArgs& a_in, const RcVariant& v, int grid, size_t smem, cudaStream_t s, int slot) {
  CompressArgs a = a_in;
  a.chains4 = true;
  void* nx = nullptr;
  SMASH_CUDA(cudaGetSymbolAddress(&nx, g_compress_next));
  a.next = reinterpret_cast<int*>(nx) + slot;
  SMASH_CUDA(cudaMemsetAsync(a.next, 0, sizeof(int), s));
#ifdef SMASH_COMPRESS_PROF
  void* pp = nullptr;
  SMASH_CUDA(cudaGetSymbolAddress(&pp, g_compress_prof));
  SMASH_CUDA(cudaMemsetAsync(pp, 0, sizeof(g_compress_prof), s));
  a.prof = reinterpret_cast<unsigned long long*>(pp);
#endif
  if (a.dim == 1) launch_compress_rc_dim<1>(a, v, grid, smem, s);
  else if (a.dim == 2) launch_compress_rc_dim<2>(a, v, grid, smem, s);
  else launch_compress_rc_dim<3>(a, v, grid, smem, s);
#ifdef SMASH_COMPRESS_PROF
  unsigned long long h[8];
  SMASH_CUDA(cudaMemcpyAsync(h, pp, sizeof(h), cudaMemcpyDeviceToHost, s));
  SMASH_CUDA(cudaStreamSynchronize(s));
  const double st = h[7] ? (double)h[7] : 1.0;
  fprintf(stderr, "compress_rc nodes %d nt %d rr %d grid %d: Mcycles (thread 0 of every CTA) build %.2f qr %.2f solve %.2f reqr %.2f"
          " | per step: argmax %.0f, reflector (owner warp) %.0f, wait %.0f, update+downdate %.0f cycles (%llu steps)\n",
          a.le - a.lb, v.nt, v.rr, grid, h[0] * 1e-6, (h[1] + h[2] + h[3] + h[4]) * 1e-6, h[5] * 1e-6, h[6] * 1e-6,
          h[1] / st, h[2] / st, h[3] / st, h[4] / st, h[7]);
#endif
}

void launch_basis_single(int dim, const double* plo, const double* phi, const BasisTables& tab,
                         int r, const double* pts_soa, int64_t n, double* out, int* err,
                         cudaStream_t s) {
  (void)err;
  double l[3] = {0, 0, 0}, h[3] = {0, 0, 0};
  for (int a = 0; a < dim; ++a) { l[a] = plo[a]; h[a] = phi[a]; }
  unsigned g = cdiv(std::max<int64_t>(n, 1), 128);
  if (dim == 1) k_basis_single<1><<<g, 128, 0, s>>>(tab, r, pts_soa, n, l[0], l[1], l[2], h[0], h[1], h[2], out);
  if (dim == 2) k_basis_single<2><<<g, 128, 0, s>>>(tab, r, pts_soa, n, l[0], l[1], l[2], h[0], h[1], h[2], out);
  if (dim == 3) k_basis_single<3><<<g, 128, 0, s>>>(tab, r, pts_soa, n, l[0], l[1], l[2], h[0], h[1], h[2], out);
  SMASH_CUDA(cudaGetLastError());
}

}  // namespace smash
