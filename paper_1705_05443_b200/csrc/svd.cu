// K5: HSS nearfield block-row assembly + batched truncated SVD -- replaces the
// per-node `block(ibar, near columns)` + `truncated_svd` of build_hss
// (smash/hss.py:279-299, smash/lowrank.py:265-276).
//
// One CTA per node.  A (|ibar| x n_near) is generated from the kernel into an
// L2-resident workspace, then its left singular subspace is computed as
//   A P = Q1 R      column-pivoted Householder QR, stopped once |R_ii| falls
//                   2^3 below the fp64 noise floor (2^-56 |R_00|, SMASH_SVD_FLOOR):
//                   the discarded block perturbs the singular values by about
//                   sqrt(n) 2^-56 sigma_1, the order of LAPACK's own rounding.
//                   Stopping AT the noise floor (2^-53) made the kept vectors near
//                   the eps_svd cut ~10x less accurate (cfg 4 full size: 21 rank
//                   flips vs 1 for a LAPACK restatement; 2^-56 .. 2^-63 all give
//                   the LAPACK restatement's counts, profiles/hss_skeleton_census_r02.txt);
//   R_k^T = Q2 R2   unpivoted QR of the k' x n_near leading rows (transposed);
//   R2 V = W        one-sided (Hestenes) Jacobi on the k' x k' triangle,
//                   round-robin pair order, one warp per pair;
// so sigma_j = ||W_j|| and U(A) = Q1[:, :k'] V.  keep = #{sigma >= eps sigma_1}
// (lowrank.py:275) and S = U[:, kept] (descending sigma) is handed to the
// compression kernel as extra panel rows.  Column order and signs of S do not
// change the pivoted QR of [U_basis, S]^T in exact arithmetic.
#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"
#include "qr_device.cuh"
#include "svd.cuh"

namespace smash {

namespace {

using namespace qr;

constexpr int SVD_THREADS = 256;
constexpr int MAX_NEAR = 64;
// shared-memory area (doubles) for B = R_k^T, then J / V, then the back-transform Y
// (96 KB: two CTAs per SM; J + V fit up to rank 78)
constexpr int SVD_BIG = 12288;

struct IbarSide {
  const int* nib;       // |ibar| per BFS node (valid for the current + deeper levels)
  const int* rank;
  const int* pt_a;      // leaf point range start
  const int* pt_b;
  const double* P;      // tree-ordered points SoA
  int64_t P_stride;
  const double* Sk;     // compact skeleton points SoA
  int64_t S_stride;
  const int* skel_off;
};

struct SvdArgs {
  int lb, le, dim, kernel;
  double dx, eps_svd;
  double floor_rel, floor_leaf;  // QR truncation |R_ii| <= floor |R_00| (internal / leaf nodes)
  int transpose;  // 0: K(target, source) (row pass); 1: K(source, target) (column pass)
  const int* nchild;
  const int* child_first;
  const int* near_ptr;
  const int* near_idx;
  IbarSide self, other;
  // outputs
  int* keep;
  const int64_t* sv_off;
  double* sv;
  int* nn_out;
  // workspace
  double* gws;
  int64_t gws_stride;  // doubles per CTA
  int nmax, nnmax;
  int* err;
  long long* dbg;  // SMASH_SVD_DBG: phase cycle counts of block 0's first nodes
};

__device__ __forceinline__ int ibar_size(const IbarSide& s, const int* nchild, const int* child_first,
                                         int j) {
  if (nchild[j] == 0) return s.pt_b[j] - s.pt_a[j];
  int n = 0;
  for (int c = 0; c < nchild[j]; ++c) n += s.rank[child_first[j] + c];
  return n;
}

__device__ __forceinline__ const double* ibar_base(const IbarSide& s, const int* nchild,
                                                   const int* child_first, int j, int64_t* stride) {
  if (nchild[j] == 0) {
    *stride = s.P_stride;
    return s.P + s.pt_a[j];
  }
  *stride = s.S_stride;
  return s.Sk + s.skel_off[child_first[j]];
}

__global__ void k_near_cols(SvdArgs A) {
  int v = A.lb + blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= A.le) return;
  int nn = 0;
  for (int e = A.near_ptr[v]; e < A.near_ptr[v + 1]; ++e)
    nn += ibar_size(A.other, A.nchild, A.child_first, A.near_idx[e]);
  A.nn_out[v - A.lb] = nn;
}

// Column work by 8-lane groups: a column of the panel (column-major, stride 1) is
// split over the group's lanes (rows gl, gl + 8, ...), each lane keeping up to
// GR rows in registers between the dot product and the update; sums are
// combined by a 3-level butterfly (identical in every lane of the group).
constexpr int GR = 16;  // register-cached rows per lane (covers 128 rows below the pivot)

__device__ __forceinline__ double grp_sum(double x, unsigned gm) {
  x += __shfl_xor_sync(gm, x, 4);
  x += __shfl_xor_sync(gm, x, 2);
  x += __shfl_xor_sync(gm, x, 1);
  return x;
}

__device__ __forceinline__ double grp_sumsq(const double* c, int r0, int r1, int gl, unsigned gm) {
  double s0 = 0.0, s1 = 0.0;
  int r = r0 + gl;
  for (; r + 8 < r1; r += 16) {
    const double a = c[r], b = c[r + 8];
    s0 = fma(a, a, s0);
    s1 = fma(b, b, s1);
  }
  if (r < r1) s0 = fma(c[r], c[r], s0);
  return grp_sum(s0 + s1, gm);
}

// H_i^T applied to column c (rows i..m-1; v_i = 1, v_r = vh[r] below): the
// group's rows i+1.. are loaded once (registers), w = c_i + v^T c, c -= tau w v.
// Returns the updated c_i in every lane; x[] keeps the updated rows (row
// i + 1 + gl + 8q) for a following norm recomputation.
__device__ __forceinline__ double grp_reflect(double* c, int m, int i, double tau, const double* vh,
                                              int gl, unsigned gm, double (&x)[GR], bool store) {
  const int rb = i + 1 + gl;
#pragma unroll
  for (int q = 0; q < GR; ++q) x[q] = rb + 8 * q < m ? c[rb + 8 * q] : 0.0;
  const double ci = c[i];
  if (tau == 0.0) return ci;
  double w0 = 0.0, w1 = 0.0;
#pragma unroll
  for (int q = 0; q < GR; q += 2) {
    if (rb + 8 * q < m) w0 = fma(vh[rb + 8 * q], x[q], w0);
    if (rb + 8 * q + 8 < m) w1 = fma(vh[rb + 8 * q + 8], x[q + 1], w1);
  }
  for (int r = rb + 8 * GR; r < m; r += 8) w0 = fma(vh[r], c[r], w0);
  const double w = ci + grp_sum(w0 + w1, gm);
  const double t = -tau * w;
#pragma unroll
  for (int q = 0; q < GR; ++q) {
    const int r = rb + 8 * q;
    if (r < m) {
      x[q] = fma(t, vh[r], x[q]);
      if (store) c[r] = x[q];
    }
  }
  for (int r = rb + 8 * GR; r < m; r += 8)
    if (store) c[r] = fma(t, vh[r], c[r]);
  return ci + t;
}

template <int KER, int D>
__global__ void __launch_bounds__(SVD_THREADS, 2) k_svd(SvdArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Shared S;
  double* taus;
  double* sig;
  int* near_start;
  const double** near_base;
  int64_t* near_stride;
  int* order;
  double* big;
  {
    double* d = reinterpret_cast<double*>(smem_raw);
    S.vn1 = d; d += A.nnmax;
    S.vn2 = d; d += A.nnmax;
    S.vh = d; d += max(A.nmax, A.nnmax);
    S.rdiag = d; d += max(A.nmax, A.nnmax);
    taus = d; d += A.nmax;
    sig = d; d += A.nmax;
    S.nodes = nullptr;
    S.redv = d; d += 32;
    S.misc = d; d += 8;
    near_base = reinterpret_cast<const double**>(d); d += MAX_NEAR;
    near_stride = reinterpret_cast<int64_t*>(d); d += MAX_NEAR;
    int* ip = reinterpret_cast<int*>(d);
    S.redi = ip; ip += 32;
    S.imisc = ip; ip += 8;
    near_start = ip; ip += MAX_NEAR + 1;
    order = ip; ip += A.nmax;
    S.jpvt = ip; ip += A.nnmax;
    big = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(ip) + 15) & ~uintptr_t(15));
  }
  const int tid = threadIdx.x, NT = blockDim.x;
  const int lane = tid & 31;
  // 8-lane groups: one column (or Jacobi pair) per group
  const int g8 = tid >> 3, gl = tid & 7, ngr = NT >> 3;
  const unsigned gm = 0xffu << (lane & ~7);
  double* W = A.gws + (size_t)blockIdx.x * A.gws_stride;
  int dbg_n = 0;
  for (int v = A.lb + blockIdx.x; v < A.le; v += gridDim.x) {
    const int n = A.self.nib[v];
    const int e0 = A.near_ptr[v], e1 = A.near_ptr[v + 1];
    if (tid == 0) {
      int acc = 0, cnt = 0;
      for (int e = e0; e < e1 && cnt < MAX_NEAR; ++e) {
        const int j = A.near_idx[e];
        const int sz = ibar_size(A.other, A.nchild, A.child_first, j);
        if (sz == 0) continue;  // hss.py:283 drops empty neighbour sets
        near_start[cnt] = acc;
        near_base[cnt] = ibar_base(A.other, A.nchild, A.child_first, j, &near_stride[cnt]);
        acc += sz;
        ++cnt;
      }
      near_start[cnt] = acc;
      S.imisc[0] = cnt;
      S.imisc[1] = acc;
      if (e1 - e0 > MAX_NEAR) atomicOr(A.err, DEV_CAPACITY);
    }
    __syncthreads();
    const int nnear = S.imisc[0], nn = S.imisc[1];
    if (n == 0 || nn == 0) {
      if (tid == 0) A.keep[v] = 0;
      __syncthreads();
      continue;
    }
    const bool dbg = A.dbg && blockIdx.x < 4 && tid == 0 && dbg_n == 0;  // first node of blocks 0-3
    long long tsv[6];
    if (dbg) tsv[0] = clock64();
    // ---- assemble A (n x nn), column-major in W (one column per nearfield point)
    int64_t ts;
    const double* tb = ibar_base(A.self, A.nchild, A.child_first, v, &ts);
    const int ldp = n;
    {
      int g = 0;
      for (int b = tid / n, a = tid % n; b < nn;) {
        while (g + 1 < nnear && near_start[g + 1] <= b) ++g;
        const int bl = b - near_start[g];
        double x[D], y[D];
#pragma unroll
        for (int d = 0; d < D; ++d) {
          x[d] = tb[(int64_t)d * ts + a];
          y[d] = near_base[g][(int64_t)d * near_stride[g] + bl];
        }
        W[(size_t)b * ldp + a] = A.transpose ? kval<KER, D>(y, x, A.dx) : kval<KER, D>(x, y, A.dx);
        a += NT;
        while (a >= n) { a -= n; ++b; }
      }
    }
    __syncthreads();
    if (dbg) tsv[1] = clock64();
    // ---- column-pivoted QR of A, truncated at the noise floor
    double* P = W;
    const int kmax = min(n, nn);
    for (int j = g8; j < nn; j += ngr) {
      const double nr = __dsqrt_rn(grp_sumsq(P + (size_t)j * ldp, 0, n, gl, gm));
      if (gl == 0) {
        S.vn1[j] = nr;
        S.vn2[j] = nr;
      }
    }
    __syncthreads();
    const double floor_v = A.nchild[v] ? A.floor_rel : A.floor_leaf;
    int kp = 0;
    for (int i = 0; i < kmax; ++i) {
      double bv = -1.0;
      int bi = 0x7fffffff;
      for (int j = i + tid; j < nn; j += NT)
        if (S.vn1[j] > bv) { bv = S.vn1[j]; bi = j; }
      const int pvt = block_argmax_1bar(bv, bi, S);
      if (pvt != i) {
        double* ci = P + (size_t)i * ldp;
        double* cp = P + (size_t)pvt * ldp;
        for (int row = tid; row < n; row += NT) {
          const double t = cp[row];
          cp[row] = ci[row];
          ci[row] = t;
        }
        if (tid == 0) {
          S.vn1[pvt] = S.vn1[i];
          S.vn2[pvt] = S.vn2[i];
        }
      }
      __syncthreads();
      householder(P + (size_t)i * ldp - i, 1, n, i, S);  // column i (stride 1)
      __syncthreads();
      const double tau = S.misc[0];
      if (tid == 0) taus[i] = tau;
      const double r0 = fabs(S.rdiag[0]);
      if (r0 == 0.0 || !(fabs(S.rdiag[i]) > floor_v * r0)) break;
      kp = i + 1;
      for (int j = i + 1 + g8; j < nn; j += ngr) {
        double* c = P + (size_t)j * ldp;
        double x[GR];
        const double rij = grp_reflect(c, n, i, tau, S.vh, gl, gm, x, true);
        if (gl == 0 && tau != 0.0) c[i] = rij;
        // norm downdate (dlaqp2), exact recomputation when cancellation is severe
        const double v1 = S.vn1[j];
        if (v1 != 0.0) {
          const double q = fabs(rij) / v1;
          const double temp = fmax(1.0 - q * q, 0.0);
          const double q2 = v1 / S.vn2[j];
          if (temp * (q2 * q2) <= TOL3Z) {
            double s0 = 0.0;
#pragma unroll
            for (int qq = 0; qq < GR; ++qq) s0 = fma(x[qq], x[qq], s0);
            for (int r = i + 1 + gl + 8 * GR; r < n; r += 8) s0 = fma(c[r], c[r], s0);
            const double nv = i + 1 < n ? sqrt(grp_sum(s0, gm)) : 0.0;
            if (gl == 0) {
              S.vn1[j] = nv;
              S.vn2[j] = nv;
            }
          } else if (gl == 0) {
            S.vn1[j] = v1 * sqrt(temp);
          }
        }
      }
      __syncthreads();
    }
    __syncthreads();
    if (kp == 0) {
      if (tid == 0) A.keep[v] = 0;
      __syncthreads();
      continue;
    }
    if (dbg) tsv[2] = clock64();
    // ---- B = R_k^T (nn x kp, column-major), unpivoted QR -> R2 (kp x kp); B in
    // shared memory when it fits
    const bool bsm = (int64_t)nn * kp <= SVD_BIG;
    double* B = bsm ? big : W + (size_t)n * nn;
    double* T = W + (size_t)n * nn;  // global staging (free once B is in shared memory / consumed)
    const int ldb = nn;
    for (int e = tid; e < nn * kp; e += NT) {
      const int j = e / nn, b = e - j * nn;
      B[(size_t)j * ldb + b] = b >= j ? P[(size_t)b * ldp + j] : 0.0;
    }
    __syncthreads();
    for (int i = 0; i < kp; ++i) {
      householder(B + (size_t)i * ldb - i, 1, nn, i, S);
      __syncthreads();
      const double tau = S.misc[0];
      if (tau != 0.0)
        for (int j = i + 1 + g8; j < kp; j += ngr) {
          double* c = B + (size_t)j * ldb;
          double x[GR];
          const double rij = grp_reflect(c, nn, i, tau, S.vh, gl, gm, x, true);
          if (gl == 0) c[i] = rij;
        }
      __syncthreads();
    }
    // ---- one-sided Jacobi on R2's columns (column-major J: J[c*kp + r]), V accumulated;
    // J and V in shared memory when they fit (R2 staged through global scratch when
    // B occupies that area).  Column norms are kept up to date through the rotation
    // (one dot product per pair) and refreshed exactly at every sweep.
    const bool jsm = 2 * kp * kp <= SVD_BIG;
    double* J = jsm ? big : W + (size_t)n * nn + (size_t)nn * kp;
    double* V = J + (size_t)kp * kp;
    double* nrm = sig;  // squared column norms (reuses the sigma scratch)
    if (bsm && jsm) {
      for (int e = tid; e < kp * kp; e += NT) {
        const int c = e / kp, r = e - c * kp;
        T[e] = r <= c ? B[(size_t)c * ldb + r] : 0.0;
      }
      __syncthreads();
      for (int e = tid; e < kp * kp; e += NT) J[e] = T[e];
    } else {
      for (int e = tid; e < kp * kp; e += NT) {
        const int c = e / kp, r = e - c * kp;
        J[e] = r <= c ? B[(size_t)c * ldb + r] : 0.0;
      }
    }
    for (int e = tid; e < kp * kp; e += NT) V[e] = (e % (kp + 1)) == 0 ? 1.0 : 0.0;
    __syncthreads();
    const int np = kp + (kp & 1);  // round-robin over an even count (dummy = kp)
    if (dbg) tsv[3] = clock64();
    int sweeps_done = 0;
    for (int sweep = 0; sweep < 40; ++sweep) {
      sweeps_done = sweep + 1;
      for (int c = g8; c < kp; c += ngr) {  // exact squared norms
        double s2 = 0.0;
        for (int r = gl; r < kp; r += 8) s2 = fma(J[(size_t)c * kp + r], J[(size_t)c * kp + r], s2);
        s2 = grp_sum(s2, gm);
        if (gl == 0) nrm[c] = s2;
      }
      if (tid == 0) S.imisc[2] = 0;
      __syncthreads();
      for (int rnd = 0; rnd < np - 1; ++rnd) {
        for (int pr = g8; pr < np / 2; pr += ngr) {
          // circle method: position 0 fixed, others rotate
          int a = pr == 0 ? 0 : 1 + (pr - 1 + rnd) % (np - 1);
          int b = 1 + (np - 2 - pr + rnd) % (np - 1);
          if (a >= kp || b >= kp) continue;
          double* ja = J + (size_t)a * kp;
          double* jb = J + (size_t)b * kp;
          double ga = 0;
          long long jt0 = 0, jt1 = 0, jt2 = 0;
          if (dbg) jt0 = clock64();
          for (int r = gl; r < kp; r += 8) ga = fma(ja[r], jb[r], ga);
          ga = grp_sum(ga, gm);
          if (dbg) jt1 = clock64();
          const double al = nrm[a], be = nrm[b];
          if (ga * ga > 1e-30 * (al * be) && ga != 0.0) {
            const double zeta = (be - al) / (2.0 * ga);
            const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double c = rsqrt(1.0 + t * t), s = c * t;
            if (dbg) jt2 = clock64();
            double* va = V + (size_t)a * kp;
            double* vb = V + (size_t)b * kp;
            for (int r = gl; r < kp; r += 8) {
              const double x = ja[r], y = jb[r];
              ja[r] = c * x - s * y;
              jb[r] = s * x + c * y;
              const double p = va[r], q = vb[r];
              va[r] = c * p - s * q;
              vb[r] = s * p + c * q;
            }
            __syncwarp(gm);
            if (gl == 0) {
              nrm[a] = fmax(al - t * ga, 0.0);
              nrm[b] = be + t * ga;
              S.imisc[2] = 1;
            }
            if (dbg && tid == 0) {
              const long long jt3 = clock64();
              A.dbg[34] += jt1 - jt0; A.dbg[35] += jt2 - jt1; A.dbg[36] += jt3 - jt2; A.dbg[38] += 1;
            }
          }
        }
        long long jb0 = 0;
        if (dbg && tid == 0) jb0 = clock64();
        __syncthreads();
        if (dbg && tid == 0) { A.dbg[37] += clock64() - jb0; A.dbg[39] += 1; }
      }
      if (S.imisc[2] == 0) break;
      __syncthreads();
    }
    if (dbg) tsv[4] = clock64();
    if (A.dbg && tid == 0) {  // every node: max sweeps, nodes at the sweep cap
      atomicMax(reinterpret_cast<unsigned long long*>(A.dbg + 32), (unsigned long long)sweeps_done);
      if (sweeps_done >= 40) atomicAdd(reinterpret_cast<unsigned long long*>(A.dbg + 33), 1ull);
    }
    // ---- singular values, keep count, descending order
    for (int c = g8; c < kp; c += ngr) {
      double s2 = 0.0;
      for (int r = gl; r < kp; r += 8) s2 = fma(J[(size_t)c * kp + r], J[(size_t)c * kp + r], s2);
      s2 = grp_sum(s2, gm);
      if (gl == 0) sig[c] = sqrt(s2);
    }
    __syncthreads();
    if (tid == 0) {
      double smax = 0.0;
      for (int c = 0; c < kp; ++c) smax = fmax(smax, sig[c]);
      int keep = 0;
      if (smax > 0.0) {
        // selection of sigma >= eps * sigma_1 in descending order
        for (int c = 0; c < kp; ++c) order[c] = c;
        for (int c = 1; c < kp; ++c) {  // insertion sort by sigma descending (kp small)
          int x = order[c];
          int p = c - 1;
          while (p >= 0 && sig[order[p]] < sig[x]) { order[p + 1] = order[p]; --p; }
          order[p + 1] = x;
        }
        const double thr = A.eps_svd * smax;
        for (int c = 0; c < kp; ++c) keep += sig[c] >= thr ? 1 : 0;
      }
      S.imisc[3] = keep;
      A.keep[v] = keep;
    }
    __syncthreads();
    const int keep = S.imisc[3];
    if (keep == 0) continue;
    // ---- U = Q1[:, :kp] V[:, kept]  (n x keep): Y staged in shared memory (over
    // the J/V area, through registers) when it fits, reflectors applied by
    // 8-lane groups per column
    double* Yg = A.sv + A.sv_off[v];
    const bool ysm = n * (keep | 1) <= SVD_BIG;
    double* Y = ysm ? big : Yg;
    const int ldy = ysm ? (keep | 1) : keep;
    {
      // kept columns of V (descending sigma) -> T (global staging: Y may overlap V)
      for (int e = tid; e < kp * keep; e += NT) {
        const int a = e / keep, c = e - a * keep;
        T[e] = V[(size_t)order[c] * kp + a];
      }
      __syncthreads();
      for (int e = tid; e < n * ldy; e += NT) {
        const int a = e / ldy, c = e - a * ldy;
        Y[e] = (a < kp && c < keep) ? T[a * keep + c] : 0.0;
      }
    }
    __syncthreads();
    for (int i = kp - 1; i >= 0; --i) {
      const double tau = taus[i];
      if (tau == 0.0) continue;
      for (int row = i + 1 + tid; row < n; row += NT) S.vh[row] = P[(size_t)i * ldp + row];
      __syncthreads();
      for (int c = g8; c < keep; c += ngr) {
        double w = 0.0;
        for (int row = i + gl; row < n; row += 8)
          w = fma(row == i ? 1.0 : S.vh[row], Y[(size_t)row * ldy + c], w);
        w = grp_sum(w, gm);
        const double t = -tau * w;
        for (int row = i + gl; row < n; row += 8)
          Y[(size_t)row * ldy + c] = fma(t, row == i ? 1.0 : S.vh[row], Y[(size_t)row * ldy + c]);
      }
      __syncthreads();
    }
    if (ysm) {
      for (int e = tid; e < n * keep; e += NT) Yg[e] = Y[(e / keep) * ldy + e % keep];
      __syncthreads();
    }
    if (dbg) {
      tsv[5] = clock64();
      long long* o = A.dbg + blockIdx.x * 8;
      for (int q = 0; q < 5; ++q) o[q] = tsv[q + 1] - tsv[q];
      o[5] = kp; o[6] = keep + 1000 * sweeps_done; o[7] = n * 1000 + nn;
    }
    ++dbg_n;
  }
}

template <typename F>
void cub_call(F f, DBuf<char>& tmp, cudaStream_t s) {
  size_t bytes = 0;
  SMASH_CUDA(f((void*)nullptr, bytes));
  if (bytes > tmp.n) tmp.alloc(bytes, s);
  SMASH_CUDA(f((void*)tmp.p, bytes));
}

__global__ void k_sv_cap(int lb, int le, const int* nib, const int* nn, int64_t* cap) {
  int v = lb + blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= le) return;
  int a = nib[v], b = nn[v - lb];
  cap[v - lb] = (int64_t)a * min(a, b);
}

__global__ void k_sv_off(int lb, int le, const int64_t* loc, int64_t* off) {
  int v = lb + blockIdx.x * blockDim.x + threadIdx.x;
  if (v < le) off[v] = loc[v - lb];
}

__global__ void k_max_keep(int lb, int le, const int* keep, int* out) {
  int m = 0;
  for (int v = lb + blockIdx.x * blockDim.x + threadIdx.x; v < le; v += gridDim.x * blockDim.x)
    m = max(m, keep[v]);
  for (int off = 16; off; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

IbarSide ibar_side(MatrixImpl* M, int side) {
  TreeImpl* t = M->tree;
  SideFactors& F = side == 0 ? M->rowf : *M->colf;
  const bool col = side == 1 && !t->shared;
  IbarSide s;
  s.nib = F.nib.p;
  s.rank = F.rank.p;
  s.pt_a = col ? t->col_a.p : t->row_a.p;
  s.pt_b = col ? t->col_b.p : t->row_b.p;
  s.P = col ? t->pts_col.p : t->pts_row.p;
  s.P_stride = col ? t->ny : t->nx;
  s.Sk = F.skel_pts.p;
  s.S_stride = F.skel_stride;
  s.skel_off = F.skel_off.p;
  return s;
}

}  // namespace

int hss_level_svd(MatrixImpl* M, int side, int level, NearSets* near, int nmax, SvdWorkspace& ws,
                  cudaStream_t s, int sub_lb, int sub_le) {
  TreeImpl* t = M->tree;
  const int n_nodes = t->n_nodes;
  const int lb = t->level_begin(level), le = t->level_end(level), cnt = le - lb;
  // sharded build: the SVDs of this rank's node range only (capacities stay level-wide)
  const int run_lb = sub_lb >= 0 ? sub_lb : lb, run_le = sub_lb >= 0 ? sub_le : le;
  if (ws.keep.n < (size_t)n_nodes) {
    ws.keep.alloc(n_nodes, s);
    ws.keep.zero(s);
    ws.sv_off.alloc(n_nodes, s);
    ws.sv_off.zero(s);
  }
  SvdArgs A{};
  A.lb = lb; A.le = le; A.dim = t->dim; A.kernel = M->p.kernel;
  A.dx = M->p.kernel == SMASH_KERNEL_EXP ? 1.0 : M->p.dx;
  A.eps_svd = M->p.eps_svd;
  static const int floor_exp = getenv("SMASH_SVD_FLOOR") ? atoi(getenv("SMASH_SVD_FLOOR")) : 60;
  static const int floor_leaf = getenv("SMASH_SVD_FLOOR_LEAF") ? atoi(getenv("SMASH_SVD_FLOOR_LEAF")) : 56;
  A.floor_rel = ldexp(1.0, -floor_exp);
  A.floor_leaf = ldexp(1.0, -floor_leaf);
  A.transpose = side;
  A.nchild = t->nchild.p; A.child_first = t->child_first.p;
  A.near_ptr = near->ptr.p; A.near_idx = near->idx.p;
  A.self = ibar_side(M, side);
  A.other = ibar_side(M, 1 - side);
  A.keep = ws.keep.p;
  DBuf<int> nn;
  nn.alloc(cnt, s);
  A.nn_out = nn.p;
  k_near_cols<<<cdiv(cnt, 128), 128, 0, s>>>(A);
  // S capacity: |ibar| x min(|ibar|, n_near) per node
  DBuf<int64_t> cap, off;
  cap.alloc(cnt + 1, s); off.alloc(cnt + 1, s);
  SMASH_CUDA(cudaMemsetAsync(cap.p + cnt, 0, 8, s));
  k_sv_cap<<<cdiv(cnt, 128), 128, 0, s>>>(lb, le, A.self.nib, nn.p, cap.p);
  DBuf<char> tmp;
  cub_call([&](void* tp, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(tp, b, cap.p, off.p, cnt + 1, s);
  }, tmp, s);
  DBuf<int> dmax;
  dmax.alloc(1, s);
  dmax.zero(s);
  int64_t total = 0;
  d2h(&total, off.p + cnt, 1, s);
  std::vector<int> hnn(cnt);
  d2h(hnn.data(), nn.p, cnt, s);
  sync(s);
  int nnmax = 1;
  for (int x : hnn) nnmax = std::max(nnmax, x);
  ws.sv.alloc(std::max<int64_t>(total, 1), s);
  k_sv_off<<<cdiv(cnt, 128), 128, 0, s>>>(lb, le, off.p, ws.sv_off.p);
  A.sv_off = ws.sv_off.p;
  A.sv = ws.sv.p;
  A.nmax = std::max(nmax, 1);
  A.nnmax = nnmax;
  const int kpmax = std::min(A.nmax, A.nnmax);
  A.gws_stride = (int64_t)A.nmax * A.nnmax + (int64_t)A.nnmax * kpmax + 2 * (int64_t)kpmax * kpmax;
  int dev = 0, nsm = 0;
  SMASH_CUDA(cudaGetDevice(&dev));
  SMASH_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  static const int svd_per_sm = getenv("SMASH_SVD_PER_SM") ? atoi(getenv("SMASH_SVD_PER_SM")) : 2;
  const int grid = std::min(cnt, nsm * svd_per_sm);
  DBuf<double> gws;
  gws.alloc((size_t)grid * A.gws_stride, s);
  A.gws = gws.p;
  DBuf<int> err;
  err.alloc(1, s);
  err.zero(s);
  A.err = err.p;
  static const bool svd_dbg = getenv("SMASH_SVD_DBG") != nullptr;
  DBuf<long long> dbgbuf;
  A.dbg = nullptr;
  if (svd_dbg) {
    dbgbuf.alloc(40, s);
    dbgbuf.zero(s);
    A.dbg = dbgbuf.p;
  }
  const int mx = std::max(A.nmax, A.nnmax);
  size_t smem = 8 * ((size_t)2 * A.nnmax + 2 * mx + 2 * A.nmax + 32 + 8 + 2 * MAX_NEAR) +
                4 * ((size_t)32 + 8 + MAX_NEAR + 1 + A.nmax + A.nnmax) + 64 + 16 +
                8 * (size_t)SVD_BIG;
  SMASH_CHECK(smem <= 200 * 1024, SMASH_ERR_INVALID, "HSS nearfield block too large");
  dispatch_kernel_dim(A.kernel, A.dim, [&]<int KER, int D>() {
    SMASH_CUDA(cudaFuncSetAttribute(k_svd<KER, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
    SvdArgs Ar = A;
    Ar.lb = run_lb;
    Ar.le = run_le;
    if (run_le > run_lb) k_svd<KER, D><<<std::min(grid, run_le - run_lb), SVD_THREADS, smem, s>>>(Ar);
  });
  SMASH_CUDA(cudaGetLastError());
  if (run_le > run_lb)
    k_max_keep<<<std::min<unsigned>(cdiv(run_le - run_lb, 256), 64), 256, 0, s>>>(run_lb, run_le, ws.keep.p,
                                                                                dmax.p);
  int hk = 0, he = 0;
  d2h(&hk, dmax.p, 1, s);
  d2h(&he, err.p, 1, s);
  sync(s);
  SMASH_CHECK(he == 0, SMASH_ERR_INVALID, "nearfield set larger than the supported cap");
  if (svd_dbg) {
    long long h[40];
    d2h(h, dbgbuf.p, 40, s);
    sync(s);
    fprintf(stderr, "svd level %d side %d cnt %d:", level, side, cnt);
    for (int q = 0; q < 4; ++q)
      fprintf(stderr, " [asm %lld qr %lld qr2 %lld jac %lld back %lld kp %lld keep %lld n.nn %lld]", h[q * 8], h[q * 8 + 1],
              h[q * 8 + 2], h[q * 8 + 3], h[q * 8 + 4], h[q * 8 + 5], h[q * 8 + 6], h[q * 8 + 7]);
    fprintf(stderr, " max_sweeps %lld capped %lld | jacobi (thread 0 of traced nodes): dot %.0f scalar %.0f rotate %.0f per rotation (%lld), barrier wait %.0f per round (%lld)\n", h[32], h[33],
            h[38] ? (double)h[34] / h[38] : 0.0, h[38] ? (double)h[35] / h[38] : 0.0, h[38] ? (double)h[36] / h[38] : 0.0, h[38],
            h[39] ? (double)h[37] / h[39] : 0.0, h[39]);
  }
  return hk;
}

}  // namespace smash
