// HSS ULV factorisation and solve on the GPU (replaces
// smash/apply.py:168-354, _reduce_node / ulv_factor / ulv_solve).
//
// The reference walks the nodes in postorder; every node only needs its
// children, so here one level of the tree is one batch: one CTA per node,
// levels bottom-up for the factorisation and the upward solve, top-down for
// the downward solve.  A host-side plan (sizes from the tree and the factor
// ranks) gives every node fixed slots in a handful of flat HBM buffers:
//
//   D   (m_r x m_c)  the node's diagonal block; after the reduction it holds
//                    Dtrans = (Q^T D)[:m_r-t] Qz (Dcorr | D_red) on top and the
//                    LQ factor L plus the Qz reflectors in its last t rows
//   U   (m_r x k_r)  the row basis; after the reduction R (upper) + Q reflectors
//   VT  (k_c x m_c)  V^T; after the reduction Mfull = V^T Qz (Mcorr | V_red^T)
//   CP  (m_red x k_c(sibling))  U_red B_(c,sibling), kept for the solve
//
// Row-basis QR = Householder on the columns of U (dlarfg convention), applied
// to D from the left; the elimination of the t local equations is the LQ of
// the bottom t rows of Q^T D (= QR of Bbot^T in the reference), applied to the
// other rows of D and to V^T from the right.  Matrices are row-major; every
// reflector application is one warp per vector with a shuffle-reduced dot.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "smash_impl.cuh"

namespace smash {

namespace {

constexpr int ULV_THREADS = 256;
constexpr int ULV_PF = 8;  // reflector entries per lane held in registers (rows up to 256)
constexpr double PIVOT_RTOL = 1e-13;  // apply.py:18

struct UlvNode {
  int mr, mc, kr, kc, t;
  int leaf;
  int c1, c2;        // BFS children (HSS: binary), -1 for leaves
  int parent, pos;   // BFS parent; row offset of this node's reduced columns in the parent's x
  int64_t oD, oU, oVT, otU, otZ, oCP;
  int64_t ob, ox, og;  // solve workspaces (units of nrhs)
  int row_a, col_a;    // leaf point ranges (tree order)
  int post;
};

__device__ __forceinline__ double warp_sum(double x) {
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// dlarfg on x[0], x[s], ..., x[(n-1)s] by one warp: x[0] <- beta, x[1:] <- v[1:],
// returns tau (0 when nothing to annihilate).
__device__ double warp_larfg(double* x, int64_t s, int n) {
  const int lane = threadIdx.x & 31;
  double ss = 0.0;
  for (int i = 1 + lane; i < n; i += 32) {
    double v = x[i * s];
    ss = fma(v, v, ss);
  }
  ss = warp_sum(ss);
  const double alpha = x[0];
  if (n <= 1 || ss == 0.0) return 0.0;
  const double xnorm = sqrt(ss);
  const double beta = -copysign(hypot(alpha, xnorm), alpha);
  const double tau = (beta - alpha) / beta;
  const double scal = 1.0 / (alpha - beta);
  for (int i = 1 + lane; i < n; i += 32) x[i * s] *= scal;
  __syncwarp();
  if (lane == 0) x[0] = beta;
  __syncwarp();
  return tau;
}

// y <- (I - tau v v^T) y with v[0] = 1, v[1:] = vs[1:] (vs in shared memory),
// y[i] at y[i * sy], n entries; one warp.
__device__ __forceinline__ void warp_apply(const double* vs, int n, double tau, double* y,
                                           int64_t sy) {
  const int lane = threadIdx.x & 31;
  double w = 0.0;
  for (int i = lane; i < n; i += 32) w = fma(i == 0 ? 1.0 : vs[i], y[i * sy], w);
  w = warp_sum(w) * tau;
  for (int i = lane; i < n; i += 32) y[i * sy] -= w * (i == 0 ? 1.0 : vs[i]);
  __syncwarp();
}

// expand() entry (lowrank.py:222-229): row q of P[I; G] for a node with local
// inverse permutation inv (ibar position -> perm position), rank k.
__device__ __forceinline__ double expand_at(const int* inv, const double* G, int k, int q, int c) {
  const int j = inv[q];
  return j < k ? (j == c ? 1.0 : 0.0) : G[(int64_t)(j - k) * k + c];
}

struct FacView {
  const int* perm;
  const double* G;
  const int* skel;
  const int64_t* ib_off;
  const int64_t* g_off;
  const int* skel_off;
  const int* nib;
};

__device__ void load_inv(const FacView& F, int v, int* inv) {
  const int n = F.nib[v];
  const int* p = F.perm + F.ib_off[v];
  for (int j = threadIdx.x; j < n; j += blockDim.x) inv[p[j]] = j;
}

struct UlvArgs {
  const UlvNode* nd;
  int lb, le, root;
  double* D;
  double* U;
  double* VT;
  double* tauU;
  double* tauZ;
  double* CP;
  FacView R, C;
  const double* prow;  // tree-ordered SoA points (rows / cols)
  const double* pcol;
  int64_t nrow, ncol;
  double dx;
  int* err;  // [0] = flag, [1] = postorder node id
  int vs_cap;         // reflector buffer (doubles) at the start of k_ulv_reduce's shared memory
  int64_t stage_cap;  // nodes with |D| + |U| + |V^T| <= stage_cap are reduced in shared memory
};

__device__ __forceinline__ void flag_singular(const UlvArgs& A, int post) {
  if (atomicCAS(A.err, 0, 1) == 0) A.err[1] = post;
}

// ---- assembly ------------------------------------------------------------------------
template <int KER, int DIM>
__global__ void __launch_bounds__(ULV_THREADS) k_ulv_assemble(UlvArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int v = A.lb + blockIdx.x;
  if (v >= A.le) return;
  const UlvNode& N = A.nd[v];
  const int tid = threadIdx.x, NT = blockDim.x;
  double* D = A.D + N.oD;
  if (N.leaf) {
    int* invr = reinterpret_cast<int*>(smem);
    int* invc = invr + N.mr;
    if (v != A.root) {
      load_inv(A.R, v, invr);
      load_inv(A.C, v, invc);
    }
    for (int e = tid; e < N.mr * N.mc; e += NT) {
      const int r = e / N.mc, c = e % N.mc;
      double x[DIM], y[DIM];
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        x[a] = A.prow[(int64_t)a * A.nrow + N.row_a + r];
        y[a] = A.pcol[(int64_t)a * A.ncol + N.col_a + c];
      }
      D[e] = kval<KER, DIM>(x, y, A.dx);
    }
    if (v == A.root) return;
    __syncthreads();
    const double* Gr = A.R.G + A.R.g_off[v];
    const double* Gc = A.C.G + A.C.g_off[v];
    for (int e = tid; e < N.mr * N.kr; e += NT)
      A.U[N.oU + e] = expand_at(invr, Gr, N.kr, e / N.kr, e % N.kr);
    for (int e = tid; e < N.kc * N.mc; e += NT) {
      const int a = e / N.mc, c = e % N.mc;
      A.VT[N.oVT + e] = expand_at(invc, Gc, N.kc, c, a);
    }
    return;
  }
  // internal node: children's reduced blocks (apply.py:246-266)
  const UlvNode& N1 = A.nd[N.c1];
  const UlvNode& N2 = A.nd[N.c2];
  const int m1 = N1.mr - N1.t, n1 = N1.mc - N1.t, m2 = N2.mr - N2.t, n2 = N2.mc - N2.t;
  double* B12 = reinterpret_cast<double*>(smem);  // kr1 x kc2
  double* B21 = B12 + N1.kr * N2.kc;              // kr2 x kc1
  int* invr = reinterpret_cast<int*>(B21 + N2.kr * N1.kc);
  int* invc = invr + N1.kr + N2.kr;
  // coupling blocks at the skeletons (hss.py:106-150)
  auto skel_pt = [&](const FacView& F, const double* P, int64_t stride, int node, int a, double* x) {
    const int lab = F.skel[F.skel_off[node] + a];
#pragma unroll
    for (int d = 0; d < DIM; ++d) x[d] = P[(int64_t)d * stride + lab];
  };
  for (int e = tid; e < N1.kr * N2.kc; e += NT) {
    double x[DIM], y[DIM];
    skel_pt(A.R, A.prow, A.nrow, N.c1, e / N2.kc, x);
    skel_pt(A.C, A.pcol, A.ncol, N.c2, e % N2.kc, y);
    B12[e] = kval<KER, DIM>(x, y, A.dx);
  }
  for (int e = tid; e < N2.kr * N1.kc; e += NT) {
    double x[DIM], y[DIM];
    skel_pt(A.R, A.prow, A.nrow, N.c2, e / N1.kc, x);
    skel_pt(A.C, A.pcol, A.ncol, N.c1, e % N1.kc, y);
    B21[e] = kval<KER, DIM>(x, y, A.dx);
  }
  if (v != A.root) {
    load_inv(A.R, v, invr);
    load_inv(A.C, v, invc);
  }
  __syncthreads();
  // U_red of a child: [R; 0] after a reduction, U itself when nothing was eliminated
  auto ured = [&](const UlvNode& C, int r, int a) -> double {
    const double u = A.U[C.oU + (int64_t)r * C.kr + a];
    return C.t > 0 ? (r <= a ? u : 0.0) : u;
  };
  // CP = U_red B (kept for the solve), stored with the child
  double* CP1 = A.CP + N1.oCP;
  double* CP2 = A.CP + N2.oCP;
  for (int e = tid; e < m1 * N2.kc; e += NT) {
    const int r = e / N2.kc, b = e % N2.kc;
    double s = 0.0;
    for (int a = 0; a < N1.kr; ++a) s = fma(ured(N1, r, a), B12[a * N2.kc + b], s);
    CP1[e] = s;
  }
  for (int e = tid; e < m2 * N1.kc; e += NT) {
    const int r = e / N1.kc, b = e % N1.kc;
    double s = 0.0;
    for (int a = 0; a < N2.kr; ++a) s = fma(ured(N2, r, a), B21[a * N1.kc + b], s);
    CP2[e] = s;
  }
  __syncthreads();
  const double* D1 = A.D + N1.oD;
  const double* D2 = A.D + N2.oD;
  const double* V1 = A.VT + N1.oVT;  // V_red^T = VT[:, t:]
  const double* V2 = A.VT + N2.oVT;
  for (int e = tid; e < N.mr * N.mc; e += NT) {
    const int r = e / N.mc, c = e % N.mc;
    double val;
    if (r < m1 && c < n1) {
      val = D1[(int64_t)r * N1.mc + N1.t + c];
    } else if (r >= m1 && c >= n1) {
      val = D2[(int64_t)(r - m1) * N2.mc + N2.t + (c - n1)];
    } else if (r < m1) {  // CP1 V2_red^T
      double s = 0.0;
      for (int b = 0; b < N2.kc; ++b)
        s = fma(CP1[(int64_t)r * N2.kc + b], V2[(int64_t)b * N2.mc + N2.t + (c - n1)], s);
      val = s;
    } else {
      double s = 0.0;
      for (int b = 0; b < N1.kc; ++b)
        s = fma(CP2[(int64_t)(r - m1) * N1.kc + b], V1[(int64_t)b * N1.mc + N1.t + c], s);
      val = s;
    }
    D[e] = val;
  }
  if (v == A.root) return;
  // U = [U1_red R_c1; U2_red R_c2], V^T = [W_c1^T V1_red^T, W_c2^T V2_red^T]
  const double* Gr = A.R.G + A.R.g_off[v];
  const double* Gc = A.C.G + A.C.g_off[v];
  for (int e = tid; e < N.mr * N.kr; e += NT) {
    const int r = e / N.kr, c = e % N.kr;
    double s = 0.0;
    if (r < m1)
      for (int a = 0; a < N1.kr; ++a) s = fma(ured(N1, r, a), expand_at(invr, Gr, N.kr, a, c), s);
    else
      for (int a = 0; a < N2.kr; ++a)
        s = fma(ured(N2, r - m1, a), expand_at(invr, Gr, N.kr, N1.kr + a, c), s);
    A.U[N.oU + e] = s;
  }
  for (int e = tid; e < N.kc * N.mc; e += NT) {
    const int a = e / N.mc, c = e % N.mc;
    double s = 0.0;
    if (c < n1)
      for (int b = 0; b < N1.kc; ++b)
        s = fma(expand_at(invc, Gc, N.kc, b, a), V1[(int64_t)b * N1.mc + N1.t + c], s);
    else
      for (int b = 0; b < N2.kc; ++b)
        s = fma(expand_at(invc, Gc, N.kc, N1.kc + b, a), V2[(int64_t)b * N2.mc + N2.t + (c - n1)], s);
    A.VT[N.oVT + e] = s;
  }
}

// ---- reduction (_reduce_node, apply.py:196-234) -------------------------------------------
// Apply reflectors 0..nref-1, in order, to one vector y (n <= 32*ULV_PF entries,
// y[j] at y[j*sy]) held by one warp in registers: reflector i is
// v_i[j] = 1 (j == i), vat(i, j) (j > i), 0 (j < i), with tau taus[i]; the next
// reflector is prefetched while the current one is applied.
template <int PF, class VF>
__device__ __forceinline__ void warp_apply_all(double* y, int64_t sy, int n, int nref,
                                               const double* taus, VF vat) {
  const int lane = threadIdx.x & 31;
  double yr[PF], cur[PF], nxt[PF];
#pragma unroll
  for (int k = 0; k < PF; ++k) {
    const int j = lane + 32 * k;
    yr[k] = j < n ? y[j * sy] : 0.0;
  }
  auto load = [&](int i, double* dst) {
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      const int j = lane + 32 * k;
      dst[k] = j < n ? (j > i ? vat(i, j) : (j == i ? 1.0 : 0.0)) : 0.0;
    }
  };
  load(0, cur);
  double tau = taus[0];
  for (int i = 0; i < nref; ++i) {
    double tau_n = 0.0;
    if (i + 1 < nref) {
      load(i + 1, nxt);
      tau_n = taus[i + 1];
    }
    double w = 0.0;
#pragma unroll
    for (int k = 0; k < PF; ++k) w = fma(cur[k], yr[k], w);
    w = warp_sum(w) * tau;
#pragma unroll
    for (int k = 0; k < PF; ++k) yr[k] = fma(-w, cur[k], yr[k]);
#pragma unroll
    for (int k = 0; k < PF; ++k) cur[k] = nxt[k];
    tau = tau_n;
  }
#pragma unroll
  for (int k = 0; k < PF; ++k) {
    const int j = lane + 32 * k;
    if (j < n) y[j * sy] = yr[k];
  }
}

__global__ void __launch_bounds__(ULV_THREADS) k_ulv_reduce(UlvArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* vs = reinterpret_cast<double*>(smem);
  __shared__ double s_tau, s_norm;
  const int v = A.lb + blockIdx.x;
  if (v >= A.le || v == A.root) return;
  const UlvNode& N = A.nd[v];
  if (N.t == 0) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, NW = blockDim.x >> 5;
  const int mr = N.mr, mc = N.mc, kr = N.kr, kc = N.kc, t = N.t;
  // Stage D, U and V^T in shared memory when they fit (all reflector traffic then
  // stays on chip; the row-major layouts and leading dimensions are unchanged).
  const int64_t nD = (int64_t)mr * mc, nU = (int64_t)mr * kr, nV = (int64_t)kc * mc;
  const bool stage = nD + nU + nV <= A.stage_cap;
  double* Dg = A.D + N.oD;
  double* Ug = A.U + N.oU;
  double* Vg = A.VT + N.oVT;
  double* sb = vs + A.vs_cap;
  double* D = stage ? sb : Dg;
  double* U = stage ? sb + nD : Ug;
  double* VT = stage ? sb + nD + nU : Vg;
  if (stage) {
    for (int64_t e = tid; e < nD; e += blockDim.x) D[e] = Dg[e];
    for (int64_t e = tid; e < nU; e += blockDim.x) U[e] = Ug[e];
    for (int64_t e = tid; e < nV; e += blockDim.x) VT[e] = Vg[e];
    __syncthreads();
  }
  // register-resident application of whole reflector sequences (rows / columns up
  // to 32*ULV_PF entries); otherwise every reflector is applied as it is formed
  const bool fast = mr <= 32 * ULV_PF && mc <= 32 * ULV_PF;
  // 1. Householder QR of U, applied to D from the left (Q^T D)
  for (int i = 0; i < kr; ++i) {
    if (wid == 0) {
      double tau = warp_larfg(U + (int64_t)i * kr + i, kr, mr - i);
      if (lane == 0) { s_tau = tau; A.tauU[N.otU + i] = tau; }
    }
    __syncthreads();
    for (int r = i + 1 + tid; r < mr; r += blockDim.x) vs[r - i] = U[(int64_t)r * kr + i];
    __syncthreads();
    const double tau = s_tau;
    if (tau != 0.0) {
      if (fast) {  // U's own columns now, D's columns after the factorisation
        for (int j = wid; j < kr - i - 1; j += NW)
          warp_apply(vs, mr - i, tau, U + (int64_t)i * kr + (i + 1 + j), kr);
      } else {
        for (int j = wid; j < (kr - i - 1) + mc; j += NW) {
          if (j < kr - i - 1) warp_apply(vs, mr - i, tau, U + (int64_t)i * kr + (i + 1 + j), kr);
          else warp_apply(vs, mr - i, tau, D + (int64_t)i * mc + (j - (kr - i - 1)), mc);
        }
      }
    }
    __syncthreads();
  }
  if (fast && kr > 0) {
    // Q^T D: one warp per column of D, the column in registers, all kr reflectors
    const double* taus = A.tauU + N.otU;
    const double* Uc = U;
    const int ldu = kr;
    auto uat = [Uc, ldu](int i, int j) { return Uc[j * ldu + i]; };
    for (int c = wid; c < mc; c += NW) {
      if (mr <= 128) warp_apply_all<4>(D + c, mc, mr, kr, taus, uat);
      else warp_apply_all<ULV_PF>(D + c, mc, mr, kr, taus, uat);
    }
    __syncthreads();
  }
  // 2. LQ of Bbot = the last t rows of Q^T D (QR of Bbot^T), applied from the right
  //    to the other rows of D (Dtrans) and to V^T (Mfull)
  const int r0 = mr - t;
  if (wid == 0) {  // ||Bbot||_inf before the elimination (singularity test, apply.py:218-221)
    double mx = 0.0;
    for (int r = 0; r < t; ++r) {
      double s = 0.0;
      for (int c = lane; c < mc; c += 32) s += fabs(D[(int64_t)(r0 + r) * mc + c]);
      s = warp_sum(s);
      mx = fmax(mx, s);
    }
    if (lane == 0) s_norm = mx;
  }
  __syncthreads();
  for (int i = 0; i < t; ++i) {
    double* row = D + (int64_t)(r0 + i) * mc;
    if (wid == 0) {
      double tau = warp_larfg(row + i, 1, mc - i);
      if (lane == 0) { s_tau = tau; A.tauZ[N.otZ + i] = tau; }
    }
    __syncthreads();
    for (int c = i + 1 + tid; c < mc; c += blockDim.x) vs[c - i] = row[c];
    __syncthreads();
    const double tau = s_tau;
    if (tau != 0.0) {
      const int nrows = fast ? (t - i - 1) : (t - i - 1) + r0 + kc;
      for (int j = wid; j < nrows; j += NW) {
        double* y;
        if (j < t - i - 1) y = D + (int64_t)(r0 + i + 1 + j) * mc;
        else if (j < t - i - 1 + r0) y = D + (int64_t)(j - (t - i - 1)) * mc;
        else y = VT + (int64_t)(j - (t - i - 1) - r0) * mc;
        warp_apply(vs, mc - i, tau, y + i, 1);
      }
    }
    __syncthreads();
  }
  if (fast) {
    // Dtrans = Dtop Qz and Mfull = V^T Qz: one warp per row, the row in registers,
    // all t reflectors (stored in the LQ rows of D)
    const double* taus = A.tauZ + N.otZ;
    const double* Lz = D + (int64_t)r0 * mc;
    const int ldz = mc;
    auto vat = [Lz, ldz](int i, int j) { return Lz[i * ldz + j]; };
    for (int j = wid; j < r0 + kc; j += NW) {
      double* y = j < r0 ? D + (int64_t)j * mc : VT + (int64_t)(j - r0) * mc;
      if (mc <= 128) warp_apply_all<4>(y, 1, mc, t, taus, vat);
      else warp_apply_all<ULV_PF>(y, 1, mc, t, taus, vat);
    }
    __syncthreads();
  }
  if (tid == 0) {
    double dmin = INFINITY;
    for (int i = 0; i < t; ++i) dmin = fmin(dmin, fabs(D[(int64_t)(r0 + i) * mc + i]));
    if (dmin <= PIVOT_RTOL * fmax(s_norm, 1e-300)) flag_singular(A, N.post);
  }
  if (stage) {
    __syncthreads();
    for (int64_t e = tid; e < nD; e += blockDim.x) Dg[e] = D[e];
    for (int64_t e = tid; e < nU; e += blockDim.x) Ug[e] = U[e];
    for (int64_t e = tid; e < nV; e += blockDim.x) Vg[e] = VT[e];
  }
}

// ---- root LU with partial pivoting (sla.lu_factor, apply.py:270-283) -------------------------
__global__ void __launch_bounds__(ULV_THREADS) k_ulv_root_lu(UlvArgs A, int* piv) {
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ double s_norm;
  const UlvNode& N = A.nd[A.root];
  const int m = N.mr, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, NW = blockDim.x >> 5;
  double* D = A.D + N.oD;
  if (wid == 0) {
    double mx = 0.0;
    for (int r = 0; r < m; ++r) {
      double s = 0.0;
      for (int c = lane; c < m; c += 32) s += fabs(D[(int64_t)r * m + c]);
      mx = fmax(mx, warp_sum(s));
    }
    if (lane == 0) s_norm = mx;
  }
  for (int k = 0; k < m; ++k) {
    // pivot: first row of max |D[r][k]|, r >= k
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int r = k + tid; r < m; r += blockDim.x) {
      double a = fabs(D[(int64_t)r * m + k]);
      if (a > bv) { bv = a; bi = r; }
    }
    for (int o = 16; o; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { red_v[wid] = bv; red_i[wid] = bi; }
    __syncthreads();
    bv = red_v[0]; bi = red_i[0];
    for (int w = 1; w < NW; ++w)
      if (red_v[w] > bv || (red_v[w] == bv && red_i[w] < bi)) { bv = red_v[w]; bi = red_i[w]; }
    if (tid == 0) piv[k] = bi;
    if (bi != k)
      for (int c = tid; c < m; c += blockDim.x) {
        double x = D[(int64_t)k * m + c];
        D[(int64_t)k * m + c] = D[(int64_t)bi * m + c];
        D[(int64_t)bi * m + c] = x;
      }
    __syncthreads();
    const double p = D[(int64_t)k * m + k];
    if (p != 0.0)
      for (int r = k + 1 + tid; r < m; r += blockDim.x) D[(int64_t)r * m + k] /= p;
    __syncthreads();
    for (int e = tid; e < (m - k - 1) * (m - k - 1); e += blockDim.x) {
      const int r = k + 1 + e / (m - k - 1), c = k + 1 + e % (m - k - 1);
      D[(int64_t)r * m + c] -= D[(int64_t)r * m + k] * D[(int64_t)k * m + c];
    }
    __syncthreads();
  }
  if (tid == 0 && m > 0) {
    double dmin = INFINITY;
    for (int i = 0; i < m; ++i) dmin = fmin(dmin, fabs(D[(int64_t)i * m + i]));
    if (dmin <= PIVOT_RTOL * fmax(s_norm, 1e-300)) flag_singular(A, N.post);
  }
}

// ---- solve ------------------------------------------------------------------------------------
struct SolveArgs {
  UlvArgs A;
  const double* b;   // caller order, n_row x R
  double* x;         // caller order, n_col x R
  const int64_t* perm_row;  // tree position -> caller index (int64, device)
  const int64_t* perm_col;
  double* wb;        // per node mr x R
  double* wx;        // per node mc x R  ([z1; xvec])
  double* wg;        // per node kc x R
  const int* piv;
  int R;
  int stage;         // this level's per-node vectors fit shared memory (after the vs buffer)
  int vs_cap;        // doubles reserved for the reflector buffer at the start of shared memory
};

// upward pass of one level (apply.py:300-330); the root also runs the LU solve
__global__ void __launch_bounds__(ULV_THREADS) k_ulv_up(SolveArgs S) {
  extern __shared__ __align__(16) unsigned char smem[];
  const UlvArgs& A = S.A;
  const int v = A.lb + blockIdx.x;
  if (v >= A.le) return;
  const UlvNode& N = A.nd[v];
  const int R = S.R, tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, wid = tid >> 5,
            NW = NT >> 5;
  double* b = S.wb + N.ob * R;
  double* g = S.wg + N.og * R;
  int* invc = reinterpret_cast<int*>(smem);
  // bcur
  if (N.leaf) {
    for (int e = tid; e < N.mr * R; e += NT) {
      const int r = e / R, c = e % R;
      b[e] = S.b[S.perm_row[N.row_a + r] * R + c];
    }
    for (int e = tid; e < N.kc * R; e += NT) g[e] = 0.0;
  } else {
    const UlvNode& N1 = A.nd[N.c1];
    const UlvNode& N2 = A.nd[N.c2];
    const int m1 = N1.mr - N1.t;
    const double* b1 = S.wb + N1.ob * R;
    const double* b2 = S.wb + N2.ob * R;
    const double* g1 = S.wg + N1.og * R;
    const double* g2 = S.wg + N2.og * R;
    const double* CP1 = A.CP + N1.oCP;
    const double* CP2 = A.CP + N2.oCP;
    for (int e = tid; e < N.mr * R; e += NT) {
      const int r = e / R, c = e % R;
      double s;
      if (r < m1) {
        s = b1[(int64_t)r * R + c];
        for (int q = 0; q < N2.kc; ++q) s -= CP1[(int64_t)r * N2.kc + q] * g2[(int64_t)q * R + c];
      } else {
        s = b2[(int64_t)(r - m1) * R + c];
        for (int q = 0; q < N1.kc; ++q)
          s -= CP2[(int64_t)(r - m1) * N1.kc + q] * g1[(int64_t)q * R + c];
      }
      b[e] = s;
    }
    if (v != A.root) {  // gpre = W_c1^T g1 + W_c2^T g2
      load_inv(A.C, v, invc);
      __syncthreads();
      const double* Gc = A.C.G + A.C.g_off[v];
      for (int e = tid; e < N.kc * R; e += NT) {
        const int a = e / R, c = e % R;
        double s = 0.0;
        for (int q = 0; q < N1.kc; ++q) s = fma(expand_at(invc, Gc, N.kc, q, a), g1[(int64_t)q * R + c], s);
        for (int q = 0; q < N2.kc; ++q)
          s = fma(expand_at(invc, Gc, N.kc, N1.kc + q, a), g2[(int64_t)q * R + c], s);
        g[e] = s;
      }
    }
  }
  __syncthreads();
  if (v == A.root) {  // LU solve (sla.lu_solve): P, L (unit), U
    const int m = N.mr;
    const double* LU = A.D + N.oD;
    double* xr = S.wx + N.ox * R;
    for (int c = wid; c < R; c += NW) {
      if (lane == 0) {
        for (int k = 0; k < m; ++k) {
          const int p = S.piv[k];
          if (p != k) { double q = b[(int64_t)k * R + c]; b[(int64_t)k * R + c] = b[(int64_t)p * R + c]; b[(int64_t)p * R + c] = q; }
        }
        for (int i = 0; i < m; ++i) {
          double s = b[(int64_t)i * R + c];
          for (int j = 0; j < i; ++j) s -= LU[(int64_t)i * m + j] * xr[(int64_t)j * R + c];
          xr[(int64_t)i * R + c] = s;
        }
        for (int i = m - 1; i >= 0; --i) {
          double s = xr[(int64_t)i * R + c];
          for (int j = i + 1; j < m; ++j) s -= LU[(int64_t)i * m + j] * xr[(int64_t)j * R + c];
          xr[(int64_t)i * R + c] = s / LU[(int64_t)i * m + i];
        }
      }
    }
    if (N.leaf) {  // single-leaf tree: the root system is the whole matrix
      __syncthreads();
      for (int e = tid; e < N.mc * R; e += NT) {
        const int r = e / R, c = e % R;
        S.x[S.perm_col[N.col_a + r] * R + c] = xr[e];
      }
    }
    return;
  }
  if (N.t == 0) return;  // bred = bcur, g = gpre
  const double* U = A.U + N.oU;
  const double* D = A.D + N.oD;
  const double* VT = A.VT + N.oVT;
  const int mr = N.mr, mc = N.mc, kr = N.kr, t = N.t, r0 = mr - t;
  double* vs = reinterpret_cast<double*>(smem);
  if (S.stage) {
    // the node's right-hand sides and z1 in shared memory: Q^T b, the forward
    // substitution (left-looking, coalesced rows of L) and the corrections run
    // on chip; bred, z1 and g go back to HBM for the parent / the downward pass
    double* sb = vs + S.vs_cap;
    double* sz = sb + (int64_t)mr * R;
    for (int e = tid; e < mr * R; e += NT) sb[e] = b[e];
    double* su = sz + (int64_t)t * R;  // U (reflectors below the diagonal), coalesced copy
    for (int e = tid; e < mr * kr; e += NT) su[e] = U[e];
    __syncthreads();
    if (mr <= 32 * ULV_PF) {
      // Q^T b with each warp's column in registers (entry j = lane + 32k) and the
      // next reflector (column i+1 of U below the diagonal) prefetched
      for (int c = wid; c < R; c += NW) {
        double yr[ULV_PF], cur[ULV_PF], nxt[ULV_PF];
#pragma unroll
        for (int k = 0; k < ULV_PF; ++k) {
          const int j = lane + 32 * k;
          yr[k] = j < mr ? sb[(int64_t)j * R + c] : 0.0;
        }
        auto load_col = [&](int ii, double* dst) {
#pragma unroll
          for (int k = 0; k < ULV_PF; ++k) {
            const int j = lane + 32 * k;
            dst[k] = j < mr ? (j > ii ? su[j * kr + ii] : (j == ii ? 1.0 : 0.0)) : 0.0;
          }
        };
        load_col(0, cur);
        double tau = A.tauU[N.otU];
        for (int i = 0; i < kr; ++i) {
          double tau_n = 0.0;
          if (i + 1 < kr) {
            load_col(i + 1, nxt);
            tau_n = A.tauU[N.otU + i + 1];
          }
          double w = 0.0;
#pragma unroll
          for (int k = 0; k < ULV_PF; ++k) w = fma(cur[k], yr[k], w);
          w = warp_sum(w) * tau;
#pragma unroll
          for (int k = 0; k < ULV_PF; ++k) yr[k] = fma(-w, cur[k], yr[k]);
#pragma unroll
          for (int k = 0; k < ULV_PF; ++k) cur[k] = nxt[k];
          tau = tau_n;
        }
#pragma unroll
        for (int k = 0; k < ULV_PF; ++k) {
          const int j = lane + 32 * k;
          if (j < mr) sb[(int64_t)j * R + c] = yr[k];
        }
      }
      __syncthreads();
    } else {
      for (int i = 0; i < kr; ++i) {
        for (int r = i + 1 + tid; r < mr; r += NT) vs[r - i] = U[(int64_t)r * kr + i];
        __syncthreads();
        const double tau = A.tauU[N.otU + i];
        if (tau != 0.0)
          for (int c = wid; c < R; c += NW) warp_apply(vs, mr - i, tau, sb + (int64_t)i * R + c, R);
        __syncthreads();
      }
    }
    for (int c = wid; c < R; c += NW) {
      for (int i = 0; i < t; ++i) {
        const double* Li = D + (int64_t)(r0 + i) * mc;
        double acc = 0.0;
        for (int j = lane; j < i; j += 32) acc = fma(Li[j], sz[(int64_t)j * R + c], acc);
        acc = warp_sum(acc);
        if (lane == 0) sz[(int64_t)i * R + c] = (sb[(int64_t)(r0 + i) * R + c] - acc) / Li[i];
        __syncwarp();
      }
    }
    __syncthreads();
    double* z = S.wx + N.ox * R;
    for (int e = tid; e < t * R; e += NT) z[e] = sz[e];
    for (int e = tid; e < r0 * R; e += NT) {
      const int r = e / R, c = e % R;
      double sacc = sb[e];
      for (int j = 0; j < t; ++j) sacc -= D[(int64_t)r * mc + j] * sz[(int64_t)j * R + c];
      b[e] = sacc;
    }
    for (int e = tid; e < N.kc * R; e += NT) {
      const int a = e / R, c = e % R;
      double sacc = g[e];
      for (int j = 0; j < t; ++j) sacc = fma(VT[(int64_t)a * mc + j], sz[(int64_t)j * R + c], sacc);
      g[e] = sacc;
    }
    return;
  }
  // bp = Q^T bcur
  for (int i = 0; i < kr; ++i) {
    for (int r = i + 1 + tid; r < mr; r += NT) vs[r - i] = U[(int64_t)r * kr + i];
    __syncthreads();
    const double tau = A.tauU[N.otU + i];
    if (tau != 0.0)
      for (int c = wid; c < R; c += NW) warp_apply(vs, mr - i, tau, b + (int64_t)i * R + c, R);
    __syncthreads();
  }
  // z1 = L^-1 bp[r0:], kept in x[0:t) for the downward pass
  // (right-looking forward substitution, one warp per right-hand side: lane 0
  // finishes z_i, the warp subtracts its column of L from the rows below)
  double* z = S.wx + N.ox * R;
  for (int c = wid; c < R; c += NW) {
    for (int i = 0; i < t; ++i) {
      double zi = 0.0;
      if (lane == 0) {
        zi = b[(int64_t)(r0 + i) * R + c] / D[(int64_t)(r0 + i) * mc + i];
        z[(int64_t)i * R + c] = zi;
      }
      zi = __shfl_sync(0xffffffffu, zi, 0);
      for (int j = i + 1 + lane; j < t; j += 32)
        b[(int64_t)(r0 + j) * R + c] -= D[(int64_t)(r0 + j) * mc + i] * zi;
      __syncwarp();
    }
  }
  __syncthreads();
  // bred = bp[:r0] - Dcorr z1 ; g += Mcorr z1
  for (int e = tid; e < r0 * R; e += NT) {
    const int r = e / R, c = e % R;
    double s = b[e];
    for (int j = 0; j < t; ++j) s -= D[(int64_t)r * mc + j] * z[(int64_t)j * R + c];
    b[e] = s;
  }
  for (int e = tid; e < N.kc * R; e += NT) {
    const int a = e / R, c = e % R;
    double s = g[e];
    for (int j = 0; j < t; ++j) s = fma(VT[(int64_t)a * mc + j], z[(int64_t)j * R + c], s);
    g[e] = s;
  }
}

// downward pass of one level (apply.py:332-348): x_v = Qz [z1; xvec]
__global__ void __launch_bounds__(ULV_THREADS) k_ulv_down(SolveArgs S) {
  extern __shared__ __align__(16) unsigned char smem[];
  const UlvArgs& A = S.A;
  const int v = A.lb + blockIdx.x;
  if (v >= A.le || v == A.root) return;
  const UlvNode& N = A.nd[v];
  const UlvNode& Pn = A.nd[N.parent];
  const int R = S.R, tid = threadIdx.x, NT = blockDim.x, wid = tid >> 5, NW = NT >> 5;
  double* xg = S.wx + N.ox * R;
  const double* xp = S.wx + Pn.ox * R;
  const int n_red = N.mc - N.t;
  // [z1; xvec] assembled in shared memory when the level fits (else in place in HBM)
  double* xv = S.stage ? reinterpret_cast<double*>(smem) + S.vs_cap : xg;
  if (S.stage)
    for (int e = tid; e < N.t * R; e += NT) xv[e] = xg[e];
  for (int e = tid; e < n_red * R; e += NT) xv[(int64_t)N.t * R + e] = xp[(int64_t)N.pos * R + e];
  __syncthreads();
  if (N.t > 0 && N.mc <= 32 * ULV_PF) {
    // Each warp applies the reflectors to its own right-hand-side columns with
    // the column held in registers (entry j = lane + 32k in yr[k]) and no block
    // barriers; reflector i-1's row (and tau) are prefetched while reflector i is
    // applied.  The row's entry at the diagonal is replaced by the implicit 1.
    const double* D = A.D + N.oD;
    const int mc = N.mc, r0 = N.mr - N.t, lane = tid & 31;
    for (int c = wid; c < R; c += NW) {
      double yr[ULV_PF], cur[ULV_PF], nxt[ULV_PF];
#pragma unroll
      for (int k = 0; k < ULV_PF; ++k) {
        const int j = lane + 32 * k;
        yr[k] = j < mc ? xv[(int64_t)j * R + c] : 0.0;
      }
      auto load_row = [&](int ii, double* dst) {
        const double* row = D + (int64_t)(r0 + ii) * mc;
#pragma unroll
        for (int k = 0; k < ULV_PF; ++k) {
          const int j = lane + 32 * k;
          dst[k] = j < mc ? (j > ii ? row[j] : (j == ii ? 1.0 : 0.0)) : 0.0;
        }
      };
      int i = N.t - 1;
      load_row(i, cur);
      double tau = A.tauZ[N.otZ + i];
      for (; i >= 0; --i) {
        double tau_n = 0.0;
        if (i > 0) {
          load_row(i - 1, nxt);
          tau_n = A.tauZ[N.otZ + i - 1];
        }
        double w = 0.0;
#pragma unroll
        for (int k = 0; k < ULV_PF; ++k) w = fma(cur[k], yr[k], w);
        w = warp_sum(w) * tau;
#pragma unroll
        for (int k = 0; k < ULV_PF; ++k) yr[k] = fma(-w, cur[k], yr[k]);
#pragma unroll
        for (int k = 0; k < ULV_PF; ++k) cur[k] = nxt[k];
        tau = tau_n;
      }
#pragma unroll
      for (int k = 0; k < ULV_PF; ++k) {
        const int j = lane + 32 * k;
        if (j < mc) xv[(int64_t)j * R + c] = yr[k];
      }
    }
    __syncthreads();
  } else if (N.t > 0) {
    const double* D = A.D + N.oD;
    double* vs = reinterpret_cast<double*>(smem);
    const int mc = N.mc, r0 = N.mr - N.t;
    for (int i = N.t - 1; i >= 0; --i) {
      const double* row = D + (int64_t)(r0 + i) * mc;
      for (int c = i + 1 + tid; c < mc; c += NT) vs[c - i] = row[c];
      __syncthreads();
      const double tau = A.tauZ[N.otZ + i];
      if (tau != 0.0)
        for (int c = wid; c < R; c += NW) warp_apply(vs, mc - i, tau, xv + (int64_t)i * R + c, R);
      __syncthreads();
    }
  }
  if (N.leaf) {
    for (int e = tid; e < N.mc * R; e += NT) {
      const int r = e / R, c = e % R;
      S.x[S.perm_col[N.col_a + r] * R + c] = xv[e];
    }
  } else if (S.stage) {
    __syncthreads();
    for (int e = tid; e < N.mc * R; e += NT) xg[e] = xv[e];
  }
}

}  // namespace

struct UlvImpl {
  MatrixImpl* M = nullptr;
  std::vector<UlvNode> h;
  DBuf<UlvNode> d;
  DBuf<double> D, U, VT, tauU, tauZ, CP;
  DBuf<int> piv, err;
  DBuf<int64_t> perm_row, perm_col;
  int root = 0;
  int64_t nb = 0, nx = 0, ng = 0;
  int vs_cap = 1;
  size_t smem_asm = 0, smem_red = 0, smem_up = 0;
  DBuf<double> wb, wx, wg;
  int64_t ws_nrhs = 0;
  // solves share the workspaces: each waits for the previous one (any stream), and the
  // factorisation is freed only after its last solve completes
  cudaEvent_t last_use = nullptr;
  ~UlvImpl() {
    if (last_use) {
      cudaEventSynchronize(last_use);
      cudaEventDestroy(last_use);
    }
  }
};

namespace {

UlvArgs make_args(UlvImpl* F, int lb, int le) {
  MatrixImpl* M = F->M;
  TreeImpl* t = M->tree;
  auto view = [](const SideFactors& S) {
    return FacView{S.perm.p, S.G.p, S.skel.p, S.ib_off.p, S.g_off.p, S.skel_off.p, S.nib.p};
  };
  UlvArgs A;
  A.nd = F->d.p; A.lb = lb; A.le = le; A.root = F->root;
  A.D = F->D.p; A.U = F->U.p; A.VT = F->VT.p; A.tauU = F->tauU.p; A.tauZ = F->tauZ.p; A.CP = F->CP.p;
  A.R = view(M->rowf); A.C = view(*M->colf);
  A.prow = t->pts_row.p;
  A.pcol = t->shared ? t->pts_row.p : t->pts_col.p;
  A.nrow = t->nx; A.ncol = t->shared ? t->nx : t->ny;
  A.dx = M->p.dx;
  A.err = F->err.p;
  A.vs_cap = F->vs_cap;
  A.stage_cap = 0;
  return A;
}

void check_err(UlvImpl* F, cudaStream_t s) {
  int h[2] = {0, 0};
  d2h(h, F->err.p, 2, s);
  sync(s);
  SMASH_CHECK(h[0] == 0, SMASH_ERR_NUMERICAL,
              "ULV elimination hit a singular local block at node " + std::to_string(h[1]));
}

}  // namespace

UlvImpl* ulv_factor(MatrixImpl* M, cudaStream_t s) {
  SMASH_CHECK(M->p.structure == SMASH_STRUCT_HSS, SMASH_ERR_INVALID,
              "ULV factorization expects an HSS matrix");
  TreeImpl* t = M->tree;
  const int n = t->n_nodes, L = t->n_levels;
  std::unique_ptr<UlvImpl> F(new UlvImpl());
  F->M = M;
  std::vector<int> nch(n), cf(n), par(n), post(n), ra(n), rb(n), ca(n), cb(n), kr(n), kc(n);
  d2h(nch.data(), t->nchild.p, n, s);
  d2h(cf.data(), t->child_first.p, n, s);
  d2h(par.data(), t->parent.p, n, s);
  d2h(post.data(), t->post.p, n, s);
  d2h(ra.data(), t->row_a.p, n, s);
  d2h(rb.data(), t->row_b.p, n, s);
  d2h(ca.data(), t->shared ? t->row_a.p : t->col_a.p, n, s);
  d2h(cb.data(), t->shared ? t->row_b.p : t->col_b.p, n, s);
  d2h(kr.data(), M->rowf.rank.p, n, s);
  d2h(kc.data(), M->colf->rank.p, n, s);
  sync(s);
  F->root = t->level_begin(1);
  std::vector<UlvNode>& H = F->h;
  H.assign(n, UlvNode{});
  int64_t oD = 0, oU = 0, oVT = 0, otU = 0, otZ = 0, oCP = 0, ob = 0, ox = 0, og = 0;
  size_t sm_asm = 16, sm_red = 16, sm_up = 16;
  int vs_cap = 1;
  std::vector<int64_t> lvl_need(L + 2, 0);  // per level: largest staged reduction (doubles)
  for (int l = L; l >= 1; --l) {
    for (int v = t->level_begin(l); v < t->level_end(l); ++v) {
      UlvNode& N = H[v];
      const bool root = v == F->root;
      N.leaf = nch[v] == 0;
      N.post = post[v];
      N.parent = root ? -1 : par[v];
      N.row_a = ra[v];
      N.col_a = ca[v];
      N.kr = root ? 0 : kr[v];
      N.kc = root ? 0 : kc[v];
      if (N.leaf) {
        N.c1 = N.c2 = -1;
        N.mr = rb[v] - ra[v];
        N.mc = cb[v] - ca[v];
      } else {
        SMASH_CHECK(nch[v] == 2, SMASH_ERR_INVALID, "ULV expects a binary (HSS) tree");
        N.c1 = cf[v]; N.c2 = cf[v] + 1;
        const UlvNode &A1 = H[N.c1], &A2 = H[N.c2];
        N.mr = (A1.mr - A1.t) + (A2.mr - A2.t);
        N.mc = (A1.mc - A1.t) + (A2.mc - A2.t);
        sm_asm = std::max(sm_asm, 8 * (size_t)(A1.kr * A2.kc + A2.kr * A1.kc) +
                                      4 * (size_t)(A1.kr + A2.kr + A1.kc + A2.kc) + 16);
        sm_up = std::max(sm_up, 4 * (size_t)(A1.kc + A2.kc) + 16);
      }
      if (N.leaf) sm_asm = std::max(sm_asm, 4 * (size_t)(N.mr + N.mc) + 16);
      const int e = N.mr - N.kr;
      N.t = (!root && e > 0) ? std::min(e, N.mc) : 0;
      if (root)
        SMASH_CHECK(N.mr == N.mc, SMASH_ERR_NUMERICAL,
                    "ULV root system is " + std::to_string(N.mr) + "x" + std::to_string(N.mc) +
                        ", not square");
      N.oD = oD; oD += (int64_t)N.mr * N.mc;
      N.oU = oU; oU += (int64_t)N.mr * N.kr;
      N.oVT = oVT; oVT += (int64_t)N.kc * N.mc;
      N.otU = otU; otU += N.kr;
      N.otZ = otZ; otZ += N.t;
      N.ob = ob; ob += N.mr;
      N.ox = ox; ox += N.mc;
      N.og = og; og += N.kc;
      sm_red = std::max(sm_red, 8 * (size_t)std::max(N.mr, N.mc) + 16);
      vs_cap = std::max(vs_cap, std::max(N.mr, N.mc));
      if (!root && N.t > 0)
        lvl_need[l] = std::max<int64_t>(lvl_need[l], (int64_t)N.mr * N.mc + (int64_t)N.mr * N.kr +
                                                         (int64_t)N.kc * N.mc);
      sm_up = std::max(sm_up, 8 * (size_t)std::max(N.mr, N.mc) + 16);
    }
  }
  // CP slots (child c: m_red(c) x k_c(sibling)) and x offsets of the children
  for (int v = 0; v < n; ++v) {
    UlvNode& N = H[v];
    if (N.leaf) continue;
    UlvNode &A1 = H[N.c1], &A2 = H[N.c2];
    A1.oCP = oCP; oCP += (int64_t)(A1.mr - A1.t) * A2.kc;
    A2.oCP = oCP; oCP += (int64_t)(A2.mr - A2.t) * A1.kc;
    A1.pos = 0;
    A2.pos = A1.mc - A1.t;
  }
  SMASH_CHECK(sm_asm <= 200 * 1024 && sm_red <= 200 * 1024, SMASH_ERR_INVALID,
              "ULV: node blocks too large for one CTA");
  // reduce: reflector buffer + staging area, capped at 48 KB so that >= 4 CTAs
  // share an SM (measured: cfg 1's nodes gain 1.5x in shared memory, while
  // cfg 4's 128 x 128 leaves run faster from L2 with 8 CTAs per SM than
  // staged with 1 CTA per SM)
  vs_cap = (vs_cap + 1) & ~1;
  F->vs_cap = vs_cap;
  sm_red = 8 * (size_t)vs_cap + 64;  // unstaged levels
  F->smem_asm = sm_asm; F->smem_red = sm_red; F->smem_up = sm_up;
  F->nb = ob; F->nx = ox; F->ng = og;
  F->d.alloc(n, s);
  h2d(F->d.p, H.data(), n, s);
  F->D.alloc(std::max<int64_t>(oD, 1), s);
  F->U.alloc(std::max<int64_t>(oU, 1), s);
  F->VT.alloc(std::max<int64_t>(oVT, 1), s);
  F->tauU.alloc(std::max<int64_t>(otU, 1), s);
  F->tauZ.alloc(std::max<int64_t>(otZ, 1), s);
  F->CP.alloc(std::max<int64_t>(oCP, 1), s);
  F->piv.alloc(std::max(H[F->root].mr, 1), s);
  F->err.alloc(2, s);
  F->err.zero(s);
  F->perm_row.alloc(t->nx, s);
  F->perm_col.alloc(t->shared ? t->nx : t->ny, s);
  {
    std::vector<int> pr(t->nx), pc(t->shared ? t->nx : t->ny);
    d2h(pr.data(), t->perm_row.p, pr.size(), s);
    d2h(pc.data(), t->shared ? t->perm_row.p : t->perm_col.p, pc.size(), s);
    sync(s);
    std::vector<int64_t> a(pr.begin(), pr.end()), b(pc.begin(), pc.end());
    h2d(F->perm_row.p, a.data(), a.size(), s);
    h2d(F->perm_col.p, b.data(), b.size(), s);
    sync(s);
  }
  const int dim = t->dim;
  for (int l = L; l >= 1; --l) {
    const int lb = t->level_begin(l), le = t->level_end(l);
    UlvArgs A = make_args(F.get(), lb, le);
    dispatch_kernel_dim(M->p.kernel, dim, [&]<int KER, int DIM>() {
      auto k = k_ulv_assemble<KER, DIM>;
      SMASH_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_asm));
      k<<<le - lb, ULV_THREADS, sm_asm, s>>>(A);
    });
    SMASH_CUDA(cudaGetLastError());
    if (l > 1) {
      // a level is staged in shared memory when its largest node fits 48 KB (>= 4 CTAs/SM)
      static const bool no_stage = getenv("SMASH_ULV_NOSTAGE") != nullptr;
      const int64_t cap = (48 * 1024 - 8 * (int64_t)F->vs_cap - 64) / 8;
      A.stage_cap = (!no_stage && lvl_need[l] <= cap) ? lvl_need[l] : 0;
      const size_t sm = sm_red + 8 * (size_t)A.stage_cap;
      SMASH_CUDA(cudaFuncSetAttribute(k_ulv_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)std::max<size_t>(sm, 48 * 1024)));
      k_ulv_reduce<<<le - lb, ULV_THREADS, sm, s>>>(A);
      SMASH_CUDA(cudaGetLastError());
    }
  }
  k_ulv_root_lu<<<1, ULV_THREADS, 0, s>>>(make_args(F.get(), F->root, F->root + 1), F->piv.p);
  SMASH_CUDA(cudaGetLastError());
  check_err(F.get(), s);
  return F.release();
}

void ulv_solve(UlvImpl* F, const double* b, double* x, int64_t R, cudaStream_t s) {
  SMASH_CHECK(R >= 1, SMASH_ERR_INVALID, "nrhs must be positive");
  TreeImpl* t = F->M->tree;
  if (!F->last_use) SMASH_CUDA(cudaEventCreateWithFlags(&F->last_use, cudaEventDisableTiming));
  SMASH_CUDA(cudaStreamWaitEvent(s, F->last_use, 0));
  if (F->ws_nrhs < R) {
    // the old workspaces may still be read by a solve on another stream: free after it
    SMASH_CUDA(cudaEventSynchronize(F->last_use));
    F->wb.alloc(std::max<int64_t>(F->nb * R, 1), s);
    F->wx.alloc(std::max<int64_t>(F->nx * R, 1), s);
    F->wg.alloc(std::max<int64_t>(F->ng * R, 1), s);
    F->ws_nrhs = R;
  }
  SolveArgs S;
  S.b = b; S.x = x; S.perm_row = F->perm_row.p; S.perm_col = F->perm_col.p;
  S.wb = F->wb.p; S.wx = F->wx.p; S.wg = F->wg.p; S.piv = F->piv.p; S.R = (int)R;
  const size_t sm = F->smem_up;
  // per level: stage the nodes' vectors in shared memory when they fit 64 KB
  static const bool no_stage = getenv("SMASH_ULV_NOSTAGE") != nullptr;
  const int L = t->n_levels;
  std::vector<int> vcap(L + 2, 1);
  std::vector<int64_t> need_up(L + 2, 0), need_dn(L + 2, 0);
  for (int l = 1; l <= L; ++l)
    for (int v = t->level_begin(l); v < t->level_end(l); ++v) {
      const UlvNode& N = F->h[v];
      vcap[l] = std::max(vcap[l], (std::max(N.mr, N.mc) + 1) & ~1);
      need_up[l] = std::max<int64_t>(need_up[l], (int64_t)(N.mr + N.t) * R + (int64_t)N.mr * N.kr);
      need_dn[l] = std::max<int64_t>(need_dn[l], (int64_t)N.mc * R);
    }
  auto lvl_smem = [&](int l, int64_t need, int* stage) {
    const size_t want = 8 * ((size_t)vcap[l] + (size_t)need) + 64;
    *stage = !no_stage && want <= 64 * 1024;
    return *stage ? std::max(sm, want) : sm;
  };
  SMASH_CUDA(cudaFuncSetAttribute(k_ulv_up, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::max<size_t>(sm, 64 * 1024 + 64)));
  SMASH_CUDA(cudaFuncSetAttribute(k_ulv_down, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::max<size_t>(sm, 64 * 1024 + 64)));
  static const bool timing = getenv("SMASH_ULV_TIMING") != nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timing) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
  }
  auto tick = [&](const char* what, int l) {
    if (!timing) return;
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    fprintf(stderr, "ulv_solve %s level %d: %.3f ms\n", what, l, ms);
    cudaEventRecord(e0, s);
  };
  if (timing) cudaEventRecord(e0, s);
  for (int l = t->n_levels; l >= 1; --l) {
    S.A = make_args(F, t->level_begin(l), t->level_end(l));
    S.vs_cap = vcap[l];
    const size_t smu = lvl_smem(l, need_up[l], &S.stage);
    k_ulv_up<<<t->level_end(l) - t->level_begin(l), ULV_THREADS, smu, s>>>(S);
    tick("up", l);
  }
  for (int l = 2; l <= t->n_levels; ++l) {
    S.A = make_args(F, t->level_begin(l), t->level_end(l));
    S.vs_cap = vcap[l];
    const size_t smd = lvl_smem(l, need_dn[l], &S.stage);
    k_ulv_down<<<t->level_end(l) - t->level_begin(l), ULV_THREADS, smd, s>>>(S);
    tick("down", l);
  }
  if (timing) {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  SMASH_CUDA(cudaGetLastError());
  SMASH_CUDA(cudaEventRecord(F->last_use, s));
}

void ulv_free(UlvImpl* F) { delete F; }

}  // namespace smash
