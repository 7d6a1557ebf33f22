// K5 host side: level plan and launches of the HSS nearfield SVD (device code and the
// algorithm notes: svd_kernels.cuh; k_svd instantiations: svd_<kernel>.cu).
#include "svd_kernels.cuh"

namespace smash {
namespace svdk {

// explicit instantiations live in svd_log.cu / svd_invr.cu / svd_exp.cu / svd_cauchy.cu
extern template void svd_launch<SMASH_KERNEL_LOG>(int, const SvdLaunch&);
extern template void svd_launch<SMASH_KERNEL_INV_R>(int, const SvdLaunch&);
extern template void svd_launch<SMASH_KERNEL_EXP>(int, const SvdLaunch&);
extern template void svd_launch<SMASH_KERNEL_CAUCHY>(int, const SvdLaunch&);

namespace {

void svd_launch_kernel(int ker, int dim, const SvdLaunch& L) {
  switch (ker) {
    case SMASH_KERNEL_LOG: svd_launch<SMASH_KERNEL_LOG>(dim, L); break;
    case SMASH_KERNEL_INV_R: svd_launch<SMASH_KERNEL_INV_R>(dim, L); break;
    case SMASH_KERNEL_EXP: svd_launch<SMASH_KERNEL_EXP>(dim, L); break;
    case SMASH_KERNEL_CAUCHY: svd_launch<SMASH_KERNEL_CAUCHY>(dim, L); break;
    default: throw Error(SMASH_ERR_INVALID, "unsupported kernel / dimension combination");
  }
}

__global__ void k_near_cols(SvdArgs A) {
  int v = A.lb + blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= A.le) return;
  int nn = 0;
  for (int e = A.near_ptr[v]; e < A.near_ptr[v + 1]; ++e)
    nn += ibar_size(A.other, A.nchild, A.child_first, A.near_idx[e]);
  A.nn_out[v - A.lb] = nn;
}

__global__ void __launch_bounds__(SVD_THREADS, 4) k_jacobi(JacArgs A) {
  extern __shared__ __align__(16) double jac_smem[];
  double* Js = jac_smem;
  double* nrm = jac_smem + JAC_KP * JAC_KP + SVD_SLACK;
  Shared S{};
  S.imisc = reinterpret_cast<int*>(nrm + 256);
  const int tid = threadIdx.x, NT = blockDim.x;
  for (int v = A.lb + blockIdx.x; v < A.le; v += gridDim.x) {
    const int kp = A.kp_g[v - A.ws_lb];
    if (kp == 0) continue;
    double* Jg = A.gws + (size_t)(v - A.ws_lb) * A.gws_stride + A.joff_g[v - A.ws_lb];
    if (kp <= JAC_KP) {
      for (int e = tid; e < kp * kp; e += NT) Js[e] = Jg[e];
      __syncthreads();
      jacobi_sweeps<8>(Js, kp, nrm, S, nullptr, false);
      __syncthreads();
      for (int e = tid; e < kp * kp; e += NT) Jg[e] = Js[e];
    } else {
      __syncthreads();
      jacobi_sweeps<16>(Jg, kp, nrm, S, nullptr, false);
    }
    __syncthreads();
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

void svd_launch_jacobi(const JacArgs& a, int grid, cudaStream_t s) {
  constexpr size_t jac_smem = JAC_SMEM_DOUBLES * sizeof(double);
  static const bool jac_attr = [] {
    SMASH_CUDA(cudaFuncSetAttribute(k_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)jac_smem));
    return true;
  }();
  (void)jac_attr;
  k_jacobi<<<grid, SVD_THREADS, jac_smem, s>>>(a);
}

}  // namespace svdk

using namespace svdk;

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
  static const int floor_exp = getenv("SMASH_SVD_FLOOR") ? atoi(getenv("SMASH_SVD_FLOOR")) : 57;
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
  A.gws_stride = (int64_t)A.nmax * A.nnmax + (int64_t)A.nnmax * kpmax + 2 * (int64_t)kpmax * kpmax + 2 * SVD_SLACK;
  int dev = 0, nsm = 0;
  SMASH_CUDA(cudaGetDevice(&dev));
  SMASH_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  static const int svd_per_sm_env = getenv("SMASH_SVD_PER_SM") ? atoi(getenv("SMASH_SVD_PER_SM")) : 0;
  static const bool hyb_on = !(getenv("SMASH_SVD_HYB") && atoi(getenv("SMASH_SVD_HYB")) == 0);
  static const bool gq0_on = !(getenv("SMASH_SVD_GQ0") && atoi(getenv("SMASH_SVD_GQ0")) == 0);
  static const int big_waves = getenv("SMASH_SVD_BIGW") ? atoi(getenv("SMASH_SVD_BIGW")) : 4;
  const int64_t panel = (int64_t)A.nmax * A.nnmax;
  const int mx = std::max(A.nmax, A.nnmax);
  const size_t smem_small = 8 * ((size_t)3 * A.nnmax + 2 * mx + 2 * A.nmax + 32 + 8 + 2 * MAX_NEAR) +
                            4 * ((size_t)32 + 8 + MAX_NEAR + 1 + A.nmax + A.nnmax) + 64 + 16;
  // work area: the largest that leaves two CTAs per SM (about 96 KB)
  SMASH_CHECK(smem_small + 8 * 4096 <= SVD_SMEM_MAX / 2 - 1024, SMASH_ERR_INVALID, "HSS nearfield block too large");
  const int big2 = (int)(((SVD_SMEM_MAX / 2 - 1024) - smem_small) / 8) & ~1;
  A.big = big2;
  A.gq0 = gq0_on;
  // level shapes: (a) at most 80 rows with every column of the panel in the two-per-SM work
  // area: all-shared group-column QR; (b) up to 128 x 256 (config 4's leaf blocks and its
  // middle levels): the HYB kernel, one CTA per SM, two register columns per group;
  // (c) anything else on the swap-based QR -- panel in the work area if it fits, widened to
  // one CTA per SM on levels of few nodes, else in the L2-resident workspace
  const int slots = (A.nnmax + 31) & ~31;
  const bool shape_a = gq0_on && A.nmax <= 80 && A.nnmax <= 32 * HQ_KC && (int64_t)slots * (A.nmax <= 72 ? 72 : 80) <= big2;
  const bool hyb = hyb_on && !shape_a && panel > big2 && A.nmax <= HQ_ROWS && A.nnmax <= 32 * HQ_KC &&
                   smem_small + 8 * (size_t)HQ_BIG <= SVD_SMEM_MAX;
  if (hyb) {
    A.big = HQ_BIG;
  } else if (panel > big2 && run_le - run_lb <= big_waves * nsm) {
    A.big = (int)std::min<int64_t>(panel, (int64_t)((SVD_SMEM_MAX - smem_small) / 8));
  }
  const int svd_per_sm = svd_per_sm_env ? svd_per_sm_env : (A.big > big2 ? 1 : 2);
  static const bool split_on = !(getenv("SMASH_SVD_SPLIT") && atoi(getenv("SMASH_SVD_SPLIT")) == 0);
  static const int split_chunk = getenv("SMASH_SVD_CHUNK") ? atoi(getenv("SMASH_SVD_CHUNK")) : 8;
  const int run_cnt = run_le - run_lb;
  // a wide HYB level is split: QR launches of one CTA per SM, the later phases at two
  const bool split = hyb && split_on && run_cnt > 2 * nsm;
  // wide levels also hand the Jacobi sweeps to k_jacobi (four CTAs per SM)
  static const bool jsplit_on = !(getenv("SMASH_SVD_JSPLIT") && atoi(getenv("SMASH_SVD_JSPLIT")) == 0);
  const bool jsplit = jsplit_on && run_cnt > 2 * nsm && (split || (!hyb && A.big == big2));
  const int grid = std::min(cnt, nsm * svd_per_sm);
  // per-node workspaces: every chunked level works inside the same 1 GB block (allocated once
  // per build, always the same size: the stream-ordered pool hands the block back instead of
  // mapping fresh memory for each level's different size, which cost sporadic 0.2 - 0.7 s)
  constexpr int64_t WS_DOUBLES = (int64_t)1 << 27;
  int chunk = 0;
  if (split || jsplit) {
    const int64_t fit = std::max<int64_t>(1, WS_DOUBLES / A.gws_stride);
    const int64_t unit = 2 * nsm;
    chunk = (int)std::min<int64_t>(run_cnt, fit >= unit ? fit / unit * unit : fit);
    if (split) chunk = std::min(chunk, split_chunk * nsm);
  }
  DBuf<double> gws_local;
  if (chunk) {
    if (ws.gws.n < (size_t)WS_DOUBLES) ws.gws.alloc(WS_DOUBLES, s);
    A.gws = ws.gws.p;
  } else {
    gws_local.alloc((size_t)grid * A.gws_stride, s);
    A.gws = gws_local.p;
  }
  DBuf<int> kp_g;
  DBuf<double> taus_g;
  DBuf<int64_t> joff_g;
  if (chunk) {
    kp_g.alloc(chunk, s);
    taus_g.alloc((size_t)chunk * A.nmax, s);
    joff_g.alloc(chunk, s);
    A.kp_g = kp_g.p;
    A.taus_g = taus_g.p;
    A.joff_g = joff_g.p;
  }
  DBuf<int> err;
  err.alloc(1, s);
  err.zero(s);
  A.err = err.p;
  static const bool svd_dbg = getenv("SMASH_SVD_DBG") != nullptr;
  DBuf<long long> dbgbuf;
  A.dbg = nullptr;
  if (svd_dbg) {
    dbgbuf.alloc(48, s);
    dbgbuf.zero(s);
    A.dbg = dbgbuf.p;
  }
  const size_t smem = smem_small + 8 * (size_t)A.big;
  const size_t smem2 = smem_small + 8 * (size_t)big2;
  if (run_le > run_lb) {
    SvdLaunch Lc{A, run_lb, run_le, chunk, nsm, grid, big2, split, jsplit, hyb, smem, smem2, s};
    svd_launch_kernel(A.kernel, A.dim, Lc);
  }
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
    long long h[48];
    d2h(h, dbgbuf.p, 48, s);
    sync(s);
    fprintf(stderr, "svd level %d side %d cnt %d:", level, side, cnt);
    for (int q = 0; q < 4; ++q)
      fprintf(stderr, " [asm %lld qr %lld qr2 %lld jac %lld back %lld kp %lld keep %lld n.nn %lld]", h[q * 8], h[q * 8 + 1],
              h[q * 8 + 2], h[q * 8 + 3], h[q * 8 + 4], h[q * 8 + 5], h[q * 8 + 6], h[q * 8 + 7]);
    fprintf(stderr, " max_sweeps %lld capped %lld | jacobi (thread 0 of traced nodes): dot %.0f scalar %.0f rotate %.0f per rotation (%lld), barrier wait %.0f per round (%lld) | group QR per step: scalars + update %.0f, write-back + argmax %.0f (%lld) | second QR per step: scalars %.0f columns %.0f barrier %.0f (%lld)\n", h[32], h[33],
            h[38] ? (double)h[34] / h[38] : 0.0, h[38] ? (double)h[35] / h[38] : 0.0, h[38] ? (double)h[36] / h[38] : 0.0, h[38],
            h[39] ? (double)h[37] / h[39] : 0.0, h[39], h[43] ? (double)h[40] / h[43] : 0.0,
            h[43] ? (double)h[42] / h[43] : 0.0, h[43], h[47] ? (double)h[44] / h[47] : 0.0,
            h[47] ? (double)h[45] / h[47] : 0.0, h[47] ? (double)h[46] / h[47] : 0.0, h[47]);
  }
  return hk;
}


}  // namespace smash
