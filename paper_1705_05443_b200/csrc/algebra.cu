// HSS algebra of the reference (smash/hss.py:317-400) on the
// device: diag_scale, hss_add and cauchy_like_hss produce matrices whose generators
// are block-diagonal stacks of diagonally scaled copies of built matrices,
//   S = sum_t diag(dl_t) A_t diag(dr_t)
// (hss_add concatenates bases and stacks R / W / B block-diagonally, diag_scale scales
// the leaf bases and diagonal blocks).  Their product is therefore
//   S q = sum_t dl_t o (A_t (dr_t o q)),
// evaluated here with ONE device matvec per distinct base A_t over all of its terms'
// scaled right-hand sides at once (a cauchy_like_hss with p generator columns and
// nrhs right-hand sides is one p*nrhs-column product of the Cauchy HSS matrix), then
// one combine kernel.
#include "smash_impl.cuh"

namespace smash {

namespace {

// Qs[i, j*R + c] = dr_j[i] * q[i, c] for the group's terms j (dr rows stacked [T][n])
__global__ void k_prescale(const double* q, int64_t n, int R, const double* dr, const int* terms,
                           int m, double* Qs) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)m * R;
  if (e >= n * per) return;
  const int64_t i = e / per;
  const int jc = (int)(e - i * per);
  const int j = jc / R, c = jc - j * R;
  Qs[e] = dr[(int64_t)terms[j] * n + i] * q[i * R + c];
}

struct TermSrc {
  const double* Z;  // the group's product (n_row x ld)
  int ld;           // m * R
  int slot;         // this term's column block in it
};

// z[i, c] = sum_t dl_t[i] * (A_t (dr_t o q))[i, c], terms in order
__global__ void k_combine(const TermSrc* src, int T, const double* dl, int64_t n, int R,
                          double* z) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * R) return;
  const int64_t i = e / R;
  const int c = (int)(e - i * R);
  double acc = 0.0;
  for (int t = 0; t < T; ++t) {
    const TermSrc s = src[t];
    acc = fma(dl[(int64_t)t * n + i], s.Z[i * s.ld + (int64_t)s.slot * R + c], acc);
  }
  z[e] = acc;
}

}  // namespace

void sum_matvec(int T, MatrixImpl* const* bases, const double* dl, const double* dr,
                const double* q, double* z, int64_t R, int levelwise, cudaStream_t s) {
  SMASH_CHECK(T >= 1, SMASH_ERR_INVALID, "a scaled sum needs at least one term");
  SMASH_CHECK(R >= 1, SMASH_ERR_INVALID, "nrhs must be positive");
  TreeImpl* t0 = bases[0]->tree;
  for (int t = 0; t < T; ++t)
    SMASH_CHECK(bases[t] && bases[t]->tree == t0, SMASH_ERR_INVALID,
                "operands must share one cluster tree");
  const int64_t nr = t0->nx, nc = t0->ny;
  // group the terms by base, in order of first appearance
  std::vector<MatrixImpl*> gb;
  std::vector<std::vector<int>> gt;
  for (int t = 0; t < T; ++t) {
    size_t g = 0;
    while (g < gb.size() && gb[g] != bases[t]) ++g;
    if (g == gb.size()) {
      gb.push_back(bases[t]);
      gt.emplace_back();
    }
    gt[g].push_back(t);
  }
  std::vector<DBuf<double>> Qs(gb.size()), Zs(gb.size());
  std::vector<DBuf<int>> idx(gb.size());
  std::vector<TermSrc> src(T);
  for (size_t g = 0; g < gb.size(); ++g) {
    const int m = (int)gt[g].size();
    idx[g].alloc(m, s);
    h2d(idx[g].p, gt[g].data(), m, s);
    Qs[g].alloc((size_t)nc * m * R, s);
    Zs[g].alloc((size_t)nr * m * R, s);
    const int64_t work = nc * m * R;
    k_prescale<<<cdiv(work, 256), 256, 0, s>>>(q, nc, (int)R, dr, idx[g].p, m, Qs[g].p);
    SMASH_CUDA(cudaGetLastError());
    if (levelwise) matvec_levelwise(gb[g], Qs[g].p, Zs[g].p, (int64_t)m * R, s);
    else matvec(gb[g], Qs[g].p, Zs[g].p, (int64_t)m * R, s);
    for (int j = 0; j < m; ++j) src[gt[g][j]] = TermSrc{Zs[g].p, (int)(m * R), j};
  }
  DBuf<TermSrc> dsrc;
  dsrc.alloc(T, s);
  h2d(dsrc.p, src.data(), T, s);
  k_combine<<<cdiv(nr * R, 256), 256, 0, s>>>(dsrc.p, T, dl, nr, (int)R, z);
  SMASH_CUDA(cudaGetLastError());
  // pageable h2d copies are staged before they return; the temporaries are freed
  // stream-ordered after the combine
}

}  // namespace smash
