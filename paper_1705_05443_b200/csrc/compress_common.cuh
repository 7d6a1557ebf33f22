// Device helpers shared by the two compression kernels (compress.cu, compress_rc.cuh):
// numpy's pairwise row sum, the Lagrange cardinal functions, the ibar point source of a node.
#pragma once

#include "compress.cuh"
#include "qr_device.cuh"

namespace smash {
namespace cmn {

constexpr int MAX_SWAPS = 200;                     // lowrank.py:171

// numpy's pairwise summation (8 accumulators, n <= 128) over terms f(0..n-1);
// this is the order of `terms.sum(axis=1)` in lowrank.py:116.
template <typename F>
__device__ __forceinline__ double np_pairwise_sum(int n, F f) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, f(i));
    return r;
  }
  double a0 = f(0), a1 = f(1), a2 = f(2), a3 = f(3), a4 = f(4), a5 = f(5), a6 = f(6), a7 = f(7);
  int i = 8;
  const int lim = n - (n % 8);
  for (; i < lim; i += 8) {
    a0 = __dadd_rn(a0, f(i + 0)); a1 = __dadd_rn(a1, f(i + 1));
    a2 = __dadd_rn(a2, f(i + 2)); a3 = __dadd_rn(a3, f(i + 3));
    a4 = __dadd_rn(a4, f(i + 4)); a5 = __dadd_rn(a5, f(i + 5));
    a6 = __dadd_rn(a6, f(i + 6)); a7 = __dadd_rn(a7, f(i + 7));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3)),
                         __dadd_rn(__dadd_rn(a4, a5), __dadd_rn(a6, a7)));
  for (; i < n; ++i) res = __dadd_rn(res, f(i));
  return res;
}

// Lagrange cardinal functions of one axis at x (lowrank.py:108-120), written to L[0..m).
__device__ __forceinline__ void lagrange_axis(double x, const double* nd, const double* w, int m,
                                              double* L) {
  bool exact = false;
  for (int k = 0; k < m; ++k) exact |= (__dsub_rn(x, nd[k]) == 0.0);
  if (exact) {
    for (int k = 0; k < m; ++k) L[k] = (__dsub_rn(x, nd[k]) == 0.0) ? 1.0 : 0.0;
    return;
  }
  double S = np_pairwise_sum(m, [&](int k) { return __ddiv_rn(w[k], __dsub_rn(x, nd[k])); });
  for (int k = 0; k < m; ++k) L[k] = __ddiv_rn(__ddiv_rn(w[k], __dsub_rn(x, nd[k])), S);
}

// ---------------------------------------------------------------------------
// ibar point access
// ---------------------------------------------------------------------------
struct NodeSrc {
  const double* base;  // coordinate SoA base for this node's ibar
  int64_t stride;
  const int* lab;      // labels (nullptr -> leaf: label = lab0 + c)
  int lab0;
};

__device__ __forceinline__ NodeSrc node_src(const CompressArgs& A, int v) {
  NodeSrc s;
  if (A.nchild[v] == 0) {
    int a = A.pt_a[v];
    s.base = A.P + a;
    s.stride = A.P_stride;
    s.lab = nullptr;
    s.lab0 = a;
  } else {
    int o = A.skel_off[A.child_first[v]];
    s.base = A.Sk + o;
    s.stride = A.S_stride;
    s.lab = A.Slab + o;
    s.lab0 = 0;
  }
  return s;
}

}  // namespace cmn
}  // namespace smash
