// Shared helpers for the SMASH B200 library (sm_100a).
//
// Exactness: every floating-point operation whose result must match the CPU
// reference bit for bit (tree bisection midpoints, admissibility, the
// Chebyshev/Lagrange basis) is written with explicit round-to-nearest
// intrinsics (__dadd_rn / __dmul_rn / __fma_rn / IEEE division and sqrt), so
// nvcc cannot contract or reassociate them.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/smash_b200.h"

// Checked build (SMASH_CHECKED=1 in _build.py -> libsmash_b200_checked.so): device-side
// bounds / invariant asserts and bounded spin waits that trap instead of hanging -- the
// stand-in for compute-sanitizer, which this GPU pool does not allow.
#ifdef SMASH_CHECKED
#include <cassert>
#define SMASH_DASSERT(cond) assert(cond)
#else
#define SMASH_DASSERT(cond) ((void)0)
#endif

namespace smash {

// ---------------------------------------------------------------------------
// errors: C-ABI status codes mirror the reference CLI's exit codes
// (smash/cli.py:266-278): 2 = invalid argument (ValueError), 3 = numerical
// failure (RuntimeError, e.g. the sRRQR swap cap or an unsplittable cluster).
// ---------------------------------------------------------------------------
struct Error : public std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

#define SMASH_CUDA(call)                                                                   \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      throw ::smash::Error(SMASH_ERR_CUDA, std::string("CUDA error: ") +                   \
                                               cudaGetErrorString(e_) + " at " __FILE__ ":" + \
                                               std::to_string(__LINE__));                  \
  } while (0)

#define SMASH_CHECK(cond, code, msg)                     \
  do {                                                   \
    if (!(cond)) throw ::smash::Error((code), (msg));    \
  } while (0)

// device error flags (set by kernels, read back by the host orchestration)
enum DevErr : int {
  DEV_OK = 0,
  DEV_UNSPLITTABLE = 1,    // points coincide beyond the key depth (cluster.py:340-341)
  DEV_DEGENERATE_BOX = 2,  // interp_basis degenerate box (lowrank.py:131-134)
  DEV_SWAP_CAP = 4,        // srrqr swap loop cap (lowrank.py:196-197)
  DEV_CAPACITY = 8,        // internal capacity exceeded
};

// ---------------------------------------------------------------------------
// stream-ordered device buffer
// ---------------------------------------------------------------------------
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t st = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), st(o.st) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; st = o.st; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count, cudaStream_t s) {
    release();
    n = count;
    st = s;
    if (count) SMASH_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T), s));
  }
  void zero(cudaStream_t s) {
    if (n) SMASH_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void release() {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
    n = 0;
  }
  operator T*() const { return p; }
};

template <typename T>
inline void d2h(T* dst, const T* src, size_t n, cudaStream_t s) {
  if (n) SMASH_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, s));
}
template <typename T>
inline void h2d(T* dst, const T* src, size_t n, cudaStream_t s) {
  if (n) SMASH_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
}
template <typename T>
inline void d2d(T* dst, const T* src, size_t n, cudaStream_t s) {
  if (n) SMASH_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToDevice, s));
}
inline void sync(cudaStream_t s) { SMASH_CUDA(cudaStreamSynchronize(s)); }

inline unsigned cdiv(size_t a, size_t b) { return (unsigned)((a + b - 1) / b); }

// Keep freed stream-ordered allocations in the device pool (the default release
// threshold of 0 hands memory back to the driver at every synchronisation,
// which turns each per-level cudaMallocAsync into a real allocation).
inline void init_pool() {
  static bool done = false;
  if (done) return;
  int dev = 0;
  SMASH_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  SMASH_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t thr = ~0ULL;
  SMASH_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  done = true;
}

// ---------------------------------------------------------------------------
// exact geometry (smash/cluster.py:64-85)
// ---------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ double norm_fma(const double* v) {
  // np.linalg.norm of a 1..3-vector == sqrt(fma(v2,v2,fma(v1,v1,v0*v0)))
  double s = __dmul_rn(v[0], v[0]);
#pragma unroll
  for (int k = 1; k < D; ++k) s = __fma_rn(v[k], v[k], s);
  return __dsqrt_rn(s);
}

__device__ __forceinline__ double norm_fma_dyn(const double* v, int d) {
  double s = __dmul_rn(v[0], v[0]);
  for (int k = 1; k < d; ++k) s = __fma_rn(v[k], v[k], s);
  return __dsqrt_rn(s);
}

// Box centre (lo+hi)/2 and radius 0.5*||hi-lo||.
__device__ __forceinline__ void box_center_radius(const double* lo, const double* hi, int d,
                                                  double* c, double* rad) {
  double w[3];
  for (int k = 0; k < d; ++k) {
    c[k] = __dmul_rn(__dadd_rn(lo[k], hi[k]), 0.5);
    w[k] = __dsub_rn(hi[k], lo[k]);
  }
  *rad = __dmul_rn(0.5, norm_fma_dyn(w, d));
}

// well_separated: rA + rB <= tau * ||cA - cB|| (smash/cluster.py:81-85)
__device__ __forceinline__ bool well_separated(const double* cA, double rA, const double* cB,
                                               double rB, int d, double tau) {
  double v[3];
  for (int k = 0; k < d; ++k) v[k] = __dsub_rn(cA[k], cB[k]);
  double dist = norm_fma_dyn(v, d);
  return __dadd_rn(rA, rB) <= __dmul_rn(tau, dist);
}

}  // namespace smash
