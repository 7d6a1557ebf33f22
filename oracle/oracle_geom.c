/*
 * TEST INFRASTRUCTURE ONLY -- part of the CPU oracle (see oracle/__init__.py).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library.  The product path never does.
 *
 * Exact fused multiply-add helpers for the oracle's box geometry.
 *
 * The reference measures box radii and centre distances with np.linalg.norm
 * (smash/cluster.py:68-71, :81-85), which for a 1-3 element float64 vector is
 * an OpenBLAS ddot whose scalar tail contracts to an FMA chain:
 *     norm(v) = sqrt(fma(v2, v2, fma(v1, v1, v0 * v0)))
 * (probe p8).  numpy has no fma, so the oracle calls
 * these C helpers; gcc's fma() is the correctly rounded IEEE operation, the
 * same one the CUDA kernels issue with __fma_rn.
 *
 * Build: gcc -O2 -fPIC -shared -ffp-contract=off -o oracle/_build/liboracle_geom.so oracle/oracle_geom.c -lm
 */
#include <math.h>
#include <stdint.h>

/* out[i] = || v[i, 0:d] ||_2 with the FMA-chain summation order. */
void or_norm_rows(const double* v, int64_t n, int d, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    const double* r = v + i * d;
    double s = r[0] * r[0];
    for (int k = 1; k < d; ++k) s = fma(r[k], r[k], s);
    out[i] = sqrt(s);
  }
}

/* out[i] = fma(a[i], b[i], c[i]) */
void or_fma(const double* a, const double* b, const double* c, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = fma(a[i], b[i], c[i]);
}
