"""Golden container files written by the REAL reference (development container only).

Builds two small matrices with the unmodified reference package
(/root/reference/pkg/src/smash, imported read-only, never copied) in its own
kernel family (the real 1-D Cauchy kernel, Chebyshev interpolation basis) and
writes them with the reference's own ``smash.container.save_matrix``
(container.py:58-128), next to the reference's matvec of a seeded vector:

  container/ref_cauchy_hss.smash  -- HSS, x_i = i/n, y_j = (j + 0.5)/n (cfg-4 geometry), n = 512
  container/ref_cauchy_h2.smash   -- H2 on the same points
  container/ref_container.npz     -- q and z = matvec_nodewise(M, q) for both

tests/test_container.py loads the files with paper_1705_05443_b200.load_matrix
(GPU) and checks the device matvec against z; the CPU tests parse them.

Usage:  python tests/golden/make_container_golden.py
"""
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
import smash  # noqa: E402  (the reference)
from smash.container import save_matrix  # noqa: E402

n = 512
x = (np.arange(n) / n)[:, None]
y = ((np.arange(n) + 0.5) / n)[:, None]
X, Y = smash.PointSet(x), smash.PointSet(y, role="col")
spec = smash.KernelSpec("cauchy")
q = np.random.default_rng(44).standard_normal(n)
out = {"q": q}
for kind in ("hss", "h2"):
    tree = smash.build_tree(X, Y, nu0=32, mode="binary", tau=0.6)
    params = smash.BuildParams(r=12, tau=0.6, basis="interp", eps_svd=1e-11)
    build = smash.build_hss if kind == "hss" else smash.build_h2
    M = build(tree, spec, X, Y, params)
    out["z_" + kind] = smash.matvec_nodewise(M, q)
    if kind == "hss":
        F = smash.ulv_factor(M)
        out["x_hss"] = smash.ulv_solve(F, q)
        out["B3"] = np.random.default_rng(45).standard_normal((n, 3))
        out["X3_hss"] = smash.ulv_solve(F, out["B3"])
    save_matrix(M, os.path.join(HERE, "container", "ref_cauchy_%s.smash" % kind))
np.savez_compressed(os.path.join(HERE, "container", "ref_container.npz"), **out)
print("ok", {k: v.shape for k, v in out.items()})
