"""Golden fixture for the HSS algebra (hss_add / diag_scale / cauchy_like_hss,
smash/hss.py:317-400) from the REAL reference (development container only).

Inputs follow the reference's own tests: the nearly coincident interval pair of
pkg/tests/conftest.py (restated: x_i = i/(n+1), y = x + 1e-7 U(0,1)), generator
columns w, v ~ U(0,1) (pkg/tests/test_apply.py:166-180), the Chebyshev basis
(basis="interp": the B200 path has no Taylor basis).  Stores the products of the
reference's generator-form results, their ranks and the exact products.

Usage:  python tests/golden/make_algebra_golden.py
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import smash, orc  # noqa: E402  (reference import path + oracle)
from smash.hss import cauchy_like_hss  # noqa: E402


def main(n=400, p=2, seed=11):
    x = (np.arange(1, n + 1) / (n + 1.0)).reshape(-1, 1)
    y = x + 1e-7 * np.random.default_rng(0).random((n, 1))
    X, Y = smash.PointSet(x), smash.PointSet(y, role="col")
    rng = np.random.default_rng(seed)
    w, v = rng.random((n, p)), rng.random((n, p))
    q = rng.standard_normal((n, 3))
    dl, dr = 0.5 + rng.random(n), 0.5 + rng.random(n)
    tree = smash.build_tree(X, Y, nu0=50, tau=0.6)
    params = smash.BuildParams(r=25, tau=0.6, eps_svd=1e-9, basis="interp")
    M = cauchy_like_hss(tree, X, Y, w, v, params)
    base = smash.build_hss(tree, smash.KernelSpec("cauchy"), X, Y, params)
    S = smash.diag_scale(base, dl, dr)
    T = smash.hss_add(base, S)
    C = orc.kernel_block("cauchy", x, y)
    A = sum(w[:, l][:, None] * C * v[:, l][None, :] for l in range(p))
    out = dict(x=x, y=y, w=w, v=v, q=q, dl=dl, dr=dr,
               z_like=smash.matvec_nodewise(M, q), z_like_level=smash.matvec_levelwise(M, q),
               z_scaled=smash.matvec_nodewise(S, q), z_sum=smash.matvec_nodewise(T, q),
               exact_like=A @ q, exact_scaled=(dl[:, None] * C * dr[None, :]) @ q,
               exact_sum=(C + dl[:, None] * C * dr[None, :]) @ q,
               rank_row_like=np.array([M.rank_row(i) if i != tree.root else 0 for i in range(len(tree.nodes))]),
               rank_col_like=np.array([M.rank_col(i) if i != tree.root else 0 for i in range(len(tree.nodes))]))
    os.makedirs(os.path.join(HERE, "algebra"), exist_ok=True)
    np.savez_compressed(os.path.join(HERE, "algebra", "cauchy_like.npz"), **out)
    rel = np.linalg.norm(out["z_like"] - out["exact_like"]) / np.linalg.norm(out["exact_like"])
    print("cauchy_like n=%d p=%d nodes=%d relerr_vs_exact %.2e" % (n, p, len(tree.nodes), rel))


if __name__ == "__main__":
    main()
