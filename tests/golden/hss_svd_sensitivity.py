"""How far the reference's HSS output moves under an equally valid fp64 SVD
(test infrastructure; development container only).

The HSS candidate [U_hat, S] (hss.py:274-299) carries S = the kept left singular
vectors of the nearfield block row (lowrank.py:265-276, LAPACK gesdd).  Singular
vectors whose singular value sits near the cut eps_svd * sigma_1 are determined
only to ~eps * sigma_1 / gap by ANY backward-stable fp64 SVD, and they enter the
candidate unscaled, so the skeleton order and G of the reference are themselves
sensitive to the SVD's rounding.  This script measures that sensitivity: it runs
the oracle's restatement of build_hss (pinned bit-exact to the reference with
gesdd, tests/test_oracle_golden.py) with the SVD replaced by another backward-
stable LAPACK route -- column-pivoted QR (dgeqp3) followed by gesvd of R, the same
QR-preconditioned structure as the GPU kernel K5 (csrc/svd.cu) -- and counts, against
the reference's own output:

  * ordered-skeleton and rank mismatches per (side, node);
  * the transfer-matrix difference e1 = ||dX|| / ||X|| on label-identical nodes;
  * the matvec difference and the error against the exact product.

Usage: python tests/golden/hss_svd_sensitivity.py [cfg4_2k cfg4_8k pair1d_hss cfg1_full] [full4]
Writes tests/golden/full/hss_svd_sensitivity.json (read by the HSS parity tests).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np
import scipy.linalg as sla

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

from oracle import smash_oracle as orc  # noqa: E402

import parity  # noqa: E402
from conftest import load_golden  # noqa: E402

OUT = os.path.join(HERE, "full", "hss_svd_sensitivity.json")


def truncated_svd_qr(M, eps):
    """Kept left singular vectors by dgeqp3 + gesvd(R) (same keep rule as lowrank.py:275)."""
    M = np.asarray(M)
    if min(M.shape) == 0:
        return np.zeros((M.shape[0], 0))
    Q, R, _ = sla.qr(M, mode="economic", pivoting=True)
    Ur, sig, _ = sla.svd(R, lapack_driver="gesvd")
    keep = 0 if sig[0] == 0 else int(np.count_nonzero(sig >= eps * sig[0]))
    return (Q @ Ur)[:, :keep]


def build_alt(X, Y, m):
    orc_tsvd = orc.truncated_svd
    orc.truncated_svd = truncated_svd_qr
    try:
        t = orc.build_tree(X, None if Y is X else Y, nu0=m["nu0"], mode=m["mode"])
        M = orc.build_hss(t, m["kernel"], m["r"], m["tau"], m["eps_svd"], rtol=m["rtol"],
                          dx=None if m["kernel"] == "exp" else 0.0)
    finally:
        orc.truncated_svd = orc_tsvd
    return M


def small(name):
    g = load_golden(name)
    m = g["meta"]
    M = build_alt(g["X"], g["Y"], m)
    order = rank = total = 0
    e1, res, ek = [], [], []
    for side, fac in (("row", M.rowfac), ("col", M.colfac)):
        skels = M.skel_row if side == "row" else M.skel_col
        for i, f in fac.items():
            ref = g["skel_%s" % side][g["skel_%s_ptr" % side][i]:g["skel_%s_ptr" % side][i + 1]]
            total += 1
            ib_r, ib_a = parity.ref_ibar(g, side, i), orc._ibar(M.tree, i, skels, side)
            if f.skel.size != ref.size:
                rank += 1
                continue
            X = parity.align_rows(f.expand(), ib_a, ib_r)
            if X is None or not np.array_equal(f.skel, ref):
                order += int(not np.array_equal(f.skel, ref))
                C = parity.ref_candidate(g, side, i)
                if C is not None and X is not None:
                    # how well the alternative factor interpolates the reference's own candidate
                    C_a = parity.align_rows(C, ib_r, ib_a)
                    res.append(np.linalg.norm(C_a - f.expand() @ C_a[f.perm[:f.rank]]) / np.linalg.norm(C))
            elif "G_row" in g:
                pr, Gr = parity.ref_factor(g, side, i)
                Xr = parity.expand(pr, Gr, f.rank)
                e1.append(np.linalg.norm(X - Xr) / max(np.linalg.norm(Xr), 1e-300))
                C = parity.ref_candidate(g, side, i)
                if C is not None and f.rank:
                    sv = np.linalg.svd(C[pr[:f.rank]], compute_uv=False)
                    ek.append(e1[-1] / (sv[0] / sv[-1]) if sv[-1] > 0 else 0.0)
    z = orc.matvec(M, g["q"])
    dz = max(np.linalg.norm(z[:, c] - g["z"][:, c]) / np.linalg.norm(g["z"][:, c]) for c in range(z.shape[1]))
    rows, ze = g["exact_rows"], g["z_exact_rows"]
    return dict(factors=total, order_mismatch=order, rank_mismatch=rank,
                G_e1_median=float(np.median(e1)) if e1 else 0.0, G_e1_max=float(np.max(e1)) if e1 else 0.0,
                G_e1_over_kappa_max=float(np.max(ek)) if ek else 0.0,
                mismatched_residual_max=float(np.max(res)) if res else 0.0,
                matvec_rel_vs_reference=float(dz),
                err_vs_exact=float(np.linalg.norm(z[rows] - ze) / np.linalg.norm(ze)),
                ref_err_vs_exact=float(np.linalg.norm(g["z"][rows] - ze) / np.linalg.norm(ze)))


def full4():
    g = dict(np.load(os.path.join(HERE, "full", "cfg4_full.npz")))
    m = dict(orc.CONFIGS[4])
    X, Y, rng = orc.make_config_points(4)
    q = rng.standard_normal((Y.shape[0], int(g["nrhs"])))
    M = build_alt(X, Y, m)
    order = rank = total = 0
    for side, fac in (("row", M.rowfac), ("col", M.colfac)):
        for i, f in fac.items():
            total += 1
            if f.skel.size != g["rank_" + side][i]:
                rank += 1
            elif int(hashlib.blake2b(np.asarray(f.skel, "<i8").tobytes(), digest_size=8).hexdigest(), 16) \
                    != int(g["skdig_" + side][i]):
                order += 1
    e1, res, ek = [], [], []
    for side, fac in (("row", M.rowfac), ("col", M.colfac)):
        ids = g["gs_%s_nodes" % side]
        skels = M.skel_row if side == "row" else M.skel_col
        for t, i in enumerate(ids):
            sl = lambda key: g["gs_%s_%s" % (side, key)][g["gs_%s_%s_ptr" % (side, key)][t]:
                                                         g["gs_%s_%s_ptr" % (side, key)][t + 1]]
            f = fac[int(i)]
            pr, Gr, ibar = sl("perm").astype(np.int64), sl("G"), sl("ibar").astype(np.int64)
            ncol = int(g["gs_%s_cand_cols" % side][t])
            k = int(g["rank_" + side][i])
            if f.rank != k:
                continue
            ib_a = orc._ibar(M.tree, int(i), skels, side)
            Xr = parity.expand(pr, Gr, k)
            X = parity.align_rows(f.expand(), ib_a, ibar)
            if X is not None and np.array_equal(f.skel, ibar[pr[:k]]):
                e1.append(np.linalg.norm(X - Xr) / max(np.linalg.norm(Xr), 1e-300))
                if ncol and k:
                    sv = np.linalg.svd(sl("cand").reshape(-1, ncol)[pr[:k]], compute_uv=False)
                    ek.append(e1[-1] / (sv[0] / sv[-1]) if sv[-1] > 0 else 0.0)
            elif X is not None and ncol:
                C = sl("cand").reshape(-1, ncol)
                C_a = parity.align_rows(C, ibar, ib_a)
                res.append(np.linalg.norm(C_a - f.expand() @ C_a[f.perm[:k]]) / np.linalg.norm(C))
    z = orc.matvec(M, q)
    rows, er = g["z_rows"].astype(np.int64), g["exact_rows"].astype(np.int64)
    dz = max(np.linalg.norm(z[rows, c] - g["z_at_rows"][:, c]) / np.linalg.norm(g["z_at_rows"][:, c])
             for c in range(z.shape[1]))
    ze = g["z_exact_rows"]
    ref_at = g["z_at_rows"][np.searchsorted(rows, er)]
    return dict(factors=total, order_mismatch=order, rank_mismatch=rank,
                G_e1_median=float(np.median(e1)) if e1 else 0.0, G_e1_max=float(np.max(e1)) if e1 else 0.0,
                G_e1_over_kappa_max=float(np.max(ek)) if ek else 0.0,
                mismatched_residual_max=float(np.max(res)) if res else 0.0,
                matvec_rel_vs_reference_sampled=float(dz),
                err_vs_exact=float(np.linalg.norm(z[er] - ze) / np.linalg.norm(ze)),
                ref_err_vs_exact=float(np.linalg.norm(ref_at - ze) / np.linalg.norm(ze)))


if __name__ == "__main__":
    res = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for a in sys.argv[1:] or ["cfg4_2k", "cfg4_8k", "pair1d_hss", "cfg1_full"]:
        res[a] = full4() if a == "full4" else small(a)
        print(a, res[a], flush=True)
        os.makedirs(os.path.dirname(OUT), exist_ok=True)
        with open(OUT, "w") as f:
            json.dump(res, f, indent=1, sort_keys=True)
