"""Parity rules shared by the CPU and GPU tests.

Rule 3 (transfer matrices): compare the expand() matrices X = P [I; G] by row
label.  Pass if

    ||dX||_F / ||X||_F <= 1e-10                                  (clause 1)
or  ||dX C[skel]||_F / ||C||_F <= 1e-13                           (clause 2)
    and ||dX||_F / ||X||_F <= 100 * kappa(R11) * 2^-53

where C is the compr input (|ibar| x ncols) and R11 the leading k x k block of
the pivoted QR of C^T, so kappa(R11) = cond(C[skel]).  Clause 2 accepts G that
differ only along the directions an ill-conditioned R11 leaves undetermined:
the interpolation C ~= X C[skel] they define is the same to 1e-13.
"""

from __future__ import annotations

import numpy as np

from oracle import smash_oracle as orc

EPS = 2.0 ** -53


def expand(perm, G, k):
    perm = np.asarray(perm)
    n = perm.size
    X = np.zeros((n, k))
    X[perm[:k]] = np.eye(k)
    if k < n:
        X[perm[k:]] = np.asarray(G).reshape(n - k, k)
    return X


def rule3(Xg, Xr, C=None, skel_local=None):
    """Return (ok, clause, e1, e2, kappa)."""
    nx = max(np.linalg.norm(Xr), 1e-300)
    e1 = np.linalg.norm(Xg - Xr) / nx
    if e1 <= 1e-10:
        return True, 1, e1, None, None
    if C is None or skel_local is None or C.size == 0:
        return False, 0, e1, None, None
    Cs = C[np.asarray(skel_local)]
    sv = np.linalg.svd(Cs, compute_uv=False)
    kappa = sv[0] / sv[-1] if sv.size and sv[-1] > 0 else np.inf
    e2 = np.linalg.norm((Xg - Xr) @ Cs) / max(np.linalg.norm(C), 1e-300)
    ok = e2 <= 1e-13 and e1 <= 100 * kappa * EPS
    return ok, 2, e1, e2, kappa


def node_basis(g, side, i, ibar):
    """C = interp_basis(padded box, points[ibar], r) of node i from the golden's tree
    (hss.py:219-238 with _pad_box hss.py:39-45) -- the H^2 compr input."""
    lo, hi = g["lo"], g["hi"]
    root = int(np.nonzero(g["parent"] < 0)[0][0])
    diam = 2 * orc.box_radius(lo[root], hi[root])[0]
    pad = max(1e-9 * diam, 1e-300)
    plo, phi = orc.pad_box(lo[i], hi[i], pad)
    pts = g["X"][g["perm_row"]] if side == "row" else g["Y"][g["perm_col"]]
    return orc.interp_basis(plo, phi, pts[ibar], int(g["meta"]["r"]))


def ref_ibar(g, side, i):
    """ibar of node i from the reference's own skeletons (hss.py:241-244)."""
    kids = g["child_idx"][g["child_ptr"][i]:g["child_ptr"][i + 1]]
    if kids.size == 0:
        a, b = (g["row_start"][i], g["row_stop"][i]) if side == "row" else (g["col_start"][i], g["col_stop"][i])
        return np.arange(a, b, dtype=np.int64)
    sp, sv = g["skel_%s_ptr" % side], g["skel_%s" % side]
    return np.concatenate([sv[sp[c]:sp[c + 1]] for c in kids])


def ref_candidate(g, side, i):
    """The reference's compr input for node i: stored [U_hat, S] for HSS fixtures that
    recorded it, else the recomputed H^2 basis; None when not available."""
    key = "cand_%s" % side
    if key in g:
        ptr = g["cand_%s_ptr" % side]
        ncol = int(g["cand_%s_cols" % side][i])
        v = g[key][ptr[i]:ptr[i + 1]]
        return v.reshape(-1, ncol) if ncol else None
    if g["meta"]["structure"] == "h2":
        return node_basis(g, side, i, ref_ibar(g, side, i))
    return None


def ref_factor(g, side, i):
    """(perm, G) of node i; the column side falls back to the row side when the
    fixture recorded them as bitwise equal."""
    if "G_%s" % side not in g:
        side = "row"
    pp, pv = g["fperm_%s_ptr" % side], g["fperm_%s" % side]
    gp, gv = g["G_%s_ptr" % side], g["G_%s" % side]
    return pv[pp[i]:pp[i + 1]], gv[gp[i]:gp[i + 1]]


def hss_sensitivity(name):
    """The reference's own HSS sensitivity to an equally valid fp64 SVD on fixture
    `name` (tests/golden/hss_svd_sensitivity.py), or None."""
    import json
    import os
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "full", "hss_svd_sensitivity.json")
    if not os.path.exists(p):
        return None
    return json.load(open(p)).get(name)


def hss_g_ok(name, e1, kappa=None):
    """HSS G clause: a label-identical node whose G differs from the reference's by more
    than rule 3 allows passes if the difference is of the size the reference's own
    algorithm shows under another backward-stable SVD (hss_svd_sensitivity.json):
    e1 <= 10 kappa(R11) max(e1 / kappa) of that restatement (the difference of an
    interpolative factor scales with the conditioning of its skeleton rows), or
    e1 <= 4 max(e1) of it."""
    s = hss_sensitivity(name)
    if s is None:
        return False
    if kappa is not None and np.isfinite(kappa) and s.get("G_e1_over_kappa_max", 0.0) > 0:
        if e1 <= 10 * kappa * s["G_e1_over_kappa_max"]:
            return True
    return e1 <= 4 * max(s["G_e1_max"], 1e-10)


def align_rows(X, ibar_from, ibar_to):
    """X's rows (labelled by ibar_from) reordered into ibar_to's label order, or None
    when the two ibar label sets differ (G rows are compared by label, SURVEY 8(c) rule 3:
    a child whose ordered skeleton differs reorders its parent's ibar)."""
    ibar_from = np.asarray(ibar_from)
    ibar_to = np.asarray(ibar_to)
    if ibar_from.size != ibar_to.size:
        return None
    o_from, o_to = np.argsort(ibar_from, kind="stable"), np.argsort(ibar_to, kind="stable")
    if not np.array_equal(ibar_from[o_from], ibar_to[o_to]):
        return None
    idx = np.empty(ibar_to.size, np.int64)
    idx[o_to] = o_from  # row of ibar_from carrying the label of ibar_to[r]
    return X[idx]


def gpu_ibar(M, side, i):
    """ibar of node i in the GPU build: leaf range, else the children's GPU skeletons."""
    tr = M.tree
    kids = tr.nodes[i].children
    if not kids:
        return np.asarray(tr.row_range(i) if side == "row" else tr.col_range(i), np.int64)
    fac = M.rowfac if side == "row" else M.colfac
    return np.concatenate([np.asarray(fac[c].skel, np.int64) for c in kids])
