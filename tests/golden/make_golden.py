"""Generate golden fixtures from the REAL reference package (development container only).

Runs /root/reference/pkg/src/smash (read-only, imported, never copied) with the
SURVEY.md 8(c) extension applied by monkeypatching module globals:

  * smash.hss.kernel_block  -> BASELINE kernels log / inv_r / exp (cauchy stays native)
  * smash.{hss,h2}.kernel_dtype -> float64 (real kernels on 2-D points)
  * smash.hss.interp_basis  -> 3-D tensor extension (d <= 2 delegates to the reference)
  * smash.{hss,h2}.compr    -> compr(..., rtol=<config tolerance>)

and stores, per case, the inputs and the reference's tree arrays, pair sets,
ordered skeletons, ranks, swap counts, transfer matrices G (small cases) and
matvec outputs as compressed .npz next to this script.  The fixtures are what
tests/test_oracle_golden.py (CPU) and tests/test_gpu_parity.py (GPU) compare
against; /root/reference is not needed at test time.

Usage:  python tests/golden/make_golden.py [case ...]
"""

from __future__ import annotations

import functools
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REPO)
sys.path.insert(0, REF_SRC)

import smash  # noqa: E402  (the reference)
import smash.h2  # noqa: E402
import smash.hss  # noqa: E402
import smash.lowrank  # noqa: E402

from oracle import smash_oracle as orc  # noqa: E402

_ORIG_KERNEL_BLOCK = smash.hss.kernel_block
_ORIG_INTERP = smash.hss.interp_basis
_ORIG_COMPR = smash.lowrank.compr


def install_extension(kind: str, rtol: float):
    """extend the reference from outside."""
    if kind == "cauchy":
        smash.hss.kernel_block = _ORIG_KERNEL_BLOCK
    else:
        def kb(spec, X, Y, rows, cols):
            return orc.kernel_block(kind, X.coords[np.asarray(rows)], Y.coords[np.asarray(cols)])
        smash.hss.kernel_block = kb
    f64 = lambda kernel, X: np.dtype(np.float64)  # noqa: E731
    smash.hss.kernel_dtype = f64
    smash.h2.kernel_dtype = f64

    def interp3(box, pts, r):
        if len(box.lo) <= 2:
            return _ORIG_INTERP(box, pts, r)
        return orc.interp_basis(np.asarray(box.lo), np.asarray(box.hi), pts, r)
    smash.hss.interp_basis = interp3
    c = functools.partial(_ORIG_COMPR, rtol=rtol)
    smash.hss.compr = c
    smash.h2.compr = c


def case_points(case):
    rng = np.random.default_rng(case["seed"])
    g = case["gen"]
    N = case["N"]
    if g == "cfg":
        X, Y, rng = orc.make_config_points(case["cfg"], N=N)
        return X, Y, rng
    if g == "uniform":
        X = rng.random((N, case["dim"]))
        return X, X, rng
    if g == "clustered2d":
        X = np.vstack([rng.random((N // 2, 2)) * 0.05, rng.random((N - N // 2, 2)) * 0.9 + 0.1])
        return X, X, rng
    if g == "pair1d":
        X = rng.random((N, 1))
        Y = rng.random((N + 7, 1))
        return X, Y, rng
    raise ValueError(g)


# name -> parameters.  cfgN_* follow BASELINE config N at reduced N.
CASES = {
    "cfg1_full": dict(gen="cfg", cfg=1, N=4096, seed=1, store_G=True, store_cand=True),
    "cfg2_4k": dict(gen="cfg", cfg=2, N=4096, seed=2, store_G=True),
    "cfg2_32k": dict(gen="cfg", cfg=2, N=32768, seed=2, store_G=False),
    "cfg3_8k": dict(gen="cfg", cfg=3, N=8192, seed=3, store_G=True),
    "cfg4_8k": dict(gen="cfg", cfg=4, N=8192, seed=4, store_G=True),
    "cfg5_16k": dict(gen="cfg", cfg=5, N=16384, seed=5, store_G=True),
    # every compr candidate [U_hat, S] of a Cauchy HSS build (gesdd's S), so the
    # GPU sRRQR can be checked on the reference's own inputs
    "cfg4_2k": dict(gen="cfg", cfg=4, N=2048, seed=4, store_G=True, store_cand=True),
    # edge cases: adaptive 2-D with deep shrinks, X != Y in 1-D, 3-D tiny
    "clustered2d": dict(gen="clustered2d", N=3000, seed=11, structure="h2", kernel="log", dim=2,
                        mode="2d", nu0=16, r=16, tau=0.7, rtol=1e-8, eps_svd=0.0, nrhs=3, store_G=True),
    "pair1d_hss": dict(gen="pair1d", N=700, seed=12, structure="hss", kernel="cauchy", dim=1,
                       mode="binary", nu0=20, r=12, tau=0.6, rtol=1e-10, eps_svd=1e-11, nrhs=2,
                       store_G=True, store_cand=True),
    "pair1d_h2": dict(gen="pair1d", N=700, seed=13, structure="h2", kernel="cauchy", dim=1,
                      mode="binary", nu0=20, r=12, tau=0.5, rtol=1e-10, eps_svd=0.0, nrhs=1,
                      store_G=True),
    "tiny_single_leaf": dict(gen="uniform", N=40, seed=14, structure="h2", kernel="inv_r", dim=2,
                             mode="2d", nu0=64, r=9, tau=0.7, rtol=1e-8, eps_svd=0.0, nrhs=1,
                             store_G=True),
    "uniform3d_small": dict(gen="uniform", N=2000, seed=15, structure="h2", kernel="exp", dim=3,
                            mode="2d", nu0=32, r=27, tau=0.7, rtol=1e-6, eps_svd=0.0, nrhs=2,
                            store_G=True),
}


def resolve(case):
    c = dict(case)
    if c["gen"] == "cfg":
        base = orc.CONFIGS[c["cfg"]]
        for k in ("structure", "kernel", "dim", "mode", "nu0", "r", "tau", "rtol", "eps_svd"):
            c.setdefault(k, base[k])
        c.setdefault("nrhs", min(2, max(base["nrhs"])))  # 2 columns pin multi-RHS; keeps fixtures small
    return c


def tree_arrays(tree):
    n = len(tree.nodes)
    child_ptr = np.zeros(n + 1, np.int64)
    kids = []
    for i, nd in enumerate(tree.nodes):
        child_ptr[i + 1] = child_ptr[i] + len(nd.children)
        kids += list(nd.children)
    return dict(
        level=np.array([nd.level for nd in tree.nodes], np.int64),
        parent=np.array([nd.parent for nd in tree.nodes], np.int64),
        child_ptr=child_ptr, child_idx=np.array(kids, np.int64),
        lo=np.array([nd.box.lo for nd in tree.nodes]), hi=np.array([nd.box.hi for nd in tree.nodes]),
        row_start=np.array([nd.row_start for nd in tree.nodes], np.int64),
        row_stop=np.array([nd.row_stop for nd in tree.nodes], np.int64),
        col_start=np.array([nd.col_start for nd in tree.nodes], np.int64),
        col_stop=np.array([nd.col_stop for nd in tree.nodes], np.int64),
        perm_row=tree.perm_row, perm_col=tree.perm_col)


def flat_dict(d, n, dtype):
    ptr = np.zeros(n + 1, np.int64)
    vals = []
    for i in range(n):
        v = np.asarray(d.get(i, np.zeros(0, dtype)), dtype)
        ptr[i + 1] = ptr[i] + v.size
        vals.append(v.ravel())
    return ptr, (np.concatenate(vals) if vals else np.zeros(0, dtype))


def run_case(name, case):
    c = resolve(case)
    X, Y, rng = case_points(c)
    q = rng.standard_normal((Y.shape[0], c["nrhs"]))
    install_extension(c["kernel"], c["rtol"])
    cands = []
    if c.get("store_cand"):
        inner = smash.hss.compr if c["structure"] == "hss" else smash.h2.compr

        def rec(C, ibar, **kw):
            cands.append(np.array(C))
            return inner(C, ibar, **kw)
        smash.hss.compr = rec
        smash.h2.compr = rec
    PX = smash.PointSet(X)
    PY = PX if Y is X else smash.PointSet(Y, role="col")
    t0 = time.time()
    tree = smash.build_tree(PX, None if Y is X else PY, nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
    params = smash.BuildParams(r=c["r"], tau=c["tau"], eps_svd=c["eps_svd"], s=2.0, basis="interp")
    spec = smash.KernelSpec("cauchy", dx=0.0)
    if c["structure"] == "h2":
        M = smash.build_h2(tree, spec, PX, PY, params)
    else:
        M = smash.build_hss(tree, spec, PX, PY, params)
    t_build = time.time() - t0
    z = smash.matvec_nodewise(M, q)
    n = len(tree.nodes)
    out = dict(X=X, Y=Y, q=q, z=z, t_build=t_build)
    try:  # the reference's level-synchronous matvec where the tree is perfect (apply.py:98-165)
        out["z_levelwise"] = smash.matvec_levelwise(M, q)
    except ValueError:
        pass
    out.update(tree_arrays(tree))
    L = np.array(M.pairs_L, np.int64).reshape(-1, 2)
    Lm = np.array(M.pairs_Lm, np.int64).reshape(-1, 2)
    out["L"] = orc._sorted_pairs(L)
    out["Lm"] = orc._sorted_pairs(Lm)
    for side, fac in (("row", M.rowfac), ("col", M.colfac)):
        ptr, sk = flat_dict({i: f.skel for i, f in fac.items()}, n, np.int64)
        out["skel_%s_ptr" % side] = ptr
        out["skel_%s" % side] = sk
        has = np.zeros(n, bool)
        has[list(fac.keys())] = True
        out["has_%s" % side] = has
        if c.get("store_G"):
            gptr, gv = flat_dict({i: f.G for i, f in fac.items()}, n, np.float64)
            pptr, pv = flat_dict({i: f.perm for i, f in fac.items()}, n, np.int64)
            if side == "col" and np.array_equal(gv, out["G_row"]) and np.array_equal(pv, out["fperm_row"]):
                out["col_factors_equal_row"] = True   # X = Y: bitwise identical (probe p12)
                continue
            out["G_%s_ptr" % side], out["G_%s" % side] = gptr, gv
            out["fperm_%s_ptr" % side], out["fperm_%s" % side] = pptr, pv
    if cands:
        # calls run row then column per node, levels L..2 (h2.py:44-53, hss.py:272-299)
        it = iter(cands)
        order = [(side, i) for lev in range(tree.n_levels, 1, -1) for i in tree.level_nodes(lev)
                 for side in ("row", "col")]
        got = {key: next(it) for key in order}
        for side in ("row", "col"):
            mats = [got.get((side, i), np.zeros((0, 0))) for i in range(n)]
            out["cand_%s_cols" % side] = np.array([m_.shape[1] if m_.ndim == 2 else 0 for m_ in mats], np.int64)
            out["cand_%s_ptr" % side], out["cand_%s" % side] = flat_dict(
                {i: m_.ravel() for i, m_ in enumerate(mats)}, n, np.float64)
    if c["structure"] == "hss":
        near = [smash.nearfield_set(tree, i, c["tau"]) for i in range(n)]
        ptr, nv = flat_dict({i: np.array(v, np.int64) for i, v in enumerate(near)}, n, np.int64)
        out["near_ptr"], out["near"] = ptr, nv
    # exact dense product on sampled rows (error vs exact, SURVEY 8(c) rule 5)
    rows = np.sort(np.random.default_rng(99).choice(X.shape[0], min(64, X.shape[0]), replace=False))
    ze = orc.dense_matvec(c["kernel"], X[rows], Y, q, dx=0.0 if c["kernel"] != "exp" else None)
    out["exact_rows"] = rows
    out["z_exact_rows"] = ze
    meta = {k: v for k, v in c.items() if isinstance(v, (int, float, str, bool))}
    out["meta_keys"] = np.array(list(meta.keys()))
    out["meta_vals"] = np.array([str(v) for v in meta.values()])
    # shrink: drop duplicates of the row side when X is Y, store indices as int32
    if Y is X:
        out["Y_is_X"] = True
        del out["Y"]
        assert np.array_equal(out["perm_col"], out["perm_row"])
        del out["perm_col"]
        if np.array_equal(out["skel_col"], out["skel_row"]) and np.array_equal(out["skel_col_ptr"], out["skel_row_ptr"]):
            out["skel_col_equal_row"] = True
            del out["skel_col"], out["skel_col_ptr"]
    for k, v in list(out.items()):
        if isinstance(v, np.ndarray) and v.dtype == np.int64:
            out[k] = v.astype(np.int32)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    rel = np.linalg.norm(z[rows] - ze) / np.linalg.norm(ze)
    print("%-18s N=%-6d nodes=%-6d |L|=%-7d |Lm|=%-6d build %.2fs  relerr_vs_exact %.2e" % (
        name, X.shape[0], n, L.shape[0], Lm.shape[0], t_build, rel))


if __name__ == "__main__":
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        run_case(nm, CASES[nm])
