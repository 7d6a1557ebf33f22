"""Full-size golden digests of the BASELINE configs from the REAL reference
(development container only; minutes to ~1 h per config, single-threaded).

Runs /root/reference/pkg/src/smash (imported read-only, never copied) with the
SURVEY.md 8(c) extension of make_golden.py on BASELINE configs 2-5 at their
full N (config 1 is already stored in full as cfg1_full.npz) and stores what a
GPU build of the same seeded inputs must reproduce, in a form small enough to
commit:

  * tree arrays: one blake2b-64 digest per array (level, parent, children,
    boxes, ranges, perms) plus node / level counts;
  * pair lists L / L-minus (sorted) and HSS nearfield sets: digests + counts;
  * ordered skeletons: per node and side the rank and a blake2b-64 digest of the
    skeleton labels (int64 LE), so a mismatch is located to the node;
  * transfer matrices: perm, ibar and G of a seeded sample of nodes (bounded
    total size), for SURVEY 8(c) rule 3 (the test rebuilds C = interp_basis on
    the GPU-independent oracle from ibar and the tree boxes);
  * the matvec: z at 1024 seeded rows, the column norms of the full z and the
    projections W^T z with W = default_rng(7).standard_normal((N, 4));
  * the exact dense product at 256 of those rows (SURVEY 8(c) rule 5).

Usage:  python tests/golden/make_golden_full.py cfg2 [cfg3 cfg4 cfg5]
Writes tests/golden/full/<cfg>_full.npz.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as mg  # noqa: E402  (installs the reference import path)
from make_golden import smash, orc  # noqa: E402

OUT = os.environ.get("SMASH_FULL_OUT", os.path.join(HERE, "full"))

NRHS = {2: 16, 3: 1, 4: 8, 5: 16}
G_BUDGET = 100_000     # sampled G (+ HSS candidate) entries per side
N_ZROWS = 1024
N_EXACT = 256


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype.kind in "iu":
        a = a.astype("<i8")
    else:
        a = a.astype("<f8")
    return hashlib.blake2b(a.tobytes(), digest_size=8).hexdigest()


def node_digests(fac: dict, n: int):
    rank = np.full(n, -1, np.int32)
    dig = np.zeros(n, np.uint64)
    for i, f in fac.items():
        rank[i] = f.skel.size
        dig[i] = int(digest(np.asarray(f.skel, np.int64)), 16)
    return rank, dig


def sample_nodes(fac: dict, rng, extra=None):
    ids = np.array(sorted(fac), np.int64)
    rng.shuffle(ids)
    out, total = [], 0
    for i in ids:
        g = fac[int(i)].G.size + (extra(int(i)) if extra else 0)
        if total + g > G_BUDGET:
            continue
        out.append(int(i))
        total += g
        if len(out) >= 400:
            break
    return sorted(out)


def _ibar_of(M, tree, side, i):
    nd = tree.nodes[i]
    if not nd.children:
        a, b = (nd.row_start, nd.row_stop) if side == "row" else (nd.col_start, nd.col_stop)
        return np.arange(a, b, dtype=np.int64)
    sk = M.skel_row if side == "row" else M.skel_col
    return np.concatenate([np.asarray(sk[c], np.int64) for c in nd.children])


def run(cfg: int):
    base = orc.CONFIGS[cfg]
    c = dict(base)
    X, Y, rng = orc.make_config_points(cfg, N=int(os.environ["SMASH_FULL_N"]) if os.environ.get("SMASH_FULL_N") else None)
    N = X.shape[0]
    nrhs = NRHS[cfg]
    q = rng.standard_normal((Y.shape[0], nrhs))
    mg.install_extension(c["kernel"], c["rtol"])
    cands = []
    if c["structure"] == "hss":
        # record the candidate [U_hat, S] of every compr call (row then column per
        # node, levels L..2, hss.py:272-299); gesdd's S is not recomputable off-host
        inner = smash.hss.compr

        def rec(C, ibar, **kw):
            cands.append(np.array(C))
            return inner(C, ibar, **kw)
        smash.hss.compr = rec
    PX = smash.PointSet(X)
    PY = PX if Y is X else smash.PointSet(Y, role="col")
    t0 = time.time()
    tree = smash.build_tree(PX, None if Y is X else PY, nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
    t_tree = time.time() - t0
    params = smash.BuildParams(r=c["r"], tau=c["tau"], eps_svd=c["eps_svd"], s=2.0, basis="interp")
    spec = smash.KernelSpec("cauchy", dx=0.0)
    t0 = time.time()
    build = smash.build_h2 if c["structure"] == "h2" else smash.build_hss
    M = build(tree, spec, PX, PY, params, use_cache=False)
    t_build = time.time() - t0
    print("cfg%d tree %.1fs build %.1fs" % (cfg, t_tree, t_build), flush=True)
    n = len(tree.nodes)
    out = dict(N=N, nrhs=nrhs, n_nodes=n, n_levels=tree.n_levels, t_tree=t_tree, t_build=t_build,
               seed=cfg)
    T = mg.tree_arrays(tree)
    for k, v in T.items():
        out["tree_" + k] = digest(v)
    L = orc._sorted_pairs(np.array(M.pairs_L, np.int64).reshape(-1, 2))
    Lm = orc._sorted_pairs(np.array(M.pairs_Lm, np.int64).reshape(-1, 2))
    out.update(n_L=L.shape[0], n_Lm=Lm.shape[0], L=digest(L), Lm=digest(Lm))
    if c["structure"] == "hss":
        near = [np.asarray(smash.nearfield_set(tree, i, c["tau"]), np.int64) for i in range(n)]
        ptr = np.zeros(n + 1, np.int64)
        ptr[1:] = np.cumsum([v.size for v in near])
        out["near_ptr"] = digest(ptr)
        out["near"] = digest(np.concatenate(near))
    cand_of = {}
    if cands:
        it = iter(cands)
        for lev in range(tree.n_levels, 1, -1):
            for i in tree.level_nodes(lev):
                cand_of[("row", i)] = next(it)
                cand_of[("col", i)] = next(it)
        del cands[:]
    srng = np.random.default_rng(1234)
    same = Y is X and sorted(M.rowfac) == sorted(M.colfac) and all(
        np.array_equal(M.rowfac[i].perm, M.colfac[i].perm) and np.array_equal(M.rowfac[i].G, M.colfac[i].G)
        for i in M.rowfac)
    out["col_equals_row"] = same   # X = Y: the reference's column factors are bitwise the row factors
    for side, fac in (("row", M.rowfac), ("col", M.colfac)):
        rank, dig = node_digests(fac, n)
        out["rank_" + side], out["skdig_" + side] = rank, dig
        if same and side == "col":
            continue
        ids = sample_nodes(fac, srng, (lambda i, s=side: cand_of[(s, i)].size) if cand_of else None)
        out["gs_%s_nodes" % side] = np.array(ids, np.int32)
        for key, fn in (("perm", lambda i: fac[i].perm), ("G", lambda i: fac[i].G.ravel()),
                        ("ibar", lambda i: _ibar_of(M, tree, side, i))):
            parts = [np.asarray(fn(i)) for i in ids]
            ptr = np.zeros(len(ids) + 1, np.int64)
            ptr[1:] = np.cumsum([p.size for p in parts])
            out["gs_%s_%s_ptr" % (side, key)] = ptr
            vals = np.concatenate(parts) if parts else np.zeros(0)
            out["gs_%s_%s" % (side, key)] = vals.astype(np.float64 if key == "G" else np.int32)
        if cand_of:
            parts = [cand_of[(side, i)] for i in ids]
            out["gs_%s_cand_cols" % side] = np.array([p.shape[1] for p in parts], np.int32)
            ptr = np.zeros(len(ids) + 1, np.int64)
            ptr[1:] = np.cumsum([p.size for p in parts])
            out["gs_%s_cand_ptr" % side] = ptr
            out["gs_%s_cand" % side] = np.concatenate([p.ravel() for p in parts])
    t0 = time.time()
    z = smash.matvec_nodewise(M, q)
    t_mv = time.time() - t0
    print("cfg%d matvec %.1fs" % (cfg, t_mv), flush=True)
    zr = np.sort(np.random.default_rng(99).choice(N, N_ZROWS, replace=False))
    out["z_rows"] = zr.astype(np.int32)
    out["z_at_rows"] = z[zr]
    out["z_colnorm"] = np.linalg.norm(z, axis=0)
    W = np.random.default_rng(7).standard_normal((N, 4))
    out["z_proj"] = W.T @ z
    out["t_matvec"] = t_mv
    er = zr[:: N_ZROWS // N_EXACT]
    dx = None if c["kernel"] == "exp" else 0.0
    out["exact_rows"] = er.astype(np.int32)
    out["z_exact_rows"] = orc.dense_matvec(c["kernel"], X[er], Y, q, dx=dx, chunk=16)
    out["swaps_note"] = "reference srrqr swap counts are not exposed"
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, "cfg%d_full.npz" % cfg), **out)
    rel = np.linalg.norm(z[er] - out["z_exact_rows"]) / np.linalg.norm(out["z_exact_rows"])
    print("cfg%d N=%d nodes=%d |L|=%d |Lm|=%d build %.1fs matvec %.1fs relerr_vs_exact %.2e" % (
        cfg, N, n, L.shape[0], Lm.shape[0], t_build, t_mv, rel), flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:]:
        run(int(a.replace("cfg", "")))
