"""Pin the CPU oracle against fixtures produced by the real reference
(tests/golden/make_golden.py).  Runs on CPU only."""

import numpy as np
import pytest

from conftest import golden_names, unflatten
from oracle import smash_oracle as orc

CASES = golden_names()


def oracle_build(g):
    m = g["meta"]
    X, Y = g["X"], g["Y"]
    sym = X is Y
    tree = orc.build_tree(X, None if sym else Y, nu0=m["nu0"], mode=m["mode"])
    return tree, sym


@pytest.mark.parametrize("name", CASES)
def test_tree_matches_reference(golden, name):
    g = golden(name)
    tree, _ = oracle_build(g)
    assert np.array_equal(tree.level, g["level"])
    assert np.array_equal(tree.parent, g["parent"])
    kids = np.concatenate([np.asarray(c, np.int64) for c in tree.children]) if tree.n_nodes else []
    assert np.array_equal(np.asarray(kids, np.int64), g["child_idx"])
    assert np.array_equal(tree.lo, g["lo"]) and np.array_equal(tree.hi, g["hi"])
    for k in ("row_start", "row_stop", "col_start", "col_stop", "perm_row", "perm_col"):
        assert np.array_equal(getattr(tree, k), g[k]), k


@pytest.mark.parametrize("name", CASES)
def test_pairs_match_reference(golden, name):
    g = golden(name)
    tree, _ = oracle_build(g)
    L, Lm = orc.leaf_sets(tree, g["meta"]["tau"], g["meta"]["structure"])
    assert np.array_equal(L, g["L"])
    assert np.array_equal(Lm, g["Lm"])
    if g["meta"]["structure"] == "hss":
        near = orc.nearfield_sets(tree, g["meta"]["tau"])
        for i in range(tree.n_nodes):
            assert near[i] == unflatten(g["near_ptr"], g["near"], i).tolist()


def _build(g):
    m = g["meta"]
    tree, sym = oracle_build(g)
    if m["structure"] == "h2":
        M = orc.build_h2(tree, m["kernel"], m["r"], m["tau"], rtol=m["rtol"],
                         dx=None if m["kernel"] == "exp" else 0.0, symmetric=sym)
    else:
        M = orc.build_hss(tree, m["kernel"], m["r"], m["tau"], m["eps_svd"], rtol=m["rtol"],
                          dx=None if m["kernel"] == "exp" else 0.0)
    return M


_BUILT = {}


def built(golden, name):
    if name not in _BUILT:
        _BUILT[name] = _build(golden(name))
    return _BUILT[name]


@pytest.mark.parametrize("name", CASES)
def test_skeletons_match_reference(golden, name):
    g = golden(name)
    M = built(golden, name)
    n = M.tree.n_nodes
    for side, fac in (("row", M.rowfac), ("col", M.colfac)):
        has = g["has_%s" % side]
        for i in range(n):
            if not has[i]:
                assert i not in fac
                continue
            ref = unflatten(g["skel_%s_ptr" % side], g["skel_%s" % side], i)
            assert np.array_equal(fac[i].skel, ref), (side, i)


@pytest.mark.parametrize("name", CASES)
def test_transfer_matrices_match_reference(golden, name):
    g = golden(name)
    if "G_row" not in g:
        pytest.skip("fixture stores no G (size)")
    M = built(golden, name)
    sides = [("row", M.rowfac)]
    if "G_col" in g:
        sides.append(("col", M.colfac))
    for side, fac in sides:
        for i in fac:
            G = unflatten(g["G_%s_ptr" % side], g["G_%s" % side], i)
            perm = unflatten(g["fperm_%s_ptr" % side], g["fperm_%s" % side], i)
            assert np.array_equal(perm[:fac[i].rank], fac[i].perm[:fac[i].rank])
            # identical LAPACK calls -> identical G (bitwise on the same host)
            np.testing.assert_allclose(fac[i].G.ravel(), G, rtol=0, atol=1e-12 * max(1.0, np.abs(G).max(initial=0)))


@pytest.mark.parametrize("name", CASES)
def test_matvec_matches_reference(golden, name):
    g = golden(name)
    M = built(golden, name)
    z = orc.matvec(M, g["q"])
    ref = g["z"]
    for c in range(ref.shape[1]):
        assert np.linalg.norm(z[:, c] - ref[:, c]) <= 1e-10 * np.linalg.norm(ref[:, c])


@pytest.mark.parametrize("name", [n for n in CASES if n in ("cfg2_4k", "cfg3_8k", "cfg5_16k", "clustered2d",
                                                          "uniform3d_small", "cfg1_full", "cfg4_2k")])
def test_parity_helpers_rebuild_reference_inputs(golden, name):
    """tests/parity.py rebuilds the reference's compr input of every node (H^2: the
    padded-box basis over the reference's ibar; HSS: the recorded [U_hat, S]); the
    reference's own factor must interpolate it (C ~= X C[skel]) -- this pins the
    helper the GPU G test (rule 3, clause 2) relies on."""
    import parity
    g = golden(name)
    for side in ("row", "col"):
        for i in np.nonzero(g["has_%s" % side])[0][:200]:
            C = parity.ref_candidate(g, side, int(i))
            pr, Gr = parity.ref_factor(g, side, int(i))
            k = unflatten(g["skel_%s_ptr" % side], g["skel_%s" % side], int(i)).size
            if C is None:
                assert k == 0
                continue
            assert C.shape[0] == pr.size
            assert np.array_equal(parity.ref_ibar(g, side, int(i))[pr[:k]],
                                  unflatten(g["skel_%s_ptr" % side], g["skel_%s" % side], int(i)))
            X = parity.expand(pr, Gr, k)
            res = np.linalg.norm(C - X @ C[pr[:k]]) / np.linalg.norm(C)
            assert res <= 1e-5, (side, i, res)
            ok, *_ = parity.rule3(X, X, C, pr[:k])
            assert ok
