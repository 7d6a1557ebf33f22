"""GPU parity: the CUDA path (through the C ABI) against the reference-generated
golden fixtures and the CPU oracle.

Bars (SURVEY.md 8(c) parity rules): tree arrays, pair sets, nearfield sets and
ordered skeletons bit-exact; matvec within 1e-10 relative per RHS column; the
error against the exact product no worse than 1.1x the reference's + 1e-12.
"""

import numpy as np
import pytest

import parity
from conftest import golden_names, unflatten

pytestmark = pytest.mark.gpu

CASES = golden_names()


@pytest.fixture(scope="module")
def smash_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1705_05443_b200 as sg
    return sg


_TREES = {}
_MATS = {}


def gpu_tree(sg, golden, name):
    if name not in _TREES:
        g = golden(name)
        m = g["meta"]
        X = sg.PointSet(g["X"])
        Y = None if g["Y"] is g["X"] else sg.PointSet(g["Y"], role="col")
        _TREES[name] = sg.build_tree(X, Y, nu0=m["nu0"], mode=m["mode"], tau=m["tau"])
    return _TREES[name]


def gpu_matrix(sg, golden, name):
    if name not in _MATS:
        g = golden(name)
        m = g["meta"]
        tree = gpu_tree(sg, golden, name)
        spec = sg.KernelSpec(m["kernel"], dx=None if m["kernel"] == "exp" else 0.0)
        params = sg.BuildParams(r=m["r"], tau=m["tau"], eps_svd=m["eps_svd"], s=2.0, basis="interp",
                                rtol=m["rtol"])
        build = sg.build_h2 if m["structure"] == "h2" else sg.build_hss
        _MATS[name] = build(tree, spec, None, None, params)
    return _MATS[name]


@pytest.mark.parametrize("name", CASES)
def test_tree_bitexact(smash_gpu, golden, name):
    g = golden(name)
    A = gpu_tree(smash_gpu, golden, name).arrays()
    for k in ("level", "parent", "child_ptr", "child_idx", "row_start", "row_stop", "col_start",
              "col_stop", "perm_row", "perm_col"):
        assert np.array_equal(A[k], g[k]), k
    assert np.array_equal(A["lo"], g["lo"]) and np.array_equal(A["hi"], g["hi"])
    assert np.array_equal(A["points_row"], g["X"][g["perm_row"]])


@pytest.mark.parametrize("name", CASES)
def test_pair_sets_bitexact(smash_gpu, golden, name):
    g = golden(name)
    m = g["meta"]
    tree = gpu_tree(smash_gpu, golden, name)
    L, Lm = smash_gpu.leaf_sets(tree, m["tau"], m["structure"])
    assert np.array_equal(np.array(L, np.int64).reshape(-1, 2), g["L"])
    assert np.array_equal(np.array(Lm, np.int64).reshape(-1, 2), g["Lm"])
    if m["structure"] == "hss":
        for i in range(len(g["level"])):
            assert smash_gpu.nearfield_set(tree, i, m["tau"]) == unflatten(g["near_ptr"], g["near"], i).tolist()


def _h2_or_skip(golden, name):
    """Both structures are built on the GPU (HSS adds the batched SVD kernel)."""
    return None


@pytest.mark.parametrize("name", CASES)
def test_skeletons_bitexact(smash_gpu, golden, name):
    _h2_or_skip(golden, name)
    g = golden(name)
    M = gpu_matrix(smash_gpu, golden, name)
    mism, total = [], 0
    for side, fac in (("row", M.rowfac), ("col", M.colfac)):
        has = g["has_%s" % side]
        assert sorted(fac) == [int(i) for i in np.nonzero(has)[0]]
        for i in fac:
            ref = unflatten(g["skel_%s_ptr" % side], g["skel_%s" % side], i)
            total += 1
            if not np.array_equal(fac[i].skel, ref):
                mism.append((side, i, fac[i].skel.size, ref.size))
    m = g["meta"]
    print("%s: %d factors, %d ordered-skeleton mismatches %s" % (name, total, len(mism), mism[:6]))
    if m["structure"] == "hss" and m["kernel"] == "cauchy":
        # The HSS candidate [U_hat, S] carries the kept left singular vectors of the
        # nearfield block (hss.py:286-287) unscaled; those near the eps_svd cut are fixed
        # only to ~eps*sigma_1/gap by ANY fp64 SVD, so near-tied pivots follow the SVD's
        # rounding.  The GPU sRRQR is bit-exact on the reference's own candidates
        # (test_hss_compr_on_reference_candidates); here ranks must agree everywhere and
        # the order mismatches stay within those of the reference's own algorithm run
        # with another backward-stable SVD (tests/golden/hss_svd_sensitivity.py), +10% + 2.
        sens = parity.hss_sensitivity(name)
        assert all(kg == kr for _, _, kg, kr in mism), mism[:10]
        bar = int(1.1 * sens["order_mismatch"]) + 2 if sens else 0
        assert len(mism) <= bar, (len(mism), bar, mism[:10])
    else:
        assert not mism, "skeleton mismatches (side, node, k_gpu, k_ref): %s" % mism[:10]


@pytest.mark.parametrize("name", CASES)
def test_transfer_G(smash_gpu, golden, name):
    """Transfer matrices by SURVEY 8(c) rule 3 (tests/parity.py) on every fixture that
    stores the reference's G, H^2 and HSS.  Nodes whose ordered skeleton differs from
    the reference (HSS-Cauchy only, see test_skeletons_bitexact) cannot be compared by
    label; for them the GPU factor must interpolate the reference's own compr input
    within 10x of the worse of the reference's own factor and the reference algorithm run
    with another backward-stable SVD (tests/golden/hss_svd_sensitivity.py)."""
    g = golden(name)
    if "G_row" not in g:
        pytest.skip("fixture stores no G (cfg2_32k: the full-size cfg2 digest samples G)")
    M = gpu_matrix(smash_gpu, golden, name)
    bad, clause2, clause3, skipped, e1max = [], 0, 0, 0, 0.0
    for side, fac in (("row", M.rowfac), ("col", M.colfac)):
        for i, f in fac.items():
            pr, Gr = parity.ref_factor(g, side, i)
            k = f.rank
            Xr = parity.expand(pr, Gr, k)
            C = parity.ref_candidate(g, side, i)
            ib_r, ib_g = parity.ref_ibar(g, side, i), parity.gpu_ibar(M, side, i)
            # rows by label (G row order follows ibar), columns by the ordered skeleton
            Xg = parity.align_rows(f.expand(), ib_g, ib_r)
            ref_skel = unflatten(g["skel_%s_ptr" % side], g["skel_%s" % side], i)
            if Xg is None or not np.array_equal(f.skel, ref_skel):
                assert g["meta"]["structure"] == "hss", (side, i)
                skipped += 1
                if C is not None and Xg is not None:
                    C_g = parity.align_rows(C, ib_r, ib_g)  # reference candidate in GPU ibar order
                    sk_g = f.perm[:k]
                    ref_res = np.linalg.norm(C - Xr @ C[pr[:k]]) / np.linalg.norm(C)
                    gpu_res = np.linalg.norm(C_g - f.expand() @ C_g[sk_g]) / np.linalg.norm(C)
                    sens = parity.hss_sensitivity(name) or {}
                    bar = max(10 * ref_res + 1e-13, 10 * sens.get("mismatched_residual_max", 0.0))
                    assert gpu_res <= bar, (side, i, gpu_res, ref_res, bar)
                continue
            ok, clause, e1, e2, kappa = parity.rule3(Xg, Xr, C, pr[:k])
            clause2 += clause == 2
            if not ok and g["meta"]["structure"] == "hss" and parity.hss_g_ok(name, e1, kappa):
                ok, clause = True, 3
                clause3 += 1
                e1max = max(e1max, e1)
            if not ok:
                bad.append((side, i, e1, e2, kappa))
    assert not bad, "rule 3 failures (side, node, e1, e2, kappa): %s" % bad[:10]
    print("%s: %d nodes by clause 2, %d by the HSS SVD-sensitivity clause (max e1 %.2e), "
          "%d label-mismatched nodes checked by residual" % (name, clause2, clause3, e1max, skipped))


@pytest.mark.parametrize("name", ["cfg4_2k", "pair1d_hss", "cfg1_full"])
def test_hss_compr_on_reference_candidates(smash_gpu, golden, name):
    """The GPU sRRQR on the reference's OWN compr inputs [U_hat, S] (S from the
    reference's gesdd, recorded by make_golden.py): ordered skeletons bit-exact and G by
    rule 3 on every node.  This isolates the sRRQR from the SVD -- any HSS skeleton
    difference of the full GPU build comes from the batched SVD's rounding."""
    g = golden(name)
    m = g["meta"]
    n = len(g["level"])
    checked = 0
    for side in ("row", "col"):
        for i in range(n):
            if not g["has_%s" % side][i]:
                continue
            C = parity.ref_candidate(g, side, i)
            ref = unflatten(g["skel_%s_ptr" % side], g["skel_%s" % side], i)
            ibar = parity.ref_ibar(g, side, i)
            if C is None:
                assert ref.size == 0
                continue
            f = smash_gpu.compr(C, ibar, s=2.0, rtol=m["rtol"])
            assert np.array_equal(f.skel, ref), (side, i, f.skel[:8], ref[:8])
            pr, Gr = parity.ref_factor(g, side, i)
            ok, clause, e1, e2, kappa = parity.rule3(f.expand(), parity.expand(pr, Gr, f.rank), C, pr[:f.rank])
            assert ok, (side, i, e1, e2, kappa)
            checked += 1
    assert checked > 0


@pytest.mark.parametrize("name", CASES)
def test_matvec_vs_reference(smash_gpu, golden, name):
    _h2_or_skip(golden, name)
    g = golden(name)
    M = gpu_matrix(smash_gpu, golden, name)
    z = smash_gpu.matvec_nodewise(M, g["q"])
    ref = g["z"]
    for c in range(ref.shape[1]):
        rel = np.linalg.norm(z[:, c] - ref[:, c]) / np.linalg.norm(ref[:, c])
        assert rel <= 1e-10, (c, rel)
    # vs exact on the sampled rows: no worse than the reference
    rows = g["exact_rows"]
    ze = g["z_exact_rows"]
    e_gpu = np.linalg.norm(z[rows] - ze) / np.linalg.norm(ze)
    e_ref = np.linalg.norm(ref[rows] - ze) / np.linalg.norm(ze)
    assert e_gpu <= 1.1 * e_ref + 1e-12


@pytest.mark.parametrize("nrhs", [1, 3, 8, 16, 21])
@pytest.mark.parametrize("name", ["cfg2_4k", "cfg5_16k", "uniform3d_small"])
def test_matvec_multi_rhs_vs_oracle(smash_gpu, golden, name, nrhs):
    """Every nrhs chunk path (DFMA for < 8 columns, DMMA for 8/16) against the
    oracle matvec on the same (reference-identical) factors."""
    from oracle import smash_oracle as orc
    g = golden(name)
    m = g["meta"]
    M = gpu_matrix(smash_gpu, golden, name)
    ot = orc.build_tree(g["X"], None, nu0=m["nu0"], mode=m["mode"])
    OM = orc.build_h2(ot, m["kernel"], m["r"], m["tau"], rtol=m["rtol"],
                      dx=None if m["kernel"] == "exp" else 0.0, symmetric=True)
    q = np.random.default_rng(nrhs).standard_normal((g["X"].shape[0], nrhs))
    z = smash_gpu.matvec_nodewise(M, q)
    zr = orc.matvec(OM, q)
    for c in range(nrhs):
        rel = np.linalg.norm(z[:, c] - zr[:, c]) / np.linalg.norm(zr[:, c])
        assert rel <= 1e-10, (c, rel)


@pytest.mark.parametrize("overlap", [False, True])
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name", ["cfg2_32k", "cfg5_16k", "pair1d_hss"])
def test_sharded_stages_single_process(smash_gpu, golden, name, world, overlap):
    """The multi-GPU stages (shard.py) emulated in one process on one GPU: one matrix per
    virtual rank, the halo exchange done by copying exactly the planned coefficient rows
    between the ranks' buffers (no inter-rank waiting on one device), stage 2 or the
    stage 3 (nearfield) + stage 4 split; the owned rows summed must equal the product."""
    import torch
    from paper_1705_05443_b200 import _lib
    from paper_1705_05443_b200.shard import _DevBuf, frontier_fixup, matvec_plan, set_partition
    import ctypes
    g = golden(name)
    mats = []
    for r in range(world):
        _MATS.pop(name, None)
        _TREES.pop(name, None)
        mats.append(gpu_matrix(smash_gpu, golden, name))
    plan = matvec_plan(mats[0], world)
    lib = _lib.load()
    nrhs = 8
    Q = torch.from_numpy(np.random.default_rng(7).standard_normal((g["Y"].shape[0], nrhs))).cuda()
    zs = []
    for r, M in enumerate(mats):
        set_partition(M, plan, r)
        z = torch.zeros((M.n_row, nrhs), dtype=torch.float64, device="cuda")
        _lib.check(lib.smash_matvec_stage(M._h, 1, _lib.ptr(Q), _lib.ptr(z), nrhs, _lib.stream_ptr()))
        if overlap:
            _lib.check(lib.smash_matvec_stage(M._h, 3, _lib.ptr(Q), _lib.ptr(z), nrhs, _lib.stream_ptr()))
        zs.append(z)
    views = []
    for M in mats:
        p, rows = ctypes.c_void_p(), _lib.c_i64()
        _lib.check(lib.smash_matvec_coeffs(M._h, ctypes.byref(p), ctypes.byref(rows)))
        views.append(torch.as_tensor(_DevBuf(p.value, rows.value * nrhs), device="cuda").view(rows.value, nrhs))
    sent = [v.clone() for v in views]  # what each rank holds after stage 1
    for r in range(world):
        for s_ in range(world):
            idx = torch.from_numpy(plan["rows"][s_][r]).cuda()
            if idx.numel():
                views[r].index_copy_(0, idx, sent[s_].index_select(0, idx))
        src, dst = frontier_fixup(plan, r)
        if src.size:
            views[r].index_copy_(0, torch.from_numpy(dst).cuda(), views[r].index_select(0, torch.from_numpy(src).cuda()))
    for M, z in zip(mats, zs):
        _lib.check(lib.smash_matvec_stage(M._h, 4 if overlap else 2, _lib.ptr(Q), _lib.ptr(z), nrhs,
                                          _lib.stream_ptr()))
    zsum = sum(zs).cpu().numpy()
    zref = smash_gpu.matvec_nodewise(mats[0], Q.cpu().numpy())
    rel = np.linalg.norm(zsum - zref) / np.linalg.norm(zref)
    assert rel <= 1e-12, rel
    _MATS.pop(name, None)
    _TREES.pop(name, None)


@pytest.mark.parametrize("mode", ["2d", "binary"])
def test_tree_bitexact_sub_2e21_cluster(smash_gpu, mode):
    """A 3-D cluster 1e-9 wide needs bisection digits past the first 21 per axis (the
    high key word), so the device tree sort must order by the low key word too; the
    tree must still equal the oracle's (the reference recursion, cluster.py:263-353)."""
    from oracle import smash_oracle as orc
    rng = np.random.default_rng(21)
    X = np.vstack([rng.random((300, 3)), 0.37 + 1e-9 * rng.random((200, 3))])
    ot = orc.build_tree(X, nu0=16, mode=mode)
    tree = smash_gpu.build_tree(smash_gpu.PointSet(X), nu0=16, mode=mode)
    A = tree.arrays()
    assert np.array_equal(A["perm_row"], ot.perm_row)
    assert np.array_equal(A["level"], ot.level) and np.array_equal(A["parent"], ot.parent)
    assert np.array_equal(A["lo"], ot.lo) and np.array_equal(A["hi"], ot.hi)
    assert np.array_equal(A["row_start"], ot.row_start) and np.array_equal(A["row_stop"], ot.row_stop)
