"""HSS ULV factorisation / solve on the GPU (smash/apply.py:168-354).

Parity: a matrix the reference built and saved (tests/golden/container) is loaded,
factored and solved on the device, and compared with the reference's own
ulv_solve of the same right-hand sides.  The reference's ULV tests
(pkg/tests/test_apply.py:120-195) are ported: residual through the matvec,
agreement with a dense solve, several right-hand sides, reuse, rejection of H2
input, singular blocks reported with the node id.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sg():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1705_05443_b200 as s
    return s


@pytest.fixture(scope="module")
def ref_hss(sg):
    M = sg.load_matrix(os.path.join(GOLDEN, "container", "ref_cauchy_hss.smash"))
    return M, np.load(os.path.join(GOLDEN, "container", "ref_container.npz"))


def test_matches_reference_ulv(sg, ref_hss):
    M, g = ref_hss
    F = sg.ulv_factor(M)
    x = sg.ulv_solve(F, g["q"])
    xr = g["x_hss"]
    assert np.linalg.norm(x - xr) <= 1e-10 * np.linalg.norm(xr)
    X3 = F.solve(g["B3"])
    assert X3.shape == (M.n_col, 3)
    assert np.linalg.norm(X3 - g["X3_hss"]) <= 1e-10 * np.linalg.norm(g["X3_hss"])


def _hss_log_1d(sg, n=4096, nu0=64):
    x = np.random.default_rng(1).random((n, 1))
    tree = sg.build_tree(sg.PointSet(x), nu0=nu0, mode="binary", tau=0.6)
    M = sg.build_hss(tree, sg.KernelSpec("log", dx=0.0), None, None,
                     sg.BuildParams(r=10, tau=0.6, basis="interp", rtol=1e-8, eps_svd=1e-9))
    return M, x


def _hss_cauchy(sg, n=2048):
    X = (np.arange(n) / n)[:, None]
    Y = ((np.arange(n) + 0.5) / n)[:, None]
    tree = sg.build_tree(sg.PointSet(X), sg.PointSet(Y, role="col"), nu0=64, mode="binary", tau=0.6)
    M = sg.build_hss(tree, sg.KernelSpec("cauchy"), None, None,
                     sg.BuildParams(r=16, tau=0.6, basis="interp", rtol=1e-10, eps_svd=1e-11))
    return M, X, Y


@pytest.mark.parametrize("case", ["log", "cauchy"])
def test_solve_then_multiply_recovers_rhs(sg, case):
    M = _hss_log_1d(sg)[0] if case == "log" else _hss_cauchy(sg)[0]
    b = np.random.default_rng(5).random(M.n_row)
    x = sg.ulv_solve(sg.ulv_factor(M), b)
    r = sg.matvec_nodewise(M, x) - b
    assert np.linalg.norm(r) <= 1e-9 * np.linalg.norm(b)


def test_solution_matches_dense_solve(sg):
    from oracle import smash_oracle as orc
    M, X, Y = _hss_cauchy(sg, n=1024)
    A = orc.kernel_block("cauchy", X, Y)
    b = np.random.default_rng(7).random(1024)
    x = sg.ulv_solve(sg.ulv_factor(M), b)
    xd = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xd) <= 1e-7 * np.linalg.norm(xd)


def test_multiple_rhs_and_reuse(sg):
    M, _ = _hss_log_1d(sg, n=2048)
    F = sg.ulv_factor(M)
    B = np.random.default_rng(8).random((2048, 3))
    Xs = sg.ulv_solve(F, B)
    assert Xs.shape == (2048, 3)
    for j in range(3):
        np.testing.assert_allclose(Xs[:, j], sg.ulv_solve(F, B[:, j]), rtol=1e-12, atol=1e-12)
    rng = np.random.default_rng(9)
    for _ in range(3):
        b = rng.random(2048)
        r = sg.matvec_nodewise(M, F.solve(b)) - b
        assert np.linalg.norm(r) <= 1e-9 * np.linalg.norm(b)


def test_single_leaf_tree(sg):
    M, x = _hss_log_1d(sg, n=50, nu0=64)
    b = np.random.default_rng(3).random(50)
    xs = sg.ulv_solve(sg.ulv_factor(M), b)
    from oracle import smash_oracle as orc
    A = orc.kernel_block("log", x, x, 0.0)
    np.testing.assert_allclose(A @ xs, b, rtol=0, atol=1e-10 * np.abs(b).max())


def test_factorization_rejects_h2_input(sg):
    X = np.random.default_rng(2).random((2000, 2))
    tree = sg.build_tree(sg.PointSet(X), nu0=32, mode="2d", tau=0.7)
    M = sg.build_h2(tree, sg.KernelSpec("inv_r", dx=0.0), None, None,
                    sg.BuildParams(r=36, tau=0.7, basis="interp", rtol=1e-8))
    with pytest.raises(ValueError):
        sg.ulv_factor(M)


def test_singular_block_reported_with_node_id(sg):
    # every point twice: duplicate rows make the local elimination singular
    x = np.repeat(np.linspace(0.0, 1.0, 512), 2)[:, None]
    tree = sg.build_tree(sg.PointSet(x), nu0=32, mode="binary", tau=0.6)
    M = sg.build_hss(tree, sg.KernelSpec("log", dx=0.0), None, None,
                     sg.BuildParams(r=10, tau=0.6, basis="interp", rtol=1e-8, eps_svd=1e-9))
    with pytest.raises(np.linalg.LinAlgError, match="node"):
        sg.ulv_factor(M)


def test_adaptive_tree_and_many_rhs(sg):
    """Leaves on several levels (clustered 1-D points) and more right-hand sides than
    warps per CTA (R = 20: shared-memory staging off for the leaf level, on above)."""
    from oracle import smash_oracle as orc
    rng = np.random.default_rng(13)
    x = np.sort(np.concatenate([rng.random(600), 0.31 + 1e-3 * rng.random(900)]))[:, None]
    tree = sg.build_tree(sg.PointSet(x), nu0=64, mode="binary", tau=0.6)
    depths = {tree.nodes[i].level for i in tree.leaves()}
    assert len(depths) > 1
    M = sg.build_hss(tree, sg.KernelSpec("log", dx=0.0), None, None,
                     sg.BuildParams(r=12, tau=0.6, basis="interp", rtol=1e-10, eps_svd=1e-11))
    A = orc.kernel_block("log", x, x, 0.0)
    B = rng.standard_normal((x.shape[0], 20))
    F = sg.ulv_factor(M)
    X = sg.ulv_solve(F, B)
    r = sg.matvec_nodewise(M, X) - B
    assert np.linalg.norm(r) <= 1e-9 * np.linalg.norm(B)
    Xd = np.linalg.solve(A, B)
    assert np.linalg.norm(X - Xd) <= 1e-6 * np.linalg.norm(Xd)
    np.testing.assert_allclose(sg.ulv_solve(F, B[:, 3]), X[:, 3], rtol=1e-11, atol=1e-11 * np.abs(X).max())
