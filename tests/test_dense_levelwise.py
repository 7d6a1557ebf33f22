"""GPU dense oracle (smash.bench.dense_matvec, bench.py:284-296) and the
level-wise matvec contract (apply.py:83-165), SURVEY.md 8(f) items 2 and 4."""

import numpy as np
import pytest

from conftest import golden_names

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sg():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1705_05443_b200 as sg
    return sg


def _np_dense(kind, X, Y, dx):
    d = X[:, None, :] - Y[None, :, :]
    if kind == "cauchy":
        diff = d[..., 0]
        with np.errstate(divide="ignore"):
            K = 1.0 / diff
        K[diff == 0] = dx
        return K
    r = np.sqrt(np.sum(d * d, axis=-1))
    with np.errstate(divide="ignore"):
        if kind == "log":
            K = np.log(r)
        elif kind == "inv_r":
            K = 1.0 / r
        else:
            return np.exp(-r)
    K[r == 0] = dx
    return K


@pytest.mark.parametrize("kind,dim", [("log", 1), ("log", 2), ("inv_r", 2), ("inv_r", 3),
                                      ("exp", 3), ("exp", 2), ("cauchy", 1)])
@pytest.mark.parametrize("nrhs", [1, 5, 16])
def test_dense_matvec_vs_numpy(sg, kind, dim, nrhs):
    rng = np.random.default_rng(7)
    X = rng.random((700, dim))
    Y = np.vstack([X[:300], rng.random((257, dim))]) if kind != "cauchy" else rng.random((557, 1)) + 0.37
    q = rng.standard_normal((Y.shape[0], nrhs))
    spec = sg.KernelSpec(kind, dx=None if kind == "exp" else 0.0)
    z = sg.dense_matvec(spec, X, Y, q)
    ze = _np_dense(kind, X, Y, spec.dx_value) @ q
    assert z.shape == ze.shape
    assert sg.relative_error(z, ze) <= 1e-13


def test_dense_matvec_shapes(sg):
    spec = sg.KernelSpec("inv_r", dx=0.0)
    X = np.random.default_rng(1).random((50, 2))
    q1 = np.ones(50)
    assert sg.dense_matvec(spec, X, X, q1).shape == (50,)
    with pytest.raises(ValueError):
        sg.dense_matvec(spec, X, X, np.ones(49))


@pytest.mark.parametrize("name", [n for n in golden_names() if n.startswith(("cfg2", "cfg3", "cfg5"))])
def test_dense_oracle_matches_golden_exact_rows(sg, golden, name):
    g = golden(name)
    if "z_exact_rows" not in g:
        pytest.skip("fixture stores no exact rows")
    m = g["meta"]
    spec = sg.KernelSpec(m["kernel"], dx=None if m["kernel"] == "exp" else 0.0)
    rows = g["exact_rows"]
    z = sg.dense_matvec(spec, g["X"][rows], g["Y"], g["q"])
    assert sg.relative_error(z, g["z_exact_rows"]) <= 1e-12


def _build(sg, cfg, N):
    from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points
    c = CONFIGS[cfg]
    X, Y, rng = make_points(cfg, N=N)
    spec, params = build_params(cfg)
    tree = sg.build_tree(sg.PointSet(X), nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
    M = (sg.build_h2 if c["structure"] == "h2" else sg.build_hss)(tree, spec, None, None, params)
    return M, X, spec, rng.standard_normal((X.shape[0], 3))


def test_levelwise_equals_nodewise_on_perfect_tree(sg):
    M, X, spec, q = _build(sg, 2, 1 << 15)  # uniform points: perfect quadtree at this N
    z1 = sg.matvec_nodewise(M, q)
    z2 = sg.matvec_levelwise(M, q)
    assert np.linalg.norm(z1 - z2) <= 1e-14 * np.linalg.norm(z1)  # apply.py / test_apply.py:59-65


def test_levelwise_rejects_adaptive_tree(sg):
    M, X, spec, q = _build(sg, 5, 1 << 14)  # clustered points: leaves on several levels
    with pytest.raises(ValueError):
        sg.matvec_levelwise(M, q)


def test_matvec_error_vs_gpu_dense_full(sg):
    """Whole-vector error against the exact product (not sampled rows) at a size
    the CPU oracle would stream for minutes."""
    M, X, spec, q = _build(sg, 2, 1 << 15)
    z = sg.matvec_nodewise(M, q)
    ze = sg.dense_matvec(spec, X, X, q)
    err = sg.relative_error(z, ze)
    assert err < 1e-5, err  # reference error 1.9e-6 .. 3.2e-6 at cfg-2 parameters
