"""Level-synchronous matvec (smash/apply.py:83-165).

GPU (-m gpu), through the C ABI smash_matvec_levelwise:
  * on every perfect-tree fixture: <= 1e-14 against the node-wise device matvec
    (the reference's own contract, pkg/tests/test_apply.py:59-65) and <= 1e-10 per
    column against the REAL reference's matvec_levelwise output;
  * on the reference's OWN factors (imported through smash_matrix_import): <= 1e-13
    against the reference's matvec_levelwise (only summation order differs);
  * every nrhs chunk path; adaptive trees rejected with ValueError (apply.py:83-95).
CPU: the oracle's level-wise restatement reproduces the reference's output.
"""

import ctypes

import numpy as np
import pytest

from conftest import golden_names, load_golden

def _perfect():
    import os
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    return [n for n in golden_names() if "z_levelwise" in np.load(os.path.join(here, n + ".npz")).files]


PERFECT = _perfect()


# ---------------------------------------------------------------- CPU: oracle pin

@pytest.mark.parametrize("name", PERFECT)
def test_oracle_levelwise_matches_reference(name):
    from oracle import smash_oracle as orc
    g = load_golden(name)
    m = g["meta"]
    X, Y = g["X"], g["Y"]
    tree = orc.build_tree(X, None if Y is X else Y, nu0=m["nu0"], mode=m["mode"])
    if m["structure"] == "h2":
        M = orc.build_h2(tree, m["kernel"], m["r"], m["tau"], rtol=m["rtol"],
                         dx=None if m["kernel"] == "exp" else 0.0, symmetric=Y is X)
    else:
        M = orc.build_hss(tree, m["kernel"], m["r"], m["tau"], m["eps_svd"], rtol=m["rtol"],
                          dx=None if m["kernel"] == "exp" else 0.0)
    z = orc.matvec_levelwise(M, g["q"])
    ref = g["z_levelwise"]
    for c in range(ref.shape[1]):
        assert np.linalg.norm(z[:, c] - ref[:, c]) <= 1e-14 * np.linalg.norm(ref[:, c])


def test_oracle_levelwise_rejects_adaptive_tree():
    from oracle import smash_oracle as orc
    g = load_golden("cfg5_16k")
    m = g["meta"]
    tree = orc.build_tree(g["X"], nu0=m["nu0"], mode=m["mode"])
    M = orc.build_h2(tree, m["kernel"], m["r"], m["tau"], rtol=m["rtol"], dx=0.0, symmetric=True)
    with pytest.raises(ValueError):
        orc.matvec_levelwise(M, g["q"])


# ---------------------------------------------------------------- GPU

@pytest.fixture(scope="module")
def sg():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1705_05443_b200 as s
    return s


def _tree_and_params(sg, g):
    m = g["meta"]
    X = sg.PointSet(g["X"])
    Y = None if g["Y"] is g["X"] else sg.PointSet(g["Y"], role="col")
    tree = sg.build_tree(X, Y, nu0=m["nu0"], mode=m["mode"], tau=m["tau"])
    spec = sg.KernelSpec(m["kernel"], dx=None if m["kernel"] == "exp" else 0.0)
    params = sg.BuildParams(r=m["r"], tau=m["tau"], eps_svd=m["eps_svd"], s=2.0, basis="interp",
                            rtol=m["rtol"])
    return tree, spec, params


def _import_reference(sg, tree, spec, params, g):
    """A device matrix holding the reference's own factors (perm, skel, G per node)."""
    from paper_1705_05443_b200 import _lib
    from paper_1705_05443_b200.h2 import H2Matrix
    from paper_1705_05443_b200.hss import HssMatrix
    m = g["meta"]
    sides = []
    for side in ("row", "col"):
        src = side if ("G_%s" % side) in g else "row"
        sp = g["skel_%s_ptr" % side].astype(np.int64)
        sides.append([np.ascontiguousarray(np.diff(sp), np.int64),
                      np.ascontiguousarray(g["fperm_%s_ptr" % src], np.int64),
                      np.ascontiguousarray(g["fperm_%s" % src], np.int64),
                      np.ascontiguousarray(sp, np.int64),
                      np.ascontiguousarray(g["skel_%s" % side], np.int64),
                      np.ascontiguousarray(g["G_%s_ptr" % src], np.int64),
                      np.ascontiguousarray(g["G_%s" % src], np.float64)])
    arr_t = ctypes.c_void_p * 2
    cols = [arr_t(*[s[j].ctypes.data for s in sides]) for j in range(7)]
    p = _lib.BuildParamsC(structure=_lib.STRUCT[m["structure"]], kernel=spec.code,
                          dx=spec.dx_value if spec.dx_value == spec.dx_value else 0.0,
                          r=int(params.r), tau=float(params.tau), s=float(params.s),
                          rtol=float(params.rtol), eps_svd=float(params.eps_svd))
    h = ctypes.c_void_p()
    _lib.check(_lib.load().smash_matrix_import(tree._h, ctypes.byref(p), 2, *cols, _lib.stream_ptr(),
                                               ctypes.byref(h)))
    cls = HssMatrix if m["structure"] == "hss" else H2Matrix
    return cls(tree, params, spec, h)


@pytest.mark.gpu
@pytest.mark.parametrize("name", PERFECT)
def test_levelwise_gpu(sg, name):
    g = load_golden(name)
    tree, spec, params = _tree_and_params(sg, g)
    build = sg.build_h2 if g["meta"]["structure"] == "h2" else sg.build_hss
    M = build(tree, spec, None, None, params)
    z1 = sg.matvec_nodewise(M, g["q"])
    z2 = sg.matvec_levelwise(M, g["q"])
    assert np.linalg.norm(z1 - z2) <= 1e-14 * np.linalg.norm(z1)  # test_apply.py:59-65
    ref = g["z_levelwise"]
    for c in range(ref.shape[1]):
        assert np.linalg.norm(z2[:, c] - ref[:, c]) <= 1e-10 * np.linalg.norm(ref[:, c])


@pytest.mark.gpu
@pytest.mark.parametrize("name", [n for n in PERFECT if n.startswith("cfg4") or n == "tiny_single_leaf"])
def test_levelwise_gpu_on_reference_factors(sg, name):
    g = load_golden(name)
    tree, spec, params = _tree_and_params(sg, g)
    M = _import_reference(sg, tree, spec, params, g)
    z = sg.matvec_levelwise(M, g["q"])
    ref = g["z_levelwise"]
    for c in range(ref.shape[1]):
        assert np.linalg.norm(z[:, c] - ref[:, c]) <= 1e-13 * np.linalg.norm(ref[:, c])
    zn = sg.matvec_nodewise(M, g["q"])
    assert np.linalg.norm(zn - g["z"]) <= 1e-13 * np.linalg.norm(g["z"])


@pytest.mark.gpu
@pytest.mark.parametrize("nrhs", [1, 3, 8, 16, 21])
def test_levelwise_gpu_chunks(sg, nrhs):
    g = load_golden("cfg2_32k")
    tree, spec, params = _tree_and_params(sg, g)
    M = sg.build_h2(tree, spec, None, None, params)
    q = np.random.default_rng(nrhs).standard_normal((g["X"].shape[0], nrhs))
    z1 = sg.matvec_nodewise(M, q)
    z2 = sg.matvec_levelwise(M, q)
    for c in range(nrhs):
        assert np.linalg.norm(z1[:, c] - z2[:, c]) <= 1e-14 * np.linalg.norm(z1[:, c])
    z3 = sg.matvec_levelwise(M, q[:, 0])
    assert z3.shape == (g["X"].shape[0],)


@pytest.mark.gpu
def test_levelwise_gpu_rejects_adaptive_tree(sg):
    g = load_golden("cfg5_16k")
    tree, spec, params = _tree_and_params(sg, g)
    M = sg.build_h2(tree, spec, None, None, params)
    with pytest.raises(ValueError):
        sg.matvec_levelwise(M, g["q"])
