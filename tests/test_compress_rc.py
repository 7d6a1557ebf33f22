"""The two compression kernels (K3 + K4) agree bit for bit.

k_compress (csrc/compress.cu: panel in shared or global memory, physical column swaps) and
k_compress_rc (csrc/compress_rc.cuh: thread per column, bottom rows in registers, positions
instead of swaps; wide nodes over thread-block clusters) run the same floating-point
operations in the same order (smash/lowrank.py:163-255 through LAPACK's dlaqp2), so every
exported factor array -- ranks, perm, G, ordered skeletons, swap counts -- must be identical.
The register-column kernel is the default; SMASH_COMPRESS_RC=0 selects k_compress.  The
parity of the default path against the reference is tests/test_gpu_parity.py and
tests/test_fullsize_parity.py.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sg():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1705_05443_b200 as sg
    return sg


def _build(sg, cfg, N, rc):
    from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points
    old = os.environ.get("SMASH_COMPRESS_RC")
    os.environ["SMASH_COMPRESS_RC"] = "1" if rc else "0"
    try:
        c = CONFIGS[cfg]
        X, Y, _ = make_points(cfg, N=N)
        spec, params = build_params(cfg)
        tree = sg.build_tree(sg.PointSet(X), None if Y is X else sg.PointSet(Y, role="col"),
                             nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
        fn = sg.build_h2 if c["structure"] == "h2" else sg.build_hss
        M = fn(tree, spec, None, None, params)
        out = {"%d_%s" % (s, k): np.asarray(v) for s in (0, 1) for k, v in M.export_side(s).items()}
        return out, M.swaps
    finally:
        if old is None:
            os.environ.pop("SMASH_COMPRESS_RC", None)
        else:
            os.environ["SMASH_COMPRESS_RC"] = old


# config 1 / 4: HSS (panel rows r + kept singular vectors); 2 / 5: 2-D H^2 (36 / 64 rows, up to
# 144 / 256 columns); 3: 3-D H^2 (125 rows: the 44- / 48-register-row variants, streamed R11,
# and nodes of up to 1000 columns on clusters of four CTAs)
@pytest.mark.parametrize("cfg,N", [(1, None), (2, 1 << 14), (4, 1 << 13), (5, 1 << 16), (3, 1 << 16)])
def test_register_column_kernel_equals_k_compress(sg, cfg, N):
    a, sa = _build(sg, cfg, N, rc=False)
    b, sb = _build(sg, cfg, N, rc=True)
    assert sa == sb
    assert a.keys() == b.keys()
    for k in a:
        x, y = a[k], b[k]
        assert x.shape == y.shape, k
        if x.dtype.kind == "f":  # compare bit patterns (-0.0 vs 0.0, NaN payloads)
            assert np.array_equal(x.view(np.int64), y.view(np.int64)), k
        else:
            assert np.array_equal(x, y), k


def _build_points(sg, X, cfg, rc):
    from paper_1705_05443_b200.workloads import CONFIGS, build_params
    old = os.environ.get("SMASH_COMPRESS_RC")
    os.environ["SMASH_COMPRESS_RC"] = "1" if rc else "0"
    try:
        c = CONFIGS[cfg]
        spec, params = build_params(cfg)
        tree = sg.build_tree(sg.PointSet(X), nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
        M = sg.build_h2(tree, spec, None, None, params)
        out = {"%d_%s" % (s, k): np.asarray(v) for s in (0, 1) for k, v in M.export_side(s).items()}
        return out, M.swaps
    finally:
        if old is None:
            os.environ.pop("SMASH_COMPRESS_RC", None)
        else:
            os.environ["SMASH_COMPRESS_RC"] = old


@pytest.mark.parametrize("cfg,dim", [(3, 3), (5, 2)])
def test_register_column_kernel_ragged_levels(sg, cfg, dim):
    """Adaptive trees: narrow and wide nodes on the same level (a level launched whole on the
    cluster kernel holds nodes that fill one of its four CTAs only), duplicated points
    (rank-deficient panels: the back substitution and swap loop of the small classes)."""
    rng = np.random.default_rng(100 + cfg)
    n = 20000
    blob = 0.5 + 0.01 * rng.standard_normal((n // 2, dim))
    X = np.vstack([rng.random((n // 2 - 200, dim)), blob, np.repeat(rng.random((20, dim)), 10, axis=0)])
    a, sa = _build_points(sg, X, cfg, rc=False)
    b, sb = _build_points(sg, X, cfg, rc=True)
    assert sa == sb
    for k in a:
        x, y = a[k], b[k]
        assert x.shape == y.shape, k
        if x.dtype.kind == "f":
            assert np.array_equal(x.view(np.int64), y.view(np.int64)), k
        else:
            assert np.array_equal(x, y), k
