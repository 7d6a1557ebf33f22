"""Container save/load (smash/container.py).

CPU: the reference-written golden containers (tests/golden/make_container_golden.py)
parse with this package's reader, and the payload writer round-trips bit-exactly.
GPU: those reference files load into device matrices whose matvec matches the
reference's; GPU-built H2 / HSS matrices survive save -> load bit-exactly.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

REF_FILES = {"hss": os.path.join(GOLDEN, "container", "ref_cauchy_hss.smash"),
             "h2": os.path.join(GOLDEN, "container", "ref_cauchy_h2.smash")}


def _container():
    from paper_1705_05443_b200 import container
    return container


# ------------------------------------------------------------------------------ CPU

@pytest.mark.parametrize("kind", ["hss", "h2"])
def test_reference_container_parses(kind):
    c = _container()
    header, arrays = c._read(REF_FILES[kind])
    assert header["kind"] == kind and header["dtype"] == "f8"
    n = len(header["tree"]["nodes"])
    root = n - 1
    for side in ("rowfac", "colfac"):
        for i in range(n):
            if i == root:
                continue
            perm, G, skel = (arrays["%s.%d.%s" % (side, i, f)] for f in ("perm", "G", "skel"))
            k = skel.size
            assert sorted(perm.tolist()) == list(range(perm.size))
            assert G.shape == (perm.size - k, k)
    assert arrays["perm_row"].dtype == np.int64 and arrays["points_row"].dtype == np.float64


def test_payload_roundtrip_bit_exact(tmp_path):
    c = _container()
    rng = np.random.default_rng(3)
    pl = c._Payload()
    a = rng.standard_normal((7, 3))
    b = rng.integers(-5, 5, 11)
    pl.add("a", a)
    pl.add("b", b)
    path = tmp_path / "x.smash"
    with open(path, "wb") as fh:
        fh.write(c._MAGIC + json.dumps({"arrays": pl.manifest}).encode() + b"\0")
        for ch in pl.chunks:
            fh.write(ch)
    _, arrs = c._read(str(path))
    assert arrs["a"].tobytes() == a.tobytes()
    assert np.array_equal(arrs["b"], b) and arrs["b"].dtype == np.int64


def test_bad_magic_rejected(tmp_path):
    c = _container()
    p = tmp_path / "bad.smash"
    p.write_bytes(b"NOT-SMASH\n{}\0")
    with pytest.raises(ValueError):
        c._read(str(p))


# ------------------------------------------------------------------------------ GPU

@pytest.fixture(scope="module")
def sg():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1705_05443_b200 as s
    return s


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["hss", "h2"])
def test_load_reference_container_matvec(sg, kind):
    """A file the reference wrote runs on the device matvec with the reference's own factors."""
    g = np.load(os.path.join(GOLDEN, "container", "ref_container.npz"))
    M = sg.load_matrix(REF_FILES[kind])
    assert M.kind == kind
    c = _container()
    _, arrays = c._read(REF_FILES[kind])
    for i, f in M.rowfac.items():
        assert np.array_equal(f.skel, arrays["rowfac.%d.skel" % i])
        assert np.array_equal(f.G, arrays["rowfac.%d.G" % i])
    for i, f in M.colfac.items():
        assert np.array_equal(f.perm, arrays["colfac.%d.perm" % i])
    z = sg.matvec_nodewise(M, g["q"])
    zr = g["z_" + kind]
    assert np.linalg.norm(z - zr) <= 1e-12 * np.linalg.norm(zr)


def _h2_2d(sg):
    X = np.random.default_rng(2).random((3000, 2))
    tree = sg.build_tree(sg.PointSet(X), nu0=32, mode="2d", tau=0.7)
    return sg.build_h2(tree, sg.KernelSpec("inv_r", dx=0.0), None, None,
                       sg.BuildParams(r=36, tau=0.7, basis="interp", rtol=1e-8)), X.shape[0]


def _hss_1d(sg):
    x = np.random.default_rng(1).random((2048, 1))
    tree = sg.build_tree(sg.PointSet(x), nu0=64, mode="binary", tau=0.6)
    return sg.build_hss(tree, sg.KernelSpec("log", dx=0.0), None, None,
                        sg.BuildParams(r=10, tau=0.6, basis="interp", rtol=1e-8, eps_svd=1e-9)), 2048


def _hss_cauchy_xy(sg):
    n = 1024
    X = sg.PointSet((np.arange(n) / n)[:, None])
    Y = sg.PointSet(((np.arange(n) + 0.5) / n)[:, None], role="col")
    tree = sg.build_tree(X, Y, nu0=64, mode="binary", tau=0.6)
    return sg.build_hss(tree, sg.KernelSpec("cauchy"), None, None,
                        sg.BuildParams(r=16, tau=0.6, basis="interp", rtol=1e-10, eps_svd=1e-11)), n


@pytest.mark.gpu
@pytest.mark.parametrize("make", [_h2_2d, _hss_1d, _hss_cauchy_xy])
def test_save_load_roundtrip_bit_exact(sg, tmp_path, make):
    M, n = make(sg)
    path = str(tmp_path / "m.smash")
    sg.save_matrix(M, path)
    M2 = sg.load_matrix(path)
    assert type(M2) is type(M)
    for side in (0, 1):
        a, b = M.export_side(side), M2.export_side(side)
        for k in ("has", "rank", "perm_ptr", "perm", "skel_ptr", "skel", "g_ptr", "G"):
            assert a[k].tobytes() == b[k].tobytes(), (side, k)
    q = np.random.default_rng(7).standard_normal((n, 3))
    z1, z2 = sg.matvec_nodewise(M, q), sg.matvec_nodewise(M2, q)
    assert z1.tobytes() == z2.tobytes()
    # the header stays readable by the reference loader: reference kernel families under
    # "kernel", the BASELINE extensions under "b200_kernel" with "kernel": null
    header, _ = _container()._read(path)
    if M.kernel.kind == "cauchy":
        assert header["kernel"]["kind"] == "cauchy"
    else:
        assert header["kernel"] is None and header["b200_kernel"]["kind"] == M.kernel.kind


@pytest.mark.gpu
def test_load_rejects_tampered_tree(sg, tmp_path):
    M, _ = _h2_2d(sg)
    path = str(tmp_path / "m.smash")
    sg.save_matrix(M, path)
    c = _container()
    raw = open(path, "rb").read()
    head = raw[len(c._MAGIC):]
    cut = head.index(b"\0")
    header = json.loads(head[:cut].decode())
    header["tree"]["nodes"][0]["rows"][1] += 1
    bad = tmp_path / "bad.smash"
    bad.write_bytes(c._MAGIC + json.dumps(header).encode() + b"\0" + head[cut + 1:])
    with pytest.raises(ValueError):
        sg.load_matrix(str(bad))


def test_oracle_ulv_matches_reference_ulv():
    """The oracle's ULV restatement (checker for tests/test_ulv.py and bench numbers)
    reproduces the reference's ulv_solve on the golden geometry."""
    from oracle import smash_oracle as orc
    g = np.load(os.path.join(GOLDEN, "container", "ref_container.npz"))
    n = 512
    x = (np.arange(n) / n)[:, None]
    y = ((np.arange(n) + 0.5) / n)[:, None]
    tree = orc.build_tree(x, y, nu0=32, mode="binary")
    M = orc.build_hss(tree, "cauchy", 12, 0.6, 1e-11)
    F = orc.ulv_factor(M)
    xs = orc.ulv_solve(F, g["q"])
    assert np.linalg.norm(xs - g["x_hss"]) <= 1e-9 * np.linalg.norm(g["x_hss"])
    X3 = orc.ulv_solve(F, g["B3"])
    assert np.linalg.norm(X3 - g["X3_hss"]) <= 1e-9 * np.linalg.norm(g["X3_hss"])
