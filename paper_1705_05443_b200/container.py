"""Binary container for GPU-built structured matrices -- drop-in for
smash/container.py (/root/reference/pkg/src/smash/container.py).

The file format is the reference's (container.py:1-7, 58-128): the magic line
``SMASH-BIN-1``, a JSON header (kind, params, tree topology, kernel, pair
lists, array manifest), a NUL byte, then little-endian f8 / i8 payloads, so a
round trip is bit-exact.  Two compatible extensions:

* ``params.rtol`` (the sRRQR tolerance, BuildParams.rtol) -- ignored by the
  reference loader;
* kernels outside the reference's families (log, 1/r, exp) are written under
  ``b200_kernel`` with ``kernel: null``, so the reference's ``load_matrix``
  still reads such a file (factors, skeletons, tree) as a kernel-less matrix.

``load_matrix`` rebuilds the cluster tree on the GPU from the stored caller
points (deterministic; checked against the stored topology node by node),
rebuilds and checks the pair lists, and uploads the stored factors through the
C ABI (``smash_matrix_import``), so a loaded matrix runs the same device
matvec as a freshly built one -- including files the reference itself wrote,
whenever their kernel family and dtype are on the B200 path.
"""

from __future__ import annotations

import ctypes
import json

import numpy as np

from . import _lib
from .cluster import PointSet, build_tree, leaf_sets
from .h2 import H2Matrix
from .hss import BuildParams, HssMatrix
from .kernel import KernelSpec

__all__ = ["save_matrix", "load_matrix"]

_MAGIC = b"SMASH-BIN-1\n"                          # container.py:22
_DT = {"f8": "<f8", "c16": "<c16", "i8": "<i8"}    # container.py:24
_REF_KINDS = ("cauchy", "cauchy_like", "laplace_dlp")  # kernel.py:220


def _tag(arr: np.ndarray) -> str:
    if arr.dtype.kind == "c":
        return "c16"
    if arr.dtype.kind in "iu":
        return "i8"
    return "f8"


class _Payload:
    """Array manifest + raw chunks (container.py:35-50)."""

    def __init__(self):
        self.manifest, self.chunks, self.offset = [], [], 0

    def add(self, name: str, arr) -> None:
        arr = np.asarray(arr)
        tag = _tag(arr)
        raw = np.ascontiguousarray(arr, dtype=_DT[tag]).tobytes()
        self.manifest.append({"name": name, "dtype": tag, "shape": list(arr.shape),
                              "offset": self.offset, "nbytes": len(raw)})
        self.chunks.append(raw)
        self.offset += len(raw)


def save_matrix(M, path) -> None:
    """Write an H2 or HSS matrix built on the GPU (container.py:58-128)."""
    if not isinstance(M, (H2Matrix, HssMatrix)):
        raise TypeError("save_matrix expects an H2Matrix or HssMatrix from this package")
    tr = M.tree
    pl = _Payload()
    pl.add("perm_row", tr.perm_row)
    pl.add("perm_col", tr.perm_col)
    pl.add("points_row", tr.points_row)
    pl.add("points_col", tr.points_col)
    for side, facs in (("rowfac", M.rowfac), ("colfac", M.colfac)):
        for i, f in facs.items():
            pl.add("%s.%d.perm" % (side, i), f.perm)
            pl.add("%s.%d.G" % (side, i), f.G)
            pl.add("%s.%d.skel" % (side, i), f.skel)
    for i, f in M.rowfac.items():
        pl.add("skel_row.%d" % i, f.skel)
    for i, f in M.colfac.items():
        pl.add("skel_col.%d" % i, f.skel)
    for i, D in M.Dblocks.items():  # HSS leaf diagonal blocks (hss.py:301-302)
        pl.add("D.%d" % i, D)

    kern = {"kind": M.kernel.kind, "dx": M.kernel.dx, "nq": 0, "curve": None}
    p = M.params
    header = {
        "kind": M.kind,
        "dtype": "f8",
        "use_cache": bool(M.use_cache),
        "params": {"r": p.r, "tau": p.tau, "eps_svd": p.eps_svd, "s": p.s, "basis": p.basis,
                   "rtol": p.rtol},
        "tree": {
            "mode": tr.mode, "nu0": tr.nu0, "tau_default": tr.tau_default,
            "nodes": [{"level": nd.level, "parent": nd.parent, "children": list(nd.children),
                       "lo": [float(x) for x in nd.box.lo], "hi": [float(x) for x in nd.box.hi],
                       "rows": [nd.row_start, nd.row_stop], "cols": [nd.col_start, nd.col_stop]}
                      for nd in tr.nodes],
        },
        "kernel": kern if M.kernel.kind in _REF_KINDS else None,
        "b200_kernel": kern,
        "pairs_L": [[int(a), int(b)] for a, b in np.asarray(M.pairs_L).reshape(-1, 2)],
        "pairs_Lm": [[int(a), int(b)] for a, b in np.asarray(M.pairs_Lm).reshape(-1, 2)],
        "arrays": pl.manifest,
    }
    with open(path, "wb") as fh:
        fh.write(_MAGIC)
        fh.write(json.dumps(header).encode())
        fh.write(b"\0")
        for chunk in pl.chunks:
            fh.write(chunk)


def _read(path):
    """Header + arrays (container.py:131-155)."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if not raw.startswith(_MAGIC):
        raise ValueError("not a structured-matrix container: %s" % path)
    raw = raw[len(_MAGIC):]
    cut = raw.index(b"\0")
    header = json.loads(raw[:cut].decode())
    buf = raw[cut + 1:]
    arrays = {}
    for ent in header["arrays"]:
        count = int(np.prod(ent["shape"], dtype=np.int64)) if ent["shape"] else 1
        a = np.frombuffer(buf, dtype=_DT[ent["dtype"]], count=count, offset=ent["offset"])
        arrays[ent["name"]] = a.reshape(ent["shape"]).copy()
    return header, arrays


def _caller_points(perm: np.ndarray, pts: np.ndarray) -> np.ndarray:
    out = np.empty_like(pts)
    out[perm] = pts
    return out


def _check_tree(tree, nodes) -> None:
    got = tree.nodes
    if len(got) != len(nodes):
        raise ValueError("container tree has %d nodes, the B200 rebuild %d" % (len(nodes), len(got)))
    for i, (a, b) in enumerate(zip(got, nodes)):
        if (a.level != b["level"] or a.parent != b["parent"] or list(a.children) != list(b["children"])
                or [a.row_start, a.row_stop] != list(b["rows"]) or [a.col_start, a.col_stop] != list(b["cols"])
                or not np.array_equal(np.asarray(a.box.lo, float), np.asarray(b["lo"], float))
                or not np.array_equal(np.asarray(a.box.hi, float), np.asarray(b["hi"], float))):
            raise ValueError("container tree node %d differs from the B200 rebuild" % i)


def _side_arrays(arrays, side: str, n: int, root: int):
    rank = np.zeros(n, np.int64)
    pp, sp, gp = (np.zeros(n + 1, np.int64) for _ in range(3))
    perm, skel, G = [], [], []
    for i in range(n):
        if i == root:
            pass
        else:
            key = "%s.%d." % (side, i)
            if key + "perm" not in arrays:
                raise ValueError("container lacks %sperm (a factor per non-root node)" % key)
            p, g, s = arrays[key + "perm"], arrays[key + "G"], arrays[key + "skel"]
            rank[i] = s.size
            perm.append(p.astype(np.int64).ravel())
            skel.append(s.astype(np.int64).ravel())
            G.append(np.asarray(g, np.float64).ravel())
        pp[i + 1] = pp[i] + (perm[-1].size if i != root else 0)
        sp[i + 1] = sp[i] + (skel[-1].size if i != root else 0)
        gp[i + 1] = gp[i] + (G[-1].size if i != root else 0)
    cat = lambda xs, dt: np.ascontiguousarray(np.concatenate(xs) if xs else np.zeros(0, dt), dtype=dt)
    return [rank, pp, cat(perm, np.int64), sp, cat(skel, np.int64), gp, cat(G, np.float64)]


def load_matrix(path, device=None):
    """Read a container into a GPU matrix (container.py:131-211)."""
    header, arrays = _read(path)
    if header.get("dtype", "f8") != "f8":
        raise ValueError("complex matrices are outside the B200 (fp64 real) path")
    kh = header.get("b200_kernel") or header.get("kernel")
    if kh is None:
        raise ValueError("matrix was saved without a kernel; the device matvec needs one")
    kernel = KernelSpec(kh["kind"], dx=kh.get("dx"))
    ph = header["params"]
    params = BuildParams(r=ph["r"], tau=ph["tau"], eps_svd=ph["eps_svd"], s=ph["s"],
                         basis=ph.get("basis"), rtol=ph.get("rtol", 1e-14))
    th = header["tree"]
    prow, pcol = arrays["perm_row"], arrays["perm_col"]
    xr, xc = arrays["points_row"], arrays["points_col"]
    shared = np.array_equal(prow, pcol) and np.array_equal(xr, xc)
    X = PointSet(_caller_points(prow, xr))
    Y = None if shared else PointSet(_caller_points(pcol, xc), role="col")
    tree = build_tree(X, Y, nu0=th["nu0"], mode=th["mode"], tau=th["tau_default"])
    _check_tree(tree, th["nodes"])
    kind = header["kind"]
    L, Lm = leaf_sets(tree, params.tau, kind)
    for name, got in (("pairs_L", L), ("pairs_Lm", Lm)):
        want = {tuple(p) for p in header[name]}
        if {tuple(int(x) for x in p) for p in np.asarray(got).reshape(-1, 2)} != want:
            raise ValueError("container %s differ from the B200 pair lists" % name)
    n, root = len(th["nodes"]), tree.root
    sides = [_side_arrays(arrays, "rowfac", n, root)]
    colfac_same = all(("rowfac" + k[6:]) in arrays and np.array_equal(arrays[k], arrays["rowfac" + k[6:]])
                      for k in arrays if k.startswith("colfac."))
    if not (shared and colfac_same):
        sides.append(_side_arrays(arrays, "colfac", n, root))
    ns = len(sides)
    keep = sides  # the host arrays must outlive the call
    arr_t = ctypes.c_void_p * ns
    cols = [arr_t(*[s[j].ctypes.data for s in keep]) for j in range(7)]
    p = _lib.BuildParamsC(structure=_lib.STRUCT[kind], kernel=kernel.code,
                          dx=kernel.dx_value if kernel.dx_value == kernel.dx_value else 0.0,
                          r=int(params.r), tau=float(params.tau), s=float(params.s),
                          rtol=float(params.rtol), eps_svd=float(params.eps_svd))
    h = ctypes.c_void_p()
    _lib.check(_lib.load().smash_matrix_import(tree._h, ctypes.byref(p), ns, *cols,
                                               _lib.stream_ptr(), ctypes.byref(h)))
    cls = HssMatrix if kind == "hss" else H2Matrix
    return cls(tree, params, kernel, h, header.get("use_cache", True))
