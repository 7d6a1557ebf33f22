"""Cluster trees and block partitions -- GPU drop-in for smash.cluster
(/root/reference/pkg/src/smash/cluster.py).

``build_tree`` (cluster.py:263), ``leaf_sets`` (:402) and ``nearfield_set``
(:374) run on the GPU through the C ABI (include/smash_b200.h); the returned
``ClusterTree`` keeps the device handle and materialises the reference's
Python-side view (``nodes``, ``perm_row`` ...) lazily on first access.
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _lib

__all__ = ["PointSet", "Box", "TreeNode", "ClusterTree", "build_tree", "well_separated",
           "leaf_sets", "nearfield_set"]


class PointSet:
    """(n, d) float64 coordinates plus a role tag (cluster.py:27-45).

    ``coords`` may be a numpy array or a torch tensor; a CUDA tensor stays on the
    device (the tree build reads it in place) and is copied to the host only if
    ``.coords`` is accessed."""

    def __init__(self, coords, role: str = "row"):
        self.role = role
        self._dev = None
        self._coords = None
        if hasattr(coords, "detach") and getattr(coords, "is_cuda", False):
            import torch
            t = coords.detach()
            if t.dim() == 1:
                t = t.reshape(1, -1)
            if t.dim() != 2:
                raise ValueError("coords must be a 2-d array")
            self._dev = t.to(torch.float64).contiguous()
        else:
            if hasattr(coords, "detach"):
                coords = coords.detach().cpu().numpy()
            c = np.atleast_2d(np.asarray(coords, dtype=np.float64))
            if c.ndim != 2:
                raise ValueError("coords must be a 2-d array")
            self._coords = c

    @property
    def coords(self) -> np.ndarray:
        if self._coords is None:
            self._coords = self._dev.cpu().numpy()
        return self._coords

    @property
    def shape(self):
        return tuple(self._dev.shape) if self._dev is not None else self._coords.shape

    @property
    def n(self) -> int:
        return self.shape[0]

    @property
    def dim(self) -> int:
        return self.shape[1]

    def device_tensor(self):
        if self._dev is None:
            self._dev = _lib.to_device(self._coords)
        return self._dev


def _fma(a: float, b: float, c: float) -> float:
    """Correctly rounded fused multiply-add (exact rational arithmetic)."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _norm_fma(v) -> float:
    """np.linalg.norm of a short vector as OpenBLAS evaluates it (FMA chain)."""
    v = [float(x) for x in v]
    s = v[0] * v[0]
    for x in v[1:]:
        s = _fma(x, x, s)
    return float(np.sqrt(s))


@dataclass(frozen=True)
class Box:
    """Axis-aligned box (cluster.py:48-78)."""

    lo: tuple
    hi: tuple

    @staticmethod
    def of(lo, hi) -> "Box":
        return Box(tuple(float(v) for v in np.atleast_1d(lo)), tuple(float(v) for v in np.atleast_1d(hi)))

    @property
    def dim(self) -> int:
        return len(self.lo)

    @property
    def center(self) -> np.ndarray:
        return (np.asarray(self.lo) + np.asarray(self.hi)) / 2.0

    @property
    def radius(self) -> float:
        return 0.5 * _norm_fma(np.asarray(self.hi) - np.asarray(self.lo))

    def contains(self, pts: np.ndarray, slack: float = 1e-12) -> bool:
        if pts.size == 0:
            return True
        return bool(np.all(pts >= np.asarray(self.lo) - slack) and np.all(pts <= np.asarray(self.hi) + slack))


def well_separated(box_a: Box, box_b: Box, tau: float) -> bool:
    """rA + rB <= tau * ||cA - cB|| (cluster.py:81-85), same rounding as the GPU kernels."""
    return box_a.radius + box_b.radius <= tau * _norm_fma(box_a.center - box_b.center)


@dataclass
class TreeNode:
    index: int
    level: int
    box: Box
    parent: int = -1
    children: tuple = ()
    row_start: int = 0
    row_stop: int = 0
    col_start: int = 0
    col_stop: int = 0

    @property
    def is_leaf(self) -> bool:
        return not self.children

    @property
    def n_row(self) -> int:
        return self.row_stop - self.row_start

    @property
    def n_col(self) -> int:
        return self.col_stop - self.col_start


class ClusterTree:
    """Postordered cluster tree held on the GPU (cluster.py:118-217 interface)."""

    def __init__(self, handle, mode: str, nu0: int, tau_default: float):
        self._h = handle
        self.mode = mode
        self.nu0 = nu0
        self.tau_default = tau_default
        n_nodes, n_lev, n_row, n_col = _lib.c_i64(), _lib.c_i32(), _lib.c_i64(), _lib.c_i64()
        dim, shared = _lib.c_i32(), _lib.c_i32()
        _lib.check(_lib.load().smash_tree_sizes(handle, ctypes.byref(n_nodes), ctypes.byref(n_lev),
                                                ctypes.byref(n_row), ctypes.byref(n_col),
                                                ctypes.byref(dim), ctypes.byref(shared)))
        self._n_nodes = n_nodes.value
        self._n_levels = n_lev.value
        self._n_row = n_row.value
        self._n_col = n_col.value
        self._dim = dim.value
        self.shared_points = bool(shared.value)
        self._arrays = None
        self._nodes = None
        self._pairs = {}
        self._near = {}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.smash_tree_free(h)
            self._h = None

    # -- lazy host view --------------------------------------------------------
    def arrays(self) -> dict:
        """All tree arrays (postorder), copied once from the device."""
        if self._arrays is None:
            n, d = self._n_nodes, self._dim
            T = {k: _lib.empty(n, "int64") for k in ("level", "parent", "row_start", "row_stop",
                                                     "col_start", "col_stop")}
            T["child_ptr"] = _lib.empty(n + 1, "int64")
            T["child_idx"] = _lib.empty(max(n - 1, 0), "int64")
            T["lo"] = _lib.empty((n, d))
            T["hi"] = _lib.empty((n, d))
            T["perm_row"] = _lib.empty(self._n_row, "int64")
            T["perm_col"] = _lib.empty(self._n_col, "int64")
            T["points_row"] = _lib.empty((self._n_row, d))
            T["points_col"] = _lib.empty((self._n_col, d))
            P = _lib.ptr
            _lib.check(_lib.load().smash_tree_export(
                self._h, P(T["level"]), P(T["parent"]), P(T["child_ptr"]), P(T["child_idx"]),
                P(T["lo"]), P(T["hi"]), P(T["row_start"]), P(T["row_stop"]), P(T["col_start"]),
                P(T["col_stop"]), P(T["perm_row"]), P(T["perm_col"]), P(T["points_row"]),
                P(T["points_col"]), _lib.stream_ptr()))
            self._arrays = {k: v.cpu().numpy() for k, v in T.items()}
        return self._arrays

    @property
    def nodes(self) -> list:
        if self._nodes is None:
            A = self.arrays()
            cp, ci = A["child_ptr"], A["child_idx"]
            self._nodes = [
                TreeNode(index=i, level=int(A["level"][i]), box=Box.of(A["lo"][i], A["hi"][i]),
                         parent=int(A["parent"][i]),
                         children=tuple(int(c) for c in ci[cp[i]:cp[i + 1]]),
                         row_start=int(A["row_start"][i]), row_stop=int(A["row_stop"][i]),
                         col_start=int(A["col_start"][i]), col_stop=int(A["col_stop"][i]))
                for i in range(self._n_nodes)]
        return self._nodes

    @property
    def perm_row(self) -> np.ndarray:
        return self.arrays()["perm_row"]

    @property
    def perm_col(self) -> np.ndarray:
        return self.arrays()["perm_col"]

    @property
    def points_row(self) -> np.ndarray:
        return self.arrays()["points_row"]

    @property
    def points_col(self) -> np.ndarray:
        return self.arrays()["points_col"]

    # -- reference accessors (cluster.py:139-183) ------------------------------
    @property
    def root(self) -> int:
        return self._n_nodes - 1

    @property
    def dim(self) -> int:
        return self._dim

    @property
    def n_levels(self) -> int:
        return self._n_levels

    @property
    def n_row(self) -> int:
        return self._n_row

    @property
    def n_col(self) -> int:
        return self._n_col

    def is_leaf(self, i: int) -> bool:
        A = self.arrays()
        return A["child_ptr"][i + 1] == A["child_ptr"][i]

    def leaves(self):
        A = self.arrays()
        return [int(i) for i in np.nonzero(np.diff(A["child_ptr"]) == 0)[0]]

    def level_nodes(self, level: int):
        return [int(i) for i in np.nonzero(self.arrays()["level"] == level)[0]]

    def row_range(self, i: int) -> np.ndarray:
        A = self.arrays()
        return np.arange(A["row_start"][i], A["row_stop"][i])

    def col_range(self, i: int) -> np.ndarray:
        A = self.arrays()
        return np.arange(A["col_start"][i], A["col_stop"][i])

    def sibling(self, i: int) -> int:
        p = self.nodes[i].parent
        if p < 0:
            raise ValueError("root has no sibling")
        sibs = [c for c in self.nodes[p].children if c != i]
        if len(sibs) != 1:
            raise ValueError("node %d has %d siblings" % (i, len(sibs)))
        return sibs[0]

    def verify(self):
        """Structural invariants of cluster.py:187-217, checked on the exported arrays."""
        nodes = self.nodes
        root = nodes[self.root]
        assert root.level == 1
        assert root.row_start == 0 and root.row_stop == self.n_row
        assert root.col_start == 0 and root.col_stop == self.n_col
        assert np.array_equal(np.sort(self.perm_row), np.arange(self.n_row))
        assert np.array_equal(np.sort(self.perm_col), np.arange(self.n_col))
        for nd in nodes:
            assert nd.row_stop >= nd.row_start and nd.col_stop >= nd.col_start
            assert nd.n_row + nd.n_col > 0, "empty node %d" % nd.index
            assert nd.box.contains(self.points_row[nd.row_start:nd.row_stop])
            assert nd.box.contains(self.points_col[nd.col_start:nd.col_stop])
            if nd.is_leaf:
                assert nd.n_row <= self.nu0 and nd.n_col <= self.nu0
            else:
                assert max(nd.n_row, nd.n_col) > self.nu0
                assert len(nd.children) >= 2
                if self.mode == "binary":
                    assert len(nd.children) == 2
                r, c = nd.row_start, nd.col_start
                for ci in nd.children:
                    ch = nodes[ci]
                    assert ch.parent == nd.index and ch.level == nd.level + 1 and ch.index < nd.index
                    assert ch.row_start == r and ch.col_start == c
                    r, c = ch.row_stop, ch.col_stop
                assert r == nd.row_stop and c == nd.col_stop

    def to_json(self) -> str:
        A = self.arrays()
        return json.dumps({
            "mode": self.mode, "nu0": self.nu0, "n_row": self.n_row, "n_col": self.n_col,
            "dim": self.dim, "perm_row": A["perm_row"].tolist(), "perm_col": A["perm_col"].tolist(),
            "nodes": [{"index": nd.index, "level": nd.level, "parent": nd.parent,
                       "children": list(nd.children), "lo": list(nd.box.lo), "hi": list(nd.box.hi),
                       "row_range": [nd.row_start, nd.row_stop], "col_range": [nd.col_start, nd.col_stop]}
                      for nd in self.nodes]})


def build_tree(points_row: PointSet, points_col: PointSet = None, nu0: int = 50,
               mode: str = "binary", tau: float = 0.6) -> ClusterTree:
    """GPU adaptive cluster tree (replaces cluster.py:263-353)."""
    if mode == "2^d":
        mode = "2d"
    if mode not in ("binary", "2d"):
        raise ValueError("mode must be 'binary' or '2d'")
    if nu0 < 1:
        raise ValueError("nu0 must be positive")
    nx, dim = points_row.shape
    if nx == 0:
        raise ValueError("row point set is empty")
    shared = points_col is None or points_col is points_row
    ny = nx if shared else points_col.shape[0]
    if not shared and points_col.shape[1] != dim:
        raise ValueError("row/column point dimensions differ")
    if not 1 <= dim <= 3:
        raise ValueError("points must have 1, 2 or 3 coordinates")
    lib = _lib.load()
    dX = points_row.device_tensor()
    dY = None if shared else points_col.device_tensor()
    h = ctypes.c_void_p()
    _lib.check(lib.smash_tree_build(_lib.ptr(dX), nx, None if shared else _lib.ptr(dY), ny, dim,
                                    nu0, _lib.MODE[mode], _lib.stream_ptr(), ctypes.byref(h)))
    return ClusterTree(h, mode, nu0, tau)


def _pairs(tree: ClusterTree, tau: float, structure: str):
    key = (float(tau) if structure == "h2" else 0.0, structure)
    if key not in tree._pairs:
        if structure not in _lib.STRUCT:
            raise ValueError("structure must be 'hss' or 'h2'")
        lib = _lib.load()
        nL, nLm = _lib.c_i64(), _lib.c_i64()
        _lib.check(lib.smash_leaf_sets(tree._h, float(tau), _lib.STRUCT[structure], _lib.stream_ptr(),
                                       ctypes.byref(nL), ctypes.byref(nLm)))
        L = _lib.empty((nL.value, 2), "int64")
        Lm = _lib.empty((nLm.value, 2), "int64")
        _lib.check(lib.smash_leaf_sets_export(tree._h, float(tau), _lib.STRUCT[structure],
                                              _lib.ptr(L), _lib.ptr(Lm), _lib.stream_ptr()))
        tree._pairs[key] = (L.cpu().numpy(), Lm.cpu().numpy())
    return tree._pairs[key]


def leaf_sets(tree: ClusterTree, tau: float = None, structure: str = "h2"):
    """(L, Lm) block partition computed on the GPU (replaces cluster.py:402-447).
    Lists of (i, j) tuples, sorted lexicographically."""
    if tau is None:
        tau = tree.tau_default
    L, Lm = _pairs(tree, tau, structure)
    return [tuple(map(int, p)) for p in L], [tuple(map(int, p)) for p in Lm]


def nearfield_set(tree: ClusterTree, i: int, tau: float = None) -> list:
    """N_i computed on the GPU for all nodes at once and cached per tau
    (replaces cluster.py:374-399)."""
    if tau is None:
        tau = tree.tau_default
    key = float(tau)
    if key not in tree._near:
        lib = _lib.load()
        tot = _lib.c_i64()
        _lib.check(lib.smash_nearfield(tree._h, key, _lib.stream_ptr(), ctypes.byref(tot)))
        ptr = _lib.empty(tree._n_nodes + 1, "int64")
        idx = _lib.empty(tot.value, "int64")
        _lib.check(lib.smash_nearfield_export(tree._h, key, _lib.ptr(ptr), _lib.ptr(idx),
                                              _lib.stream_ptr()))
        tree._near[key] = (ptr.cpu().numpy(), idx.cpu().numpy())
    p, x = tree._near[key]
    return [int(v) for v in x[p[i]:p[i + 1]]]
