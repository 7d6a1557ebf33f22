"""Structured-matrix containers and the HSS builder -- GPU drop-in for the
hot-path parts of smash.hss (/root/reference/pkg/src/smash/hss.py).

``build_hss`` (hss.py:247-303) and ``build_h2`` (h2.py:25-54) run the whole
bottom-up construction on the GPU (tree levels L..2: basis + sRRQR batched per
level).  The returned matrix keeps the device handle; the reference's
accessors (rowfac/colfac, skel_row/skel_col, U/V/R/W, B/NF, todense) are
materialised lazily from exported factors.  Couplings and nearfield blocks are
never stored -- the matvec regenerates them in registers, so ``use_cache`` is
accepted for API compatibility only.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .cluster import ClusterTree, leaf_sets
from .kernel import KernelSpec, kernel_block_coords
from .lowrank import InterpolativeFactor

__all__ = ["BuildParams", "HssMatrix", "build_hss", "build_hss_sharded", "make_matrix"]


@dataclass
class BuildParams:
    """Construction knobs (hss.py:23-32) plus ``rtol``, the sRRQR rank tolerance
    the reference hard-codes to 1e-14 (lowrank.py:19) -- BASELINE's "sRRQR
    tolerance"."""

    r: int = 20
    tau: float = 0.6
    eps_svd: float = 0.0
    s: float = 2.0
    basis: str = None  # "interp" only; None resolves to interp except for cauchy (Taylor, out of scope)
    rtol: float = 1e-14


def _resolve_basis(params: BuildParams, kernel: KernelSpec) -> str:
    basis = params.basis
    if basis is None:
        basis = "taylor" if kernel.kind == "cauchy" else "interp"
    if basis == "taylor":
        raise NotImplementedError("the Taylor basis is outside the B200 hot path; pass basis='interp' "
                                  "(BASELINE mandates Chebyshev interpolation)")
    if basis != "interp":
        raise ValueError("unknown basis %r" % basis)
    return basis


class _StructuredMatrix:
    kind = "structured"

    def __init__(self, tree: ClusterTree, params: BuildParams, kernel: KernelSpec, handle,
                 use_cache: bool = True):
        self.tree = tree
        self.params = params
        self.kernel = kernel
        self.dtype = np.dtype(np.float64)
        self.use_cache = use_cache
        self._h = handle
        self._fac = {}
        self._dblocks = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.smash_matrix_free(h)
            self._h = None

    # -- shapes ---------------------------------------------------------------
    @property
    def n_row(self) -> int:
        return self.tree.n_row

    @property
    def n_col(self) -> int:
        return self.tree.n_col

    @property
    def shape(self):
        return (self.n_row, self.n_col)

    # -- partitions -------------------------------------------------------------
    @property
    def pairs_L(self):
        return leaf_sets(self.tree, self.params.tau, self.kind)[0]

    @property
    def pairs_Lm(self):
        return leaf_sets(self.tree, self.params.tau, self.kind)[1]

    # -- factors -----------------------------------------------------------------
    def export_side(self, side: int) -> dict:
        """Raw exported factor arrays of one side (postorder CSR layout)."""
        if side not in self._fac:
            lib = _lib.load()
            has_t, ib_t, sk_t, g_t = _lib.c_i64(), _lib.c_i64(), _lib.c_i64(), _lib.c_i64()
            _lib.check(lib.smash_matrix_sizes(self._h, side, ctypes.byref(has_t), ctypes.byref(ib_t),
                                              ctypes.byref(sk_t), ctypes.byref(g_t)))
            n = len(self.tree.arrays()["level"])
            E = dict(has=_lib.empty(n, "int64"), rank=_lib.empty(n, "int64"),
                     perm_ptr=_lib.empty(n + 1, "int64"), perm=_lib.empty(ib_t.value, "int64"),
                     skel_ptr=_lib.empty(n + 1, "int64"), skel=_lib.empty(sk_t.value, "int64"),
                     g_ptr=_lib.empty(n + 1, "int64"), G=_lib.empty(g_t.value))
            P = _lib.ptr
            _lib.check(lib.smash_matrix_export(self._h, side, P(E["has"]), P(E["rank"]),
                                               P(E["perm_ptr"]), P(E["perm"]), P(E["skel_ptr"]),
                                               P(E["skel"]), P(E["g_ptr"]), P(E["G"]),
                                               _lib.stream_ptr()))
            self._fac[side] = {k: v.cpu().numpy() for k, v in E.items()}
        return self._fac[side]

    def _factors(self, side: int) -> dict:
        key = ("fac", side)
        if key not in self._fac:
            E = self.export_side(side)
            out = {}
            for i in np.nonzero(E["has"])[0]:
                i = int(i)
                perm = E["perm"][E["perm_ptr"][i]:E["perm_ptr"][i + 1]]
                k = int(E["rank"][i])
                G = E["G"][E["g_ptr"][i]:E["g_ptr"][i + 1]].reshape(perm.size - k, k)
                skel = E["skel"][E["skel_ptr"][i]:E["skel_ptr"][i + 1]]
                out[i] = InterpolativeFactor(nrows=perm.size, perm=perm, G=G, skel=skel,
                                             skel_local=perm[:k].copy())
            self._fac[key] = out
        return self._fac[key]

    @property
    def rowfac(self) -> dict:
        return self._factors(0)

    @property
    def colfac(self) -> dict:
        return self._factors(1)

    @property
    def skel_row(self) -> dict:
        return {i: f.skel for i, f in self.rowfac.items()}

    @property
    def skel_col(self) -> dict:
        return {i: f.skel for i, f in self.colfac.items()}

    @property
    def swaps(self):
        a, b = _lib.c_i64(), _lib.c_i64()
        _lib.check(_lib.load().smash_matrix_stats(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def rank_row(self, i: int) -> int:
        return self.rowfac[i].rank

    def rank_col(self, i: int) -> int:
        return self.colfac[i].rank

    # -- generator accessors (hss.py:106-162) -------------------------------------
    def U(self, i: int) -> np.ndarray:
        return self.rowfac[i].expand()

    def V(self, i: int) -> np.ndarray:
        return self.colfac[i].expand()

    def _child_slice(self, c: int, fac: dict):
        p = self.tree.nodes[c].parent
        off = 0
        for ch in self.tree.nodes[p].children:
            k = fac[ch].rank
            if ch == c:
                return p, off, off + k
            off += k
        raise KeyError(c)

    def R(self, c: int) -> np.ndarray:
        p, a, b = self._child_slice(c, self.rowfac)
        return self.rowfac[p].expand()[a:b]

    def W(self, c: int) -> np.ndarray:
        p, a, b = self._child_slice(c, self.colfac)
        return self.colfac[p].expand()[a:b]

    def B(self, i: int, j: int) -> np.ndarray:
        """Coupling block: exact kernel entries at the skeletons (GPU evaluated)."""
        return kernel_block_coords(self.kernel, self.tree.points_row[self.rowfac[i].skel],
                                   self.tree.points_col[self.colfac[j].skel])

    def NF(self, i: int, j: int) -> np.ndarray:
        """Dense nearfield block of a leaf pair (GPU evaluated)."""
        t = self.tree
        return kernel_block_coords(self.kernel, t.points_row[t.row_range(i)], t.points_col[t.col_range(j)])

    @property
    def Dblocks(self) -> dict:
        if self._dblocks is None:
            self._dblocks = {i: self.NF(i, i) for i in self.tree.leaves()} if self.kind == "hss" else {}
        return self._dblocks

    # -- dense reconstruction (checker utility, hss.py:166-187) ----------------------
    def _basis_big(self, i: int, side: str) -> np.ndarray:
        if self.tree.is_leaf(i):
            return self.U(i) if side == "row" else self.V(i)
        parts = [self._basis_big(c, side) @ (self.R(c) if side == "row" else self.W(c))
                 for c in self.tree.nodes[i].children]
        return np.vstack(parts)

    def todense(self) -> np.ndarray:
        tr = self.tree
        out = np.zeros(self.shape)
        for i, j in self.pairs_L:
            blk = self._basis_big(i, "row") @ self.B(i, j) @ self._basis_big(j, "col").T
            out[np.ix_(tr.row_range(i), tr.col_range(j))] = blk
        for i, j in self.pairs_Lm:
            out[np.ix_(tr.row_range(i), tr.col_range(j))] = self.NF(i, j)
        res = np.empty_like(out)
        res[np.ix_(tr.perm_row, tr.perm_col)] = out
        return res


class HssMatrix(_StructuredMatrix):
    kind = "hss"

    def sibling_B(self, i: int) -> np.ndarray:
        return self.B(i, self.tree.sibling(i))


def _params_c(kind: str, tree: ClusterTree, kernel: KernelSpec, params: BuildParams):
    _resolve_basis(params, kernel)
    if kernel.kind == "cauchy" and kernel.dx is None and tree.shared_points:
        raise ValueError("coincident points need a diagonal value d_x")
    return _lib.BuildParamsC(structure=_lib.STRUCT[kind], kernel=kernel.code,
                             dx=kernel.dx_value if kernel.dx_value == kernel.dx_value else 0.0,
                             r=int(params.r), tau=float(params.tau), s=float(params.s),
                             rtol=float(params.rtol), eps_svd=float(params.eps_svd))


def make_matrix(cls, tree: ClusterTree, kernel: KernelSpec, params: BuildParams, use_cache: bool):
    """Run the GPU construction for ``cls.kind`` and wrap the handle."""
    p = _params_c(cls.kind, tree, kernel, params)
    h = ctypes.c_void_p()
    _lib.check(_lib.load().smash_matrix_build(tree._h, ctypes.byref(p), _lib.stream_ptr(),
                                              ctypes.byref(h)))
    return cls(tree, params, kernel, h, use_cache)


def build_hss(tree: ClusterTree, kernel: KernelSpec, X=None, Y=None, params: BuildParams = None,
              use_cache: bool = True) -> HssMatrix:
    """GPU HSS construction (replaces hss.py:247-303).  X / Y are accepted for
    signature compatibility; the tree already holds the points."""
    params = params or BuildParams()
    if tree.mode == "2d" and tree.dim > 1:
        raise ValueError("HSS construction needs a binary tree")
    return make_matrix(HssMatrix, tree, kernel, params, use_cache)


def build_hss_sharded(tree: ClusterTree, kernel: KernelSpec, X=None, Y=None, params: BuildParams = None,
                      group=None, use_cache: bool = True) -> HssMatrix:
    """HSS construction distributed over the ranks of a torch.distributed process group
    (SURVEY.md 8(e), configs 1 and 4).  HSS levels depend on each other through the
    nearfield SVD (hss.py:279-299 reads the other side's level-(l+1) skeletons), so the
    work is split level by level: every rank runs the SVDs and sRRQRs of a contiguous
    share of the level's nodes, and one exchange per level and side sums the disjoint,
    zero-filled ranks / perm / G / ordered skeleton labels and coordinates over the ranks
    (float64 as int64 bit patterns: exact) before every rank compacts the level.  Every
    rank ends with the full matrix, bit-identical to build_hss's."""
    import torch
    import torch.distributed as dist
    from .h2 import _DevView
    params = params or BuildParams()
    if tree.mode == "2d" and tree.dim > 1:
        raise ValueError("HSS construction needs a binary tree")
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    p = _params_c("hss", tree, kernel, params)
    gloo = dist.get_backend(group) == "gloo"
    failure = []
    VIEW = {0: 0, 1: 2, 2: 2, 3: 0}  # float64 summed as its int64 bit pattern

    def exchange(ctx, n, ptrs, counts, dtypes):
        try:
            for i in range(n):
                dt = dtypes[i]
                t = torch.as_tensor(_DevView(ptrs[i], counts[i], VIEW[dt]), device="cuda")
                op = dist.ReduceOp.MAX if dt == 3 else dist.ReduceOp.SUM
                if gloo:
                    h = t.cpu()
                    dist.all_reduce(h, op=op, group=group)
                    t.copy_(h)
                else:
                    dist.all_reduce(t, op=op, group=group)
            torch.cuda.current_stream().synchronize()
            return 0
        except BaseException as e:  # surfaced after the C call returns
            failure.append(e)
            return 1

    fn = _lib.EXCHANGE_FN(exchange)
    h = ctypes.c_void_p()
    rc = _lib.load().smash_matrix_build_sharded(tree._h, ctypes.byref(p), int(rank), int(world),
                                                ctypes.cast(fn, ctypes.c_void_p), None,
                                                _lib.stream_ptr(), ctypes.byref(h))
    if failure:
        raise failure[0]
    _lib.check(rc)
    return HssMatrix(tree, params, kernel, h, use_cache)
