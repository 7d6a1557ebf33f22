"""HSS algebra -- GPU drop-in for smash.hss.hss_add / diag_scale / cauchy_like_hss
(/root/reference/pkg/src/smash/hss.py:317-400).

The reference's algebra produces generator-form HSS matrices: diag_scale scales the
leaf bases and diagonal blocks of a matrix (transfers and couplings unchanged), and
hss_add concatenates the skeletons and bases of two matrices on one tree and stacks
their transfers and couplings block-diagonally.  Every such result is therefore a
sum of diagonally scaled built matrices,

    S = sum_t diag(dl_t) A_t diag(dr_t),

and that term list is the device representation here (``ScaledSumHss``): the scalings
live on the device, the bases are the built device matrices, and the product runs
in the C ABI (smash_sum_matvec: one multi-column device matvec per distinct base,
then one combine kernel).  The reference's generator accessors (U, V, R, W, B, NF,
Dblocks, skel_row / skel_col, rank_row / rank_col, todense) are materialised from the
terms exactly as hss_add / diag_scale assemble them.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .hss import BuildParams, HssMatrix, build_hss
from .kernel import KernelSpec

__all__ = ["ScaledSumHss", "hss_add", "diag_scale", "cauchy_like_hss"]


def _blkdiag(X, Y):
    """hss.py:345-349."""
    out = np.zeros((X.shape[0] + Y.shape[0], X.shape[1] + Y.shape[1]))
    out[:X.shape[0], :X.shape[1]] = X
    out[X.shape[0]:, X.shape[1]:] = Y
    return out


def _blkdiag_all(mats):
    out = mats[0]
    for m in mats[1:]:
        out = _blkdiag(out, m)
    return out


class ScaledSumHss:
    """sum_t diag(dl_t) A_t diag(dr_t) over built HSS matrices A_t sharing one tree."""

    kind = "hss"

    def __init__(self, terms):
        torch = _lib.torch_cuda()
        self.terms = list(terms)  # [(A_t, dl_t host f64 (n_row,), dr_t host f64 (n_col,))]
        A0 = self.terms[0][0]
        self.tree = A0.tree
        self.params = A0.params
        self.kernel = None
        self.dtype = np.dtype(np.float64)
        self.use_cache = A0.use_cache
        self._dl = torch.from_numpy(np.stack([t[1] for t in self.terms])).cuda()
        self._dr = torch.from_numpy(np.stack([t[2] for t in self.terms])).cuda()
        self._dblocks = None

    # -- shapes / partition ------------------------------------------------------
    @property
    def n_row(self):
        return self.tree.n_row

    @property
    def n_col(self):
        return self.tree.n_col

    @property
    def shape(self):
        return (self.n_row, self.n_col)

    @property
    def pairs_L(self):
        return self.terms[0][0].pairs_L

    @property
    def pairs_Lm(self):
        return self.terms[0][0].pairs_Lm

    # -- skeletons (hss_add concatenates them, hss.py:327-329) --------------------
    @property
    def skel_row(self):
        return {i: np.concatenate([A.skel_row[i] for A, _, _ in self.terms]) for i in self.terms[0][0].skel_row}

    @property
    def skel_col(self):
        return {i: np.concatenate([A.skel_col[i] for A, _, _ in self.terms]) for i in self.terms[0][0].skel_col}

    def rank_row(self, i):
        return sum(A.rank_row(i) for A, _, _ in self.terms)

    def rank_col(self, i):
        return sum(A.rank_col(i) for A, _, _ in self.terms)

    # -- generators (hss.py:330-343 for sums, 366-378 for scalings) ----------------
    def _rows(self, i):
        return self.tree.row_range(i)

    def _cols(self, i):
        return self.tree.col_range(i)

    def U(self, i):
        pr = self.tree.perm_row
        return np.hstack([dl[pr][self._rows(i)][:, None] * A.U(i) for A, dl, _ in self.terms])

    def V(self, i):
        pc = self.tree.perm_col
        return np.hstack([dr[pc][self._cols(i)][:, None] * A.V(i) for A, _, dr in self.terms])

    def R(self, c):
        return _blkdiag_all([A.R(c) for A, _, _ in self.terms])

    def W(self, c):
        return _blkdiag_all([A.W(c) for A, _, _ in self.terms])

    def B(self, i, j):
        return _blkdiag_all([A.B(i, j) for A, _, _ in self.terms])

    def NF(self, i, j):
        pr, pc = self.tree.perm_row, self.tree.perm_col
        out = None
        for A, dl, dr in self.terms:
            blk = dl[pr][self._rows(i)][:, None] * A.NF(i, j) * dr[pc][self._cols(j)][None, :]
            out = blk if out is None else out + blk
        return out

    @property
    def Dblocks(self):
        if self._dblocks is None:
            self._dblocks = {i: self.NF(i, i) for i in self.tree.leaves()}
        return self._dblocks

    def _basis_big(self, i, side):
        if self.tree.is_leaf(i):
            return self.U(i) if side == "row" else self.V(i)
        return np.vstack([self._basis_big(c, side) @ (self.R(c) if side == "row" else self.W(c))
                          for c in self.tree.nodes[i].children])

    def todense(self):
        """Dense reconstruction from the generators (hss.py:175-187), a checker utility."""
        tr = self.tree
        out = np.zeros(self.shape)
        for i, j in self.pairs_L:
            out[np.ix_(tr.row_range(i), tr.col_range(j))] = \
                self._basis_big(i, "row") @ self.B(i, j) @ self._basis_big(j, "col").T
        for i, j in self.pairs_Lm:
            out[np.ix_(tr.row_range(i), tr.col_range(j))] = self.NF(i, j)
        res = np.empty_like(out)
        res[np.ix_(tr.perm_row, tr.perm_col)] = out
        return res

    # -- product on the device --------------------------------------------------------
    def matvec_device(self, Q, out=None, levelwise: bool = False):
        torch = _lib.torch_cuda()
        if Q.dim() != 2 or Q.shape[0] != self.n_col:
            raise ValueError("vector length %d does not match matrix (%d)" % (Q.shape[0], self.n_col))
        Q = Q.contiguous()
        if out is None:
            out = torch.empty((self.n_row, Q.shape[1]), dtype=torch.float64, device=Q.device)
        hs = (ctypes.c_void_p * len(self.terms))(*[A._h.value for A, _, _ in self.terms])
        _lib.check(_lib.load().smash_sum_matvec(len(self.terms), hs, _lib.ptr(self._dl), _lib.ptr(self._dr),
                                                _lib.ptr(Q), _lib.ptr(out), Q.shape[1], int(levelwise),
                                                _lib.stream_ptr()))
        return out


def _terms_of(M):
    if isinstance(M, ScaledSumHss):
        return list(M.terms)
    if getattr(M, "kind", None) != "hss" or not hasattr(M, "_h"):
        raise ValueError("expected an HSS matrix")
    return [(M, np.ones(M.n_row), np.ones(M.n_col))]


def diag_scale(M, dl, dr) -> ScaledSumHss:
    """diag(dl) @ M @ diag(dr), dl / dr in caller order (hss.py:352-381)."""
    dl = np.asarray(dl, dtype=np.float64)
    dr = np.asarray(dr, dtype=np.float64)
    if dl.shape != (M.n_row,) or dr.shape != (M.n_col,):
        raise ValueError("scaling vectors must match the matrix shape")
    return ScaledSumHss([(A, a * dl, b * dr) for A, a, b in _terms_of(M)])


def hss_add(A, B) -> ScaledSumHss:
    """Sum of two HSS matrices on the same tree (hss.py:317-342)."""
    if getattr(A, "kind", None) != "hss" or getattr(B, "kind", None) != "hss":
        raise ValueError("hss_add expects HSS matrices")
    if A.tree is not B.tree:
        raise ValueError("operands must share one cluster tree")
    return ScaledSumHss(_terms_of(A) + _terms_of(B))


def cauchy_like_hss(tree, X, Y, w, v, params: BuildParams = None) -> ScaledSumHss:
    """HSS form of sum_l diag(w[:, l]) C diag(v[:, l]), C the Cauchy matrix: one C
    build reused through diagonal scalings and sums (hss.py:384-400).  The B200 path
    builds C with the Chebyshev basis (pass basis='interp'; the Taylor basis is out of
    scope)."""
    w = np.asarray(w, dtype=float)
    v = np.asarray(v, dtype=float)
    if w.ndim != 2 or v.ndim != 2 or w.shape[1] != v.shape[1]:
        raise ValueError("generator matrices need matching column counts")
    base = build_hss(tree, KernelSpec(kind="cauchy"), X, Y, params)
    acc = None
    for l in range(w.shape[1]):
        term = diag_scale(base, w[:, l], v[:, l])
        acc = term if acc is None else hss_add(acc, term)
    return acc
