"""Low-rank primitives -- GPU drop-in for the hot-path parts of smash.lowrank
(/root/reference/pkg/src/smash/lowrank.py): the Chebyshev/Lagrange basis
(lowrank.py:123-144, extended to 3-D) and interpolative compression via strong
RRQR (lowrank.py:170-255).  Each call runs the same sm_100a kernels the batched
builders use, on a single node.  The Taylor basis is out of scope (BASELINE
mandates Chebyshev interpolation).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["InterpolativeFactor", "interp_basis", "compr"]


@dataclass
class InterpolativeFactor:
    """Row interpolation C ~= X C[skel_local], X = P [I; G] (lowrank.py:206-229)."""

    nrows: int
    perm: np.ndarray
    G: np.ndarray
    skel: np.ndarray
    skel_local: np.ndarray

    @property
    def rank(self) -> int:
        return self.skel.size

    def expand(self) -> np.ndarray:
        X = np.zeros((self.nrows, self.rank), dtype=self.G.dtype)
        X[self.perm[:self.rank]] = np.eye(self.rank, dtype=self.G.dtype)
        if self.rank < self.nrows:
            X[self.perm[self.rank:]] = self.G
        return X


def interp_basis(box, pts: np.ndarray, r: int) -> np.ndarray:
    """Lagrange basis at the box's Chebyshev nodes, evaluated at pts (GPU)."""
    pts = np.atleast_2d(np.asarray(pts, dtype=np.float64))
    lo = np.ascontiguousarray(box.lo, dtype=np.float64)
    hi = np.ascontiguousarray(box.hi, dtype=np.float64)
    if pts.shape[0] == 0:
        return np.zeros((0, r))
    if pts.shape[1] != lo.size:
        raise ValueError("point dimension does not match the box")
    d = _lib.to_device(pts)
    out = _lib.empty((pts.shape[0], r))
    P = ctypes.POINTER(ctypes.c_double)
    _lib.check(_lib.load().smash_interp_basis(lo.size, lo.ctypes.data_as(P), hi.ctypes.data_as(P),
                                              _lib.ptr(d), pts.shape[0], r, _lib.ptr(out),
                                              _lib.stream_ptr()))
    return out.cpu().numpy()


def compr(C: np.ndarray, ibar: np.ndarray, s: float = 2.0, rank: int = None,
          rtol: float = 1e-14) -> InterpolativeFactor:
    """Interpolative row compression of C labelled by ibar (lowrank.py:232-255),
    with the sRRQR of C^T run by one CTA on the GPU."""
    if rank is not None:
        raise NotImplementedError("a fixed rank cut is not used on the hot path")
    C = np.atleast_2d(np.asarray(C, dtype=np.float64))
    ibar = np.asarray(ibar, dtype=np.int64)
    if C.shape[0] != ibar.size:
        raise ValueError("row labels do not match C")
    n, m = C.shape
    perm = _lib.empty(max(n, 1), "int64")
    G = _lib.empty(max(n * max(min(n, m), 1), 1))
    k, sw = _lib.c_i64(), _lib.c_i64()
    dC = _lib.to_device(C) if C.size else None
    _lib.check(_lib.load().smash_compr(_lib.ptr(dC), n, m, float(s), float(rtol), _lib.ptr(perm),
                                       _lib.ptr(G), ctypes.byref(k), ctypes.byref(sw),
                                       _lib.stream_ptr()))
    k = k.value
    p = perm.cpu().numpy()[:n]
    g = G.cpu().numpy()[:(n - k) * k].reshape(n - k, k) if 0 < k else np.zeros((n, 0))
    return InterpolativeFactor(nrows=n, perm=p, G=g, skel=ibar[p[:k]], skel_local=p[:k].copy())
