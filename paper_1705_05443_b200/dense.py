"""Exact-product oracle on the GPU -- drop-in for smash.bench.dense_matvec
(/root/reference/pkg/src/smash/bench.py:284-296) at sizes where the streaming CPU
oracle takes hours.  K(X, Y) is evaluated tile by tile in the sm_100a kernel
k_dense (csrc/dense.cu) and never stored.  Used to check the compressed matvec
against the exact product (SURVEY.md 8(c) rule 5); not on the compressed path.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .kernel import KernelSpec

__all__ = ["dense_matvec", "relative_error"]


def _dev_coords(P):
    torch = _lib.torch_cuda()
    if hasattr(P, "_dev") and P._dev is not None:
        return P._dev
    c = P.coords if hasattr(P, "coords") else P
    if isinstance(c, torch.Tensor):
        c = c.to(device="cuda", dtype=torch.float64)
        return (c.reshape(-1, 1) if c.dim() == 1 else c).contiguous()
    c = np.asarray(c, dtype=np.float64)
    return _lib.to_device(c.reshape(-1, 1) if c.ndim == 1 else c)


def dense_matvec(spec: KernelSpec, X, Y, q, chunk: int = None):
    """Exact A @ q with A = K(X, Y) (caller order).  X / Y: PointSet, numpy or torch
    (n, d); q: (n_col,) or (n_col, nrhs).  Returns the same container / rank as q."""
    torch = _lib.torch_cuda()
    dX, dY = _dev_coords(X), _dev_coords(Y)
    if dX.shape[1] != dY.shape[1]:
        raise ValueError("X and Y have different dimensions")
    is_torch = isinstance(q, torch.Tensor)
    Q = q.to(device="cuda", dtype=torch.float64) if is_torch else _lib.to_device(np.asarray(q))
    single = Q.dim() == 1
    Q = Q.reshape(Q.shape[0], -1).contiguous()
    if Q.shape[0] != dY.shape[0]:
        raise ValueError("vector length %d does not match matrix (%d)" % (Q.shape[0], dY.shape[0]))
    Z = torch.empty((dX.shape[0], Q.shape[1]), dtype=torch.float64, device="cuda")
    _lib.check(_lib.load().smash_dense_matvec(spec.code, spec.dx_value, dX.shape[1], _lib.ptr(dX),
                                              dX.shape[0], _lib.ptr(dY), dY.shape[0], _lib.ptr(Q),
                                              Q.shape[1], _lib.ptr(Z), _lib.stream_ptr()))
    if single:
        Z = Z[:, 0]
    if is_torch:
        return Z.to(q.device)
    return Z.cpu().numpy()


def relative_error(z, z_exact) -> float:
    """||z - z_exact|| / ||z_exact|| (Frobenius over all right-hand sides)."""
    z, z_exact = np.asarray(z), np.asarray(z_exact)
    return float(np.linalg.norm(z - z_exact) / max(np.linalg.norm(z_exact), 1e-300))
