"""Kernel specifications and exact kernel blocks -- GPU drop-in for the parts of
smash.kernel (/root/reference/pkg/src/smash/kernel.py) on the hot path.

Kinds: the reference's real 1-D ``cauchy`` 1/(x-y) (kernel.py:286-298) plus the
BASELINE kernels ``log`` (log|x-y|), ``inv_r`` (1/|x-y|) and ``exp``
(exp(-|x-y|)) that the reference lacks.  ``cauchy_like`` and
``laplace_dlp`` are outside this build's scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["KernelSpec", "kernel_block"]

_OUT_OF_SCOPE = ("cauchy_like", "laplace_dlp")


@dataclass
class KernelSpec:
    """Kernel kind plus the value used at coincident points (KernelSpec, kernel.py:200-233).

    ``dx`` defaults to 0 for log / inv_r (BASELINE "diagonal set to 0"); exp keeps
    its natural diagonal exp(0) = 1; cauchy requires dx only if points coincide.
    """

    kind: str
    dx: float = None

    def __post_init__(self):
        if self.kind in _OUT_OF_SCOPE:
            raise ValueError("kernel kind %r is outside the B200 hot path (see DESIGN.md)" % self.kind)
        if self.kind not in _lib.KERNEL:
            raise ValueError("unknown kernel kind %r" % self.kind)

    @property
    def code(self) -> int:
        return _lib.KERNEL[self.kind]

    @property
    def dx_value(self) -> float:
        if self.kind == "exp":
            return 1.0
        if self.dx is None:
            return 0.0 if self.kind in ("log", "inv_r") else float("nan")
        return float(self.dx)


def kernel_block(spec: KernelSpec, X, Y, rows, cols) -> np.ndarray:
    """Exact kernel submatrix A[rows, cols] in caller order (kernel.py:278-310),
    evaluated on the GPU."""
    Xc = X.coords if hasattr(X, "coords") else np.atleast_2d(np.asarray(X, dtype=np.float64))
    Yc = Y.coords if hasattr(Y, "coords") else np.atleast_2d(np.asarray(Y, dtype=np.float64))
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    return kernel_block_coords(spec, Xc[rows], Yc[cols])


def kernel_block_coords(spec: KernelSpec, Xr: np.ndarray, Yc: np.ndarray) -> np.ndarray:
    Xr = np.ascontiguousarray(Xr, dtype=np.float64)
    Yc = np.ascontiguousarray(Yc, dtype=np.float64)
    if Xr.shape[0] == 0 or Yc.shape[0] == 0:
        return np.zeros((Xr.shape[0], Yc.shape[0]))
    dX, dY = _lib.to_device(Xr), _lib.to_device(Yc)
    out = _lib.empty((Xr.shape[0], Yc.shape[0]))
    _lib.check(_lib.load().smash_kernel_block(spec.code, spec.dx_value, Xr.shape[1], _lib.ptr(dX),
                                              Xr.shape[0], _lib.ptr(dY), Yc.shape[0], _lib.ptr(out),
                                              _lib.stream_ptr()))
    res = out.cpu().numpy()
    if spec.kind == "cauchy" and spec.dx is None and Xr.shape[1] == 1:
        if np.any(Xr[:, 0][:, None] == Yc[:, 0][None, :]):
            raise ValueError("coincident points need a diagonal value d_x")
    return res
