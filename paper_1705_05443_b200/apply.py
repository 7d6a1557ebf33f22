"""Fast matvec -- GPU drop-in for smash.apply.matvec_nodewise
(/root/reference/pkg/src/smash/apply.py:26-80)."""

from __future__ import annotations

import numpy as np

from . import _lib

__all__ = ["matvec_nodewise", "matvec_levelwise", "matvec_device", "MatvecStream",
           "UlvFactorization", "ulv_factor", "ulv_solve"]


def matvec_device(M, Q, out=None):
    """A @ Q for a CUDA float64 tensor Q of shape (n_col, nrhs); returns (n_row, nrhs)."""
    torch = _lib.torch_cuda()
    if hasattr(M, "terms"):  # algebra result (algebra.py): sum of scaled device matrices
        return M.matvec_device(Q, out)
    if getattr(M, "sharded_factors", False):
        raise ValueError("this rank holds only its share of the factors (build_h2_sharded with "
                         "replicate_factors=False): apply it with shard.ShardedMatvec")
    if Q.dim() != 2 or Q.shape[0] != M.n_col:
        raise ValueError("vector length %d does not match matrix (%d)" % (Q.shape[0], M.n_col))
    Q = Q.contiguous()
    if out is None:
        out = torch.empty((M.n_row, Q.shape[1]), dtype=torch.float64, device=Q.device)
    _lib.check(_lib.load().smash_matvec(M._h, _lib.ptr(Q), _lib.ptr(out), Q.shape[1], _lib.stream_ptr()))
    return out


def matvec_nodewise(M, q):
    """A @ q through the compressed representation, caller ordering (apply.py:34-80).
    q: (n,) or (n, nrhs), numpy or torch; the result has q's rank and container."""
    torch = _lib.torch_cuda()
    is_torch = isinstance(q, torch.Tensor)
    if not is_torch:
        q = np.asarray(q)
    if q.shape[0] != M.n_col:
        raise ValueError("vector length %d does not match matrix (%d)" % (q.shape[0], M.n_col))
    single = q.ndim == 1
    pinned = is_torch and not q.is_cuda and q.is_pinned()
    if pinned:  # host-pinned round trip: async copies on the current stream
        Q = q.to(device="cuda", dtype=torch.float64, non_blocking=True)
    else:
        Q = _lib.to_device(q)
    if single:
        Q = Q.reshape(-1, 1)
    Z = matvec_device(M, Q)
    if single:
        Z = Z[:, 0]
    if pinned:
        out = torch.empty(Z.shape, dtype=torch.float64, pin_memory=True)
        out.copy_(Z, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return out
    if is_torch:
        return Z.to(q.device)
    return Z.cpu().numpy()


def matvec_levelwise(M, q):
    """Level-synchronous matvec on perfect trees (apply.py:98-165): one device
    launch per tree level for each transfer pass, per-level coefficient blocks
    and the upward sum taken child by child (csrc/matvec_level.cu); ValueError
    unless every leaf is on the deepest level and every internal node has the
    same number of children (apply.py:83-95).  Same conventions as
    matvec_nodewise."""
    torch = _lib.torch_cuda()
    is_torch = isinstance(q, torch.Tensor)
    if not is_torch:
        q = np.asarray(q)
    if q.shape[0] != M.n_col:
        raise ValueError("vector length %d does not match matrix (%d)" % (q.shape[0], M.n_col))
    single = q.ndim == 1
    Q = _lib.to_device(q)
    if single:
        Q = Q.reshape(-1, 1)
    Q = Q.contiguous()
    if hasattr(M, "terms"):  # algebra result: every base through the level-wise product
        Z = M.matvec_device(Q, levelwise=True)
    else:
        Z = torch.empty((M.n_row, Q.shape[1]), dtype=torch.float64, device=Q.device)
        _lib.check(_lib.load().smash_matvec_levelwise(M._h, _lib.ptr(Q), _lib.ptr(Z), Q.shape[1],
                                                      _lib.stream_ptr()))
    if single:
        Z = Z[:, 0]
    if is_torch:
        return Z.to(q.device)
    return Z.cpu().numpy()


class MatvecStream:
    """Many A @ Q products with host-resident inputs and outputs, the copies of
    neighbouring products overlapped with the compute (B200 copy engines: one
    host->device and one device->host engine work concurrently with the SMs).

    ``submit(Q, Z)`` takes pinned host tensors Q (n_col, nrhs) and Z (n_row, nrhs)
    and returns at once; Z holds A @ Q once ``synchronize()`` (or the event returned
    by ``submit``) completes.  ``depth`` device buffer pairs rotate, so up to
    ``depth`` products are in flight: H2D(Q_k+1) || matvec(Q_k) || D2H(Z_k-1)."""

    def __init__(self, M, nrhs: int, depth: int = 2):
        torch = _lib.torch_cuda()
        self.M, self.nrhs, self.depth = M, int(nrhs), int(depth)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dQ = [torch.empty((M.n_col, nrhs), dtype=torch.float64, device=dev) for _ in range(depth)]
        self.dZ = [torch.empty((M.n_row, nrhs), dtype=torch.float64, device=dev) for _ in range(depth)]
        self.s_in = torch.cuda.Stream()
        self.s_mv = torch.cuda.Stream()
        self.s_out = torch.cuda.Stream()
        self.e_in = [torch.cuda.Event() for _ in range(depth)]
        self.e_mv = [torch.cuda.Event() for _ in range(depth)]
        self.e_out = [torch.cuda.Event() for _ in range(depth)]
        self.k = 0

    def submit(self, Q, Z, before=None):
        torch = _lib.torch_cuda()
        if Q.shape != (self.M.n_col, self.nrhs) or Z.shape != (self.M.n_row, self.nrhs):
            raise ValueError("MatvecStream: Q / Z shapes do not match the matrix and nrhs")
        i = self.k % self.depth
        with torch.cuda.stream(self.s_in):
            if self.k >= self.depth:
                self.s_in.wait_event(self.e_mv[i])   # slot's previous product consumed dQ[i]
            self.dQ[i].copy_(Q, non_blocking=True)
            self.e_in[i].record(self.s_in)
        with torch.cuda.stream(self.s_mv):
            self.s_mv.wait_event(self.e_in[i])
            if self.k >= self.depth:
                self.s_mv.wait_event(self.e_out[i])  # dZ[i] copied out before it is overwritten
            if before is not None:  # optional work ordered before the product (e.g. an L2 flush)
                before()
            matvec_device(self.M, self.dQ[i], self.dZ[i])
            self.e_mv[i].record(self.s_mv)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(self.e_mv[i])
            Z.copy_(self.dZ[i], non_blocking=True)
            self.e_out[i].record(self.s_out)
        self.k += 1
        return self.e_out[i]

    def synchronize(self):
        self.s_out.synchronize()


# ---------------------------------------------------------------------------
# ULV factorization and solve (apply.py:168-354) -- device factorisation
# ---------------------------------------------------------------------------


class UlvFactorization:
    """GPU ULV factorisation of an HSS matrix (UlvFactorization, apply.py:186-196).
    Holds the device handle and a reference to the matrix it factors."""

    def __init__(self, matrix, handle):
        self.matrix = matrix
        self._h = handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.smash_ulv_free(h)
            self._h = None

    def solve(self, b):
        return ulv_solve(self, b)


def ulv_factor(M) -> UlvFactorization:
    """Factor an HSS matrix for repeated solves (apply.py:237-288).  Raises
    ValueError for non-HSS input and numpy.linalg.LinAlgError when a local
    elimination block or the root system is numerically singular (the message
    names the node)."""
    import ctypes
    if getattr(M, "kind", None) != "hss":
        raise ValueError("ULV factorization expects an HSS matrix")
    if hasattr(M, "terms"):
        raise NotImplementedError("the device ULV factors built (interpolative) HSS matrices; "
                                  "algebra results (hss_add / diag_scale / cauchy_like_hss) "
                                  "are applied with matvec_nodewise only")
    h = ctypes.c_void_p()
    rc = _lib.load().smash_ulv_factor(M._h, _lib.stream_ptr(), ctypes.byref(h))
    if rc == 3:
        raise np.linalg.LinAlgError(_lib.last_error())
    _lib.check(rc)
    return UlvFactorization(M, h)


def ulv_solve(F: UlvFactorization, b):
    """Solve A x = b with a ULV factorisation (apply.py:291-348); b is (n,) or
    (n, nrhs), numpy or torch; the result has b's rank and container."""
    torch = _lib.torch_cuda()
    M = F.matrix
    is_torch = isinstance(b, torch.Tensor)
    if not is_torch:
        b = np.asarray(b)
    if b.shape[0] != M.n_row:
        raise ValueError("right-hand side length %d does not match matrix (%d)" % (b.shape[0], M.n_row))
    single = b.ndim == 1
    B = _lib.to_device(b)
    if single:
        B = B.reshape(-1, 1)
    B = B.contiguous()
    X = torch.empty((M.n_col, B.shape[1]), dtype=torch.float64, device=B.device)
    _lib.check(_lib.load().smash_ulv_solve(F._h, _lib.ptr(B), _lib.ptr(X), B.shape[1], _lib.stream_ptr()))
    if single:
        X = X[:, 0]
    if is_torch:
        return X.to(b.device)
    return X.cpu().numpy()
