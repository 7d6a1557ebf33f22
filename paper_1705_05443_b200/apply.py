"""Fast matvec -- GPU drop-in for smash.apply.matvec_nodewise
(/root/reference/pkg/src/smash/apply.py:26-80)."""

from __future__ import annotations

import numpy as np

from . import _lib

__all__ = ["matvec_nodewise", "matvec_levelwise", "matvec_device"]


def matvec_device(M, Q, out=None):
    """A @ Q for a CUDA float64 tensor Q of shape (n_col, nrhs); returns (n_row, nrhs)."""
    torch = _lib.torch_cuda()
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


def _check_perfect(tree):
    """All leaves at the deepest level and a uniform child count (apply.py:83-95)."""
    A = tree.arrays()
    depth = int(A["level"].max())
    nch = np.diff(A["child_ptr"])
    leaf = nch == 0
    if np.any(A["level"][leaf] != depth):
        raise ValueError("level-synchronous matvec needs all leaves at the deepest level")
    inner = nch[~leaf]
    if inner.size and np.any(inner != inner[0]):
        raise ValueError("level-synchronous matvec needs a perfect tree")


def matvec_levelwise(M, q):
    """Level-synchronous matvec on perfect trees (apply.py:98-165).  The device
    matvec is already level-synchronous (one persistent upward pass ordered
    deepest level first, the coupling of every node at once, one downward pass
    ordered shallowest level first), so on a perfect tree this is the same
    computation as matvec_nodewise; the reference's perfect-tree contract is kept."""
    _check_perfect(M.tree)
    return matvec_nodewise(M, q)
