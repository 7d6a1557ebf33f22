"""Multi-GPU sharding of the matvec: one process per GPU,
torch.distributed (NCCL) for the single data-path exchange.

Partition: the tree is cut at a frontier of nodes (expanded from the root,
largest row count first, until there are >= 8 frontier nodes per rank); the
frontier, taken left to right, is split into contiguous groups of roughly equal
row count.  A rank owns the subtrees of its frontier nodes (a contiguous range
of tree-order rows); the frontier's ancestors ("top" nodes) are replicated.

Matvec on rank r:
  stage 1  gather q, upward pass of the owned subtrees; coefficients of all
           other nodes are zero;
  exchange all-reduce (sum) of the coefficient buffer -- the supports are
           disjoint, so this is the all-gather of the skeleton coefficients at
           the cut level;
  stage 2  upward pass of the top nodes (replicated), coupling / downward pass
           for owned + top targets, nearfield + leaf far field for the owned
           leaves: the owned rows of z (disjoint over ranks, no reduction);
  optional all-reduce of z when every rank needs the full result.
The partition is plain host logic (numpy) and is exercised with gloo on CPU in
tests/test_shard_gloo.py.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

__all__ = ["partition", "ShardedMatvec"]


def partition(A: dict, world: int, per_rank: int = 8):
    """Frontier partition of a tree given its exported arrays (postorder ids).

    Returns (owned, top, frontier_owner): owned[r] = int64 array of rank r's
    subtree nodes, top = the replicated ancestors (incl. the root), and the
    frontier list with its owners."""
    child_ptr, child_idx = A["child_ptr"], A["child_idx"]
    rs, re = A["row_start"], A["row_stop"]
    n = len(child_ptr) - 1
    root = n - 1

    def kids(i):
        return child_idx[child_ptr[i]:child_ptr[i + 1]]

    frontier = [root]
    while len(frontier) < per_rank * world:
        internal = [f for f in frontier if child_ptr[f + 1] > child_ptr[f]]
        if not internal:
            break
        big = max(internal, key=lambda f: (re[f] - rs[f], -f))
        frontier.remove(big)
        frontier.extend(int(c) for c in kids(big))
    frontier.sort(key=lambda f: (rs[f], re[f]))
    total = max(int(re[root] - rs[root]), 1)
    owner = {}
    acc = 0
    for f in frontier:
        mid = acc + (re[f] - rs[f]) / 2.0
        owner[f] = min(world - 1, int(mid * world / total))
        acc += re[f] - rs[f]
    owned = [[] for _ in range(world)]
    in_sub = np.zeros(n, bool)
    for f in frontier:
        stack = [f]
        while stack:
            v = stack.pop()
            in_sub[v] = True
            owned[owner[f]].append(v)
            stack.extend(int(c) for c in kids(v))
    owned = [np.array(sorted(o), dtype=np.int64) for o in owned]
    top = np.nonzero(~in_sub)[0].astype(np.int64)
    return owned, top, [(f, owner[f]) for f in frontier]


class _DevBuf:
    """__cuda_array_interface__ view of a library-owned device buffer."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


class ShardedMatvec:
    """Rank-local sharded matvec of a (replicated) matrix M over a process group."""

    def __init__(self, M, group=None, per_rank: int = 8):
        import torch.distributed as dist
        self.M = M
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        owned, top, self.frontier = partition(M.tree.arrays(), self.world, per_rank)
        self.owned = owned[self.rank]
        self.top = top
        own = np.ascontiguousarray(self.owned)
        tp = np.ascontiguousarray(top)
        _lib.check(_lib.load().smash_matvec_set_partition(
            M._h, own.ctypes.data_as(ctypes.c_void_p), own.size, tp.ctypes.data_as(ctypes.c_void_p),
            tp.size, _lib.stream_ptr()))

    def coeff_view(self, nrhs: int):
        import torch
        p = ctypes.c_void_p()
        rows = _lib.c_i64()
        _lib.check(_lib.load().smash_matvec_coeffs(self.M._h, ctypes.byref(p), ctypes.byref(rows)))
        return torch.as_tensor(_DevBuf(p.value, rows.value * nrhs), device="cuda")

    def __call__(self, Q, gather_output: bool = True):
        """Q: (n_col, nrhs) CUDA float64, replicated on every rank (nrhs a power of
        two <= 16).  Returns z (n_row, nrhs): the owned rows (others 0), or the full
        product when gather_output."""
        import torch
        import torch.distributed as dist
        Q = Q.contiguous()
        nrhs = Q.shape[1]
        lib = _lib.load()
        z = torch.zeros((self.M.n_row, nrhs), dtype=torch.float64, device=Q.device)
        _lib.check(lib.smash_matvec_stage(self.M._h, 1, _lib.ptr(Q), _lib.ptr(z), nrhs, _lib.stream_ptr()))
        dist.all_reduce(self.coeff_view(nrhs), group=self.group)
        _lib.check(lib.smash_matvec_stage(self.M._h, 2, _lib.ptr(Q), _lib.ptr(z), nrhs, _lib.stream_ptr()))
        if gather_output:
            dist.all_reduce(z, group=self.group)
        return z
