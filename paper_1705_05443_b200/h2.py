"""H^2 builder -- GPU drop-in for smash.h2 (/root/reference/pkg/src/smash/h2.py)."""

from __future__ import annotations

from .cluster import ClusterTree
import ctypes

import numpy as np

from . import _lib
from .hss import BuildParams, _StructuredMatrix, _resolve_basis, make_matrix
from .kernel import KernelSpec

__all__ = ["H2Matrix", "build_h2", "build_h2_local", "build_h2_sharded"]


class H2Matrix(_StructuredMatrix):
    kind = "h2"


def build_h2(tree: ClusterTree, kernel: KernelSpec, X=None, Y=None, params: BuildParams = None,
             use_cache: bool = True) -> H2Matrix:
    """GPU bottom-up H^2 construction under strong admissibility (replaces
    h2.py:25-54).  X / Y are accepted for signature compatibility."""
    params = params or BuildParams()
    if tree.mode != "2d" and tree.dim != 1:
        raise ValueError("H2 construction expects a 2^d-mode tree")
    return make_matrix(H2Matrix, tree, kernel, params, use_cache)


class _DevView:
    """__cuda_array_interface__ view of a library-owned device buffer."""

    TYPESTR = {0: "<i4", 1: "<f8", 2: "<i8"}

    def __init__(self, ptr: int, n: int, dtype: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": self.TYPESTR[dtype],
                                         "data": (ptr, False), "version": 3, "strides": None}


class PendingH2Build:
    """Phase 1 of a sharded H^2 build (one rank's share of the levels at and below
    the cut); ``buffers()`` lists the device buffers to sum over the ranks,
    ``finish()`` compacts the cut levels, compresses the top levels and returns
    the H2Matrix (identical to build_h2's)."""

    def __init__(self, tree, params, kernel, handle, use_cache):
        self.tree, self.params, self.kernel, self._h, self.use_cache = tree, params, kernel, handle, use_cache

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.smash_matrix_free(h)
            self._h = None

    def buffers(self):
        import torch
        cap = 16
        n = _lib.c_i64()
        ptrs = (ctypes.c_void_p * cap)()
        counts = (ctypes.c_int64 * cap)()
        dts = (ctypes.c_int32 * cap)()
        _lib.check(_lib.load().smash_matrix_exchange_buffers(self._h, cap, ctypes.byref(n), ptrs, counts, dts))
        return [torch.as_tensor(_DevView(ptrs[i], counts[i], dts[i]), device="cuda") for i in range(n.value)]

    def finish(self) -> H2Matrix:
        _lib.check(_lib.load().smash_matrix_build_finish(self._h, _lib.stream_ptr()))
        M = H2Matrix(self.tree, self.params, self.kernel, self._h, self.use_cache)
        self._h = None
        return M


def build_h2_local(tree: ClusterTree, kernel: KernelSpec, params: BuildParams = None, rank: int = 0,
                   world: int = 1, cut_level: int = 0, use_cache: bool = True, cut_weight=None,
                   replicate_factors: bool = True) -> PendingH2Build:
    """Phase 1 of the sharded construction for ``rank`` of ``world``.
    cut_weight: per cut-level node (left to right) work used to balance the ranks' ranges
    (default: point counts); replicate_factors=False keeps perm / G out of the exchange."""
    params = params or BuildParams()
    if tree.mode != "2d" and tree.dim != 1:
        raise ValueError("H2 construction expects a 2^d-mode tree")
    _resolve_basis(params, kernel)
    p = _lib.BuildParamsC(structure=_lib.STRUCT["h2"], kernel=kernel.code,
                          dx=kernel.dx_value if kernel.dx_value == kernel.dx_value else 0.0,
                          r=int(params.r), tau=float(params.tau), s=float(params.s),
                          rtol=float(params.rtol), eps_svd=float(params.eps_svd))
    h = ctypes.c_void_p()
    cw = None if cut_weight is None else np.ascontiguousarray(cut_weight, np.float64)
    _lib.check(_lib.load().smash_matrix_build_local_w(
        tree._h, ctypes.byref(p), int(rank), int(world), int(cut_level),
        None if cw is None else cw.ctypes.data_as(ctypes.c_void_p), int(bool(replicate_factors)),
        _lib.stream_ptr(), ctypes.byref(h)))
    pend = PendingH2Build(tree, params, kernel, h, use_cache)
    pend.replicate_factors = bool(replicate_factors)
    return pend


def shard_cut(tree: ClusterTree, world: int, cut_level: int = 0) -> int:
    """Cut level of a sharded build over ``world`` ranks (the shallowest level with
    >= 8 nodes per rank, unless cut_level >= 2 is given)."""
    c = ctypes.c_int32()
    _lib.check(_lib.load().smash_matrix_shard_cut(tree._h, int(world), int(cut_level), ctypes.byref(c)))
    return c.value


def build_h2_sharded(tree: ClusterTree, kernel: KernelSpec, X=None, Y=None, params: BuildParams = None,
                     group=None, cut_level: int = 0, use_cache: bool = True,
                     replicate_factors: bool = False) -> H2Matrix:
    """H^2 construction sharded over the ranks of a torch.distributed process group
    (NCCL over NVLink on a B200 node).  The cut-level nodes are split into contiguous
    ranges of equal matvec work (shard.subtree_work: coupling + nearfield interactions of
    the subtrees); every rank compresses its subtrees, the cut-level exchange sums the
    disjoint, zero-filled ranks / |ibar| / ordered skeleton labels and coordinates over
    the ranks (float64 buffers summed as int64 bit patterns: bit-exact), and the top
    levels are compressed redundantly.  With replicate_factors=False (default) perm and
    G stay on their owner: each rank holds the factors of its subtrees and of the top
    levels -- what the sharded matvec (shard.ShardedMatvec, same partition) reads; with
    True every rank ends with the full matrix, bit-identical to build_h2's."""
    import torch
    import torch.distributed as dist
    from .cluster import _pairs
    from .shard import cut_partition, subtree_work
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    params = params or BuildParams()
    A = tree.arrays()
    cut = shard_cut(tree, world, cut_level)
    L, Lm = _pairs(tree, params.tau, "h2")
    w = subtree_work(A, L, Lm, params.r)
    owner, cut_nodes = cut_partition(A, world, cut, w[np.nonzero(A["level"] == cut)[0]])
    pend = build_h2_local(tree, kernel, params, rank, world, cut, use_cache,
                          cut_weight=w[cut_nodes], replicate_factors=replicate_factors)
    gloo = dist.get_backend(group) == "gloo"
    for b in pend.buffers():
        t = b.view(torch.int64) if b.dtype == torch.float64 else b  # bit patterns: exact sums
        if gloo:
            h = t.cpu()
            dist.all_reduce(h, group=group)
            t.copy_(h)
        else:
            dist.all_reduce(t, group=group)
    M = pend.finish()
    own = np.zeros(len(A["level"]), np.int64)
    _lib.check(_lib.load().smash_matrix_shard_owner(M._h, own.ctypes.data_as(ctypes.c_void_p)))
    assert np.array_equal(own, owner), "build and host partitions differ"
    M.shard_owner = own
    M.sharded_factors = not replicate_factors
    return M
