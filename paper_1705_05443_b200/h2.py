"""H^2 builder -- GPU drop-in for smash.h2 (/root/reference/pkg/src/smash/h2.py)."""

from __future__ import annotations

from .cluster import ClusterTree
import ctypes

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
                   world: int = 1, cut_level: int = 0, use_cache: bool = True) -> PendingH2Build:
    """Phase 1 of the sharded construction for ``rank`` of ``world``."""
    params = params or BuildParams()
    if tree.mode != "2d" and tree.dim != 1:
        raise ValueError("H2 construction expects a 2^d-mode tree")
    _resolve_basis(params, kernel)
    p = _lib.BuildParamsC(structure=_lib.STRUCT["h2"], kernel=kernel.code,
                          dx=kernel.dx_value if kernel.dx_value == kernel.dx_value else 0.0,
                          r=int(params.r), tau=float(params.tau), s=float(params.s),
                          rtol=float(params.rtol), eps_svd=float(params.eps_svd))
    h = ctypes.c_void_p()
    _lib.check(_lib.load().smash_matrix_build_local(tree._h, ctypes.byref(p), int(rank), int(world),
                                                    int(cut_level), _lib.stream_ptr(), ctypes.byref(h)))
    return PendingH2Build(tree, params, kernel, h, use_cache)


def build_h2_sharded(tree: ClusterTree, kernel: KernelSpec, X=None, Y=None, params: BuildParams = None,
                     group=None, cut_level: int = 0, use_cache: bool = True) -> H2Matrix:
    """H^2 construction sharded over the ranks of a torch.distributed process group
    (NCCL over NVLink on a B200 node): every rank compresses the subtrees of its
    contiguous share of the cut level, one all-reduce per factor buffer replaces
    the cut-level all-gather (the shares are disjoint and zero elsewhere), and
    the top levels are compressed redundantly.  Every rank ends with the full
    matrix, bit-identical to build_h2's."""
    import torch.distributed as dist
    pend = build_h2_local(tree, kernel, params, dist.get_rank(group), dist.get_world_size(group),
                          cut_level, use_cache)
    for b in pend.buffers():
        dist.all_reduce(b, group=group)
    return pend.finish()
