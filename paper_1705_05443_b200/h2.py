"""H^2 builder -- GPU drop-in for smash.h2 (/root/reference/pkg/src/smash/h2.py)."""

from __future__ import annotations

from .cluster import ClusterTree
from .hss import BuildParams, _StructuredMatrix, make_matrix
from .kernel import KernelSpec

__all__ = ["H2Matrix", "build_h2"]


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
