"""paper_1705_05443_b200 -- B200-native SMASH hot path (arXiv 1705.05443).

Drop-in for the reference package's tree / construct / matvec path
(``smash.build_tree``, ``leaf_sets``, ``nearfield_set``, ``build_h2``,
``build_hss``, ``matvec_nodewise`` and the objects they return).  All compute
runs in hand-written sm_100a CUDA kernels behind the C ABI in
include/smash_b200.h (libsmash_b200.so, loaded with ctypes); there is no CPU
fallback.
"""

from .cluster import (Box, ClusterTree, PointSet, TreeNode, build_tree, leaf_sets, nearfield_set,
                      well_separated)
from .kernel import KernelSpec, kernel_block
from .lowrank import InterpolativeFactor, compr, interp_basis
from .hss import BuildParams, HssMatrix, build_hss, build_hss_sharded
from .h2 import H2Matrix, build_h2, build_h2_local, build_h2_sharded
from .apply import (MatvecStream, UlvFactorization, matvec_device, matvec_levelwise, matvec_nodewise,
                    ulv_factor, ulv_solve)
from .dense import dense_matvec, relative_error
from .container import load_matrix, save_matrix
from .algebra import ScaledSumHss, cauchy_like_hss, diag_scale, hss_add

__version__ = "0.1.0"

__all__ = [
    "Box", "BuildParams", "ClusterTree", "H2Matrix", "HssMatrix", "InterpolativeFactor",
    "KernelSpec", "PointSet", "TreeNode", "build_h2", "build_h2_local", "build_h2_sharded", "build_hss", "build_hss_sharded", "build_tree", "compr",
    "interp_basis", "kernel_block", "leaf_sets", "matvec_device", "matvec_levelwise", "matvec_nodewise",
    "dense_matvec", "relative_error", "MatvecStream",
    "nearfield_set", "well_separated", "save_matrix", "load_matrix",
    "UlvFactorization", "ulv_factor", "ulv_solve",
    "ScaledSumHss", "cauchy_like_hss", "diag_scale", "hss_add",
]
