"""ctypes binding of the C ABI (include/smash_b200.h) -- the only way the Python
layer reaches the GPU.  There is no CPU fallback: if the library or a CUDA device
is missing, every compute entry point raises."""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SMASH_LIB") or os.path.join(HERE, "libsmash_b200.so")

SMASH_OK, SMASH_ERR_INVALID, SMASH_ERR_NUMERICAL, SMASH_ERR_CUDA = 0, 2, 3, 4
MODE = {"binary": 0, "2d": 1, "2^d": 1}
STRUCT = {"h2": 0, "hss": 1}
KERNEL = {"log": 0, "inv_r": 1, "exp": 2, "cauchy": 3}

c_i32, c_i64, c_dbl, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
P_i32, P_i64, P_dbl = ctypes.POINTER(c_i32), ctypes.POINTER(c_i64), ctypes.POINTER(c_dbl)


# smash_exchange_fn (include/smash_b200.h)
EXCHANGE_FN = ctypes.CFUNCTYPE(c_i32, c_vp, c_i64, ctypes.POINTER(c_vp), ctypes.POINTER(c_i64),
                               ctypes.POINTER(c_i32))


class BuildParamsC(ctypes.Structure):
    _fields_ = [("structure", c_i32), ("kernel", c_i32), ("dx", c_dbl), ("r", c_i32),
                ("tau", c_dbl), ("s", c_dbl), ("rtol", c_dbl), ("eps_svd", c_dbl)]


# symbol -> (restype, argtypes); every symbol declared in include/smash_b200.h
SIGNATURES = {
    "smash_abi_version": (c_i32, []),
    "smash_last_error": (ctypes.c_char_p, []),
    "smash_tree_build": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_i32, c_i32, c_i32, c_vp,
                                 ctypes.POINTER(c_vp)]),
    "smash_tree_sizes": (c_i32, [c_vp, P_i64, P_i32, P_i64, P_i64, P_i32, P_i32]),
    "smash_tree_export": (c_i32, [c_vp] + [c_vp] * 14 + [c_vp]),
    "smash_tree_free": (c_i32, [c_vp]),
    "smash_leaf_sets": (c_i32, [c_vp, c_dbl, c_i32, c_vp, P_i64, P_i64]),
    "smash_leaf_sets_export": (c_i32, [c_vp, c_dbl, c_i32, c_vp, c_vp, c_vp]),
    "smash_nearfield": (c_i32, [c_vp, c_dbl, c_vp, P_i64]),
    "smash_nearfield_export": (c_i32, [c_vp, c_dbl, c_vp, c_vp, c_vp]),
    "smash_matrix_build": (c_i32, [c_vp, ctypes.POINTER(BuildParamsC), c_vp, ctypes.POINTER(c_vp)]),
    "smash_matrix_build_local": (c_i32, [c_vp, ctypes.POINTER(BuildParamsC), c_i32, c_i32, c_i32,
                                         c_vp, ctypes.POINTER(c_vp)]),
    "smash_matrix_import": (c_i32, [c_vp, ctypes.POINTER(BuildParamsC), c_i32] + [c_vp] * 7 +
                            [c_vp, ctypes.POINTER(c_vp)]),
    "smash_matrix_exchange_buffers": (c_i32, [c_vp, c_i64, P_i64, c_vp, c_vp, c_vp]),
    "smash_matrix_build_finish": (c_i32, [c_vp, c_vp]),
    "smash_matrix_sizes": (c_i32, [c_vp, c_i32, P_i64, P_i64, P_i64, P_i64]),
    "smash_matrix_export": (c_i32, [c_vp, c_i32] + [c_vp] * 8 + [c_vp]),
    "smash_matrix_stats": (c_i32, [c_vp, P_i64, P_i64]),
    "smash_ulv_factor": (c_i32, [c_vp, c_vp, ctypes.POINTER(c_vp)]),
    "smash_ulv_solve": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_vp]),
    "smash_ulv_free": (c_i32, [c_vp]),
    "smash_matvec": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_vp]),
    "smash_matvec_levelwise": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_vp]),
    "smash_matrix_build_sharded": (c_i32, [c_vp, ctypes.POINTER(BuildParamsC), c_i32, c_i32, c_vp,
                                           c_vp, c_vp, ctypes.POINTER(c_vp)]),
    "smash_matrix_build_local_w": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_i32, c_vp, c_vp]),
    "smash_matrix_shard_cut": (c_i32, [c_vp, c_i32, c_i32, c_vp]),
    "smash_matrix_shard_owner": (c_i32, [c_vp, c_vp]),
    "smash_matvec_coeff_layout": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "smash_sum_matvec": (c_i32, [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp]),
    "smash_matvec_profile": (c_i32, [c_vp, c_i32, P_dbl, P_i64]),
    "smash_matvec_set_partition": (c_i32, [c_vp, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "smash_matvec_stage": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_i64, c_vp]),
    "smash_matvec_coeffs": (c_i32, [c_vp, ctypes.POINTER(c_vp), P_i64]),
    "smash_matrix_free": (c_i32, [c_vp]),
    "smash_kernel_block": (c_i32, [c_i32, c_dbl, c_i32, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "smash_dense_matvec": (c_i32, [c_i32, c_dbl, c_i32, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "smash_interp_basis": (c_i32, [c_i32, P_dbl, P_dbl, c_vp, c_i64, c_i32, c_vp, c_vp]),
    "smash_compr": (c_i32, [c_vp, c_i64, c_i64, c_dbl, c_dbl, c_vp, c_vp, P_i64, P_i64, c_vp]),
}

_lib = None


def load():
    """Load libsmash_b200.so (built by paper_1705_05443_b200._build / __graft_entry__.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libsmash_b200.so not built (run __graft_entry__.build()); "
                              "the CUDA extension is required -- there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    return load().smash_last_error().decode(errors="replace")


def check(status: int):
    if status == SMASH_OK:
        return
    msg = load().smash_last_error().decode(errors="replace")
    if status == SMASH_ERR_INVALID:
        raise ValueError(msg)
    raise RuntimeError(msg)


# ---------------------------------------------------------------------------
# torch plumbing (device buffers and streams only)
# ---------------------------------------------------------------------------

def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1705_05443_b200 needs a CUDA device (sm_100a B200); "
                           "there is no CPU fallback")
    return torch


def stream_ptr():
    torch = torch_cuda()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def to_device(a, dtype="float64"):
    """numpy / torch -> contiguous CUDA tensor (float64 or int64)."""
    torch = torch_cuda()
    tdt = torch.float64 if dtype == "float64" else torch.int64
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=tdt).contiguous()
    arr = np.ascontiguousarray(np.asarray(a), dtype=np.float64 if dtype == "float64" else np.int64)
    return torch.from_numpy(arr).to("cuda")


def empty(shape, dtype="float64"):
    torch = torch_cuda()
    tdt = torch.float64 if dtype == "float64" else torch.int64
    return torch.empty(shape, dtype=tdt, device="cuda")


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() else ctypes.c_void_p(0)
