"""Test configuration: the ``gpu`` marker and shared helpers.

CPU (``-m "not gpu"``) tests: the oracle against the reference-generated
golden fixtures, host-side logic, the C-ABI library's symbol table and the
gloo multi-rank host logic.  GPU (``-m gpu``) tests: parity of the CUDA path
(through the C ABI) against the golden fixtures and the oracle.
"""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    d = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    out = {k: d[k] for k in d.files}
    meta = dict(zip(out.pop("meta_keys").tolist(), out.pop("meta_vals").tolist()))
    conv = {}
    for k, v in meta.items():
        for typ in (int, float):
            try:
                v = typ(v)
                break
            except ValueError:
                pass
        if v in ("True", "False"):
            v = v == "True"
        conv[k] = v
    out["meta"] = conv
    for k, v in list(out.items()):
        if isinstance(v, np.ndarray) and v.dtype == np.int32:
            out[k] = v.astype(np.int64)
    if out.get("Y_is_X") is not None:
        out["Y"] = out["X"]
        out["perm_col"] = out["perm_row"]
    if out.get("skel_col_equal_row") is not None:
        out["skel_col"], out["skel_col_ptr"] = out["skel_row"], out["skel_row_ptr"]
    return out


def golden_names():
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz"))


def unflatten(ptr, vals, i):
    return vals[ptr[i]:ptr[i + 1]]


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]
    return get
