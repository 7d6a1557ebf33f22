"""C-ABI library: loads without a GPU and exports every symbol the public
header declares (no compute calls)."""

import ctypes
import os
import re

from conftest import REPO

HEADER = os.path.join(REPO, "include", "smash_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(smash_\w+)\s*\(", txt, re.M)))


def test_header_declares_the_api():
    syms = declared_symbols()
    for s in ("smash_tree_build", "smash_leaf_sets", "smash_nearfield", "smash_matrix_build",
              "smash_matvec", "smash_kernel_block", "smash_interp_basis", "smash_compr"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_1705_05443_b200 import _lib
    lib = _lib.load()
    for s in declared_symbols():
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, s
    assert lib.smash_abi_version() == 1


def test_library_is_sm100a():
    from paper_1705_05443_b200 import _lib
    data = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in data
