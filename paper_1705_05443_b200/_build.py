"""Build the sm_100a C-ABI library libsmash_b200.so in-tree with nvcc.

Each csrc/*.cu is compiled to an object (in parallel) and linked into
paper_1705_05443_b200/libsmash_b200.so next to this file, so the library
travels with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
TRACE = os.environ.get("SMASH_TRACE") == "1"  # instrumented build (tools/xfer_trace.py)
CHECKED = os.environ.get("SMASH_CHECKED") == "1"  # device asserts + bounded spin waits
_VARIANT = "_trace" if TRACE else "_checked" if CHECKED else ""
OBJ = os.path.join(REPO, "build", "obj" + _VARIANT)
LIB = os.path.join(HERE, "libsmash_b200%s.so" % _VARIANT)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++20", "--extended-lambda", "--expt-relaxed-constexpr",
         "-Xcompiler", "-fPIC,-O2", "-I" + os.path.join(REPO, "include")] + (
             ["-DSMASH_XFER_TRACE", "-DSMASH_COMPRESS_PROF"] if TRACE else
             ["-DSMASH_CHECKED"] if CHECKED else [])


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(REPO, "include", "*.h")))


def _compile(src, verbose=False):
    obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
    newest_dep = max([os.path.getmtime(src)] + [os.path.getmtime(d) for d in _deps()])
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep:
        return obj
    cmd = [NVCC] + ARCH + FLAGS + ["-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, r.stdout, r.stderr))
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    if force:
        for o in glob.glob(os.path.join(OBJ, "*.o")):
            os.remove(o)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n%s\n%s" % (r.stdout, r.stderr))
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
