"""The opt-in symmetric coupling (SMASH_COUPLING_SYM=1: each coupling block evaluated once,
csrc/p2p_kernels.cuh k_coupling_sym + k_coupling_tsum) against the default two-sided kernel
and the reference's matvec, in a subprocess (the switch is read once per process)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from conftest import load_golden
import paper_1705_05443_b200 as sg
g = load_golden(sys.argv[1]); m = g["meta"]
tree = sg.build_tree(sg.PointSet(g["X"]), nu0=m["nu0"], mode=m["mode"], tau=m["tau"])
spec = sg.KernelSpec(m["kernel"], dx=None if m["kernel"] == "exp" else 0.0)
M = sg.build_h2(tree, spec, None, None, sg.BuildParams(r=m["r"], tau=m["tau"], basis="interp", rtol=m["rtol"]))
q = np.random.default_rng(3).standard_normal((g["X"].shape[0], int(sys.argv[2])))
np.save(sys.argv[3], sg.matvec_nodewise(M, q))
"""


@pytest.mark.parametrize("nrhs", [8, 16])
@pytest.mark.parametrize("name", ["cfg2_4k", "cfg5_16k", "uniform3d_small"])
def test_symmetric_coupling_matches(tmp_path, name, nrhs):
    pytest.importorskip("torch")
    import numpy as np
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("0", "1"):
        out = str(tmp_path / ("z%s.npy" % flag))
        env = dict(os.environ, SMASH_COUPLING_SYM=flag)
        subprocess.run([sys.executable, "-c", SCRIPT, name, str(nrhs), out], cwd=repo, env=env, check=True)
        outs.append(np.load(out))
    z0, z1 = outs
    for c in range(nrhs):
        assert np.linalg.norm(z1[:, c] - z0[:, c]) <= 1e-13 * np.linalg.norm(z0[:, c])
