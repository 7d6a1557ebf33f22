"""Dump the exported factors of a golden case's GPU build (for A/B library comparisons:
SMASH_LIB=... selects the library)."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_1705_05443_b200 as sg
from conftest import load_golden
name, out = sys.argv[1], sys.argv[2]
g = load_golden(name)
m = g["meta"]
X = sg.PointSet(g["X"])
Y = None if g["Y"] is g["X"] else sg.PointSet(g["Y"], role="col")
tree = sg.build_tree(X, Y, nu0=m["nu0"], mode=m["mode"], tau=m["tau"])
spec = sg.KernelSpec(m["kernel"], dx=None if m["kernel"] == "exp" else 0.0)
params = sg.BuildParams(r=m["r"], tau=m["tau"], eps_svd=m["eps_svd"], s=2.0, basis="interp", rtol=m["rtol"])
M = (sg.build_h2 if m["structure"] == "h2" else sg.build_hss)(tree, spec, None, None, params)
d = {}
for s in (0, 1):
    for k, v in M.export_side(s).items():
        d["%d_%s" % (s, k)] = v
np.savez(out, **d)
print(name, "swaps", M.swaps)
