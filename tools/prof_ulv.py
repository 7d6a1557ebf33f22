"""One ULV factor + solve at a config (for ncu launch lists)."""
import argparse, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1705_05443_b200 as sg
from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
a = ap.parse_args()
c = CONFIGS[a.config]
X, Y, rng = make_points(a.config)
spec, params = build_params(a.config)
tree = sg.build_tree(sg.PointSet(X), None if Y is X else sg.PointSet(Y, role="col"), nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
M = sg.build_hss(tree, spec, None, None, params)
B = torch.from_numpy(rng.standard_normal((X.shape[0], max(c["nrhs"])))).cuda()
F = sg.ulv_factor(M)
Xs = sg.ulv_solve(F, B)
torch.cuda.synchronize()
print("ok")
