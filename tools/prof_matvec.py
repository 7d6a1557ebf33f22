"""Build cfg-N once and run a few matvecs (for ncu captures of the matvec kernels)."""
import argparse, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1705_05443_b200 as sg
from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--nrhs", type=int, default=16)
ap.add_argument("--N", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
c = CONFIGS[a.config]
X, Y, rng = make_points(a.config, N=a.N)
spec, params = build_params(a.config)
tree = sg.build_tree(sg.PointSet(X), None if Y is X else sg.PointSet(Y), nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
M = (sg.build_h2 if c["structure"] == "h2" else sg.build_hss)(tree, spec, None, None, params)
Q = torch.from_numpy(rng.standard_normal((X.shape[0], a.nrhs))).cuda()
for _ in range(a.reps):
    Z = sg.matvec_device(M, Q)
torch.cuda.synchronize()
print("ok", float(Z.norm()))
