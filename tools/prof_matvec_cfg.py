"""Build one config and run a few matvecs (for ncu captures of the matvec kernels)."""
import argparse, sys
import torch
sys.path.insert(0, ".")
import paper_1705_05443_b200 as sg
from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
c = CONFIGS[a.config]
X, Y, rng = make_points(a.config)
R = max(c["nrhs"])
q = rng.standard_normal((Y.shape[0], R))
spec, params = build_params(a.config)
dX = torch.from_numpy(X).cuda()
tree = sg.build_tree(sg.PointSet(dX), None if Y is X else sg.PointSet(torch.from_numpy(Y).cuda()),
                     nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
M = (sg.build_h2 if c["structure"] == "h2" else sg.build_hss)(tree, spec, None, None, params)
Q = torch.from_numpy(q).cuda()
for _ in range(a.reps):
    sg.matvec_device(M, Q)
torch.cuda.synchronize()
