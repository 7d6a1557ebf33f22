"""Build cfg-N a few times (for ncu launch lists of the construction)."""
import argparse, sys, time
import torch
sys.path.insert(0, ".")
import paper_1705_05443_b200 as sg
from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--N", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
c = CONFIGS[a.config]
X, Y, rng = make_points(a.config, N=a.N)
spec, params = build_params(a.config)
dX = torch.from_numpy(X).cuda()
dY = dX if Y is X else torch.from_numpy(Y).cuda()
for i in range(a.reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    tree = sg.build_tree(sg.PointSet(dX), None if Y is X else sg.PointSet(dY), nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
    torch.cuda.synchronize(); t1 = time.perf_counter()
    M = (sg.build_h2 if c["structure"] == "h2" else sg.build_hss)(tree, spec, None, None, params)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print("tree %.2f ms  compress %.2f ms" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3))
