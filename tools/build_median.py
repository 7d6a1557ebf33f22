"""Median build time (tree + pair lists + compression) of a config over several reps (CUDA events)."""
import argparse, statistics, sys
import torch
sys.path.insert(0, ".")
import paper_1705_05443_b200 as sg
from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points
ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", type=int, default=[5, 2, 3])
ap.add_argument("--reps", type=int, default=7)
a = ap.parse_args()
for cfg in a.configs:
    c = CONFIGS[cfg]
    X, Y, _ = make_points(cfg)
    spec, params = build_params(cfg)
    dX = torch.from_numpy(X).cuda()
    dY = dX if Y is X else torch.from_numpy(Y).cuda()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for i in range(a.reps + 2):
        e0.record()
        tree = sg.build_tree(sg.PointSet(dX), None if Y is X else sg.PointSet(dY, role="col"),
                             nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
        M = (sg.build_h2 if c["structure"] == "h2" else sg.build_hss)(tree, spec, None, None, params)
        e1.record(); e1.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
        del M, tree
    print("cfg%d build median %.2f ms (min %.2f, max %.2f)" % (cfg, statistics.median(ts), min(ts), max(ts)))
