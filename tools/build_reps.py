"""Repeated full builds (tree + matrix) of one config, CUDA-event timed, matrix kept
alive across reps like bench.py's build loop."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1705_05443_b200 as sg
from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
c = CONFIGS[cfg]
X, Y, rng = make_points(cfg)
spec, params = build_params(cfg)
dX = torch.from_numpy(X).cuda()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
out = []
M = None
for i in range(reps):
    e0.record()
    tree = sg.build_tree(sg.PointSet(dX), nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
    M = (sg.build_h2 if c["structure"] == "h2" else sg.build_hss)(tree, spec, None, None, params)
    e1.record(); e1.synchronize()
    out.append(round(e0.elapsed_time(e1), 2))
print("cfg", cfg, "build ms", out)
