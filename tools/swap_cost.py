"""Build time with and without the sRRQR swap loop (s = 2 vs s = 1e30)."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_1705_05443_b200 as sg
from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points
for cfg in [int(a) for a in sys.argv[1:]] or [2]:
    c = CONFIGS[cfg]
    X, Y, rng = make_points(cfg)
    spec, params = build_params(cfg)
    dX = torch.from_numpy(X).cuda()
    tree = sg.build_tree(sg.PointSet(dX), nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
    for s in (2.0, 1e30):
        params.s = s
        ts = []
        for it in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            M = (sg.build_h2 if c["structure"] == "h2" else sg.build_hss)(tree, spec, None, None, params)
            torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        print("cfg %d s=%g build %.2f ms swaps %s" % (cfg, s, min(ts) * 1e3, M.swaps), flush=True)
