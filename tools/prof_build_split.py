"""Wall-clock split of one device build: tree, pair lists (smash_leaf_sets, cached on
the tree), compression (build_h2 reusing the cached pairs); GPU idle = wall - kernel time."""
import argparse, ctypes, sys, time
import torch
sys.path.insert(0, ".")
import paper_1705_05443_b200 as sg
from paper_1705_05443_b200 import _lib
from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=6)
a = ap.parse_args()
c = CONFIGS[a.config]
X, Y, rng = make_points(a.config)
spec, params = build_params(a.config)
dX = torch.from_numpy(X).cuda()
for i in range(a.reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    tree = sg.build_tree(sg.PointSet(dX), nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
    torch.cuda.synchronize(); t1 = time.perf_counter()
    nL, nLm = _lib.c_i64(), _lib.c_i64()
    _lib.check(_lib.load().smash_leaf_sets(tree._h, float(c["tau"]), _lib.STRUCT[c["structure"]],
                                           _lib.stream_ptr(), ctypes.byref(nL), ctypes.byref(nLm)))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    M = sg.build_h2(tree, spec, None, None, params)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print("tree %.3f ms  pairs %.3f ms  compress %.3f ms  total %.3f ms" % (
        (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t3 - t0) * 1e3))
