"""Per-item timeline of the persistent transfer passes (instrumented build:
SMASH_TRACE=1 python paper_1705_05443_b200/_build.py, run with
SMASH_LIB=paper_1705_05443_b200/libsmash_b200_trace.so)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1705_05443_b200 as sg
from paper_1705_05443_b200 import _lib
from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = CONFIGS[cid]
X, Y, rng = make_points(cid)
spec, params = build_params(cid)
tree = sg.build_tree(sg.PointSet(X), None if Y is X else sg.PointSet(Y), nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
M = (sg.build_h2 if c["structure"] == "h2" else sg.build_hss)(tree, spec, None, None, params)
Q = torch.from_numpy(rng.standard_normal((X.shape[0], 16))).cuda()
lib = _lib.load()
f = lib.smash_debug_xfer_trace
f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
buf = np.zeros((120000, 8), np.uint64)
serial = os.environ.get("SMASH_MATVEC_SERIAL")
for rep in range(3):
    sg.matvec_device(M, Q)
    torch.cuda.synchronize()
    n = f(buf.ctypes.data, buf.shape[0], 1)
T = buf[:n].astype(np.int64)
lv = tree.arrays()["level"]
kid = T[:, 0] >> 32
for k in sorted(set(kid.tolist())):
    S = T[kid == k]
    t0 = S[:, 2].min()
    S = S[np.argsort(S[:, 2])]
    v = S[:, 0] & 0xffffffff
    print("kernel %d: %d items, span %.1f us" % (k, len(S), (S[:, 6].max() - t0) / 1e3))
    # bfs ids -> levels via post? level array is postorder-indexed in arrays(); report per-phase means
    wait = (S[:, 3] - S[:, 2]) / 1e3
    load = (S[:, 4] - S[:, 3]) / 1e3
    comp = np.maximum(S[:, 5] - S[:, 4], 0) / 1e3
    store = (S[:, 6] - np.maximum(S[:, 5], S[:, 4])) / 1e3
    print("  mean wait %.2f us, stage %.2f us, mma %.2f us, store+publish %.2f us" % (wait.mean(), load.mean(), comp.mean(), store.mean()))
    for q in (0, len(S) // 4, len(S) // 2, 3 * len(S) // 4, len(S) - 1):
        r = S[q]
        print("  item %5d node %6d sm %3d start %7.2f wait %6.2f stage %6.2f mma %6.2f store %6.2f end %7.2f" % (
            q, r[0] & 0xffffffff, r[1], (r[2] - t0) / 1e3, (r[3] - r[2]) / 1e3, (r[4] - r[3]) / 1e3,
            max(r[5] - r[4], 0) / 1e3, (r[6] - max(r[5], r[4])) / 1e3, (r[6] - t0) / 1e3))
    h = np.histogram((S[:, 2] - t0) / 1e3, bins=np.arange(0, (S[:, 6].max() - t0) / 1e3 + 5, 5))[0]
    print("  starts per 5us:", h.tolist())
