"""A/B of the two compression kernels on full-size configs: build with SMASH_COMPRESS_RC=0
(k_compress) and =1 (k_compress_rc) in one process and compare every exported factor array
bit for bit (rank, perm, G, ordered skeletons)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1705_05443_b200 as sg
from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points

VAR = os.environ.get("AB_VAR", "SMASH_COMPRESS_RC")  # the switch under test (value 0 / 1)

def build(cfg, N, rc):
    os.environ[VAR] = str(rc)
    c = CONFIGS[cfg]
    X, Y, _ = make_points(cfg, N=N)
    spec, params = build_params(cfg)
    dX = torch.from_numpy(X).cuda()
    dY = dX if Y is X else torch.from_numpy(Y).cuda()
    tree = sg.build_tree(sg.PointSet(dX), None if Y is X else sg.PointSet(dY, role="col"),
                         nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
    fn = sg.build_h2 if c["structure"] == "h2" else sg.build_hss
    M = fn(tree, spec, None, None, params)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    M2 = fn(tree, spec, None, None, params)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    del M2
    out = {}
    for s in (0, 1):
        for k, v in M.export_side(s).items():
            out["%d_%s" % (s, k)] = np.asarray(v)
    return out, M.swaps, t

bad = 0
for arg in sys.argv[1:]:
    cfg, _, N = arg.partition(":")
    cfg = int(cfg); N = int(N) if N else None
    a, sa, ta = build(cfg, N, 0)
    b, sb, tb = build(cfg, N, 1)
    diffs = []
    for k in a:
        x, y = a[k], b[k]
        if x.shape != y.shape:
            diffs.append("%s shape %s vs %s" % (k, x.shape, y.shape))
        elif x.dtype.kind == "f":
            ne = int(np.sum(x.view(np.int64) != y.view(np.int64)))
            if ne:
                nz = int(np.sum((x != y)))
                diffs.append("%s: %d of %d entries differ in bits (%d in value, max abs %.3e)" % (k, ne, x.size, nz, np.max(np.abs(x - y))))
        elif not np.array_equal(x, y):
            diffs.append("%s: %d of %d entries differ" % (k, int(np.sum(x != y)), x.size))
    print("cfg%d N=%s: swaps %s / %s, build %.2f ms (%s=0) vs %.2f ms (%s=1): %s" % (
        cfg, N, sa, sb, ta * 1e3, VAR, tb * 1e3, VAR, "IDENTICAL" if not diffs else "DIFFERENT"))
    for d in diffs:
        print("   ", d)
    bad += bool(diffs)
sys.exit(1 if bad else 0)
