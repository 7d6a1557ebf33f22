"""Full-size run of BASELINE configs on the GPU: build time, matvec time, ranks,
error vs the exact product on 64 sampled rows (SURVEY.md 8(c) rule 5 compares it
with the reference's own error from BASELINE.md section 2)."""
import argparse, json, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1705_05443_b200 as sg
from paper_1705_05443_b200.kernel import kernel_block_coords
from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points

REF_ERR = {1: 1.4e-9, 2: 1.9e-6, 3: 1.5e-6, 4: 2.7e-11, 5: 2.1e-8}
ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", type=int, default=[1, 2, 3, 4, 5])
ap.add_argument("--N", type=int, default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--full-error", action="store_true",
                help="error vs the exact product over every row (GPU dense oracle, sg.dense_matvec)")
a = ap.parse_args()
for cfg in a.configs:
    c = CONFIGS[cfg]
    X, Y, rng = make_points(cfg, N=a.N)
    R = max(c["nrhs"])
    q = rng.standard_normal((Y.shape[0], R))
    spec, params = build_params(cfg)
    dX = torch.from_numpy(X).cuda()
    dY = dX if Y is X else torch.from_numpy(Y).cuda()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    bt = []
    for it in range(a.reps):
        e0.record()
        tree = sg.build_tree(sg.PointSet(dX), None if Y is X else sg.PointSet(dY), nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
        M = (sg.build_h2 if c["structure"] == "h2" else sg.build_hss)(tree, spec, None, None, params)
        e1.record(); e1.synchronize()
        bt.append(e0.elapsed_time(e1))
    Q = torch.from_numpy(q).cuda()
    Z = sg.matvec_device(M, Q)
    mt = []
    for it in range(a.reps):
        e0.record(); sg.matvec_device(M, Q, Z); e1.record(); e1.synchronize()
        mt.append(e0.elapsed_time(e1))
    rows = np.sort(np.random.default_rng(99).choice(X.shape[0], 64, replace=False))
    K = torch.from_numpy(kernel_block_coords(spec, X[rows], Y)).cuda()
    ze = K @ Q
    err = float(torch.linalg.norm(Z[rows] - ze) / torch.linalg.norm(ze))
    err_full = None
    if a.full_error:
        e0.record()
        zf = sg.dense_matvec(spec, dX, dY, Q)
        e1.record(); e1.synchronize()
        err_full = float(torch.linalg.norm(Z - zf) / torch.linalg.norm(zf))
        dense_ms = e0.elapsed_time(e1)
    L, Lm = sg.leaf_sets(tree, c["tau"], c["structure"])
    print(json.dumps({"cfg": cfg, "N": X.shape[0], "nrhs": R, "nodes": len(tree.arrays()["level"]),
                      "levels": tree.n_levels, "L": len(L), "Lm": len(Lm),
                      "build_ms_min": min(bt), "build_ms": bt, "matvec_ms_min": min(mt),
                      "gpts_per_s": X.shape[0] * R / (min(mt) / 1e3) / 1e9,
                      "relerr_vs_exact_64rows": err, "reference_relerr": REF_ERR[cfg],
                      "relerr_vs_exact_all_rows": err_full,
                      "dense_oracle_ms": dense_ms if a.full_error else None,
                      "swaps": M.swaps}), flush=True)
    del M, tree, K
    torch.cuda.empty_cache()
