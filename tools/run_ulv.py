"""HSS ULV factorisation + solve on the GPU at the BASELINE HSS configs (1: N=4096 log,
4: N=2^20 Cauchy), next to the oracle's CPU restatement of the reference's ULV
(smash/apply.py:168-354; oracle.smash_oracle.ulv_factor/ulv_solve, 1 core) on a
bounded sample of the same geometry.  Prints one JSON line per config."""
import argparse, json, os, sys, time
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1705_05443_b200 as sg
from oracle import smash_oracle as orc
from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", type=int, default=[1, 4])
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--cpu-N", type=int, default=16384, help="oracle sample size (cfg 4)")
a = ap.parse_args()
for cfg in a.configs:
    c = CONFIGS[cfg]
    X, Y, rng = make_points(cfg)
    spec, params = build_params(cfg)
    R = max(c["nrhs"])
    tree = sg.build_tree(sg.PointSet(X), None if Y is X else sg.PointSet(Y, role="col"), nu0=c["nu0"],
                         mode=c["mode"], tau=c["tau"])
    M = sg.build_hss(tree, spec, None, None, params)
    B = torch.from_numpy(rng.standard_normal((X.shape[0], R))).cuda()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ft, st = [], []
    for _ in range(a.reps):
        e0.record(); F = sg.ulv_factor(M); e1.record(); e1.synchronize()
        ft.append(e0.elapsed_time(e1))
    for _ in range(a.reps):
        e0.record(); Xs = sg.ulv_solve(F, B); e1.record(); e1.synchronize()
        st.append(e0.elapsed_time(e1))
    resid = float(torch.linalg.norm(sg.matvec_device(M, Xs) - B) / torch.linalg.norm(B))
    # oracle (reference algorithm, CPU, 1 core) on a bounded sample
    n_cpu = X.shape[0] if X.shape[0] <= a.cpu_N else a.cpu_N
    Xc, Yc, rc = make_points(cfg, N=n_cpu)
    ot = orc.build_tree(Xc, None if Yc is Xc else Yc, nu0=c["nu0"], mode=c["mode"])
    OM = orc.build_hss(ot, c["kernel"], c["r"], params.tau, params.eps_svd, rtol=c["rtol"],
                       dx=spec.dx_value if spec.dx_value == spec.dx_value else None)
    bc = rc.standard_normal((n_cpu, R))
    t0 = time.perf_counter(); OF = orc.ulv_factor(OM); t1 = time.perf_counter()
    xo = orc.ulv_solve(OF, bc); t2 = time.perf_counter()
    # same sample on the GPU: parity of the solution
    tg = sg.build_tree(sg.PointSet(Xc), None if Yc is Xc else sg.PointSet(Yc, role="col"), nu0=c["nu0"],
                       mode=c["mode"], tau=c["tau"])
    Mg = sg.build_hss(tg, spec, None, None, params)
    xg = sg.ulv_solve(sg.ulv_factor(Mg), bc)
    print(json.dumps({"cfg": cfg, "N": X.shape[0], "nrhs": R, "ulv_factor_ms_min": min(ft),
                      "ulv_factor_ms": ft, "ulv_solve_ms_min": min(st),
                      "solve_gpts_per_s": X.shape[0] * R / (min(st) / 1e3) / 1e9,
                      "residual_rel": resid,
                      "cpu_oracle": {"N": n_cpu, "cores": 1, "factor_s": t1 - t0, "solve_s": t2 - t1},
                      "gpu_vs_oracle_x_rel": float(np.linalg.norm(xg - xo) / np.linalg.norm(xo))}),
          flush=True)
