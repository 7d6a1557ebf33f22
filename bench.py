#!/usr/bin/env python
"""Benchmark: SMASH H^2 build time + H^2 matvec Gpoints/s (fp64) on B200.

Workload (default --config 5, the largest single-GPU BASELINE config, SURVEY.md
8(d)): N = 2^21 nonuniform 2-D points (half on the unit circle with radial
N(0, 1e-3) jitter, half from a 4-component Gaussian mixture), K(x,y) =
log|x-y| (diagonal 0), adaptive quadtree nu0 = 64, tensor Chebyshev 8x8
(r = 64), eta = 0.7, sRRQR tolerance 1e-8, fp64, 16 N(0,1) right-hand sides
(seeded synthetic data; BASELINE names no dataset).

A step is one H^2 matvec (nrhs = 16) through the device API on a matrix built
once; ``value`` = N * nrhs / t_matvec in Gpoints/s, the L2 flushed (256 MiB
write, outside the event pair) before every timed product, nothing host-
synchronised inside the product.  The build (tree + pair lists + compression)
is timed separately over the same warm-up / step counts (``build_s``).
``e2e`` repeats both through the public API with pinned host buffers and the
host<->device copies inside the timed region.  Phase times come from a
separate profiled pass after the timed loop.  ``parity`` compares the timed
output with the reference's own full-size output (tests/golden/full, digests
of the real reference on the same seeded inputs) and the exact product.
``configs`` adds build / matvec numbers of every BASELINE config (cfg 3 is the
2^20-point config of the 8-GPU target).

Usage:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config C] [--nrhs R] [--N n] [--no-extras]
For N > 1 run under torchrun: the build is sharded at the cut level and the
matvec by target subtree (shard.py) with one NCCL exchange of the skeleton
coefficients per matvec -- strong scaling of the fixed problem; time = max over
ranks, value = N * nrhs / time.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# FP64 peak measured on this pool's B200 (tools/fp64_peak.cu, profiles/fp64_peak_r01.txt):
# MEASURED_PEAKS.json has no FP64 entry.  DFMA 34.1 TF/s (DMMA 37.1 TF/s).
FP64_PEAK_TFLOPS = 34.1
# DP flops per kernel evaluation c_K (DADD + DMUL + 2*DFMA of the compiled kval<> path,
# counted by ncu on k_block -- profiles/ckernel_r02.txt); 2*nrhs flops per interaction added.
C_K = {"inv_r": 14.0, "log": 41.0, "exp": 52.0, "cauchy": 7.0}
# The matvec kernels (k_coupling / k_near, all column counts) evaluate the log and exp kernels
# from shared-memory tables (kernels.cuh log_half_tab / exp_neg_tab); DP ops per evaluation
# measured by ncu on k_coupling itself (profiles/ckernel_r02.txt): log 2 DADD + 13 DFMA = 28,
# exp 4 DADD + 5 DMUL + 15 DFMA = 39.  Construction (k_svd, k_block) keeps the series above.
C_K_MATVEC = {"inv_r": 14.0, "log": 28.0, "exp": 39.0, "cauchy": 7.0}


def c_k(kernel, nrhs):
    return C_K_MATVEC[kernel]
L2_FLUSH_BYTES = 256 << 20
# dram__bytes_read.sum + dram__bytes_write.sum per launch (ncu --set full, profiles/coupling_r01.txt)
NCU_TRAFFIC = {(2, 16, "k_coupling"): 26.45e6,
               (5, 16, "k_coupling"): 1.030274e9 + 0.454930e9}  # profiles/matvec_cfg5_r02.txt


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--nrhs", type=int, default=None)
    ap.add_argument("--N", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, dev):
        self.dev = dev
        self.proc = None
        self.path = "/tmp/bench_clocks_%d_%d.csv" % (os.getpid(), dev)

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + q, "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [r.split(", ") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except OSError:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if len(r) > 3 + k and r[3 + k].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# reference arm / cpu baseline: the oracle port of the reference algorithm
# ---------------------------------------------------------------------------

def default_nrhs(cfg):
    from paper_1705_05443_b200.workloads import CONFIGS
    return max(CONFIGS[cfg]["nrhs"])


def oracle_run(cfg, N, nrhs, warmup, steps, seed=None, cached=True):
    """Reference CPU implementation (oracle port, single thread like the
    reference's serial Python loops).  cached=True keeps coupling / nearfield
    blocks across products like the reference's use_cache=True; the full-size
    configs 3 and 5 do not fit it in host RAM, so they run uncached
    (use_cache=False, what the survey timed for the reference)."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import smash_oracle as orc
    from paper_1705_05443_b200.workloads import CONFIGS, make_points
    c = CONFIGS[cfg]
    X, Y, rng = make_points(cfg, N=N, seed=seed)
    q = rng.standard_normal((Y.shape[0], nrhs))
    t0 = time.perf_counter()
    tree = orc.build_tree(X, None if Y is X else Y, nu0=c["nu0"], mode=c["mode"])
    if c["structure"] == "h2":
        M = orc.build_h2(tree, c["kernel"], c["r"], c["tau"], rtol=c["rtol"],
                         dx=None if c["kernel"] == "exp" else 0.0, symmetric=Y is X)
    else:
        M = orc.build_hss(tree, c["kernel"], c["r"], c["tau"], c["eps_svd"], rtol=c["rtol"],
                          dx=None if c["kernel"] == "exp" else 0.0)
    t_build = time.perf_counter() - t0
    cache = {} if cached else None
    for _ in range(warmup):
        orc.matvec(M, q, cache)
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        orc.matvec(M, q, cache)
        ts.append(time.perf_counter() - t0)
    return t_build, float(np.mean(ts)), X.shape[0]


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = args.config
    R = args.nrhs or default_nrhs(cfg)
    from paper_1705_05443_b200.workloads import CONFIGS
    N = args.N or CONFIGS[cfg]["N"]
    big = N > 2 ** 18  # configs 3-5 at full size: one uncached product (~2 min on one core)
    cached = not big
    steps = 1 if big else max(1, min(args.steps, 5))
    warmup = 0 if big else 1
    t_build, t_mv, n = oracle_run(cfg, N, R, warmup, steps, cached=cached)
    val = n * R / t_mv / 1e9
    sample = ("full workload (N=%d, %d RHS), oracle port of the reference algorithm (numpy/scipy "
              "LAPACK, serial like the reference); %s; %d timed product(s) after %d warm-up" % (
                  N, R, "blocks cached as use_cache=True" if cached else
                  "blocks evaluated per product (use_cache=False: the cached blocks need ~38 GB)",
                  steps, warmup))
    line = {
        "impl": "reference", "metric": "SMASH build time + H^2 matvec Gpoints/s (fp64), 1/2/4/8 B200, % roofline",
        "value": val, "unit": "Gpoints/s", "n_gpus": args.gpus, "steps": steps, "warmup": warmup,
        "ms_per_step": t_mv * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded, SURVEY.md 8(d))",
        "config": workload_config(cfg, N, R),
        "build_s": t_build,
        "cpu_baseline": {"value": val, "unit": "Gpoints/s", "cores": 1, "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": "Gpoints/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(cfg, N, nrhs):
    from paper_1705_05443_b200.workloads import CONFIGS
    c = CONFIGS[cfg]
    return {"workload": "cfg%d %s: N=%d, nu0=%d, r=%d, tau=%g, rtol=%g, nrhs=%d" % (
        cfg, c["name"], N, c["nu0"], c["r"], c["tau"], c["rtol"], nrhs),
        "config_id": cfg, "N": N, "nrhs": nrhs, "kernel": c["kernel"], "structure": c["structure"],
        "l2": "flushed between timed matvecs (256 MiB write)", "seed": cfg}


# ---------------------------------------------------------------------------
# algorithmic work
# ---------------------------------------------------------------------------

def work_counts(sg, M, c, R, owned=None, top=None):
    """Interactions, transfer bytes and sRRQR flops of a built matrix."""
    from paper_1705_05443_b200.cluster import _pairs
    Lh, Lmh = _pairs(M.tree, c["tau"], c["structure"])
    Er, Ec = M.export_side(0), M.export_side(1)
    rk_r, rk_c = Er["rank"], Ec["rank"]
    A = M.tree.arrays()
    nr = A["row_stop"] - A["row_start"]
    ncl = A["col_stop"] - A["col_start"]
    if owned is not None:  # this rank's launches: owned + top coupling targets / owned leaves
        mine = np.zeros(len(nr), bool)
        mine[owned] = True
        tp = np.zeros(len(nr), bool)
        tp[top] = True
        Lh = Lh[mine[Lh[:, 0]] | tp[Lh[:, 0]]] if Lh.size else Lh
        Lmh = Lmh[mine[Lmh[:, 0]]] if Lmh.size else Lmh
    I_coup = float(np.sum(rk_r[Lh[:, 0]] * rk_c[Lh[:, 1]])) if Lh.size else 0.0
    I_near = float(np.sum(nr[Lmh[:, 0]] * ncl[Lmh[:, 1]])) if Lmh.size else 0.0
    # transfer passes: one side's G is read per pass (upward: column factors, downward: row
    # factors), plus the child coefficient slices read and the node coefficients written
    # (8 B x nrhs each) and the 4 B perm entries; the leaf passes also read / write the
    # N x nrhs tree-order vectors once.
    def side_bytes(E):
        G = float(E["G"].size)
        ib = float(E["perm"].size)
        k = float(E["skel"].size)
        return 8 * G + 8 * R * (ib + k) + 4 * ib
    xfer_bytes = side_bytes(Ec) + side_bytes(Er) + 2 * 8.0 * R * (M.n_row + M.n_col) / 2
    sides = [Er] if (M.tree.shared_points and c["structure"] == "h2") else [Er, Ec]
    build_flops = 0.0
    m_rows = float(c["r"])
    for E in sides:
        nib = np.diff(E["perm_ptr"]).astype(np.float64)
        kk = E["rank"].astype(np.float64)
        for nv, kv in zip(nib, kk):
            if nv <= 0:
                continue
            st = int(min(m_rows, nv))
            i = np.arange(st, dtype=np.float64)
            build_flops += float(np.sum(4.0 * (m_rows - i) * np.maximum(nv - i - 1.0, 0.0)))
            build_flops += kv * kv * (nv - kv)
    return dict(I_coup=I_coup, I_near=I_near, xfer_bytes=xfer_bytes, build_flops=build_flops,
                G_entries=float(Er["G"].size))


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return 6556.2, "fallback (last MEASURED_PEAKS.json value seen)"


def golden_parity(cfg, N, R, z):
    """Timed output vs the real reference's full-size output on the same seeded inputs
    (tests/golden/full, made by make_golden_full.py) and vs the exact product."""
    path = os.path.join(REPO, "tests", "golden", "full", "cfg%d_full.npz" % cfg)
    if not os.path.exists(path):
        return None
    g = np.load(path)
    if int(g["N"]) != N or int(g["nrhs"]) != R:
        return None
    rows = g["z_rows"].astype(np.int64)
    ref = g["z_at_rows"]
    rel = max(float(np.linalg.norm(z[rows, c] - ref[:, c]) / np.linalg.norm(ref[:, c])) for c in range(R))
    er = g["exact_rows"].astype(np.int64)
    ze = g["z_exact_rows"]
    e_gpu = float(np.linalg.norm(z[er] - ze) / np.linalg.norm(ze))
    e_ref = float(np.linalg.norm(ref[np.searchsorted(rows, er)] - ze) / np.linalg.norm(ze))
    cn = np.linalg.norm(z, axis=0)
    return {"vs_reference_rel_max_col": rel, "rows": int(rows.size),
            "colnorm_rel_max": float(np.max(np.abs(cn - g["z_colnorm"]) / g["z_colnorm"])),
            "err_vs_exact": e_gpu, "reference_err_vs_exact": e_ref, "exact_rows": int(er.size),
            "pass": bool(rel <= 1e-10 and e_gpu <= 1.1 * e_ref + 1e-12),
            "source": "tests/golden/full/cfg%d_full.npz (real reference, same seeded inputs)" % cfg}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def time_config(sg, torch, cfg, R, N, steps, warmup, flush, dev):
    """Build and matvec of one config (single GPU): median build ms, mean matvec ms,
    profiled phase ms, launches per product, the matrix and the last product."""
    from paper_1705_05443_b200 import _lib
    from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points
    import ctypes
    c = CONFIGS[cfg]
    X, Y, rng = make_points(cfg, N=N)
    q = rng.standard_normal((Y.shape[0], R))
    spec, params = build_params(cfg)
    dX = torch.from_numpy(X).to(dev)
    dY = dX if Y is X else torch.from_numpy(Y).to(dev)
    dQ = torch.from_numpy(q).to(dev)
    builder = sg.build_h2 if c["structure"] == "h2" else sg.build_hss

    def build():
        tree = sg.build_tree(sg.PointSet(dX), None if Y is X else sg.PointSet(dY, role="col"),
                             nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
        return builder(tree, spec, None, None, params)

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(warmup):
        build()
    torch.cuda.synchronize()
    build_ms = []
    for _ in range(steps):
        flush.zero_()
        e0.record()
        M = build()
        e1.record()
        e1.synchronize()
        build_ms.append(e0.elapsed_time(e1))
    out = torch.empty((M.n_row, R), dtype=torch.float64, device=dev)
    for _ in range(warmup):
        sg.matvec_device(M, dQ, out)
    torch.cuda.synchronize()
    mv_ms = []
    for _ in range(steps):
        flush.zero_()
        e0.record()
        sg.matvec_device(M, dQ, out)
        e1.record()
        e1.synchronize()
        mv_ms.append(e0.elapsed_time(e1))
    # profiled passes (phase events on the launch streams; synchronise each product):
    # as timed (nearfield concurrent), and serialised (isolated per-phase kernel times)
    lib = _lib.load()
    res = []
    for mode in (1, 2):
        lib.smash_matvec_profile(M._h, mode, None, None)
        for _ in range(steps):
            flush.zero_()
            sg.matvec_device(M, dQ)
        torch.cuda.synchronize()
        phase = (ctypes.c_double * 7)()
        launches = ctypes.c_int64()
        lib.smash_matvec_profile(M._h, 0, phase, ctypes.byref(launches))
        res.append(([phase[i] / steps for i in range(7)], launches.value / steps))
    return dict(M=M, X=X, Y=Y, q=q, dQ=dQ, out=out, build_ms=build_ms, mv_ms=mv_ms,
                phase=res[0][0], phase_serial=res[1][0], launches_per_product=res[0][1],
                spec=spec, params=params, builder=builder, c=c)


def config_summary(sg, cfg, R, T, fp64_peak, hbm):
    c = T["c"]
    W = work_counts(sg, T["M"], c, R)
    mv_s = float(np.mean(T["mv_ms"])) / 1e3
    b_s = statistics.median(T["build_ms"]) / 1e3
    per_int = c_k(c["kernel"], R) + 2 * R
    return {"N": T["M"].n_row, "nrhs": R, "build_ms": b_s * 1e3, "matvec_ms": mv_s * 1e3,
            "gpoints_s": T["M"].n_row * R / mv_s / 1e9,
            "matvec_fp64_frac": (W["I_coup"] + W["I_near"]) * per_int / mv_s / 1e12 / fp64_peak,
            "build_fp64_frac": W["build_flops"] / b_s / 1e12 / fp64_peak,
            "phase_ms": dict(zip(["gather", "upward", "coupling", "downward", "nearfield_concurrent",
                                  "leaf_farfield", "matvec_profiled"], T["phase"])),
            "interactions_coupling": W["I_coup"], "interactions_near": W["I_near"]}


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        # one process per GPU; BENCH_BACKEND=gloo + device wrap-around only to exercise the
        # N > 1 code path on a single GPU (functional check, not a measurement)
        torch.cuda.set_device(local % torch.cuda.device_count())
        dist.init_process_group(os.environ.get("BENCH_BACKEND", "nccl"))
    import paper_1705_05443_b200 as sg
    from paper_1705_05443_b200 import _lib
    from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points
    import ctypes
    cfg = args.config
    R = args.nrhs or default_nrhs(cfg)
    c = CONFIGS[cfg]
    N = args.N or c["N"]
    dev = torch.device("cuda", torch.cuda.current_device())
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    hbm, hbm_src = hbm_peak()

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if ws == 1:
        with ClockSampler(torch.cuda.current_device()) as clk:
            T = time_config(sg, torch, cfg, R, N, args.steps, args.warmup, flush, dev)
        M, X, Y, q, dQ, out = T["M"], T["X"], T["Y"], T["q"], T["dQ"], T["out"]
        spec, params, builder = T["spec"], T["params"], T["builder"]
        build_ms, mv_ms, phase = T["build_ms"], T["mv_ms"], T["phase"]
        phase_serial = T["phase_serial"]
        launches_per_product = T["launches_per_product"]
        t_mv = sum(mv_ms) / 1e3
        owned = top = None
    else:
        # N > 1 (H2, shared points): sharded construction, sharded matvec (shard.py)
        X, Y, rng = make_points(cfg, N=N)
        q = rng.standard_normal((Y.shape[0], R))
        spec, params = build_params(cfg)
        dX = torch.from_numpy(X).to(dev)
        dQ = torch.from_numpy(q).to(dev)
        builder = sg.build_h2 if c["structure"] == "h2" else sg.build_hss
        sharded_build = c["structure"] == "hss" or Y is X

        def build_device():
            tree = sg.build_tree(sg.PointSet(dX), None if Y is X else sg.PointSet(torch.from_numpy(Y).to(dev)),
                                 nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
            if c["structure"] == "hss":  # level-distributed, factors replicated
                return sg.build_hss_sharded(tree, spec, None, None, params)
            if sharded_build:
                return sg.build_h2_sharded(tree, spec, None, None, params)
            return builder(tree, spec, None, None, params)
        for _ in range(args.warmup):
            build_device()
        barrier()
        build_ms = []
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            e0.record()
            M = build_device()
            e1.record()
            e1.synchronize()
            build_ms.append(e0.elapsed_time(e1))
        from paper_1705_05443_b200.shard import ShardedMatvec
        sm = ShardedMatvec(M)
        owned, top = sm.owned, sm.top
        for _ in range(args.warmup):
            sm(dQ, gather_output=False)
        barrier()
        mv_ms = []
        with ClockSampler(torch.cuda.current_device()) as clk:
            for _ in range(args.steps):
                flush.zero_()
                barrier()
                e0.record()
                out = sm(dQ, gather_output=False)
                e1.record()
                e1.synchronize()
                mv_ms.append(e0.elapsed_time(e1))
            barrier()
        t = torch.tensor([sum(mv_ms) / 1e3, statistics.median(build_ms)], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_mv = float(t[0])
        build_ms = [float(t[1])]
        lib = _lib.load()
        lib.smash_matvec_profile(M._h, 1, None, None)
        for _ in range(args.steps):
            sm(dQ, gather_output=False)
        torch.cuda.synchronize()
        ph = (ctypes.c_double * 7)()
        lc = ctypes.c_int64()
        lib.smash_matvec_profile(M._h, 0, ph, ctypes.byref(lc))
        phase = [ph[i] / args.steps for i in range(7)]
        phase_serial = phase
        launches_per_product = lc.value / args.steps
    value = args.steps * M.n_row * R / t_mv / 1e9

    # ---- e2e through the public API with pinned host buffers: every step copies its
    # right-hand sides host->device and its result device->host (inside the timed
    # region); MatvecStream overlaps those copies of neighbouring steps with the
    # compute (copy engines), as a serving loop would
    q_pin = [torch.from_numpy(q).pin_memory(), torch.from_numpy(q.copy()).pin_memory()]
    z_pin = [torch.empty((M.n_row, R), dtype=torch.float64).pin_memory() for _ in range(2)]
    if ws > 1:
        e2e_mv = []
        for i in range(args.warmup + args.steps):
            flush.zero_()
            e0.record()
            zg = sm(q_pin[0].to(dev, non_blocking=True), gather_output=True)
            z = torch.empty(zg.shape, dtype=torch.float64, pin_memory=True)
            z.copy_(zg, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            e1.record()
            e1.synchronize()
            if i >= args.warmup:
                e2e_mv.append(e0.elapsed_time(e1))
        t_e2e = float(np.mean(e2e_mv)) / 1e3
    else:
        pipe = sg.MatvecStream(M, R, depth=2)
        for i in range(args.warmup):
            pipe.submit(q_pin[i % 2], z_pin[i % 2])
        pipe.synchronize()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(pipe.s_in)
        for i in range(args.steps):  # L2 flushed before every timed product, as for `value`
            pipe.submit(q_pin[i % 2], z_pin[i % 2], before=flush.zero_)
        s1.record(pipe.s_out)
        s1.synchronize()
        t_e2e = s0.elapsed_time(s1) / 1e3 / args.steps
        z = z_pin[(args.steps - 1) % 2]
    e2e_build = []
    for i in range(args.warmup + args.steps):
        e0.record()
        tree_h = sg.build_tree(sg.PointSet(X), None if Y is X else sg.PointSet(Y, role="col"), nu0=c["nu0"],
                               mode=c["mode"], tau=c["tau"])
        builder(tree_h, spec, None, None, params)
        e1.record()
        e1.synchronize()
        if i >= args.warmup:
            e2e_build.append(e0.elapsed_time(e1))
    if ws > 1:
        t = torch.tensor([t_e2e], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_e2e = float(t[0])
    e2e_val = M.n_row * R / t_e2e / 1e9

    # ---- parity of the timed output
    if ws == 1:
        zd = out.cpu().numpy()
        assert np.array_equal(zd, z.numpy()), "device and e2e results differ"
        parity = golden_parity(cfg, N, R, zd)
    else:  # sharded (full, gathered) vs a single-GPU build + matvec on this rank
        tree1 = sg.build_tree(sg.PointSet(dX), None if Y is X else sg.PointSet(torch.from_numpy(Y).to(dev)),
                              nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
        R1 = builder(tree1, spec, None, None, params)
        zf = sg.matvec_device(R1, dQ).cpu().numpy()
        del R1
        rel = np.linalg.norm(z.numpy() - zf) / np.linalg.norm(zf)
        assert rel <= 1e-12, "sharded matvec differs from the single-GPU one: %g" % rel
        parity = {"sharded_vs_single_gpu_rel": float(rel),
                  "halo_bytes_per_matvec": int(sm.halo_bytes(R)),
                  "all_gather_bytes_per_matvec": int(sm.half * R * 8 * (ws - 1))}
        parity.update(golden_parity(cfg, N, R, z.numpy()) or {})

    # ---- rooflines: dominant FP64 kernel, transfer passes (HBM), construction
    W = work_counts(sg, M, c, R, owned, top)
    per_int = c_k(c["kernel"], R) + 2 * R
    ms_coup, ms_near = phase_serial[2], phase_serial[4]  # isolated kernel times
    if ms_coup >= ms_near:
        dom, flops, ms = "k_coupling", W["I_coup"] * per_int, ms_coup
    else:
        dom, flops, ms = "k_near", W["I_near"] * per_int, ms_near
    achieved = flops / (ms / 1e3) / 1e12
    total_flops = (W["I_coup"] + W["I_near"]) * per_int
    roofline = {"bound": "fp64", "kernel": dom, "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
                "traffic": NCU_TRAFFIC.get((cfg, R, dom)),
                "peak_source": "measured DFMA microbenchmark (profiles/fp64_peak_r01.txt); "
                               "MEASURED_PEAKS.json has no FP64 entry",
                "flops_per_launch": flops, "ms_per_launch": ms,
                "c_K": c_k(c["kernel"], R), "interactions_coupling": W["I_coup"], "interactions_near": W["I_near"],
                "matvec_total_frac": total_flops / (t_mv / args.steps) / 1e12 / FP64_PEAK_TFLOPS,
                "scope": "rank 0's share" if ws > 1 else "whole matvec"}
    xfer_ms = phase_serial[1] + phase_serial[3] + phase_serial[5]
    transfer_roofline = {"bound": "hbm", "kernels": "k_up_leaves + k_upward + k_downward + k_down_leaves",
                         "bytes": W["xfer_bytes"], "ms": xfer_ms,
                         "achieved": W["xfer_bytes"] / (xfer_ms / 1e3) / 1e9 if xfer_ms > 0 else None,
                         "peak": hbm, "unit": "GB/s", "peak_source": hbm_src,
                         "frac": W["xfer_bytes"] / (xfer_ms / 1e3) / 1e9 / hbm if xfer_ms > 0 else None,
                         "note": "algorithmic bytes (G once per pass, coefficient slices, perms, "
                                 "tree-order vectors) over the upward + downward + leaf far-field phase "
                                 "times of the serialised profiling pass (no nearfield overlap)"}
    b_s = statistics.median(build_ms) / 1e3
    build_roofline = {"bound": "fp64", "flops": W["build_flops"], "achieved": W["build_flops"] / b_s / 1e12,
                      "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                      "frac": W["build_flops"] / b_s / 1e12 / FP64_PEAK_TFLOPS,
                      "note": "algorithmic sRRQR flops (QR + G solve) over the whole build time "
                              "(tree + pair lists + basis + sRRQR)"}

    # ---- every BASELINE config (single GPU): build + matvec at full size
    extras = None
    if ws == 1 and not args.no_extras:
        extras = {}
        del T
        for cx in (1, 2, 3, 4):
            if cx == cfg:
                continue
            Rx = default_nrhs(cx)
            Tx = time_config(sg, torch, cx, Rx, None, min(args.steps, 5), min(args.warmup, 3), flush, dev)
            extras["cfg%d" % cx] = config_summary(sg, cx, Rx, Tx, FP64_PEAK_TFLOPS, hbm)
            del Tx
            torch.cuda.synchronize()

    # ---- CPU baseline (oracle port) on a bounded sample, rank 0, N = 1 only
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        n_s = min(N, 2 ** 16)
        tb, tm, n_used = oracle_run(cfg, n_s, R, 1, 2)
        cpu = {"value": n_used * R / tm / 1e9, "unit": "Gpoints/s", "cores": 1, "kind": "port",
               "sample": "cfg%d geometry at N=%d (of %d), %d RHS, 2 cached matvecs after 1 warm-up; "
                         "oracle build %.2f s" % (cfg, n_used, N, R, tb),
               "build_s_sample": tb}

    if rank == 0:
        line = {
            "metric": "SMASH build time + H^2 matvec Gpoints/s (fp64), 1/2/4/8 B200, % roofline",
            "value": value, "unit": "Gpoints/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_mv * 1e3 / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY.md 8(d))",
            "config": workload_config(cfg, N, R),
            "build_s": b_s,
            "build_mode": ("single" if ws == 1 else
                           "sharded (HSS): level-distributed, one exchange per level and side"
                           if c["structure"] == "hss" else
                           "sharded: work-balanced cut, skeleton exchange, factors kept on their owner"),
            "phase_ms": {"gather": phase[0], "upward": phase[1], "coupling": phase[2], "downward": phase[3],
                         "nearfield_concurrent": phase[4], "leaf_farfield": phase[5],
                         "matvec_profiled": phase[6],
                         "note": "separate profiled pass (per-phase events, host-synchronised); "
                                 "the timed loop runs unprofiled"},
            "phase_ms_serial": {"gather": phase_serial[0], "upward": phase_serial[1],
                                "coupling": phase_serial[2], "downward": phase_serial[3],
                                "nearfield": phase_serial[4], "leaf_farfield": phase_serial[5],
                                "matvec": phase_serial[6],
                                "note": "profiled pass with the nearfield on the main stream: isolated "
                                        "kernel times (roofline denominators)"},
            "roofline": roofline,
            "transfer_roofline": transfer_roofline,
            "build_roofline": build_roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "Gpoints/s", "h2d_bytes_per_step": int(q.nbytes),
                    "mode": "MatvecStream: pinned host Q/Z per step, copies overlapped with the compute "
                            "of neighbouring steps (2 buffer pairs), L2 flushed before each product" if ws == 1 else "synchronous per step",
                    "d2h_bytes_per_step": int(M.n_row * R * 8),
                    "build_s": statistics.median(e2e_build) / 1e3,
                    "build_h2d_bytes": int(X.nbytes)},
            "parity": parity,
            "gpu_launches": int(round(launches_per_product * args.steps)),
            "clocks": clk.summary(),
            "swaps": list(M.swaps),
            "configs": extras,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
