#!/usr/bin/env python
"""Benchmark: SMASH H^2 build time + H^2 matvec Gpoints/s (fp64) on B200.

Workload (BASELINE.json configs[1]): config 2 -- N = 2^17
uniform points in the unit square, K(x,y) = 1/|x-y| (diagonal 0), adaptive
quadtree nu0 = 64, tensor Chebyshev 6x6 (r = 36), eta = 0.7, sRRQR tolerance
1e-8, fp64, 16 N(0,1) right-hand sides (seeded synthetic data).

A step is one H^2 matvec (nrhs = 16) through the device API on a matrix built
once; ``value`` = N * nrhs / t_matvec in Gpoints/s.  The build (tree + pair
lists + compression) is timed separately over the same warm-up / step counts
and reported as ``build_s``.  ``e2e`` repeats both through the public API with
host (pinned) buffers and the host<->device copies inside the timed region.

Usage:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config C] [--nrhs R] [--N n]
For N > 1 run under torchrun: every rank builds the (replicated) matrix; the
matvec is sharded by subtree (shard.py) with one NCCL exchange of the skeleton
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
# counted by ncu on k_block -- profiles/ckernel_r01.txt); 2*nrhs flops per interaction added.
C_K = {"inv_r": 14.0, "log": 51.0, "exp": 52.0, "cauchy": 11.0}
L2_FLUSH_BYTES = 256 << 20
# dram__bytes_read.sum + dram__bytes_write.sum per launch (ncu --set full, profiles/coupling_r01.txt)
NCU_TRAFFIC = {(2, 16, "k_coupling"): 26.45e6}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--nrhs", type=int, default=16)
    ap.add_argument("--N", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
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

def oracle_run(cfg, N, nrhs, warmup, steps, seed=None):
    """Reference CPU implementation (oracle port, single thread like the
    reference's serial Python loops; blocks cached like use_cache=True)."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import smash_oracle as orc
    from paper_1705_05443_b200.workloads import CONFIGS, make_points
    c = CONFIGS[cfg]
    X, Y, rng = make_points(cfg, N=N, seed=seed)
    q = rng.standard_normal((X.shape[0], nrhs))
    t0 = time.perf_counter()
    tree = orc.build_tree(X, None if Y is X else Y, nu0=c["nu0"], mode=c["mode"])
    if c["structure"] == "h2":
        M = orc.build_h2(tree, c["kernel"], c["r"], c["tau"], rtol=c["rtol"],
                         dx=None if c["kernel"] == "exp" else 0.0, symmetric=Y is X)
    else:
        M = orc.build_hss(tree, c["kernel"], c["r"], c["tau"], c["eps_svd"], rtol=c["rtol"],
                          dx=None if c["kernel"] == "exp" else 0.0)
    t_build = time.perf_counter() - t0
    cache = {}
    for _ in range(max(warmup, 1)):
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
    from paper_1705_05443_b200.workloads import CONFIGS
    N = args.N or CONFIGS[cfg]["N"]
    steps = max(1, min(args.steps, 5))
    t_build, t_mv, n = oracle_run(cfg, N, args.nrhs, 1, steps)
    val = n * args.nrhs / t_mv / 1e9
    line = {
        "impl": "reference", "metric": "SMASH build time + H^2 matvec Gpoints/s (fp64), 1/2/4/8 B200, % roofline",
        "value": val, "unit": "Gpoints/s", "n_gpus": args.gpus, "steps": steps, "warmup": 1,
        "ms_per_step": t_mv * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded, SURVEY.md 8(d))",
        "config": workload_config(cfg, N, args.nrhs),
        "build_s": t_build,
        "cpu_baseline": {"value": val, "unit": "Gpoints/s", "cores": 1, "kind": "port",
                         "sample": "full workload, oracle port of the reference algorithm "
                                   "(numpy/scipy, serial like the reference; blocks cached "
                                   "as use_cache=True; %d timed matvecs after 1 warm-up)" % steps},
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
# our arm
# ---------------------------------------------------------------------------

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
    cfg, R = args.config, args.nrhs
    c = CONFIGS[cfg]
    N = args.N or c["N"]
    X, Y, rng = make_points(cfg, N=N)
    q = rng.standard_normal((X.shape[0], R))
    spec, params = build_params(cfg)
    dev = torch.device("cuda", torch.cuda.current_device())
    dX = torch.from_numpy(X).to(dev)
    dQ = torch.from_numpy(q).to(dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    builder = sg.build_h2 if c["structure"] == "h2" else sg.build_hss

    # N > 1 (H2, shared points): sharded construction -- every rank compresses its
    # share of the levels at and below the cut, one NCCL all-reduce per factor buffer,
    # top levels redundant; the result is the full matrix on every rank
    sharded_build = ws > 1 and c["structure"] == "h2" and Y is X

    def build_device():
        tree = sg.build_tree(sg.PointSet(dX), None if Y is X else sg.PointSet(torch.from_numpy(Y).to(dev)),
                             nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
        if sharded_build:
            return tree, sg.build_h2_sharded(tree, spec, None, None, params)
        return tree, builder(tree, spec, None, None, params)

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- build: W warm-up + K timed (CUDA events on the launch stream)
    for _ in range(args.warmup):
        build_device()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    build_ms = []
    for _ in range(args.steps):
        flush.zero_()
        e0.record()
        tree, M = build_device()
        e1.record()
        e1.synchronize()
        build_ms.append(e0.elapsed_time(e1))
    barrier()
    if ws > 1:  # build time = max over ranks
        tb = torch.tensor([statistics.median(build_ms)], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tb, op=torch.distributed.ReduceOp.MAX)
        build_ms = [float(tb[0])]

    # ---- matvec: W warm-up + K timed, L2 flushed between timed matvecs.
    # N > 1: the sharded matvec (strong scaling of the fixed problem): every rank
    # holds the replicated matrix and q, computes its owned rows, and the skeleton
    # coefficients are exchanged once per matvec over NCCL (shard.py).
    out = torch.empty((M.n_row, R), dtype=torch.float64, device=dev)
    if ws > 1:
        from paper_1705_05443_b200.shard import ShardedMatvec
        sm = ShardedMatvec(M)

        def apply():
            return sm(dQ, gather_output=False)
    else:
        def apply():
            return sg.matvec_device(M, dQ, out)
    for _ in range(args.warmup):
        apply()
    lib = _lib.load()
    import ctypes
    lib.smash_matvec_profile(M._h, 1, None, None)
    barrier()
    mv_ms = []
    with ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(args.steps):
            flush.zero_()
            barrier() if ws > 1 else None
            e0.record()
            res = apply()
            e1.record()
            e1.synchronize()
            mv_ms.append(e0.elapsed_time(e1))
        barrier()
    if ws > 1:
        out = res
    phase = (ctypes.c_double * 7)()
    launches = ctypes.c_int64()
    lib.smash_matvec_profile(M._h, 0, phase, ctypes.byref(launches))
    t_mv = sum(mv_ms) / 1e3
    # max over ranks
    if ws > 1:
        t = torch.tensor([t_mv, max(build_ms)], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_mv = float(t[0])
    value = args.steps * M.n_row * R / t_mv / 1e9

    # ---- e2e through the public API with pinned host buffers: every step copies its
    # right-hand sides host->device and its result device->host (inside the timed
    # region); MatvecStream overlaps those copies of neighbouring steps with the
    # compute (copy engines), as a serving loop would
    q_pin = [torch.from_numpy(q).pin_memory(), torch.from_numpy(q.copy()).pin_memory()]
    z_pin = [torch.empty((M.n_row, R), dtype=torch.float64).pin_memory() for _ in range(2)]
    X_host = X
    e2e_mv = []
    if ws > 1:
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
        tree_h = sg.build_tree(sg.PointSet(X_host), None if Y is X else sg.PointSet(Y), nu0=c["nu0"],
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

    # ---- parity spot check of the timed output (device result vs public-API result)
    if ws == 1:
        zd = out.cpu().numpy()
        assert np.allclose(zd, z.numpy(), rtol=0, atol=0), "device and e2e results differ"
    else:  # sharded (full, gathered) vs the single-GPU matvec
        zf = sg.matvec_device(M, dQ).cpu().numpy()
        rel = np.linalg.norm(z.numpy() - zf) / np.linalg.norm(zf)
        assert rel <= 1e-12, "sharded matvec differs from the single-GPU one: %g" % rel

    # ---- roofline of the dominant kernel (coupling or leaf P2P)
    L, Lm = sg.leaf_sets(M.tree, c["tau"], c["structure"])
    Er = M.export_side(0)
    Ec = M.export_side(1)
    rk_r, rk_c = Er["rank"], Ec["rank"]
    Lh = np.array(L, dtype=np.int64).reshape(-1, 2)
    Lmh = np.array(Lm, dtype=np.int64).reshape(-1, 2)
    A = M.tree.arrays()
    nr = A["row_stop"] - A["row_start"]
    ncl = A["col_stop"] - A["col_start"]
    if ws > 1:  # this rank's launches cover its owned + top coupling targets / owned leaves
        mine = np.zeros(len(nr), bool)
        mine[sm.owned] = True
        top = np.zeros(len(nr), bool)
        top[sm.top] = True
        Lh = Lh[mine[Lh[:, 0]] | top[Lh[:, 0]]] if Lh.size else Lh
        Lmh = Lmh[mine[Lmh[:, 0]]] if Lmh.size else Lmh
    I_coup = float(np.sum(rk_r[Lh[:, 0]] * rk_c[Lh[:, 1]])) if Lh.size else 0.0
    I_near = float(np.sum(nr[Lmh[:, 0]] * ncl[Lmh[:, 1]])) if Lmh.size else 0.0
    per_int = C_K[c["kernel"]] + 2 * R
    ms_coup = phase[2] / args.steps
    ms_near = phase[4] / args.steps
    if ms_coup >= ms_near:
        dom, flops, ms = "k_coupling", I_coup * per_int, ms_coup
    else:
        dom, flops, ms = "k_near", I_near * per_int, ms_near
    achieved = flops / (ms / 1e3) / 1e12
    total_flops = (I_coup + I_near) * per_int
    # DRAM traffic per launch of the dominant kernel from one ncu --set full capture
    # (profiles/coupling_r01.txt; only measured for the default cfg2 / 16-RHS workload)
    traffic = NCU_TRAFFIC.get((cfg, R, dom))
    roofline = {"bound": "fp64", "kernel": dom, "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                "peak_source": "measured DFMA microbenchmark (profiles/fp64_peak_r01.txt); "
                               "MEASURED_PEAKS.json has no FP64 entry",
                "flops_per_launch": flops, "ms_per_launch": ms,
                "c_K": C_K[c["kernel"]], "interactions_coupling": I_coup, "interactions_near": I_near,
                "matvec_total_frac": total_flops / (t_mv / args.steps) / 1e12 / FP64_PEAK_TFLOPS,
                "scope": "rank 0's share" if ws > 1 else "whole matvec"}

    # ---- construction roofline: algorithmic FP64 work of the batched sRRQR
    # (per compr call on an m x n panel, sum_{i<min(m,n)} 4(m-i)(n-i-1)
    # for the pivoted QR plus k^2 (n-k) for G = (R11^-1 R12)^T), one side when the
    # column factors alias the row factors, over the whole build time
    build_flops = 0.0
    sides = [Er] if (Y is X and c["structure"] == "h2") else [Er, Ec]
    for E in sides:
        nib = np.diff(E["perm_ptr"]).astype(np.float64)
        kk = E["rank"].astype(np.float64)
        m_rows = float(c["r"])
        for nv, kv in zip(nib, kk):
            if nv <= 0:
                continue
            steps = int(min(m_rows, nv))
            i = np.arange(steps, dtype=np.float64)
            build_flops += float(np.sum(4.0 * (m_rows - i) * np.maximum(nv - i - 1.0, 0.0)))
            build_flops += kv * kv * (nv - kv)
    b_s = statistics.median(build_ms) / 1e3
    build_roofline = {"bound": "fp64", "flops": build_flops, "achieved": build_flops / b_s / 1e12,
                      "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                      "frac": build_flops / b_s / 1e12 / FP64_PEAK_TFLOPS,
                      "note": "algorithmic sRRQR flops (QR + G solve) over the whole build time "
                              "(tree + pair lists + basis + sRRQR)"}

    # ---- CPU baseline (oracle port) on a bounded sample, rank 0, N = 1 only
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        n_s = min(N, 2 ** 14)
        tb, tm, n_used = oracle_run(cfg, n_s, R, 1, 3)
        cpu = {"value": n_used * R / tm / 1e9, "unit": "Gpoints/s", "cores": 1, "kind": "port",
               "sample": "cfg%d geometry at N=%d (of %d), %d RHS, 3 cached matvecs after 1 warm-up; "
                         "oracle build %.2f s" % (cfg, n_used, N, R, tb),
               "build_s_sample": tb}

    if rank == 0:
        line = {
            "metric": "SMASH build time + H^2 matvec Gpoints/s (fp64), 1/2/4/8 B200, % roofline",
            "value": value, "unit": "Gpoints/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_mv * 1e3 / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY.md 8(d))",
            "config": workload_config(cfg, N, R),
            "build_s": statistics.median(build_ms) / 1e3,
            "build_mode": "sharded (NCCL all-reduce at the cut level)" if sharded_build else "single",
            "phase_ms": {"gather": phase[0] / args.steps, "upward": phase[1] / args.steps,
                         "coupling": ms_coup, "downward": phase[3] / args.steps,
                         "nearfield_concurrent": ms_near, "leaf_farfield": phase[5] / args.steps,
                         "matvec": phase[6] / args.steps},
            "roofline": roofline,
            "build_roofline": build_roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "Gpoints/s", "h2d_bytes_per_step": int(q.nbytes),
                    "mode": "MatvecStream: pinned host Q/Z per step, copies overlapped with the compute "
                            "of neighbouring steps (2 buffer pairs), L2 flushed before each product" if ws == 1 else "synchronous per step",
                    "d2h_bytes_per_step": int(M.n_row * R * 8),
                    "build_s": statistics.median(e2e_build) / 1e3,
                    "build_h2d_bytes": int(X.nbytes)},
            "gpu_launches": int(launches.value),
            "clocks": clk.summary(),
            "swaps": list(M.swaps),
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
