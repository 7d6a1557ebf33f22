"""Sharded H^2 construction: every rank compresses its contiguous
share of the levels at and below the cut, the disjoint factor buffers are summed
over the ranks, and the top levels are compressed redundantly.  The result must
equal the single-GPU build bit for bit (same kernels on the same data).

GPU tests: ranks simulated in one process (sum of the exchanged buffers done with
torch), and a real 2-process group (gloo, both ranks on cuda:0: the exchange is
a host-driven collective, no kernel waits on another rank's kernel).
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sg():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1705_05443_b200 as sg
    return sg


def _case(sg, cfg, N):
    from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points
    c = CONFIGS[cfg]
    X, Y, rng = make_points(cfg, N=N)
    spec, params = build_params(cfg)
    tree = sg.build_tree(sg.PointSet(X), nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
    q = rng.standard_normal((X.shape[0], 4))
    return tree, spec, params, q


def _same(M, R):
    for side in (0, 1):
        a, b = M.export_side(side), R.export_side(side)
        for k in ("has", "rank", "perm_ptr", "skel_ptr", "g_ptr"):
            assert np.array_equal(a[k], b[k]), k
        n = a["perm_ptr"][-1]
        assert np.array_equal(a["perm"][:n], b["perm"][:n])
        ns = a["skel_ptr"][-1]
        assert np.array_equal(a["skel"][:ns], b["skel"][:ns])
        ng = a["g_ptr"][-1]
        assert np.array_equal(a["G"][:ng], b["G"][:ng])


@pytest.mark.parametrize("cfg,N,world,cut", [(2, 1 << 14, 2, 0), (2, 1 << 14, 3, 0), (5, 1 << 15, 4, 0),
                                             (3, 1 << 13, 2, 0), (2, 1 << 14, 2, 3), (1, 4096, 1, 0)])
def test_sharded_equals_single(sg, cfg, N, world, cut):
    import torch
    tree, spec, params, q = _case(sg, cfg, N)  # cfg 1: its 1-D binary tree built as H^2
    ref = sg.build_h2(tree, spec, None, None, params)
    pend = [sg.build_h2_local(tree, spec, params, r, world, cut) for r in range(world)]
    bufs = [p.buffers() for p in pend]
    for i in range(len(bufs[0])):
        tot = sum(b[i] for b in bufs)
        for b in bufs:
            b[i].copy_(tot)
    mats = [p.finish() for p in pend]
    zr = sg.matvec_nodewise(ref, q)
    for M in mats:
        _same(M, ref)
        assert tuple(M.swaps) == tuple(ref.swaps)
        assert np.array_equal(sg.matvec_nodewise(M, q), zr)
    torch.cuda.synchronize()


def _worker(rank, world, port, cfg, N, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1705_05443_b200 as sg
    tree, spec, params, q = _case(sg, cfg, N)
    M = sg.build_h2_sharded(tree, spec, None, None, params, replicate_factors=True)
    R = sg.build_h2(tree, spec, None, None, params)
    ok = True
    try:
        _same(M, R)
        ok = np.array_equal(sg.matvec_nodewise(M, q), sg.matvec_nodewise(R, q))
    except AssertionError:
        ok = False
    out.put((rank, ok))
    dist.destroy_process_group()


def test_sharded_two_processes_gloo(sg):
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 2, 1 << 14, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


def _worker_sharded(rank, world, port, cfg, N, out):
    """Sharded factors (replicate_factors=False) + ShardedMatvec with the halo all-to-all:
    the owned + top factors equal the single-GPU build's bit for bit, and the gathered
    product equals the single-GPU matvec."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1705_05443_b200 as sg
    from paper_1705_05443_b200.shard import ShardedMatvec
    tree, spec, params, q = _case(sg, cfg, N)
    M = sg.build_h2_sharded(tree, spec, None, None, params)
    R = sg.build_h2(tree, spec, None, None, params)
    res = {}
    try:
        sm = ShardedMatvec(M)
        mine = set(int(v) for v in np.nonzero((M.shard_owner == rank) | (M.shard_owner < 0))[0])
        ok = True
        for side in (0, 1):
            a, b = M.export_side(side), R.export_side(side)
            for v in mine:
                if not a["has"][v]:
                    continue
                for key, ptr in (("perm", "perm_ptr"), ("G", "g_ptr"), ("skel", "skel_ptr")):
                    ok &= bool(np.array_equal(a[key][a[ptr][v]:a[ptr][v + 1]], b[key][b[ptr][v]:b[ptr][v + 1]]))
        Q = torch.from_numpy(q).cuda()
        z = sm(Q, gather_output=True).cpu().numpy()
        zr = sg.matvec_nodewise(R, q)
        rel = float(np.linalg.norm(z - zr) / np.linalg.norm(zr))
        try:
            sg.matvec_nodewise(M, q)
            guarded = False
        except ValueError:
            guarded = True
        res = dict(ok=ok, rel=rel, guarded=guarded, halo=sm.halo_rows_total,
                   rows=int(sm.half))
    except Exception as e:  # report instead of hanging the other rank
        res = dict(err=repr(e))
    out.put((rank, res))
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,N,world", [(2, 1 << 14, 2), (5, 1 << 15, 2), (3, 1 << 13, 3)])
def test_sharded_factors_and_matvec_processes_gloo(sg, cfg, N, world):
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_sharded, args=(r, world, port, cfg, N, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert "err" not in res[r], res[r]
        assert res[r]["ok"] and res[r]["guarded"], res[r]
        assert res[r]["rel"] <= 1e-13, res[r]
        assert res[r]["halo"] < 2 * res[r]["rows"]  # the halo is not an all-gather


def _same_hss(M, R):
    _same(M, R)
    assert tuple(M.swaps) == tuple(R.swaps)


def _worker_hss(rank, world, port, cfg, N, out):
    """Level-distributed HSS construction (build_hss_sharded): every rank compresses a
    share of each level and the level's outputs are summed through the exchange
    callback; every rank must hold build_hss's matrix bit for bit."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1705_05443_b200 as sg
    res = {}
    try:
        tree, spec, params, q = _case(sg, cfg, N)
        M = sg.build_hss_sharded(tree, spec, None, None, params)
        R = sg.build_hss(tree, spec, None, None, params)
        _same_hss(M, R)
        res = dict(ok=bool(np.array_equal(sg.matvec_nodewise(M, q), sg.matvec_nodewise(R, q))))
    except AssertionError as e:
        res = dict(ok=False, why=repr(e))
    except Exception as e:  # report instead of hanging the other rank
        res = dict(err=repr(e))
    out.put((rank, res))
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,N,world", [(1, 1 << 14, 2), (4, 1 << 14, 2), (1, 1 << 13, 3)])
def test_hss_sharded_processes_gloo(sg, cfg, N, world):
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_hss, args=(r, world, port, cfg, N, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert res[r].get("ok"), res[r]
