"""Multi-rank host logic of the sharded matvec (paper_1705_05443_b200/shard.py),
run with torch.distributed gloo, world_size 2 and 3, on CPU.

Each rank executes the same staged algorithm the GPU path runs (work-balanced cut
partition -> local upward of owned subtrees -> halo all-to-all of exactly the
coefficient rows halo_rows() lists -> top upward, coupling / downward for owned +
top targets, nearfield + far field for owned leaves -> all-reduce of z), with numpy
on the oracle's factors; the result must equal the single-process oracle matvec.
Coefficients that are neither owned, replicated nor received stay NaN, so a missing
halo row cannot go unnoticed."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import load_golden
from oracle import smash_oracle as orc
from paper_1705_05443_b200.shard import cut_partition, halo_rows, own_top_leaves, partition, subtree_work


def tree_arrays(t):
    n = t.n_nodes
    cp = np.zeros(n + 1, np.int64)
    for i, c in enumerate(t.children):
        cp[i + 1] = cp[i] + len(c)
    ci = np.array([c for ch in t.children for c in ch], np.int64)
    return dict(child_ptr=cp, child_idx=ci, row_start=t.row_start, row_stop=t.row_stop,
                col_start=t.col_start, col_stop=t.col_stop, level=t.level, parent=t.parent)


def staged_matvec(M, q, owner, rank, world):
    """One rank's stages (numpy mirror of smash_matvec_stage 1 / halo / 2)."""
    tr = M.tree
    n = tr.n_nodes
    root = tr.root
    owned = np.nonzero(owner == rank)[0]
    top = np.nonzero(owner < 0)[0]
    qt = q[tr.perm_col]
    R = q.shape[1]
    kcol = np.array([M.colfac[v].rank if v in M.colfac else 0 for v in range(n)], np.int64)
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(kcol)
    row_off = np.where(kcol > 0, off[:-1], -1)
    buf = np.full((off[-1], R), np.nan)

    def up(v):
        if tr.is_leaf(v):
            iv = qt[tr.col_start[v]:tr.col_stop[v]]
        else:
            iv = np.concatenate([buf[off[c]:off[c + 1]] for c in tr.children[v]])
        buf[off[v]:off[v + 1]] = M.colfac[v].expand().T @ iv

    for v in sorted((v for v in owned if v != root), key=lambda v: -tr.level[v]):
        up(v)
    rows, _ = halo_rows(owner, tr.parent, M.pairs_L, row_off, kcol, world)
    send = torch.from_numpy(np.ascontiguousarray(
        np.concatenate([buf[rows[rank][s_]] for s_ in range(world)]).reshape(-1)))
    recv_rows = np.concatenate([rows[s_][rank] for s_ in range(world)])
    recv = torch.empty(recv_rows.size * R, dtype=torch.float64)
    dist.all_to_all_single(recv, send, [rows[s_][rank].size * R for s_ in range(world)],
                           [rows[rank][s_].size * R for s_ in range(world)])
    buf[recv_rows] = recv.numpy().reshape(-1, R)
    for v in sorted((v for v in top if v != root), key=lambda v: -tr.level[v]):
        up(v)
    targets = set(int(v) for v in owned) | set(int(v) for v in top)
    targets.discard(root)
    Xr, Xc = tr.points_row, tr.points_col
    zhat = {}
    for v in targets:
        z = np.zeros((M.rowfac[v].rank, R))
        for i, j in M.pairs_L:
            if i == v:
                z += orc.kernel_block(M.kernel, Xr[M.skel_row[i]], Xc[M.skel_col[j]], M.dx) @ buf[off[j]:off[j + 1]]
        zhat[v] = z
    for v in sorted((v for v in targets if not tr.is_leaf(v)), key=lambda v: tr.level[v]):
        y = M.rowfac[v].expand() @ zhat[v]
        o = 0
        for c in tr.children[v]:
            k = M.rowfac[c].rank
            if c in zhat:  # children owned by another rank are not needed here
                zhat[c] = zhat[c] + y[o:o + k]
            o += k
    zt = np.zeros((tr.perm_row.size, R))
    for v in (int(v) for v in owned if tr.is_leaf(int(v))):
        a, b = tr.row_start[v], tr.row_stop[v]
        if v != root:
            zt[a:b] += M.rowfac[v].expand() @ zhat[v]
        for i, j in M.pairs_Lm:
            if i == v:
                zt[a:b] += orc.kernel_block(M.kernel, Xr[a:b], Xc[tr.col_start[j]:tr.col_stop[j]], M.dx) @ qt[tr.col_start[j]:tr.col_stop[j]]
    z = np.zeros_like(zt)
    z[tr.perm_row] = zt
    t = torch.from_numpy(z)
    dist.all_reduce(t)  # disjoint rows
    return t.numpy()


def _worker(rank, world, port, name, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = load_golden(name)
        m = g["meta"]
        tree = orc.build_tree(g["X"], None, nu0=m["nu0"], mode=m["mode"])
        M = orc.build_h2(tree, m["kernel"], m["r"], m["tau"], rtol=m["rtol"],
                         dx=None if m["kernel"] == "exp" else 0.0, symmetric=True)
        A = tree_arrays(tree)
        L, Lm = np.asarray(M.pairs_L), np.asarray(M.pairs_Lm)
        w = subtree_work(A, L, Lm, m["r"])
        cut = next((l for l in range(2, tree.n_levels + 1) if np.sum(A["level"] == l) >= 8 * world),
                   tree.n_levels)
        owner, cut_nodes = cut_partition(A, world, cut, w[A["level"] == cut])
        owner = own_top_leaves(A, owner, world, w)
        z = staged_matvec(M, g["q"], owner, rank, world)
        if rank == 0:
            zr = orc.matvec(M, g["q"])
            ret.put((float(np.linalg.norm(z - zr) / np.linalg.norm(zr)),
                     [int(np.sum(owner == r)) for r in range(world)], len(cut_nodes)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["cfg2_4k", "clustered2d"])
def test_sharded_matvec_gloo(name, world):
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, ret)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    rel, sizes, nf = ret.get(timeout=10)
    assert rel <= 1e-13, rel
    assert all(s > 0 for s in sizes) and nf >= 8 * world


def test_cut_partition_balances_work():
    """Work-balanced cut partition (the rule smash_matrix_build_local_w applies): every
    node owned once or replicated, owned subtrees contiguous, and the ranks' matvec work
    within the granularity of one cut-level subtree of each other."""
    g = load_golden("cfg5_16k")
    m = g["meta"]
    tree = orc.build_tree(g["X"], None, nu0=m["nu0"], mode=m["mode"])
    A = tree_arrays(tree)
    OM = orc.build_h2(tree, m["kernel"], m["r"], m["tau"], rtol=m["rtol"], dx=0.0, symmetric=True)
    w = subtree_work(A, np.asarray(OM.pairs_L), np.asarray(OM.pairs_Lm), m["r"])
    for world in (2, 4, 8):
        cut = next(l for l in range(2, tree.n_levels + 1) if np.sum(A["level"] == l) >= 8 * world)
        owner, cut_nodes = cut_partition(A, world, cut, w[A["level"] == cut])
        for v in range(tree.n_nodes):  # subtrees inherit their cut node's owner
            if owner[v] >= 0 and tree.level[v] > cut:
                assert owner[v] == owner[tree.parent[v]]
        per = np.array([w[cut_nodes][owner[cut_nodes] == r].sum() for r in range(world)])
        assert per.min() > 0
        assert per.max() - per.min() <= 2 * w[cut_nodes].max() + 1e-9
        o2 = own_top_leaves(A, owner, world, w)
        leaves = np.array([tree.is_leaf(v) for v in range(tree.n_nodes)])
        assert np.all(o2[leaves] >= 0)


def test_partition_covers_every_node_once():
    g = load_golden("cfg5_16k")
    m = g["meta"]
    tree = orc.build_tree(g["X"], None, nu0=m["nu0"], mode=m["mode"])
    A = tree_arrays(tree)
    for world in (1, 2, 4, 8):
        owned, top, frontier = partition(A, world)
        allv = np.concatenate(owned + [top])
        assert np.array_equal(np.sort(allv), np.arange(tree.n_nodes))
        # owned subtrees cover contiguous, increasing row ranges
        last = 0
        for r in range(world):
            fr = [f for f, o in frontier if o == r]
            for f in fr:
                assert tree.row_start[f] == last
                last = tree.row_stop[f]
        assert last == tree.perm_row.size
