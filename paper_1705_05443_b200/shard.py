"""Multi-GPU sharding: one process per GPU, torch.distributed
(NCCL over NVLink on a B200 node) for the data-path exchanges.

Partition.  The tree is cut at a level (the shallowest with >= 8 nodes per rank;
smash_matrix_shard_cut); the cut-level nodes, left to right, are split into
contiguous groups of roughly equal WORK -- the coupling interactions
sum_{j in L(i)} k_i k_j and nearfield interactions sum_{j in Lm(i)} n_i n_j of the
targets i in each subtree (``subtree_work``, ranks estimated as min(r, points)
before the build).  A rank owns the subtrees of its group; the nodes above the cut
("top") are replicated.  A sharded build (h2.build_h2_sharded) and the sharded
matvec use the same partition, so with ``replicate_factors=False`` each rank only
ever holds -- and needs -- the interpolative factors of its own subtrees and of the
top levels.

Matvec on rank r (ShardedMatvec):
  stage 1  gather q, upward pass of the owned subtrees;
  halo     all-to-all of skeleton coefficients: every rank receives exactly the
           coefficient rows its stage 2 reads from other ranks' subtrees -- the
           coupling sources of its owned + top targets, and the cut-level nodes
           (inputs of the replicated top upward pass) -- nothing else; the owned
           leaves' nearfield (stage 3, needs only q) runs on a side stream meanwhile;
  stage 2  upward pass of the top nodes, coupling / downward pass for owned + top
           targets, nearfield + leaf far field for the owned leaves: the owned rows
           of z (disjoint over ranks, no reduction);
  optional all-reduce of z when every rank needs the full result.
The plan is plain host logic (numpy), exercised with gloo on CPU in
tests/test_shard_gloo.py.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

__all__ = ["partition", "subtree_work", "cut_partition", "own_top_leaves", "halo_rows", "matvec_plan",
           "set_partition", "frontier_fixup", "ShardedMatvec"]


def subtree_work(A: dict, L: np.ndarray, Lm: np.ndarray, r: int, ranks=None) -> np.ndarray:
    """Per node (postorder): matvec work of the targets in its subtree -- coupling
    interactions k_i k_j over L and nearfield n_i n_j over Lm.  ``ranks`` (postorder)
    defaults to the estimate min(r, points)."""
    n = len(A["child_ptr"]) - 1
    pts = (A["row_stop"] - A["row_start"]).astype(np.float64)
    pc = (A["col_stop"] - A["col_start"]).astype(np.float64)
    k = np.minimum(float(r), pts) if ranks is None else np.asarray(ranks, np.float64)
    w = np.zeros(n)
    if len(L):
        np.add.at(w, L[:, 0], k[L[:, 0]] * k[L[:, 1]])
    if len(Lm):
        np.add.at(w, Lm[:, 0], pts[Lm[:, 0]] * pc[Lm[:, 1]])
    parent = A["parent"] if "parent" in A else None
    if parent is None:
        parent = np.full(n, -1, np.int64)
        cp, ci = A["child_ptr"], A["child_idx"]
        for v in range(n):
            parent[ci[cp[v]:cp[v + 1]]] = v
    for v in range(n):  # postorder: children before parents
        if parent[v] >= 0:
            w[parent[v]] += w[v]
    return w


def cut_partition(A: dict, world: int, cut: int, weights: np.ndarray):
    """Owner (postorder) of every node: contiguous left-to-right groups of the
    cut-level nodes balanced by ``weights`` (the rule of smash_matrix_build_local_w),
    descendants inherit, nodes above the cut (and leaves above it) get -1."""
    n = len(A["child_ptr"]) - 1
    level = A["level"]
    cut_nodes = np.nonzero(level == cut)[0]  # postorder within a level = left to right
    w = np.asarray(weights, np.float64)
    total = max(w.sum(), 1e-300)
    mid = np.cumsum(w) - 0.5 * w
    owner = np.full(n, -1, np.int64)
    owner[cut_nodes] = np.minimum(world - 1, (mid * world / total).astype(np.int64))
    cp, ci = A["child_ptr"], A["child_idx"]
    for v in range(n - 1, -1, -1):  # parents before children (reverse postorder)
        if owner[v] >= 0:
            owner[ci[cp[v]:cp[v + 1]]] = owner[v]
    return owner, cut_nodes


def own_top_leaves(A: dict, owner: np.ndarray, world: int, weights: np.ndarray) -> np.ndarray:
    """Leaves above the cut (adaptive trees) are replicated in the build; the matvec
    gives each to one rank (left to right, balanced by ``weights``) so its nearfield
    and far field are computed exactly once."""
    owner = owner.copy()
    nch = np.diff(A["child_ptr"])
    tl = np.nonzero((owner < 0) & (nch == 0))[0]
    if tl.size:
        tl = tl[np.argsort(A["row_start"][tl], kind="stable")]
        w = np.asarray(weights, np.float64)[tl]
        mid = np.cumsum(w) - 0.5 * w
        owner[tl] = np.minimum(world - 1, (mid * world / max(w.sum(), 1e-300)).astype(np.int64))
    return owner


def partition(A: dict, world: int, per_rank: int = 8, weights: np.ndarray = None):
    """Frontier partition of a tree given its exported arrays (postorder ids), for a
    replicated matrix: the frontier is expanded from the root (largest first) until
    there are >= per_rank frontier nodes per rank, then split left to right into
    contiguous groups of equal work (``weights`` per node, default row counts).

    Returns (owned, top, frontier_owner)."""
    child_ptr, child_idx = A["child_ptr"], A["child_idx"]
    rs, re = A["row_start"], A["row_stop"]
    n = len(child_ptr) - 1
    root = n - 1
    wt = (re - rs).astype(np.float64) if weights is None else np.asarray(weights, np.float64)

    def kids(i):
        return child_idx[child_ptr[i]:child_ptr[i + 1]]

    frontier = [root]
    while len(frontier) < per_rank * world:
        internal = [f for f in frontier if child_ptr[f + 1] > child_ptr[f]]
        if not internal:
            break
        big = max(internal, key=lambda f: (wt[f], -f))
        frontier.remove(big)
        frontier.extend(int(c) for c in kids(big))
    frontier.sort(key=lambda f: (rs[f], re[f]))
    total = max(float(sum(wt[f] for f in frontier)), 1e-300)
    owner = {}
    acc = 0.0
    for f in frontier:
        mid = acc + wt[f] / 2.0
        owner[f] = min(world - 1, int(mid * world / total))
        acc += wt[f]
    owned = [[] for _ in range(world)]
    in_sub = np.zeros(n, bool)
    for f in frontier:
        stack = [f]
        while stack:
            v = stack.pop()
            in_sub[v] = True
            owned[owner[f]].append(v)
            stack.extend(int(c) for c in kids(v))
    owned = [np.array(sorted(o), dtype=np.int64) for o in owned]
    top = np.nonzero(~in_sub)[0].astype(np.int64)
    return owned, top, [(f, owner[f]) for f in frontier]


def _rows_of(nodes, row_off, kcol):
    nodes = np.asarray(nodes, np.int64)
    nodes = nodes[(row_off[nodes] >= 0) & (kcol[nodes] > 0)]
    if nodes.size == 0:
        return np.zeros(0, np.int64)
    return np.concatenate([np.arange(row_off[v], row_off[v] + kcol[v], dtype=np.int64) for v in nodes])


def halo_rows(owner: np.ndarray, parent: np.ndarray, L: np.ndarray, row_off: np.ndarray,
              kcol: np.ndarray, world: int):
    """Coefficient rows each rank must receive from each other rank: rank s needs,
    from rank r != s, the rows of r's nodes that are coupling sources of s's targets
    (owned + replicated top nodes) or frontier nodes (owned nodes whose parent is
    replicated: the inputs of the top upward pass).  owner: per node the owning rank
    (-1: replicated); L: coupling pairs (target, source); row_off / kcol: coefficient
    rows [row_off, row_off + k) per node.  Returns rows[r][s] (sorted int64 arrays:
    rank r sends them to rank s) and the frontier nodes."""
    n = owner.size
    frontier = np.nonzero((owner >= 0) & ((parent < 0) | (owner[np.maximum(parent, 0)] < 0)))[0]
    rows = [[np.zeros(0, np.int64) for _ in range(world)] for _ in range(world)]
    for s in range(world):
        tgt = (owner == s) | (owner < 0)
        need = np.zeros(n, bool)
        if len(L):
            need[L[tgt[L[:, 0]], 1]] = True
        need[frontier] = True
        need &= (owner >= 0) & (owner != s)
        for r in range(world):
            if r != s:
                rows[r][s] = _rows_of(np.nonzero(need & (owner == r))[0], row_off, kcol)
    return rows, frontier


class _DevBuf:
    """__cuda_array_interface__ view of a library-owned device buffer."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


def matvec_plan(M, world: int, per_rank: int = 8) -> dict:
    """Host plan of a sharded matvec of M over ``world`` ranks (no communication):
    owner per node (M.shard_owner of a sharded build, else a work-balanced frontier
    partition; leaves above the cut handed to one rank each), the coefficient layout
    (row_off per node, up_pos per coefficient row, half = rows per half of the buffer)
    and the halo rows[r][s] rank r sends to rank s."""
    from .cluster import _pairs
    A = M.tree.arrays()
    L, Lm = _pairs(M.tree, M.params.tau, M.kind)
    kcol = M.export_side(1)["rank"]
    n = len(A["level"])
    owner = getattr(M, "shard_owner", None)
    w = subtree_work(A, L, Lm, M.params.r, kcol)
    if owner is None:
        owned, _, _ = partition(A, world, per_rank, w)
        owner = np.full(n, -1, np.int64)
        for r_, o in enumerate(owned):
            owner[o] = r_
    owner = own_top_leaves(A, np.asarray(owner, np.int64), world, w)
    lib = _lib.load()
    row_off = np.zeros(n, np.int64)
    half = _lib.c_i64()
    _lib.check(lib.smash_matvec_coeff_layout(M._h, row_off.ctypes.data_as(ctypes.c_void_p), None,
                                             ctypes.byref(half), _lib.stream_ptr()))
    up_pos = np.zeros(half.value, np.int64)
    _lib.check(lib.smash_matvec_coeff_layout(M._h, row_off.ctypes.data_as(ctypes.c_void_p),
                                             up_pos.ctypes.data_as(ctypes.c_void_p),
                                             ctypes.byref(half), _lib.stream_ptr()))
    rows, frontier = halo_rows(owner, A["parent"], L, row_off, kcol, world)
    return dict(owner=owner, row_off=row_off, up_pos=up_pos, half=half.value, rows=rows,
                frontier=frontier, kcol=kcol)


def set_partition(M, plan: dict, rank: int):
    """Hand rank's owned / replicated node lists to the device matvec (stage kernels)."""
    owner = plan["owner"]
    own = np.ascontiguousarray(np.nonzero(owner == rank)[0].astype(np.int64))
    tp = np.ascontiguousarray(np.nonzero(owner < 0)[0].astype(np.int64))
    _lib.check(_lib.load().smash_matvec_set_partition(
        M._h, own.ctypes.data_as(ctypes.c_void_p), own.size, tp.ctypes.data_as(ctypes.c_void_p),
        tp.size, _lib.stream_ptr()))
    return own, tp


def frontier_fixup(plan: dict, rank: int):
    """(src, dst) coefficient rows: received cut-level rows copied into the parent-ibar
    half of the buffer, the input order of the top upward pass."""
    owner, fr = plan["owner"], plan["frontier"]
    m = np.zeros(plan["half"], bool)
    m[_rows_of(fr[owner[fr] != rank], plan["row_off"], plan["kcol"])] = True
    src = np.nonzero(m & (plan["up_pos"] >= 0))[0]
    return src, plan["half"] + plan["up_pos"][src]


class ShardedMatvec:
    """Rank-local sharded matvec over a process group.  M is either a matrix built by
    h2.build_h2_sharded (its partition and sharded factors are used) or a replicated
    matrix (a work-balanced frontier partition is computed)."""

    def __init__(self, M, group=None, per_rank: int = 8):
        import torch
        import torch.distributed as dist
        self.M = M
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        plan = matvec_plan(M, self.world, per_rank)
        self.owner = plan["owner"]
        self.owned, self.top = set_partition(M, plan, self.rank)
        self.half = plan["half"]
        rows = plan["rows"]
        self.frontier_nodes = plan["frontier"]
        self.send_counts = [int(rows[self.rank][s].size) for s in range(self.world)]
        self.recv_counts = [int(rows[s][self.rank].size) for s in range(self.world)]
        cat = lambda xs: np.concatenate(xs) if xs else np.zeros(0, np.int64)  # noqa: E731
        dev = torch.device("cuda", torch.cuda.current_device())
        self.send_idx = torch.from_numpy(cat([rows[self.rank][s] for s in range(self.world)])).to(dev)
        self.recv_idx = torch.from_numpy(cat([rows[s][self.rank] for s in range(self.world)])).to(dev)
        src, dst = frontier_fixup(plan, self.rank)
        self.fr_src = torch.from_numpy(src).to(dev)
        self.fr_dst = torch.from_numpy(dst).to(dev)
        self.halo_rows_total = int(sum(rows[r][s].size for r in range(self.world) for s in range(self.world)))

    def coeff_view(self, nrhs: int):
        import torch
        p = ctypes.c_void_p()
        rows = _lib.c_i64()
        _lib.check(_lib.load().smash_matvec_coeffs(self.M._h, ctypes.byref(p), ctypes.byref(rows)))
        return torch.as_tensor(_DevBuf(p.value, rows.value * nrhs), device="cuda").view(rows.value, nrhs)

    def halo_bytes(self, nrhs: int) -> int:
        """Coefficient bytes moved over the whole group per matvec."""
        return self.halo_rows_total * nrhs * 8

    def exchange(self, nrhs: int):
        """The halo all-to-all of skeleton coefficients between the stages."""
        import torch
        import torch.distributed as dist
        C = self.coeff_view(nrhs)
        send = C.index_select(0, self.send_idx).reshape(-1)
        recv = torch.empty(sum(self.recv_counts) * nrhs, dtype=torch.float64, device=C.device)
        ins = [c * nrhs for c in self.send_counts]
        outs = [c * nrhs for c in self.recv_counts]
        if self.backend == "gloo":  # host-staged (the CPU test backend)
            rh = recv.cpu()
            dist.all_to_all_single(rh, send.cpu(), outs, ins, group=self.group)
            recv.copy_(rh)
        else:
            dist.all_to_all_single(recv, send, outs, ins, group=self.group)
        C.index_copy_(0, self.recv_idx, recv.view(-1, nrhs))
        if self.fr_src.numel():
            C.index_copy_(0, self.fr_dst, C.index_select(0, self.fr_src))

    def __call__(self, Q, gather_output: bool = True, overlap: bool = True):
        """Q: (n_col, nrhs) CUDA float64, replicated on every rank (nrhs a power of
        two <= 16).  Returns z (n_row, nrhs): the owned rows (others 0), or the full
        product when gather_output.  overlap: the owned leaves' nearfield (stage 3, it
        needs only q) runs on a side stream during the halo exchange."""
        import torch
        import torch.distributed as dist
        Q = Q.contiguous()
        nrhs = Q.shape[1]
        lib = _lib.load()
        z = torch.zeros((self.M.n_row, nrhs), dtype=torch.float64, device=Q.device)
        main = torch.cuda.current_stream()
        _lib.check(lib.smash_matvec_stage(self.M._h, 1, _lib.ptr(Q), _lib.ptr(z), nrhs, _lib.stream_ptr()))
        if overlap:
            if not hasattr(self, "_side"):
                self._side = torch.cuda.Stream()
            self._side.wait_stream(main)
            with torch.cuda.stream(self._side):
                _lib.check(lib.smash_matvec_stage(self.M._h, 3, _lib.ptr(Q), _lib.ptr(z), nrhs,
                                                  _lib.stream_ptr()))
            self.exchange(nrhs)
            main.wait_stream(self._side)
            _lib.check(lib.smash_matvec_stage(self.M._h, 4, _lib.ptr(Q), _lib.ptr(z), nrhs, _lib.stream_ptr()))
        else:
            self.exchange(nrhs)
            _lib.check(lib.smash_matvec_stage(self.M._h, 2, _lib.ptr(Q), _lib.ptr(z), nrhs, _lib.stream_ptr()))
        if gather_output:
            if self.backend == "gloo":
                zh = z.cpu()
                dist.all_reduce(zh, group=self.group)
                z.copy_(zh)
            else:
                dist.all_reduce(z, group=self.group)
        return z
