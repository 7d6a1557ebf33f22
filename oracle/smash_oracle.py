"""CPU oracle (TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

A plain numpy/scipy restatement of the reference SMASH hot path.  Every
function cites the reference file:line whose semantics it reproduces.  Data is
kept in flat arrays (node-indexed, postorder like the reference) rather than in
the reference's dataclasses, so the oracle can be compared array-for-array with
the GPU build.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla

__all__ = [
    "OTree", "OMatrix", "norm_rows", "box_center", "box_radius", "separated",
    "build_tree", "leaf_sets", "nearfield_sets", "cheb_nodes", "lagrange_cols",
    "interp_basis", "srrqr", "compr", "truncated_svd", "kernel_block",
    "build_h2", "build_hss", "matvec", "matvec_levelwise", "dense_matvec", "Factor",
    "make_config_points", "CONFIGS",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _geom_lib():
    """Load (building on first use, gcc only) the exact-FMA helper."""
    global _LIB
    if _LIB is None:
        out = os.path.join(_HERE, "_build", "liboracle_geom.so")
        src = os.path.join(_HERE, "oracle_geom.c")
        if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
            os.makedirs(os.path.dirname(out), exist_ok=True)
            subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                                   "-o", out, src, "-lm"])
        lib = ctypes.CDLL(out)
        lib.or_norm_rows.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                     ctypes.c_void_p]
        lib.or_norm_rows.restype = None
        _LIB = lib
    return _LIB


# ---------------------------------------------------------------------------
# geometry  (smash/cluster.py:48-85)
# ---------------------------------------------------------------------------


def norm_rows(v: np.ndarray) -> np.ndarray:
    """Row 2-norms with np.linalg.norm's FMA-chain order."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    if v.ndim == 1:
        v = v[None, :]
    out = np.empty(v.shape[0])
    if v.shape[0]:
        _geom_lib().or_norm_rows(v.ctypes.data, v.shape[0], v.shape[1], out.ctypes.data)
    return out


def box_center(lo, hi):
    """(lo + hi) / 2, smash/cluster.py:64-66."""
    return (np.asarray(lo, dtype=np.float64) + np.asarray(hi, dtype=np.float64)) / 2.0


def box_radius(lo, hi):
    """0.5 * ||hi - lo||, smash/cluster.py:68-71."""
    return 0.5 * norm_rows(np.asarray(hi, dtype=np.float64) - np.asarray(lo, dtype=np.float64))


def separated(loA, hiA, loB, hiB, tau: float) -> np.ndarray:
    """Vectorised well_separated (smash/cluster.py:81-85):
    radius(A) + radius(B) <= tau * ||center(A) - center(B)||."""
    dist = norm_rows(box_center(loA, hiA) - box_center(loB, hiB))
    return box_radius(loA, hiA) + box_radius(loB, hiB) <= tau * dist


# ---------------------------------------------------------------------------
# cluster tree  (smash/cluster.py:247-353)
# ---------------------------------------------------------------------------


@dataclass
class OTree:
    mode: str
    nu0: int
    dim: int
    level: np.ndarray        # int64[n]
    parent: np.ndarray       # int64[n], -1 at the root
    children: list           # list of tuples, child order
    lo: np.ndarray           # float64[n, d]
    hi: np.ndarray           # float64[n, d]
    row_start: np.ndarray
    row_stop: np.ndarray
    col_start: np.ndarray
    col_stop: np.ndarray
    perm_row: np.ndarray
    perm_col: np.ndarray
    points_row: np.ndarray
    points_col: np.ndarray
    _near: dict = field(default_factory=dict, repr=False)

    @property
    def n_nodes(self):
        return len(self.children)

    @property
    def root(self):
        return self.n_nodes - 1

    @property
    def n_levels(self):
        return int(self.level.max())

    def is_leaf(self, i):
        return len(self.children[i]) == 0

    def leaves(self):
        return [i for i in range(self.n_nodes) if not self.children[i]]

    def level_nodes(self, lev):
        return [int(i) for i in np.nonzero(self.level == lev)[0]]


def _cells(lo, hi, axes):
    """Sub-boxes of (lo, hi) from bisecting each axis in ``axes`` in turn,
    ordered lexicographically with the first axis most significant
    (smash/cluster.py:247-260 applied per axis as in :325-331)."""
    boxes = [(lo.copy(), hi.copy(), [])]
    for a in axes:
        nxt = []
        for blo, bhi, bits in boxes:
            mid = 0.5 * (blo[a] + bhi[a])
            l_hi = bhi.copy(); l_hi[a] = mid
            h_lo = blo.copy(); h_lo[a] = mid
            nxt.append((blo, l_hi, bits + [(a, mid, True)]))
            nxt.append((h_lo, bhi, bits + [(a, mid, False)]))
        boxes = nxt
    return boxes


def build_tree(X, Y=None, nu0: int = 50, mode: str = "binary", max_shrinks: int = 200) -> OTree:
    """Adaptive midpoint-bisection tree (smash/cluster.py:263-353).

    Same rules as the reference: leaf iff max(#row, #col) <= nu0; a split
    that leaves only one occupied cell shrinks the node box to that cell and
    retries (axis advances in binary mode); nodes are emitted in postorder
    and leaves append their points, in original index order, to the perms.
    """
    if mode == "2^d":
        mode = "2d"
    if mode not in ("binary", "2d"):
        raise ValueError("mode must be 'binary' or '2d'")
    if nu0 < 1:
        raise ValueError("nu0 must be positive")
    X = np.atleast_2d(np.asarray(X, dtype=np.float64))
    Y = X if Y is None else np.atleast_2d(np.asarray(Y, dtype=np.float64))
    if X.shape[0] == 0:
        raise ValueError("row point set is empty")
    if X.shape[1] != Y.shape[1]:
        raise ValueError("row/column point dimensions differ")
    d = X.shape[1]
    both = np.vstack([X, Y])
    root_lo, root_hi = both.min(axis=0), both.max(axis=0)

    level, parent, children, los, his = [], [], [], [], []
    rs, re, cs, ce = [], [], [], []
    prow, pcol = [], []

    def new_node(lev, lo, hi, kids, r0, r1, c0, c1):
        idx = len(level)
        level.append(lev); parent.append(-1); children.append(tuple(kids))
        los.append(lo.copy()); his.append(hi.copy())
        rs.append(r0); re.append(r1); cs.append(c0); ce.append(c1)
        for k in kids:
            parent[k] = idx
        return idx

    def grow(lev, lo, hi, xs, ys, axis):
        if max(xs.size, ys.size) <= nu0:
            r0, c0 = len(prow), len(pcol)
            prow.extend(xs.tolist()); pcol.extend(ys.tolist())
            return new_node(lev, lo, hi, (), r0, len(prow), c0, len(pcol))
        for _ in range(max_shrinks):
            axes = [axis] if mode == "binary" else list(range(d))
            nxt_axis = (axis + 1) % d if mode == "binary" else axis
            occupied = []
            for blo, bhi, bits in _cells(lo, hi, axes):
                mx = np.ones(xs.size, bool)
                my = np.ones(ys.size, bool)
                for a, mid, low in bits:
                    mx &= (X[xs, a] <= mid) == low
                    my &= (Y[ys, a] <= mid) == low
                if mx.any() or my.any():
                    occupied.append((blo, bhi, xs[mx], ys[my]))
            if len(occupied) >= 2:
                kids = [grow(lev + 1, blo, bhi, sx, sy, nxt_axis)
                        for blo, bhi, sx, sy in occupied]
                return new_node(lev, lo, hi, kids, rs[kids[0]], re[kids[-1]],
                                cs[kids[0]], ce[kids[-1]])
            lo, hi = occupied[0][0], occupied[0][1]
            axis = nxt_axis
        raise RuntimeError("box subdivision failed to separate points")

    grow(1, root_lo, root_hi, np.arange(X.shape[0]), np.arange(Y.shape[0]), 0)
    prow = np.asarray(prow, dtype=np.int64)
    pcol = np.asarray(pcol, dtype=np.int64)
    return OTree(mode=mode, nu0=nu0, dim=d, level=np.asarray(level, np.int64),
                 parent=np.asarray(parent, np.int64), children=children,
                 lo=np.asarray(los), hi=np.asarray(his),
                 row_start=np.asarray(rs, np.int64), row_stop=np.asarray(re, np.int64),
                 col_start=np.asarray(cs, np.int64), col_stop=np.asarray(ce, np.int64),
                 perm_row=prow, perm_col=pcol, points_row=X[prow], points_col=Y[pcol])


# ---------------------------------------------------------------------------
# block partitions  (smash/cluster.py:374-447)
# ---------------------------------------------------------------------------


def leaf_sets(tree: OTree, tau: float, structure: str = "h2"):
    """(L, Lm) as int64 (n, 2) arrays, each sorted lexicographically.

    h2: the reference's dual recursion from (root, root) (cluster.py:428-446),
    evaluated breadth-first -- the resulting sets are identical.
    hss: sibling pairs + leaf diagonal (cluster.py:415-424)."""
    if structure == "hss":
        L, Lm = [], []
        for i, kids in enumerate(tree.children):
            if kids:
                if len(kids) != 2:
                    raise ValueError("hss structure needs a binary tree")
                L += [(kids[0], kids[1]), (kids[1], kids[0])]
            else:
                Lm.append((i, i))
        return _sorted_pairs(L), _sorted_pairs(Lm)
    if structure != "h2":
        raise ValueError("structure must be 'hss' or 'h2'")
    L, Lm = [], []
    front = np.array([[tree.root, tree.root]], dtype=np.int64)
    leaf = np.array([not k for k in tree.children])
    while front.size:
        I, J = front[:, 0], front[:, 1]
        sep = separated(tree.lo[I], tree.hi[I], tree.lo[J], tree.hi[J], tau)
        L.append(front[sep])
        rest = front[~sep]
        nxt = []
        for i, j in rest:
            li, lj = leaf[i], leaf[j]
            if li and lj:
                Lm.append(np.array([[i, j]]))
            elif li:
                nxt += [(i, c) for c in tree.children[j]]
            elif lj:
                nxt += [(c, j) for c in tree.children[i]]
            else:
                nxt += [(a, b) for a in tree.children[i] for b in tree.children[j]]
        front = np.array(nxt, dtype=np.int64).reshape(-1, 2)
    cat = lambda xs: np.concatenate(xs) if xs else np.zeros((0, 2), np.int64)
    return _sorted_pairs(cat(L)), _sorted_pairs(cat(Lm))


def _sorted_pairs(P):
    P = np.asarray(P, dtype=np.int64).reshape(-1, 2)
    if P.shape[0] == 0:
        return P
    return P[np.lexsort((P[:, 1], P[:, 0]))]


def nearfield_sets(tree: OTree, tau: float) -> list:
    """N_i for every node (smash/cluster.py:374-399): top-down over a stable
    sort by level; candidates are the siblings (child order) then, per member
    k of the parent's set, k itself if a leaf else k's children; keep the
    ones not well separated from i."""
    if tau in tree._near:
        return tree._near[tau]
    n = tree.n_nodes
    near = [None] * n
    near[tree.root] = []
    for j in sorted(range(n), key=lambda k: tree.level[k]):
        if j == tree.root:
            continue
        p = tree.parent[j]
        cand = [c for c in tree.children[p] if c != j]
        for k in near[p]:
            cand += [k] if not tree.children[k] else list(tree.children[k])
        if cand:
            c = np.asarray(cand)
            ok = ~separated(np.repeat(tree.lo[j:j + 1], c.size, 0), np.repeat(tree.hi[j:j + 1], c.size, 0),
                            tree.lo[c], tree.hi[c], tau)
            near[j] = [int(x) for x in c[ok]]
        else:
            near[j] = []
    tree._near[tau] = near
    return near


# ---------------------------------------------------------------------------
# interpolation basis  (smash/lowrank.py:103-144)
# ---------------------------------------------------------------------------


def cheb_nodes(a: float, b: float, m: int) -> np.ndarray:
    """0.5(a+b) + 0.5(b-a) cos((2k+1) pi / 2m), lowrank.py:103-105."""
    k = np.arange(m)
    return 0.5 * (a + b) + 0.5 * (b - a) * np.cos((2 * k + 1) * np.pi / (2 * m))


def lagrange_cols(x: np.ndarray, nodes: np.ndarray) -> np.ndarray:
    """Barycentric cardinal functions at x (lowrank.py:108-120); rows where
    x hits a node exactly are one-hot."""
    m = nodes.size
    k = np.arange(m)
    w = (-1.0) ** k * np.sin((2 * k + 1) * np.pi / (2 * m))
    diff = x[:, None] - nodes[None, :]
    with np.errstate(divide="ignore", invalid="ignore"):
        t = w[None, :] / diff
        out = t / t.sum(axis=1)[:, None]
    hit = diff == 0
    rows = hit.any(axis=1)
    if rows.any():
        out[rows] = hit[rows].astype(np.float64)
    return out


def tensor_order(m: int, d: int, r: int):
    """Tensor index tuples sorted by (total degree, i, j[, k]), first r.
    d = 2 follows lowrank.py:143; d = 3 is this project's documented
    extension (the reference raises for d = 3)."""
    if d == 1:
        return [(i,) for i in range(r)]
    if d == 2:
        return [t[1:] for t in sorted((i + j, i, j) for i in range(m) for j in range(m))[:r]]
    return [t[1:] for t in sorted((i + j + k, i, j, k) for i in range(m)
                                  for j in range(m) for k in range(m))[:r]]


def grid_m(r: int, d: int) -> int:
    """Nodes per axis: r (1-D), ceil(sqrt(r)) (2-D, lowrank.py:140), the
    smallest m with m^3 >= r (3-D extension)."""
    if d == 1:
        return r
    if d == 2:
        return math.ceil(math.sqrt(r))
    m = 1
    while m ** 3 < r:
        m += 1
    return m


def interp_basis(lo, hi, pts: np.ndarray, r: int) -> np.ndarray:
    """Lagrange basis at Chebyshev nodes of the box (lowrank.py:123-144)."""
    pts = np.atleast_2d(np.asarray(pts, dtype=np.float64))
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    scale = max(np.max(hi - lo), 1.0)
    for a, b in zip(lo, hi):
        if not b - a > 1e-14 * scale:
            raise ValueError("degenerate box dimension; interpolation nodes would coincide")
    d = lo.size
    if d > 3:
        raise ValueError("interpolation basis supports d <= 3")
    m = grid_m(r, d)
    Ls = [lagrange_cols(pts[:, a], cheb_nodes(lo[a], hi[a], m)) for a in range(d)]
    if d == 1:
        return Ls[0]
    cols = []
    for idx in tensor_order(m, d, r):
        c = Ls[0][:, idx[0]] * Ls[1][:, idx[1]]
        if d == 3:
            c = c * Ls[2][:, idx[2]]
        cols.append(c)
    return np.column_stack(cols) if cols else np.zeros((pts.shape[0], 0))


def pad_box(lo, hi, pad):
    """Widen box dimensions thinner than pad by pad/2 each side (hss.py:39-45)."""
    lo = np.array(lo, dtype=np.float64)
    hi = np.array(hi, dtype=np.float64)
    thin = hi - lo < pad
    lo[thin] -= pad / 2
    hi[thin] += pad / 2
    return lo, hi


# ---------------------------------------------------------------------------
# strong RRQR and interpolative compression  (smash/lowrank.py:163-255)
# ---------------------------------------------------------------------------


def _rank_of(rdiag, kmax, rtol):
    """Count of |R_ii| > rtol |R_00|, capped (lowrank.py:163-167)."""
    if rdiag.size == 0 or rdiag[0] == 0:
        return 0
    return int(min(kmax, np.count_nonzero(np.abs(rdiag) > rtol * abs(rdiag[0]))))


@dataclass
class SrrqrOut:
    perm: np.ndarray
    R: np.ndarray
    rank: int
    swaps: int


def srrqr(M: np.ndarray, s: float = 2.0, rtol: float = 1e-14, max_swaps: int = 200) -> SrrqrOut:
    """LAPACK dgeqp3 + numerical rank + bounded-entry swap loop with
    unpivoted refactorisation (lowrank.py:170-203)."""
    M = np.asarray(M, dtype=np.float64)
    m, n = M.shape
    if min(m, n) == 0:
        return SrrqrOut(np.arange(n), np.zeros((0, n)), 0, 0)
    R, piv = sla.qr(M, mode="r", pivoting=True)
    R = R[:min(m, n)]
    k = _rank_of(np.diag(R), min(m, n), rtol)
    swaps = 0
    while 0 < k < n:
        W = sla.solve_triangular(R[:k, :k], R[:k, k:], lower=False)
        a = np.abs(W)
        if a.max() <= s:
            break
        if swaps >= max_swaps:
            raise RuntimeError("srrqr swap loop exceeded %d iterations" % max_swaps)
        i, j = divmod(int(np.argmax(a)), W.shape[1])
        piv = piv.copy()
        piv[i], piv[k + j] = piv[k + j], piv[i]
        R = sla.qr(M[:, piv], mode="r")[0][:min(m, n)]
        swaps += 1
    return SrrqrOut(np.asarray(piv, np.int64), R, k, swaps)


@dataclass
class Factor:
    """Interpolative row factor X = P [I; G] (lowrank.py:206-229)."""
    nrows: int
    perm: np.ndarray
    G: np.ndarray
    skel: np.ndarray
    skel_local: np.ndarray
    swaps: int = 0

    @property
    def rank(self):
        return int(self.skel.size)

    def expand(self):
        X = np.zeros((self.nrows, self.rank))
        X[self.perm[:self.rank]] = np.eye(self.rank)
        if self.rank < self.nrows:
            X[self.perm[self.rank:]] = self.G
        return X


def compr(C: np.ndarray, ibar: np.ndarray, s: float = 2.0, rtol: float = 1e-14) -> Factor:
    """Row ID of C labelled by ibar: srrqr(C^T), G = (R11^-1 R12)^T
    (lowrank.py:232-255)."""
    C = np.asarray(C, dtype=np.float64)
    ibar = np.asarray(ibar, dtype=np.int64)
    if C.shape[0] != ibar.size:
        raise ValueError("row labels do not match C")
    res = srrqr(C.T, s=s, rtol=rtol)
    k = res.rank
    if k:
        G = sla.solve_triangular(res.R[:k, :k], res.R[:k, k:], lower=False).T
    else:
        G = np.zeros((C.shape[0], 0))
    return Factor(C.shape[0], res.perm, np.ascontiguousarray(G), ibar[res.perm[:k]],
                  res.perm[:k].copy(), res.swaps)


def truncated_svd(M: np.ndarray, eps: float) -> np.ndarray:
    """Left singular vectors with sigma >= eps * sigma_1 (lowrank.py:265-276)."""
    M = np.asarray(M)
    if min(M.shape) == 0:
        return np.zeros((M.shape[0], 0))
    U, sig, _ = sla.svd(M, full_matrices=False)
    keep = 0 if sig[0] == 0 else int(np.count_nonzero(sig >= eps * sig[0]))
    return U[:, :keep]


# ---------------------------------------------------------------------------
# kernels  (smash/kernel.py:278-310 for cauchy; the others are the BASELINE
# extension of SURVEY.md 8(c))
# ---------------------------------------------------------------------------

KERNELS = ("log", "inv_r", "exp", "cauchy")


def kernel_block(kind: str, Xc: np.ndarray, Yc: np.ndarray, dx: float = None) -> np.ndarray:
    """Dense K(Xc[a], Yc[b]).

    log:    0.5*log(r^2), r^2 = sum dx_k^2; diagonal (r == 0) -> dx (default 0)
    inv_r:  1/sqrt(r^2); diagonal -> dx (default 0)
    exp:    exp(-sqrt(r^2)); natural diagonal 1
    cauchy: 1/(x - y) for 1-D points (kernel.py:286-298); coincident -> dx
    """
    Xc = np.atleast_2d(Xc)
    Yc = np.atleast_2d(Yc)
    if kind == "cauchy":
        if Xc.shape[1] != 1:
            raise ValueError("real cauchy kernel needs 1-D points")
        diff = Xc[:, 0][:, None] - Yc[:, 0][None, :]
        hit = diff == 0
        with np.errstate(divide="ignore", invalid="ignore"):
            K = 1.0 / diff
        if hit.any():
            if dx is None:
                raise ValueError("coincident points need a diagonal value d_x")
            K[hit] = dx
        return K
    r2 = np.zeros((Xc.shape[0], Yc.shape[0]))
    for a in range(Xc.shape[1]):
        t = Xc[:, a][:, None] - Yc[:, a][None, :]
        r2 = r2 + t * t
    hit = r2 == 0
    with np.errstate(divide="ignore", invalid="ignore"):
        if kind == "log":
            K = 0.5 * np.log(r2)
        elif kind == "inv_r":
            K = 1.0 / np.sqrt(r2)
        elif kind == "exp":
            return np.exp(-np.sqrt(r2))
        else:
            raise ValueError("unknown kernel %r" % kind)
    if hit.any():
        K[hit] = 0.0 if dx is None else dx
    return K


# ---------------------------------------------------------------------------
# builders  (smash/h2.py:25-54, smash/hss.py:219-303)
# ---------------------------------------------------------------------------


@dataclass
class OMatrix:
    kind: str
    tree: OTree
    kernel: str
    dx: float
    r: int
    tau: float
    s: float
    rtol: float
    eps_svd: float
    pairs_L: np.ndarray
    pairs_Lm: np.ndarray
    rowfac: dict
    colfac: dict
    skel_row: dict
    skel_col: dict


def _ibar(tree, i, skels, side):
    """Leaf: own tree-order range; else concatenated child skeletons (hss.py:241-244)."""
    if tree.is_leaf(i):
        a, b = (tree.row_start[i], tree.row_stop[i]) if side == "row" else (tree.col_start[i], tree.col_stop[i])
        return np.arange(a, b, dtype=np.int64)
    parts = [skels[c] for c in tree.children[i]]
    return np.concatenate(parts) if parts else np.zeros(0, np.int64)


def _pad(tree):
    """pad = max(1e-9 * diam, 1e-300), diam = 2 * root radius (hss.py:221-222)."""
    diam = 2 * box_radius(tree.lo[tree.root], tree.hi[tree.root])[0]
    return max(1e-9 * diam, 1e-300)


def _basis(tree, i, ibar, side, r, pad):
    pts = tree.points_row if side == "row" else tree.points_col
    lo, hi = pad_box(tree.lo[i], tree.hi[i], pad)
    return interp_basis(lo, hi, pts[ibar], r)


def build_h2(tree: OTree, kernel: str, r: int, tau: float, s: float = 2.0, rtol: float = 1e-14,
             dx: float = None, symmetric: bool = None) -> OMatrix:
    """Level loop L..2, row then column compr per node (h2.py:44-53).
    With symmetric=True (X is Y) the column factors alias the row factors;
    SURVEY.md 7 (probe p12) shows they are bitwise identical."""
    if tree.mode != "2d" and tree.dim != 1:
        raise ValueError("H2 construction expects a 2^d-mode tree")
    L, Lm = leaf_sets(tree, tau, "h2")
    M = OMatrix("h2", tree, kernel, dx, r, tau, s, rtol, 0.0, L, Lm, {}, {}, {}, {})
    if symmetric is None:
        symmetric = tree.points_row is tree.points_col or (
            tree.points_row.shape == tree.points_col.shape and np.array_equal(tree.perm_row, tree.perm_col)
            and np.array_equal(tree.points_row, tree.points_col))
    pad = _pad(tree)
    for lev in range(tree.n_levels, 1, -1):
        for i in tree.level_nodes(lev):
            ib = _ibar(tree, i, M.skel_row, "row")
            f = compr(_basis(tree, i, ib, "row", r, pad), ib, s=s, rtol=rtol)
            M.rowfac[i], M.skel_row[i] = f, f.skel
            if symmetric:
                M.colfac[i], M.skel_col[i] = f, f.skel
            else:
                ib = _ibar(tree, i, M.skel_col, "col")
                f = compr(_basis(tree, i, ib, "col", r, pad), ib, s=s, rtol=rtol)
                M.colfac[i], M.skel_col[i] = f, f.skel
    return M


def build_hss(tree: OTree, kernel: str, r: int, tau: float, eps_svd: float, s: float = 2.0,
              rtol: float = 1e-14, dx: float = None) -> OMatrix:
    """HSS: farfield basis + truncated SVD of the nearfield block row,
    compressed together (hss.py:274-299)."""
    for kids in tree.children:
        if kids and len(kids) != 2:
            raise ValueError("HSS construction needs a binary tree")
    L, Lm = leaf_sets(tree, tau, "hss")
    M = OMatrix("hss", tree, kernel, dx, r, tau, s, rtol, eps_svd, L, Lm, {}, {}, {}, {})
    pad = _pad(tree)
    near = nearfield_sets(tree, tau)
    Xr, Xc = tree.points_row, tree.points_col
    for lev in range(tree.n_levels, 1, -1):
        for i in tree.level_nodes(lev):
            ib_r = _ibar(tree, i, M.skel_row, "row")
            ib_c = _ibar(tree, i, M.skel_col, "col")
            cand = [_basis(tree, i, ib_r, "row", r, pad)]
            cols = [c for c in (_ibar(tree, j, M.skel_col, "col") for j in near[i]) if c.size]
            if cols and ib_r.size:
                A = kernel_block(kernel, Xr[ib_r], Xc[np.concatenate(cols)], dx)
                cand.append(truncated_svd(A, eps_svd))
            f = compr(np.hstack(cand), ib_r, s=s, rtol=rtol)
            M.rowfac[i], M.skel_row[i] = f, f.skel
            cand = [_basis(tree, i, ib_c, "col", r, pad)]
            rows = [c for c in (_ibar(tree, j, M.skel_row, "row") for j in near[i]) if c.size]
            if rows and ib_c.size:
                A = kernel_block(kernel, Xr[np.concatenate(rows)], Xc[ib_c], dx)
                cand.append(truncated_svd(A.T, eps_svd))
            f = compr(np.hstack(cand), ib_c, s=s, rtol=rtol)
            M.colfac[i], M.skel_col[i] = f, f.skel
    return M


# ---------------------------------------------------------------------------
# matvec  (smash/apply.py:26-80)
# ---------------------------------------------------------------------------


def matvec(M: OMatrix, q: np.ndarray, cache: dict = None) -> np.ndarray:
    """Upward sweep, skeleton couplings, downward sweep, dense nearfield
    (apply.py:34-80).  Blocks are evaluated on the fly, or kept in ``cache``
    across calls like the reference's use_cache=True (hss.py:138-162)."""
    def block(key, fn):
        if cache is None:
            return fn()
        b = cache.get(key)
        if b is None:
            b = cache[key] = fn()
        return b
    tr = M.tree
    q = np.asarray(q, dtype=np.float64)
    single = q.ndim == 1
    Q = q[:, None] if single else q
    if Q.shape[0] != tr.perm_col.size:
        raise ValueError("vector length %d does not match matrix (%d)" % (Q.shape[0], tr.perm_col.size))
    qt = Q[tr.perm_col]
    nr = Q.shape[1]
    Xr, Xc = tr.points_row, tr.points_col
    qhat = {}
    for lev in range(tr.n_levels, 1, -1):
        for i in tr.level_nodes(lev):
            if tr.is_leaf(i):
                v = qt[tr.col_start[i]:tr.col_stop[i]]
            else:
                v = np.concatenate([qhat[c] for c in tr.children[i]], axis=0)
            qhat[i] = M.colfac[i].expand().T @ v
    zhat = {}
    for i, j in M.pairs_L:
        blk = block(("B", i, j), lambda: kernel_block(M.kernel, Xr[M.skel_row[i]], Xc[M.skel_col[j]], M.dx))
        e = blk @ qhat[j]
        zhat[i] = zhat[i] + e if i in zhat else e
    zt = np.zeros((tr.perm_row.size, nr))
    for lev in range(2, tr.n_levels + 1):
        for i in tr.level_nodes(lev):
            zi = zhat.get(i)
            if zi is None:
                zi = np.zeros((M.rowfac[i].rank, nr))
            y = M.rowfac[i].expand() @ zi
            if tr.is_leaf(i):
                zt[tr.row_start[i]:tr.row_stop[i]] += y
            else:
                off = 0
                for c in tr.children[i]:
                    k = M.rowfac[c].rank
                    zhat[c] = zhat[c] + y[off:off + k] if c in zhat else y[off:off + k]
                    off += k
    for i, j in M.pairs_Lm:
        blk = block(("NF", i, j), lambda: kernel_block(
            M.kernel, Xr[tr.row_start[i]:tr.row_stop[i]], Xc[tr.col_start[j]:tr.col_stop[j]], M.dx))
        zt[tr.row_start[i]:tr.row_stop[i]] += blk @ qt[tr.col_start[j]:tr.col_stop[j]]
    z = np.empty_like(zt)
    z[tr.perm_row] = zt
    return z[:, 0] if single else z


def _check_perfect(tr):
    """All leaves on the deepest level and one child count (apply.py:83-95)."""
    width = None
    for i in range(tr.n_nodes):
        if tr.is_leaf(i):
            if tr.level[i] != tr.n_levels:
                raise ValueError("level-synchronous matvec needs all leaves at the deepest level")
        else:
            if width is None:
                width = len(tr.children[i])
            elif len(tr.children[i]) != width:
                raise ValueError("level-synchronous matvec needs a perfect tree")


def matvec_levelwise(M: OMatrix, q: np.ndarray) -> np.ndarray:
    """Level-synchronous matvec on perfect trees (apply.py:98-165): per-level
    coefficient blocks; a parent's coefficients are the sum over its children of
    W(c)^T qbuf[c] (one product per child); couplings, then the downward sweep
    zbuf[c] += R(c) zbuf[p] and the leaf far field, then the nearfield."""
    tr = M.tree
    _check_perfect(tr)
    q = np.asarray(q, dtype=np.float64)
    single = q.ndim == 1
    Q = q[:, None] if single else q
    if Q.shape[0] != tr.perm_col.size:
        raise ValueError("vector length %d does not match matrix (%d)" % (Q.shape[0], tr.perm_col.size))
    qt = Q[tr.perm_col]
    nr = Q.shape[1]
    Xr, Xc = tr.points_row, tr.points_col
    qbuf = {}
    for lev in range(tr.n_levels, 1, -1):
        for i in tr.level_nodes(lev):
            if tr.is_leaf(i):
                qbuf[i] = M.colfac[i].expand().T @ qt[tr.col_start[i]:tr.col_stop[i]]
            else:
                e = None
                for c in tr.children[i]:
                    term = _child_rows(M, M.colfac, c).T @ qbuf[c]
                    e = term if e is None else e + term
                qbuf[i] = e
    zbuf = {i: np.zeros((M.rowfac[i].rank, nr)) for lev in range(2, tr.n_levels + 1)
            for i in tr.level_nodes(lev)}
    for i, j in M.pairs_L:
        zbuf[i] += kernel_block(M.kernel, Xr[M.skel_row[i]], Xc[M.skel_col[j]], M.dx) @ qbuf[j]
    zt = np.zeros((tr.perm_row.size, nr))
    for lev in range(2, tr.n_levels + 1):
        for i in tr.level_nodes(lev):
            if tr.is_leaf(i):
                zt[tr.row_start[i]:tr.row_stop[i]] += M.rowfac[i].expand() @ zbuf[i]
            else:
                for c in tr.children[i]:
                    zbuf[c] += _child_rows(M, M.rowfac, c) @ zbuf[i]
    for i, j in M.pairs_Lm:
        zt[tr.row_start[i]:tr.row_stop[i]] += kernel_block(
            M.kernel, Xr[tr.row_start[i]:tr.row_stop[i]], Xc[tr.col_start[j]:tr.col_stop[j]], M.dx) \
            @ qt[tr.col_start[j]:tr.col_stop[j]]
    z = np.empty_like(zt)
    z[tr.perm_row] = zt
    return z[:, 0] if single else z


def dense_matvec(kind: str, X, Y, q, dx=None, rows=None, chunk: int = 256):
    """Exact A @ q (optionally only the given rows), streamed in row chunks
    (the pattern of smash/bench.py:284-296)."""
    X = np.atleast_2d(X)
    Y = np.atleast_2d(Y)
    rows = np.arange(X.shape[0]) if rows is None else np.asarray(rows)
    out = []
    for a in range(0, rows.size, chunk):
        out.append(kernel_block(kind, X[rows[a:a + chunk]], Y, dx) @ q)
    return np.concatenate(out, axis=0)


# ---------------------------------------------------------------------------
# BASELINE configurations and their seeded inputs
# ---------------------------------------------------------------------------

CONFIGS = {
    1: dict(name="hss_log_1d", structure="hss", kernel="log", dim=1, mode="binary", nu0=64, r=10,
            tau=0.6, rtol=1e-8, eps_svd=1e-9, nrhs=(1,), N=4096),
    2: dict(name="h2_invr_2d", structure="h2", kernel="inv_r", dim=2, mode="2d", nu0=64, r=36,
            tau=0.7, rtol=1e-8, eps_svd=0.0, nrhs=(1, 16), N=2 ** 17),
    3: dict(name="h2_exp_3d", structure="h2", kernel="exp", dim=3, mode="2d", nu0=128, r=125,
            tau=0.7, rtol=1e-6, eps_svd=0.0, nrhs=(1,), N=2 ** 20),
    4: dict(name="hss_cauchy_1d", structure="hss", kernel="cauchy", dim=1, mode="binary", nu0=128,
            r=16, tau=0.6, rtol=1e-10, eps_svd=1e-11, nrhs=(8,), N=2 ** 20),
    5: dict(name="h2_log_2d_nonuniform", structure="h2", kernel="log", dim=2, mode="2d", nu0=64,
            r=64, tau=0.7, rtol=1e-8, eps_svd=0.0, nrhs=(16,), N=2 ** 21),
}


def make_config_points(cfg: int, N: int = None, seed: int = None):
    """Seeded synthetic inputs of SURVEY.md 8(d) (seed = config id).

    Returns (X, Y, rng) where Y is X for the symmetric configs; the rng is
    positioned after the point draws so right-hand sides follow them."""
    c = CONFIGS[cfg]
    N = c["N"] if N is None else N
    rng = np.random.default_rng(cfg if seed is None else seed)
    if cfg == 1:
        X = rng.random((N, 1))
        return X, X, rng
    if cfg == 2:
        X = rng.random((N, 2))
        return X, X, rng
    if cfg == 3:
        X = rng.random((N, 3))
        return X, X, rng
    if cfg == 4:
        X = (np.arange(N, dtype=np.float64) / N).reshape(-1, 1)
        Y = ((np.arange(N, dtype=np.float64) + 0.5) / N).reshape(-1, 1)
        return X, Y, rng
    if cfg == 5:
        h = N // 2
        ang = rng.random(h) * 2 * np.pi
        rad = 1 + rng.normal(0, 1e-3, h)
        circle = np.column_stack([rad * np.cos(ang), rad * np.sin(ang)])
        centres = rng.random((4, 2))
        lab = rng.integers(0, 4, N - h)
        off = rng.normal(0, 0.02, (N - h, 2))
        X = np.vstack([circle, centres[lab] + off])
        return X, X, rng
    raise ValueError("unknown config %r" % cfg)


# ---------------------------------------------------------------------------
# ULV factorisation / solve (smash/apply.py:168-354) -- checker for the GPU ULV
# ---------------------------------------------------------------------------

ULV_PIVOT_RTOL = 1e-13  # apply.py:18


def _child_rows(M: OMatrix, fac: dict, c: int) -> np.ndarray:
    """R(c) / W(c): rows of the parent's expand() for child c's slice (hss.py:116-136)."""
    tr = M.tree
    p = tr.parent[c]
    off = 0
    for ch in tr.children[p]:
        k = fac[ch].rank
        if ch == c:
            return fac[p].expand()[off:off + k]
        off += k
    raise KeyError(c)


def _ulv_reduce(D, U, V):
    """_reduce_node (apply.py:196-234): returns (record, D_red, U_red, V_red)."""
    import scipy.linalg as sla
    m_r, k_r = U.shape
    m_c = D.shape[1]
    e = m_r - k_r
    t = min(e, m_c) if e > 0 else 0
    rec = {"t": t, "mc_red": m_c}
    if t == 0:
        return rec, D, U, V
    Q, _ = sla.qr(U, mode="full")
    Dp = Q.T @ D
    Bbot = Dp[m_r - t:]
    Qz, Rt = sla.qr(Bbot.T, mode="full")
    Ltri = Rt[:t].T
    dmin = np.min(np.abs(np.diag(Ltri)))
    if dmin <= ULV_PIVOT_RTOL * max(np.linalg.norm(Bbot, np.inf), 1e-300):
        raise np.linalg.LinAlgError("singular local block")
    Dtrans = Dp[:m_r - t] @ Qz
    Mfull = V.T @ Qz
    rec.update(Q=Q, Qz=Qz, Ltri=Ltri, Dcorr=Dtrans[:, :t], Mcorr=Mfull[:, :t], mc_red=m_c - t)
    return rec, Dtrans[:, t:], (Q.T @ U)[:m_r - t], Mfull[:, t:].T


def ulv_factor(M: OMatrix) -> dict:
    """ulv_factor (apply.py:237-288), postorder over the HSS tree."""
    import scipy.linalg as sla
    if M.kind != "hss":
        raise ValueError("ULV factorization expects an HSS matrix")
    tr = M.tree
    Xr, Xc = tr.points_row, tr.points_col
    blk = lambda rows, cols: kernel_block(M.kernel, Xr[rows], Xc[cols], M.dx)  # noqa: E731
    F = {"nodes": {}, "M": M}
    red = {}
    for i in range(tr.n_nodes):
        if tr.is_leaf(i):
            D = blk(np.arange(tr.row_start[i], tr.row_stop[i]), np.arange(tr.col_start[i], tr.col_stop[i]))
            U = M.rowfac[i].expand() if i != tr.root else None
            V = M.colfac[i].expand() if i != tr.root else None
        else:
            c1, c2 = tr.children[i]
            r1, r2 = red.pop(c1), red.pop(c2)
            CP1 = r1["U"] @ blk(M.skel_row[c1], M.skel_col[c2])
            CP2 = r2["U"] @ blk(M.skel_row[c2], M.skel_col[c1])
            F["nodes"][c1]["CP"], F["nodes"][c2]["CP"] = CP1, CP2
            D = np.block([[r1["D"], CP1 @ r2["V"].T], [CP2 @ r1["V"].T, r2["D"]]])
            if i != tr.root:
                U = np.vstack([r1["U"] @ _child_rows(M, M.rowfac, c1), r2["U"] @ _child_rows(M, M.rowfac, c2)])
                V = np.vstack([r1["V"] @ _child_rows(M, M.colfac, c1), r2["V"] @ _child_rows(M, M.colfac, c2)])
                F["nodes"][c1]["W"] = _child_rows(M, M.colfac, c1)
                F["nodes"][c2]["W"] = _child_rows(M, M.colfac, c2)
        if i == tr.root:
            F["root"] = sla.lu_factor(D) if D.shape[0] else None
            F["root_n"] = D.shape[0]
        else:
            rec, Dr, Ur, Vr = _ulv_reduce(D, U, V)
            F["nodes"][i] = rec
            red[i] = {"D": Dr, "U": Ur, "V": Vr}
    return F


def ulv_solve(F: dict, b: np.ndarray) -> np.ndarray:
    """ulv_solve (apply.py:291-348)."""
    import scipy.linalg as sla
    M = F["M"]
    tr = M.tree
    b = np.asarray(b, dtype=np.float64)
    single = b.ndim == 1
    B = b[:, None] if single else b
    bt = B[tr.perm_row]
    nc = bt.shape[1]
    z1s, gs, bred, xroot = {}, {}, {}, None
    for i in range(tr.n_nodes):
        if tr.is_leaf(i):
            bcur, gpre = bt[tr.row_start[i]:tr.row_stop[i]], None
        else:
            c1, c2 = tr.children[i]
            n1, n2 = F["nodes"][c1], F["nodes"][c2]
            b1, b2, g1, g2 = bred.pop(c1), bred.pop(c2), gs.pop(c1), gs.pop(c2)
            bcur = np.vstack([b1 - n1["CP"] @ g2, b2 - n2["CP"] @ g1])
            gpre = None if i == tr.root else n1["W"].T @ g1 + n2["W"].T @ g2
        if i == tr.root:
            xroot = sla.lu_solve(F["root"], bcur) if F["root_n"] else np.zeros((0, nc))
            break
        rec = F["nodes"][i]
        if rec["t"] > 0:
            bp = rec["Q"].T @ bcur
            z1 = sla.solve_triangular(rec["Ltri"], bp[-rec["t"]:], lower=True)
            z1s[i] = z1
            bred[i] = bp[:-rec["t"]] - rec["Dcorr"] @ z1
            gown = rec["Mcorr"] @ z1
        else:
            bred[i] = bcur
            gown = np.zeros((M.colfac[i].rank, nc))
        gs[i] = gown if gpre is None else gpre + gown
    xt = np.zeros((tr.perm_col.size, nc))

    def descend(i, xv):
        rec = F["nodes"].get(i)
        if rec is not None and rec["t"] > 0:
            xv = rec["Qz"] @ np.vstack([z1s[i], xv])
        if tr.is_leaf(i):
            xt[tr.col_start[i]:tr.col_stop[i]] = xv
            return
        pos = 0
        for c in tr.children[i]:
            w = F["nodes"][c]["mc_red"]
            descend(c, xv[pos:pos + w])
            pos += w

    descend(tr.root, xroot)
    x = np.empty_like(xt)
    x[tr.perm_col] = xt
    return x[:, 0] if single else x
