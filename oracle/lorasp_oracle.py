"""ORACLE for the LoRaSp level sweep (arxiv 1510.07363) — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` leg may import this module.  The product path (the C-ABI
library `liblorasp` and its Python binding) never calls it; there is no CPU
fallback anywhere.  This file shares no code with the CUDA path: it imports
only numpy/scipy and the seeded input generators in `synth/`.

It is a plain, slow, step-by-step transcription of the paper, in float64:

  * Def. nested partitionings by recursive coordinate
    bisection (reading Z17);
  * Def. adjacency graph (l.73-76) / adjacent clusters (l.247-249) as
    symmetrised quotient graphs; Def. distance (l.506-508);
  * Alg. 1 (l.265-289): MergeRedNodes (l.295-313), Compress (l.319-394:
    Eq. lra, Eqs. anterpol/interpol, the five edge rules l.383-389,
    Eq. rhszero), Eliminate (l.101-106, l.396-399);
  * truncation sigma_k / sigma_0 >= eps (Eq. cutOff1, l.580-584);
  * Alg. 2-4 (l.407-500): SetRHS, SolveL, SolveU, SplitVar;
  * Krylov consumers (l.651-669): PCG for SPD inputs and right-preconditioned
    GMRES(restart); the paper's preconditioned residual (Eq. GMRES_residual)
    is reported alongside.

Order within a level (the paper leaves it generic, l.281 / l.843): reading
Z1/Z2 — colour-major order of a validated distance-2 lattice colouring,
ascending cluster index within a colour, greedy distance-2 fallback.  The
paper's literal ascending order ("natural") is kept for the Appendix-A trace.

Pinned by tests/test_oracle_*.py.  Every
function below cites the passage it follows.
"""
from __future__ import annotations

import dataclasses
import math
from collections import defaultdict
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import scipy.linalg as sla
from threadpoolctl import threadpool_limits

# The oracle is sequential, like the paper's implementation (P:l.794): BLAS runs
# on one thread (multi-threaded BLAS on these small blocks is ~20x slower).
ORACLE_THREADS = 1

# Node ids are tuples:  ('r', k, c)  red node of cluster c of P_k
#                       ('s', i, c)  super-node s_c^[i]  (cluster c of P_{i-1})
#                       ('b', i, c)  black node  b_c^[i]  (cluster c of P_{i-1})
# P(b_c^[i]) = ('r', i-1, c)                       (Def. hierarchical tree l.224-227)
Node = Tuple[str, int, int]

KIND_RANK = {"s": 0, "b": 1, "r": 2}


class SingularPivot(RuntimeError):
    pass


# ---------------------------------------------------------------------------
# Nested partitionings: recursive coordinate bisection       (P:l.214-216, Z17)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class Tree:
    depth: int
    clusters: List[List[np.ndarray]]     # clusters[k][c] = ascending member indices
    axis: List[np.ndarray]               # axis[k][c] = split axis of cluster c of P_k (k<depth)
    leaf_of: np.ndarray                  # leaf cluster id of each dof


def bisection_tree(coords: np.ndarray, depth: int) -> Tree:
    """P_0..P_l, n_{P_i} = 2^i; cluster c of P_k has children 2c, 2c+1 in P_{k+1}.

    Split rule (reading Z17): the axis of largest coordinate extent; ties
    (extents within a relative 1e-9 of the largest, so that rounding in the
    coordinates cannot break them) go to the lowest axis; members sorted by (coordinate, original index); the low half
    (first floor(|C|/2)) is child 2c.  Members are kept in ascending original
    index (reading Z16).
    """
    coords = np.asarray(coords, dtype=np.float64)
    n, dim = coords.shape
    clusters = [[np.arange(n, dtype=np.int64)]]
    axes = []
    for k in range(depth):
        nxt, ax = [], np.zeros(2 ** k, dtype=np.int64)
        for c, mem in enumerate(clusters[k]):
            if mem.size == 0:
                a = 0
                lo = hi = mem
            else:
                pts = coords[mem]
                ext = pts.max(axis=0) - pts.min(axis=0)
                a = int(np.nonzero(ext >= ext.max() * (1.0 - 1e-9))[0][0])
                srt = mem[np.lexsort((mem, pts[:, a]))]
                h = mem.size // 2
                lo, hi = np.sort(srt[:h]), np.sort(srt[h:])
            ax[c] = a
            nxt += [lo, hi]
        axes.append(ax)
        clusters.append(nxt)
    leaf_of = np.empty(n, dtype=np.int64)
    for c, mem in enumerate(clusters[depth]):
        leaf_of[mem] = c
    return Tree(depth=depth, clusters=clusters, axis=axes, leaf_of=leaf_of)


def bisection_tree_algebraic(row_ptr, col_idx, depth: int) -> Tree:
    """nested partitionings from the graph of A alone (no
    coordinates; the paper used SCOTCH, P:l.560, P:l.838).  Split rule (reading
    F4): breadth-first level structure of the cluster's induced subgraph from a
    pseudo-peripheral vertex — BFS from the smallest member, take the smallest
    vertex of the last level, BFS again — members ordered by (level, index),
    vertices unreachable from it last (by index); the first floor(|C|/2) form
    child 2c.  The split axis is recorded as 0 (the colouring's lattice rule then
    sees one axis and usually falls back to the greedy rule)."""
    row_ptr = np.asarray(row_ptr, np.int64)
    col_idx = np.asarray(col_idx, np.int64)
    n = row_ptr.size - 1
    INF = 1 << 60

    def levels_from(src, inset):
        lev = {src: 0}
        frontier = [src]
        while frontier:
            nxt = []
            for v in frontier:
                for j in col_idx[row_ptr[v]:row_ptr[v + 1]]:
                    j = int(j)
                    if j != v and j in inset and j not in lev:
                        lev[j] = lev[v] + 1
                        nxt.append(j)
            frontier = nxt
        return lev

    clusters = [[np.arange(n, dtype=np.int64)]]
    axes = []
    for k in range(depth):
        nxt = []
        for mem in clusters[k]:
            if mem.size == 0:
                nxt += [mem, mem]
                continue
            inset = set(int(v) for v in mem)
            l1 = levels_from(int(mem[0]), inset)
            far = max(l1.values())
            p = min(v for v, l in l1.items() if l == far)
            l2 = levels_from(p, inset)
            order = sorted((int(v) for v in mem), key=lambda v: (l2.get(v, INF), v))
            h = mem.size // 2
            nxt += [np.array(sorted(order[:h]), dtype=np.int64), np.array(sorted(order[h:]), dtype=np.int64)]
        axes.append(np.zeros(2 ** k, dtype=np.int64))
        clusters.append(nxt)
    leaf_of = np.empty(n, dtype=np.int64)
    for c, mem in enumerate(clusters[depth]):
        leaf_of[mem] = c
    return Tree(depth=depth, clusters=clusters, axis=axes, leaf_of=leaf_of)


# ---------------------------------------------------------------------------
# Quotient graphs and distances                    (P:l.73-76, l.247-249, l.506-512)
# ---------------------------------------------------------------------------
def quotient_graph(row_ptr, col_idx, cluster_of: np.ndarray, ncl: int) -> List[set]:
    """Adjacency graph of A under a partitioning, symmetrised (Def. adj. clusters)."""
    n = row_ptr.shape[0] - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(row_ptr))
    a = cluster_of[rows]
    b = cluster_of[col_idx]
    keep = a != b
    pairs = np.unique(np.stack([a[keep], b[keep]], axis=1), axis=0) if keep.any() else np.zeros((0, 2), np.int64)
    adj = [set() for _ in range(ncl)]
    for p, q in pairs:
        adj[int(p)].add(int(q))
        adj[int(q)].add(int(p))
    return adj


def distance_sets(adj: List[set]) -> Tuple[List[set], List[set]]:
    """N1[c] (distance exactly 1) and N2[c] (distance exactly 2), by BFS."""
    N1 = [set(s) for s in adj]
    N2 = []
    for c, s in enumerate(adj):
        two = set()
        for q in s:
            two |= adj[q]
        two -= s
        two.discard(c)
        N2.append(two)
    return N1, N2


# ---------------------------------------------------------------------------
# Order within a level (Z1, Z2): validated lattice colouring, greedy fallback
# ---------------------------------------------------------------------------
def lattice_index(tree: Tree, k: int, c: int, dim: int) -> List[int]:
    """g_a(c): cluster c's index along axis a, read off its bisection path."""
    g = [0] * dim
    for t in range(k):
        anc = c >> (k - t)
        bit = (c >> (k - 1 - t)) & 1
        a = int(tree.axis[t][anc])
        g[a] = 2 * g[a] + bit
    return g


def colour_level(tree: Tree, k: int, dim: int, N1: List[set], N2: List[set]) -> List[int]:
    """Distance-2 colouring of the clusters of P_k.

    Lattice rule (Z2): colour = (sum_a (a+1) g_a) mod (2 dim + 1); accepted only
    if no two clusters at distance 1 or 2 share a colour, else greedy: ascending
    index, smallest colour unused by lower-indexed clusters within distance 2.
    """
    ncl = 2 ** k
    col = []
    for c in range(ncl):
        g = lattice_index(tree, k, c, dim)
        col.append(sum((a + 1) * g[a] for a in range(dim)) % (2 * dim + 1))
    ok = all(col[c] != col[q] for c in range(ncl) for q in (N1[c] | N2[c]))
    if ok:
        return col
    col = [-1] * ncl
    for c in range(ncl):
        used = {col[q] for q in (N1[c] | N2[c]) if q < c}
        x = 0
        while x in used:
            x += 1
        col[c] = x
    return col


# ---------------------------------------------------------------------------
# The H-tree state and Alg. 1
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class Factorization:
    n: int
    depth: int
    eps: float
    tree: Tree
    size: Dict[Node, int]
    M: Dict[Tuple[Node, Node], np.ndarray]      # Mat(e_{u->v}) keyed (u, v), shape |v| x |u|
    out: Dict[Node, set]
    inn: Dict[Node, set]
    order: Dict[Node, int]                       # Order(p)  (P:l.500)
    level_order: Dict[int, List[int]]            # clusters of P_{i-1} in processing order
    pivots: Dict[Node, tuple]                    # frozen LU of Mat(p->p)
    rank: Dict[Tuple[int, int], int]             # (level i, cluster c) -> r of s_c^[i]
    sigma: Dict[Tuple[int, int], np.ndarray]     # singular values of each compressed stack
    partners: Dict[Tuple[int, int], List[Node]]
    n1: Dict[Tuple[int, int], List[Node]]        # uneliminated neighbours of s at elimination
    trace: List[tuple]
    max_edge_distance: int = 0
    singular_checks: int = 0


def _cluster_level(u: Node) -> Tuple[int, int]:
    """The (level of P, cluster) a node corresponds to (Def. hierarchical tree)."""
    kind, lev, c = u
    return (lev, c) if kind == "r" else (lev - 1, c)


class _Factorizer:
    def __init__(self, n, row_ptr, col_idx, values, coords, depth, eps,
                 order="coloured", symmetric_stack=False, trace=False, compressor="svd",
                 partition="coordinates"):
        self.n = n
        self.l = depth
        self.eps = float(eps)
        if compressor not in ("svd", "rrqr"):
            raise ValueError(compressor)
        self.compressor = compressor
        self.symmetric_stack = symmetric_stack
        self.want_trace = trace
        coords = np.asarray(coords, dtype=np.float64).reshape(n, -1)
        self.dim = coords.shape[1]
        if partition == "algebraic":
            self.dim = 1
            self.tree = bisection_tree_algebraic(row_ptr, col_idx, depth)
        else:
            self.tree = bisection_tree(coords, depth)
        self.N1, self.N2 = {}, {}
        for k in range(depth + 1):
            cl_of = self.tree.leaf_of >> (depth - k)
            adj = quotient_graph(row_ptr, col_idx, cl_of, 2 ** k)
            self.N1[k], self.N2[k] = distance_sets(adj)
        self.order_mode = order
        self.size: Dict[Node, int] = {}
        self.M: Dict[Tuple[Node, Node], np.ndarray] = {}
        self.out: Dict[Node, set] = defaultdict(set)
        self.inn: Dict[Node, set] = defaultdict(set)
        self.eliminated: set = set()
        self.order: Dict[Node, int] = {}
        self.counter = 0
        self.pivots = {}
        self.rank, self.sigma, self.partners, self.n1 = {}, {}, {}, {}
        self.level_order = {}
        self.trace: List[tuple] = []
        self.max_edge_distance = 0
        self._init_leaves(row_ptr, col_idx, values)

    # -- block store helpers -------------------------------------------------
    def _set(self, u: Node, v: Node, blk: np.ndarray):
        self.M[(u, v)] = blk
        self.out[u].add(v)
        self.inn[v].add(u)
        if u != v:
            self._check_distance(u, v)

    def _del(self, u: Node, v: Node):
        self.M.pop((u, v), None)
        self.out[u].discard(v)
        self.inn[v].discard(u)

    def _get_or_zero(self, u: Node, v: Node) -> np.ndarray:
        if (u, v) not in self.M:
            self._set(u, v, np.zeros((self.size[v], self.size[u])))
        return self.M[(u, v)]

    def distance(self, u: Node, v: Node) -> int:
        """Def. distance (l.506-508): lift the deeper cluster, BFS at the shallower level."""
        (ku, cu), (kv, cv) = _cluster_level(u), _cluster_level(v)
        k = min(ku, kv)
        cu >>= ku - k
        cv >>= kv - k
        if cu == cv:
            return 0
        if cv in self.N1[k][cu]:
            return 1
        if cv in self.N2[k][cu]:
            return 2
        return 3  # "greater than 2"

    def _check_distance(self, u, v):
        d = self.distance(u, v)
        if d > self.max_edge_distance:
            self.max_edge_distance = d

    # -- Initialize(l)  (P:l.291-293) ----------------------------------------
    def _init_leaves(self, row_ptr, col_idx, values):
        l = self.l
        leaf_of = self.tree.leaf_of
        for c, mem in enumerate(self.tree.clusters[l]):
            self.size[("r", l, c)] = int(mem.size)
        pos = np.empty(self.n, dtype=np.int64)
        for c, mem in enumerate(self.tree.clusters[l]):
            pos[mem] = np.arange(mem.size)
        n = self.n
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(row_ptr))
        for i, j, a in zip(rows, col_idx, values):
            # entry A[i, j]: row i in cluster v = leaf_of[i], column j in u = leaf_of[j]
            # -> Mat(e_{u->v}) = A_{v,u}   (Def. adjacency graph, l.75 / l.81)
            u = ("r", l, int(leaf_of[j]))
            v = ("r", l, int(leaf_of[i]))
            blk = self._get_or_zero(u, v)
            blk[pos[i], pos[j]] += a

    # -- MergeRedNodes  (P:l.295-313) ----------------------------------------
    def merge(self, i: int):
        nsup = 2 ** (i - 1)
        for c in range(nsup):
            s = ("s", i, c)
            self.size[s] = self.size.get(("r", i, 2 * c), 0) + self.size.get(("r", i, 2 * c + 1), 0)
        reds = [("r", i, c) for c in range(2 ** i)]
        red_set = set(reds)
        moved = [(u, v) for (u, v) in list(self.M.keys()) if u in red_set and v in red_set]
        for (u, v) in moved:
            blk = self.M[(u, v)]
            su, sv = ("s", i, u[2] // 2), ("s", i, v[2] // 2)
            # Eq. merge: Mat(s_j -> s_j') = [[r0->r0', r1->r0'], [r0->r1', r1->r1']]
            ro = 0 if v[2] % 2 == 0 else self.size.get(("r", i, v[2] - 1), 0)
            co = 0 if u[2] % 2 == 0 else self.size.get(("r", i, u[2] - 1), 0)
            tgt = self._get_or_zero(su, sv)
            tgt[ro:ro + blk.shape[0], co:co + blk.shape[1]] += blk
            self._del(u, v)
        if self.want_trace:
            self.trace.append(("merge", i))

    # -- Order within level i --------------------------------------------------
    def level_sequence(self, i: int) -> List[int]:
        k = i - 1
        ncl = 2 ** k
        if self.order_mode == "natural":
            return list(range(ncl))
        col = colour_level(self.tree, k, self.dim, self.N1[k], self.N2[k])
        return sorted(range(ncl), key=lambda c: (col[c], c))

    # -- Compress  (P:l.319-394) -----------------------------------------------
    def compress(self, i: int, c: int):
        s = ("s", i, c)
        b, P = ("b", i, c), ("r", i - 1, c)
        m = self.size[s]
        nb = (self.out[s] | self.inn[s]) - {s}
        partners = [u for u in nb if u not in self.eliminated and self.size.get(u, 0) > 0
                    and self.distance(s, u) >= 2]
        partners.sort(key=lambda u: (KIND_RANK[u[0]], u[1], u[2]))
        self.partners[(i, c)] = partners
        if m == 0 or not partners:
            self.size[b] = self.size[P] = 0
            self.rank[(i, c)] = 0
            self.sigma[(i, c)] = np.zeros(0)
            return
        # Eq. (lra): stack A_k = Mat(s->p_k) (m_k x m) and B_k with B_k^T = Mat(p_k->s)
        A = [self.M.get((s, p), np.zeros((self.size[p], m))) for p in partners]
        B = [self.M.get((p, s), np.zeros((m, self.size[p]))).T for p in partners]
        stack = np.vstack(A if self.symmetric_stack else A + B)
        if self.compressor == "rrqr":
            r, sig, V = self._rrqr(stack, m)
        else:
            # thin SVD when the stack has >= m rows (V is m x m either way)
            _, sig, Vt = np.linalg.svd(stack, full_matrices=stack.shape[0] < m)
            sig0 = float(sig[0]) if sig.size else 0.0
            if sig0 == 0.0:
                r = 0                                   # reading Z4
            elif self.eps == 0.0:
                r = m                                   # reading Z3: nothing is truncated
            else:
                r = int(np.count_nonzero(sig >= self.eps * sig0))   # Eq. cutOff1, ties kept (Z5)
            V = Vt[:r].T                                # m x r
        self.rank[(i, c)] = r
        self.sigma[(i, c)] = sig
        if self.want_trace:
            self.trace.append(("compress", s, tuple(partners)))
        # edge rule 1: remove edges s -> p_k and p_k -> s
        for p in partners:
            self._del(s, p)
            self._del(p, s)
        self.size[b] = self.size[P] = r
        if r == 0:
            return
        for p, Ak, Bk in zip(partners, A, B):
            Rk = Ak @ V                             # A_k ~= R_k V^T
            Qk = Bk @ V                             # B_k ~= Q_k V^T
            self._set(P, p, Rk)                     # rule 2: P(b) -> p_k with R_k
            self._set(p, P, Qk.T)                   # rule 3: p_k -> P(b) with Q_k^T
        self._set(s, b, V.T.copy())                 # rule 4: s -> b with V^T
        self._set(b, s, V.copy())                   #         b -> s with V
        I = np.eye(r)
        self._set(b, P, -I)                         # rule 5: b <-> P(b) with -I_r
        self._set(P, b, -I.copy())
        # RHS(b) = RHS(P(b)) = 0 (Eq. rhszero) -- applied in SetRHS

    def _rrqr(self, stack: np.ndarray, m: int):
        """SURVEY 8(f) f1, the paper's proposed cheaper compressor (P:l.616,
        P:l.840): column-pivoted (Businger-Golub) QR  stack P = Q R,  truncated
        at the first k with |R_kk| < eps |R_00| (reading F1: the
        rank-revealing analogue of Eq. cutOff1); the kept row space is that of
        R[:r, :] P^T, returned as an orthonormal basis V (m x r).  Any basis of
        that span gives the same preconditioner (the black-node coordinates
        only change by an r x r rotation)."""
        Rq, piv = sla.qr(stack, mode="r", pivoting=True)
        d = np.abs(np.diag(Rq))
        sig = np.zeros(m)
        sig[:d.size] = d
        if d.size == 0 or d[0] == 0.0:
            return 0, sig, np.zeros((m, 0))          # reading Z4
        if self.eps == 0.0:
            r = m                                    # reading Z3
        else:
            small = np.nonzero(d < self.eps * d[0])[0]
            r = int(small[0]) if small.size else d.size
        if r == 0:
            return 0, sig, np.zeros((m, 0))
        W = np.zeros((m, r))
        if r <= d.size:
            W[piv, :] = Rq[:r, :].T                  # rows of R P^T, transposed
        if r > d.size:                               # eps = 0 with fewer rows than columns
            W = np.eye(m)[:, :r]
        V, _ = np.linalg.qr(W)
        return r, sig, V

    # -- Eliminate  (P:l.101-106, l.396-399) ------------------------------------
    def eliminate(self, p: Node):
        if self.size.get(p, 0) == 0:
            self.eliminated.add(p)
            self.order[p] = self.counter
            self.counter += 1
            return
        if (p, p) not in self.M:
            raise SingularPivot(f"node {p} has no pivot block")
        piv = self.M[(p, p)]
        lu = sla.lu_factor(piv, check_finite=True)
        dU = np.abs(np.diag(lu[0]))
        if dU.min() < 1e-13 * max(np.abs(piv).max(), 1e-300):   # reading Z11
            raise SingularPivot(f"singular pivot at node {p}")
        self.pivots[p] = lu
        ins = [k for k in self.inn[p] if k != p and k not in self.eliminated]
        outs = [j for j in self.out[p] if j != p and j not in self.eliminated]
        ins.sort(key=lambda u: (KIND_RANK[u[0]], u[1], u[2]))
        outs.sort(key=lambda u: (KIND_RANK[u[0]], u[1], u[2]))
        for k in ins:
            Xk = sla.lu_solve(lu, self.M[(k, p)])          # Mat(p->p)^{-1} Mat(k->p)
            for j in outs:
                upd = self.M[(p, j)] @ Xk                  # Mat(p->j) Mat(p->p)^{-1} Mat(k->p)
                tgt = self._get_or_zero(k, j)
                tgt -= upd
        self.eliminated.add(p)
        self.order[p] = self.counter
        self.counter += 1
        if self.want_trace:
            self.trace.append(("eliminate", p))

    # -- Alg. 1  (P:l.265-289) -------------------------------------------------
    def run(self) -> Factorization:
        for i in range(self.l, 0, -1):
            self.merge(i)
            seq = self.level_sequence(i)
            self.level_order[i] = seq
            for c in seq:
                s = ("s", i, c)
                self.compress(i, c)
                nb = (self.out[s] | self.inn[s]) - {s}
                self.n1[(i, c)] = sorted((u for u in nb if u not in self.eliminated),
                                         key=lambda u: (KIND_RANK[u[0]], u[1], u[2]))
                self.eliminate(s)
                self.eliminate(("b", i, c))
        return Factorization(
            n=self.n, depth=self.l, eps=self.eps, tree=self.tree, size=self.size, M=self.M,
            out=self.out, inn=self.inn, order=self.order, level_order=self.level_order,
            pivots=self.pivots, rank=self.rank, sigma=self.sigma, partners=self.partners,
            n1=self.n1, trace=self.trace, max_edge_distance=self.max_edge_distance)


def factorize(n, row_ptr, col_idx, values, coords, depth, eps, order="coloured",
              symmetric_stack=False, trace=False, compressor="svd", partition="coordinates") -> Factorization:
    """Alg. 1 on the CSR matrix A (row_ptr, col_idx, values) with point coordinates.
    compressor: "svd" (Eq. lra + Eq. cutOff1) or "rrqr" (f1, column-pivoted QR)."""
    with threadpool_limits(ORACLE_THREADS):
        return _factorize(n, row_ptr, col_idx, values, coords, depth, eps, order, symmetric_stack, trace,
                          compressor, partition)


def _factorize(n, row_ptr, col_idx, values, coords, depth, eps, order, symmetric_stack, trace,
               compressor="svd", partition="coordinates"):
    return _Factorizer(n, np.asarray(row_ptr, np.int64), np.asarray(col_idx, np.int64),
                       np.asarray(values, np.float64), coords, depth, eps, order=order,
                       symmetric_stack=symmetric_stack, trace=trace, compressor=compressor,
                       partition=partition).run()


# ---------------------------------------------------------------------------
# Alg. 2-4: solve                                              (P:l.401-500)
# ---------------------------------------------------------------------------
def _ord(f: Factorization, q: Node) -> float:
    # reds are never eliminated as such: they are eliminated as part of the super-node
    # of the next level, i.e. after every node that can reach them through an edge.
    return f.order.get(q, math.inf) if q[0] != "r" else math.inf


def solve(f: Factorization, b: np.ndarray) -> np.ndarray:
    """x ~= A^{-1} b by Alg. 2 (forward SolveL / backward SolveU in Order)."""
    with threadpool_limits(ORACLE_THREADS):
        return _solve(f, b)


def _solve(f: Factorization, b: np.ndarray) -> np.ndarray:
    l = f.depth
    rhs: Dict[Node, np.ndarray] = {}
    var: Dict[Node, np.ndarray] = {}
    for c, mem in enumerate(f.tree.clusters[l]):            # SetRHS: leaves get b
        rhs[("r", l, c)] = np.array(b[mem], dtype=np.float64)

    def R(u):
        if u not in rhs:
            rhs[u] = np.zeros(f.size.get(u, 0))             # non-leaf RHS = 0 (Eq. rhszero)
        return rhs[u]

    def solve_l(p):                                          # Alg. 3
        if f.size.get(p, 0) == 0:
            return
        fv = sla.lu_solve(f.pivots[p], R(p))
        for q in f.out[p]:
            if q != p and _ord(f, q) > f.order[p]:
                R(q)[...] -= f.M[(p, q)] @ fv

    def solve_u(p):                                          # Alg. 4
        if f.size.get(p, 0) == 0:
            var[p] = np.zeros(0)
            return
        v = R(p).copy()
        for q in f.inn[p]:
            if q != p and _ord(f, q) > f.order[p]:
                v -= f.M[(q, p)] @ var[q]
        var[p] = sla.lu_solve(f.pivots[p], v)

    for i in range(l, 0, -1):                                # forward substitution
        for c in range(2 ** (i - 1)):                        # Eq. concatRHS
            rhs[("s", i, c)] = np.concatenate([R(("r", i, 2 * c)), R(("r", i, 2 * c + 1))])
        for c in f.level_order[i]:
            solve_l(("s", i, c))
            solve_l(("b", i, c))
    for i in range(1, l + 1):                                # backward substitution
        for c in reversed(f.level_order[i]):
            solve_u(("b", i, c))
            solve_u(("s", i, c))
            s = var[("s", i, c)]                             # SplitVar (Eq. concatX)
            n0 = f.size.get(("r", i, 2 * c), 0)
            var[("r", i, 2 * c)] = s[:n0]
            var[("r", i, 2 * c + 1)] = s[n0:]
    x = np.zeros(f.n)
    for c, mem in enumerate(f.tree.clusters[l]):
        x[mem] = var[("r", l, c)]
    return x


# ---------------------------------------------------------------------------
# Krylov consumers                                             (P:l.651-669)
# ---------------------------------------------------------------------------
def spmv(row_ptr, col_idx, values, x):
    n = row_ptr.shape[0] - 1
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    return np.bincount(rows, weights=values * x[col_idx], minlength=n)


@dataclasses.dataclass
class KrylovResult:
    x: np.ndarray
    iters: int
    relres: float             # ||b - A x|| / ||b||   (Eq. accres)
    converged: bool
    history: List[float]
    breakdown: bool = False


def pcg(matvec, precond, b, tol=1e-10, maxit=500) -> KrylovResult:
    """Preconditioned CG (P:l.652 remark; readings Z21/Z24/Z27): x0 = 0,
    stop when ||r_k||_2 / ||b||_2 <= tol; iters = number of A-products."""
    nb = float(np.linalg.norm(b))
    x = np.zeros_like(b)
    if nb == 0.0:
        return KrylovResult(x, 0, 0.0, True, [0.0])
    r = b.copy()
    z = precond(r)
    p = z.copy()
    rz = float(r @ z)
    hist = [1.0]
    for it in range(1, maxit + 1):
        q = matvec(p)
        pq = float(p @ q)
        if pq <= 0.0 or rz <= 0.0:
            return KrylovResult(x, it - 1, float(np.linalg.norm(b - matvec(x))) / nb, False, hist, True)
        alpha = rz / pq
        x += alpha * p
        r -= alpha * q
        rel = float(np.linalg.norm(r)) / nb
        hist.append(rel)
        if rel <= tol:
            return KrylovResult(x, it, float(np.linalg.norm(b - matvec(x))) / nb, True, hist)
        z = precond(r)
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return KrylovResult(x, maxit, float(np.linalg.norm(b - matvec(x))) / nb, False, hist)


def gmres(matvec, precond, b, tol=1e-10, restart=50, maxit=500) -> KrylovResult:
    """Right-preconditioned GMRES(restart), MGS Arnoldi + Givens (reading Z21):
    solves A M y = b, x = M y; stops when the recurrence residual estimate
    ||b - A x|| / ||b|| <= tol; iters = number of Arnoldi steps."""
    nb = float(np.linalg.norm(b))
    x = np.zeros_like(b)
    if nb == 0.0:
        return KrylovResult(x, 0, 0.0, True, [0.0])
    hist = [1.0]
    it = 0
    while it < maxit:
        r = b - matvec(x)
        beta = float(np.linalg.norm(r))
        if beta / nb <= tol:
            return KrylovResult(x, it, beta / nb, True, hist)
        Vb = [r / beta]
        Z = []
        H = np.zeros((restart + 1, restart))
        cs, sn = np.zeros(restart), np.zeros(restart)
        g = np.zeros(restart + 1); g[0] = beta
        k_used = 0
        done = False
        for k in range(restart):
            z = precond(Vb[k]); Z.append(z)
            w = matvec(z)
            for j in range(k + 1):                       # modified Gram-Schmidt
                H[j, k] = float(w @ Vb[j])
                w = w - H[j, k] * Vb[j]
            H[k + 1, k] = float(np.linalg.norm(w))
            for j in range(k):                           # apply previous Givens
                t = cs[j] * H[j, k] + sn[j] * H[j + 1, k]
                H[j + 1, k] = -sn[j] * H[j, k] + cs[j] * H[j + 1, k]
                H[j, k] = t
            den = math.hypot(H[k, k], H[k + 1, k])
            cs[k], sn[k] = (1.0, 0.0) if den == 0.0 else (H[k, k] / den, H[k + 1, k] / den)
            H[k, k] = cs[k] * H[k, k] + sn[k] * H[k + 1, k]
            H[k + 1, k] = 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            it += 1
            k_used = k + 1
            hist.append(abs(g[k + 1]) / nb)
            if abs(g[k + 1]) / nb <= tol or it >= maxit:
                done = True
                break
            if H[k + 1, k] == 0.0 and den == 0.0:
                done = True
                break
            Vb.append(w / (float(np.linalg.norm(w)) if np.linalg.norm(w) > 0 else 1.0))
        y = sla.solve_triangular(H[:k_used, :k_used], g[:k_used])
        for j in range(k_used):
            x = x + y[j] * Z[j]
        if done:
            rel = float(np.linalg.norm(b - matvec(x))) / nb
            return KrylovResult(x, it, rel, rel <= tol * 10 or abs(g[k_used]) / nb <= tol, hist)
    rel = float(np.linalg.norm(b - matvec(x))) / nb
    return KrylovResult(x, it, rel, rel <= tol, hist)


def paper_preconditioned_residual(matvec, precond, b, x) -> float:
    """Eq. GMRES_residual (l.665-669): ||Ã b - Ã A x|| / ||Ã b||."""
    ab = precond(b)
    return float(np.linalg.norm(ab - precond(matvec(x))) / np.linalg.norm(ab))


# ---------------------------------------------------------------------------
# Convenience: per-level rank summaries, dense materialisation for pins
# ---------------------------------------------------------------------------
def ranks_by_level(f: Factorization) -> Dict[int, List[int]]:
    out = {}
    for (i, c), r in f.rank.items():
        out.setdefault(i, [0] * (2 ** (i - 1)))[c] = r
    return out


def extended_dense(f: Factorization):
    """Dense matrix of the factored extended system in Order (tiny cases only):
    returns (L, U, index map) such that A_e = L U with L_qp = Mat(p->q) Piv_p^{-1},
    U_pq = Mat(q->p) for Order(q) > Order(p), U_pp = Piv_p (block LU of A_e).
    Used by T-materialise."""
    nodes = [p for p in sorted(f.order, key=lambda u: f.order[u]) if f.size.get(p, 0) > 0]
    offs, tot = {}, 0
    for p in nodes:
        offs[p] = tot
        tot += f.size[p]
    L = np.eye(tot)
    U = np.zeros((tot, tot))

    def rng(p):
        return slice(offs[p], offs[p] + f.size[p])

    def owner(q):
        # reds map into the super-node that later contains them
        if q[0] != "r":
            return q, 0
        kind, k, c = q
        if k == 0:
            return None, 0
        sup = ("s", k, c // 2)
        o = 0 if c % 2 == 0 else f.size.get(("r", k, c - 1), 0)
        return sup, o

    for p in nodes:
        piv = f.M[(p, p)]
        U[rng(p), rng(p)] = piv
        for q in f.out[p]:
            if q == p or _ord(f, q) <= f.order[p]:
                continue
            oq, o = owner(q)
            if oq is None or f.size.get(q, 0) == 0:
                continue
            rows = slice(offs[oq] + o, offs[oq] + o + f.size[q])
            L[rows, rng(p)] = f.M[(p, q)] @ np.linalg.inv(piv)
        for q in f.inn[p]:
            if q == p or _ord(f, q) <= f.order[p]:
                continue
            oq, o = owner(q)
            if oq is None or f.size.get(q, 0) == 0:
                continue
            cols = slice(offs[oq] + o, offs[oq] + o + f.size[q])
            U[rng(p), cols] = f.M[(q, p)]
    return L, U, offs, nodes
