"""Pins of the CPU oracle against what the paper and the mathematics fix.

None of these compare the oracle with itself: each checks a closed form, a
brute-force dense computation, a paper-printed value, or an invariant stated
by the paper (citations per test).  Marked `not gpu` (no marker): they run on
the CPU box in the driver's `-m "not gpu"` pass.
"""
import math
import os

import numpy as np
import pytest
import scipy.linalg as sla

from conftest import ring_problem
from oracle import lorasp_oracle as O
from synth import csr_to_dense, make_problem

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _dense(p):
    return csr_to_dense(p.n, p.row_ptr, p.col_idx, p.values)


# ---------------------------------------------------------------------------
# eps = 0 is exact: the solve equals a brute-force dense LU solve (BASELINE
# north_star; "equivalent ... up to the accuracy of Eq. lra")
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,dims,kind,depth,order", [
    ("p2d", (16, 16), "poisson", 4, "coloured"),
    ("p2d_nat", (16, 16), "poisson", 4, "natural"),
    ("p3d", (8, 8, 8), "poisson", 5, "coloured"),
    ("vc3d", (8, 8, 8), "varcoef", 5, "coloured"),
    ("upw2d", (16, 16), "upwind", 4, "coloured"),
    ("p2d_rect", (24, 16), "poisson", 4, "coloured"),
])
def test_eps0_matches_dense_lu(name, dims, kind, depth, order):
    p = make_problem("cfg1", dims=dims, kind=kind, depth=depth)
    A = _dense(p)
    f = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, depth, 0.0, order=order)
    x = O.solve(f, p.b)
    lu = sla.lu_factor(A)
    xd = sla.lu_solve(lu, p.b)
    assert np.linalg.norm(x - xd) / np.linalg.norm(xd) <= 1e-10
    # compression really happened (so exactness is not vacuous)
    assert sum(f.rank.values()) > 0


def test_eps0_ring_exact():
    rp, ci, va, xy = ring_problem(64)
    A = csr_to_dense(64, rp, ci, va)
    b = np.sin(np.arange(64.0))
    f = O.factorize(64, rp, ci, va, xy, 3, 0.0, order="natural")
    x = O.solve(f, b)
    assert np.linalg.norm(x - np.linalg.solve(A, b)) <= 1e-12 * np.linalg.norm(x)


# ---------------------------------------------------------------------------
# Appendix A golden trace
# ---------------------------------------------------------------------------
def _load_trace():
    steps = []
    with open(os.path.join(GOLDEN, "appendix_a_trace.txt")) as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                steps.append(line)
    return steps


def _fmt(step):
    if step[0] == "merge":
        return f"merge {step[1]}"
    if step[0] == "eliminate":
        k, i, c = step[1]
        return f"eliminate {k} {i} {c}"
    k, i, c = step[1]
    parts = " ".join(f"{a} {b_} {d}" for (a, b_, d) in step[2])
    return f"compress {k} {i} {c} : {parts}"


def test_appendix_a_trace():
    rp, ci, va, xy = ring_problem(64)
    f = O.factorize(64, rp, ci, va, xy, 3, 1e-8, order="natural", trace=True)
    assert [_fmt(s) for s in f.trace] == _load_trace()
    # P(b_1), P(b_3) have size 0: never partners; level-1 super-node has size 0
    assert f.size[("r", 2, 0)] == 0 and f.size[("r", 2, 2)] == 0
    assert f.size[("s", 1, 0)] == 0


# ---------------------------------------------------------------------------
# Section 2.3 key idea: the full-rank extended system of
# Eq. (extend), eliminated "starting from the right", gives back Eq. (example1).
# Pins the sign conventions the oracle's edge rules use (-I, V, V^T).
# ---------------------------------------------------------------------------
def test_extended_sparsification_identity():
    rng = np.random.default_rng(3)
    m, k = 6, 5
    X = rng.standard_normal((m, m)); S = X @ X.T + m * np.eye(m)
    B = rng.standard_normal((m, k)); C = rng.standard_normal((m, k))
    Y = rng.standard_normal((k, k)); P = Y @ Y.T + 5 * np.eye(k)
    Z = rng.standard_normal((k, k)); Q = Z @ Z.T + 5 * np.eye(k)
    Si = np.linalg.inv(S)
    D = -B.T @ Si @ C
    Pp, Qp = P - B.T @ Si @ B, Q - C.T @ Si @ C
    U, K, Vt = np.linalg.svd(D)
    V = Vt.T
    K = np.diag(K)
    Zr = np.zeros((k, k)); I = np.eye(k)
    # rows/cols: x2, x3, z2, z3, y2, y3   (Eq. extend, l.171-197)
    E = np.block([
        [Pp, Zr, U, Zr, Zr, Zr],
        [Zr, Qp, Zr, V, Zr, Zr],
        [U.T, Zr, Zr, Zr, -I, Zr],
        [Zr, V.T, Zr, Zr, Zr, -I],
        [Zr, Zr, -I, Zr, Zr, K],
        [Zr, Zr, Zr, -I, K.T, Zr],
    ])
    keep = slice(0, 2 * k)
    aux = slice(2 * k, 6 * k)
    schur = E[keep, keep] - E[keep, aux] @ np.linalg.solve(E[aux, aux], E[aux, keep])
    target = np.block([[Pp, D], [D.T, Qp]])
    assert np.linalg.norm(schur - target) <= 1e-12 * np.linalg.norm(target)


# ---------------------------------------------------------------------------
# Elimination: scalar 2-node case 2 - 1*(1/2)*1 = 1.5
# and a 3-node random block graph vs dense Gaussian elimination.
# ---------------------------------------------------------------------------
def _bare_factorizer():
    rp, ci, va, xy = ring_problem(8)
    fz = O._Factorizer(8, rp, ci, va, xy, 1, 0.0)
    fz.M.clear(); fz.out.clear(); fz.inn.clear(); fz.size.clear()
    # hand-built graphs below are not tied to the ring's cluster tree
    fz._check_distance = lambda u, v: None
    return fz


def test_eliminate_scalar_two_node():
    fz = _bare_factorizer()
    u, v = ("s", 1, 0), ("s", 1, 1)
    fz.size.update({u: 1, v: 1})
    fz._set(u, u, np.array([[2.0]])); fz._set(u, v, np.array([[1.0]]))
    fz._set(v, u, np.array([[1.0]])); fz._set(v, v, np.array([[2.0]]))
    fz.eliminate(u)
    assert fz.M[(v, v)][0, 0] == pytest.approx(1.5, abs=1e-15)


def test_eliminate_matches_dense_schur():
    rng = np.random.default_rng(7)
    fz = _bare_factorizer()
    nodes = [("s", 1, 0), ("s", 1, 1), ("r", 0, 0)]
    sz = [3, 2, 4]
    for nd, s in zip(nodes, sz):
        fz.size[nd] = s
    n = sum(sz)
    A = rng.standard_normal((n, n)) + n * np.eye(n)
    off = np.cumsum([0] + sz)
    for a, u in enumerate(nodes):
        for b_, v in enumerate(nodes):
            # Mat(u -> v) = A_{v,u}
            fz._set(u, v, A[off[b_]:off[b_ + 1], off[a]:off[a + 1]].copy())
    fz.eliminate(nodes[0])
    S = A[3:, 3:] - A[3:, :3] @ np.linalg.solve(A[:3, :3], A[:3, 3:])
    got = np.block([[fz.M[(nodes[1], nodes[1])], fz.M[(nodes[2], nodes[1])]],
                    [fz.M[(nodes[1], nodes[2])], fz.M[(nodes[2], nodes[2])]]])
    assert np.linalg.norm(got - S) <= 1e-12 * np.linalg.norm(S)


# ---------------------------------------------------------------------------
# Compress: reconstruction error = dropped energy, the
# constructed-spectrum rank, and the edge rules.
# ---------------------------------------------------------------------------
def _compress_case(eps, spectrum=None, seed=11):
    rng = np.random.default_rng(seed)
    fz = _bare_factorizer()
    fz.eps = eps
    m = 8
    s = ("s", 1, 0)
    p1, p2 = ("s", 1, 1), ("r", 0, 1)
    # fake a level-0 cluster graph where s (cluster 0 of P_0...) is at distance 2
    fz.distance = lambda u, v: 2
    fz.size.update({s: m, p1: 5, p2: 6})
    decay = np.diag(0.4 ** np.arange(m))          # graded columns -> decaying sigma
    if spectrum is None:
        A1 = rng.standard_normal((5, m)) @ decay; A2 = rng.standard_normal((6, m)) @ decay
    else:
        Q1, _ = np.linalg.qr(rng.standard_normal((11, 11)))
        Q2, _ = np.linalg.qr(rng.standard_normal((m, m)))
        Mfull = Q1[:, :m] @ np.diag(spectrum) @ Q2.T
        A1, A2 = Mfull[:5], Mfull[5:]
    B1 = rng.standard_normal((5, m)) @ decay if spectrum is None else A1.copy()
    B2 = rng.standard_normal((6, m)) @ decay if spectrum is None else A2.copy()
    fz._set(s, s, np.eye(m) * 10)
    fz._set(s, p1, A1.copy()); fz._set(p1, s, B1.T.copy())
    fz._set(s, p2, A2.copy()); fz._set(p2, s, B2.T.copy())
    fz.compress(1, 0)
    return fz, (A1, A2, B1, B2)


def test_compress_reconstruction_equals_dropped_energy():
    fz, (A1, A2, B1, B2) = _compress_case(0.3)
    r = fz.rank[(1, 0)]
    sig = fz.sigma[(1, 0)]
    assert 0 < r < 8
    s, b, P = ("s", 1, 0), ("b", 1, 0), ("r", 0, 0)
    p1, p2 = ("s", 1, 1), ("r", 0, 1)
    V = fz.M[(b, s)]                                  # rule 4: b -> s with V
    assert np.allclose(fz.M[(s, b)], V.T)
    assert np.allclose(V.T @ V, np.eye(r), atol=1e-12)
    R1, R2 = fz.M[(P, p1)], fz.M[(P, p2)]              # rule 2: P(b) -> p_k with R_k
    Q1, Q2 = fz.M[(p1, P)].T, fz.M[(p2, P)].T          # rule 3: p_k -> P(b) with Q_k^T
    stack = np.vstack([A1, A2, B1, B2])
    approx = np.vstack([R1, R2, Q1, Q2]) @ V.T
    err = np.linalg.norm(stack - approx)
    assert err == pytest.approx(math.sqrt(float(np.sum(sig[r:] ** 2))), rel=1e-10)
    # rule 1: s <-> p_k removed; rule 5: -I between b and P(b)
    assert (s, p1) not in fz.M and (p2, s) not in fz.M
    assert np.array_equal(fz.M[(b, P)], -np.eye(r)) and np.array_equal(fz.M[(P, b)], -np.eye(r))
    assert fz.size[b] == fz.size[P] == r


def test_compress_constructed_spectrum_rank():
    # [A; A] stack of Q1 diag(1, 1e-1, ..., 1e-7) Q2^T; sigma_k/sigma_0 >= 1e-3 -> r = 4
    spec = 10.0 ** -np.arange(8.0)
    fz, _ = _compress_case(1e-3, spectrum=spec)
    assert fz.rank[(1, 0)] == 4
    sig = fz.sigma[(1, 0)]
    assert np.allclose(sig[:8] / sig[0], spec, rtol=1e-8, atol=1e-15)


def test_compress_zero_stack_rank_zero():
    fz = _bare_factorizer()
    fz.distance = lambda u, v: 2
    s, p1 = ("s", 1, 0), ("s", 1, 1)
    fz.size.update({s: 4, p1: 3})
    fz._set(s, s, np.eye(4)); fz._set(s, p1, np.zeros((3, 4))); fz._set(p1, s, np.zeros((4, 3)))
    fz.compress(1, 0)
    assert fz.rank[(1, 0)] == 0 and fz.size[("r", 0, 0)] == 0
    assert (s, p1) not in fz.M


def test_symmetric_stack_shortcut_same_ranks():
    # for symmetric A, A_k = B_k and only the A's need stacking
    p = make_problem("cfg1", dims=(32, 32), depth=6)
    f1 = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 6, 1e-2)
    f2 = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 6, 1e-2, symmetric_stack=True)
    assert f1.rank == f2.rank
    x1, x2 = O.solve(f1, p.b), O.solve(f2, p.b)
    assert np.linalg.norm(x1 - x2) <= 1e-9 * np.linalg.norm(x1)


# ---------------------------------------------------------------------------
# Theorem (preservation of sparsity): never an edge at
# distance > 2.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dims,kind,depth,eps", [
    ((32, 32), "poisson", 6, 1e-2), ((16, 16, 8), "poisson", 7, 1e-2),
    ((32, 32), "upwind", 6, 1e-3), ((8, 8, 8), "varcoef", 5, 1e-2)])
def test_sparsity_theorem(dims, kind, depth, eps):
    import scipy.sparse as sp
    from scipy.sparse.csgraph import shortest_path
    p = make_problem("cfg1", dims=dims, kind=kind, depth=depth)
    f = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, depth, eps)
    assert f.max_edge_distance <= 2
    # independent check of every surviving block with scipy's BFS on the
    # quotient graph of A at the shallower level (Def. distance l.506-508)
    rows = np.repeat(np.arange(p.n), np.diff(p.row_ptr))
    dist = {}
    for k in range(depth + 1):
        cl = f.tree.leaf_of >> (depth - k)
        G = sp.coo_matrix((np.ones(rows.size), (cl[rows], cl[p.col_idx])), shape=(2 ** k, 2 ** k))
        dist[k] = shortest_path(G.tocsr(), unweighted=True, directed=False)

    def where(u):
        kind_, lev, c = u
        return (lev, c) if kind_ == "r" else (lev - 1, c)

    for (u, v) in f.M:
        (ku, cu), (kv, cv) = where(u), where(v)
        k = min(ku, kv)
        assert dist[k][cu >> (ku - k), cv >> (kv - k)] <= 2, (u, v)


# ---------------------------------------------------------------------------
# epsilon behaviour (BASELINE north_star): the stand-alone
# residual falls as eps shrinks; per-level retained ranks do not grow with eps.
# ---------------------------------------------------------------------------
def test_residual_falls_with_eps():
    p = make_problem("cfg1", dims=(32, 32), depth=6)
    A = _dense(p)
    res = []
    ranks = []
    for eps in [1e-1, 1e-2, 1e-3, 1e-4]:
        f = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 6, eps)
        x = O.solve(f, p.b)
        res.append(np.linalg.norm(A @ x - p.b) / np.linalg.norm(p.b))
        ranks.append({i: sum(v) for i, v in O.ranks_by_level(f).items()})
    assert all(res[k + 1] < res[k] for k in range(3)), res
    for k in range(3):       # smaller eps -> per-level total rank not smaller
        for i in ranks[k]:
            assert ranks[k + 1][i] >= ranks[k][i], (k, i, ranks)


def test_first_compressing_wave_ranks_monotone_per_node():
    # leaf wave 1 stacks hold only exact fill from wave 0 (r = 0 there), so the
    # stack is eps-independent and each node's rank is monotone in eps exactly.
    p = make_problem("cfg1", dims=(32, 32), depth=6)
    fs = [O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 6, e) for e in (1e-1, 1e-2, 1e-3)]
    l = 6
    seq = fs[0].level_order[l]
    first = [c for c in seq if fs[0].partners[(l, c)]][0]
    # every node before it had r = 0, so its stack is exact fill (eps-independent)
    r = [f.rank[(l, first)] for f in fs]
    assert 0 < r[0] <= r[1] <= r[2], r


# ---------------------------------------------------------------------------
# Paper-printed accuracy: 2D Poisson, eps = 1e-4, average
# leaf super-node 64 -> "relative error ~1e-4".  The caption's "residual less
# than 1e-6" (and l.603 "residual smaller than the error") depend on the
# paper's unstated right-hand side and partitioner and are not reproduced with
# the seeded uniform[-1,1] RHS (reading R3): parity unpinned there.
# ---------------------------------------------------------------------------
def test_paper_2d_eps1e4_accuracy():
    p = make_problem("cfg1", dims=(64, 64), depth=7)         # 32-dof reds -> 64-dof supers
    A = _dense(p)
    f = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 7, 1e-4)
    x = O.solve(f, p.b)
    xd = np.linalg.solve(A, p.b)
    err = np.linalg.norm(x - xd) / np.linalg.norm(xd)
    res = np.linalg.norm(A @ x - p.b) / np.linalg.norm(p.b)
    assert 1e-5 < err < 5e-4
    assert res < 1e-3


# ---------------------------------------------------------------------------
# Solve: linearity, identity matrix, and T-materialise: the solve
# equals the x-part of A_e^{-1} [b; 0] for the block LU of the extended system
# assembled from the frozen blocks (brute force, tiny case).
# ---------------------------------------------------------------------------
def test_solve_linearity_and_identity():
    p = make_problem("cfg1", dims=(16, 16), depth=4)
    f = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 4, 1e-2)
    rng = np.random.default_rng(0)
    b1, b2 = rng.standard_normal(p.n), rng.standard_normal(p.n)
    lhs = O.solve(f, 2.0 * b1 - 3.0 * b2)
    rhs = 2.0 * O.solve(f, b1) - 3.0 * O.solve(f, b2)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)
    n = 64
    rp = np.arange(n + 1, dtype=np.int64); ci = np.arange(n, dtype=np.int64)
    fI = O.factorize(n, rp, ci, np.ones(n), np.arange(n, dtype=float).reshape(-1, 1), 3, 0.5)
    assert np.array_equal(O.solve(fI, np.arange(n, dtype=float)), np.arange(n, dtype=float))


def test_materialised_extended_lu():
    p = make_problem("cfg1", dims=(16, 16), depth=4)
    A = _dense(p)
    for eps in (0.0, 1e-2):
        f = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 4, eps)
        L, U, offs, nodes = O.extended_dense(f)
        Ae = L @ U
        N = Ae.shape[0]
        # original dofs live in the leaf supers: position of dof q
        pos = np.full(p.n, -1)
        l = f.depth
        for c, mem in enumerate(f.tree.clusters[l]):
            sup = ("s", l, c // 2)
            o = 0 if c % 2 == 0 else f.size[("r", l, c - 1)]
            pos[mem] = offs[sup] + o + np.arange(mem.size)
        be = np.zeros(N); be[pos] = p.b
        xe = np.linalg.solve(Ae, be)
        assert np.linalg.norm(xe[pos] - O.solve(f, p.b)) <= 1e-10 * np.linalg.norm(xe[pos])
        # Schur complement of A_e onto the original dofs
        aux = np.setdiff1d(np.arange(N), pos)
        Sx = Ae[np.ix_(pos, pos)] - Ae[np.ix_(pos, aux)] @ np.linalg.solve(Ae[np.ix_(aux, aux)], Ae[np.ix_(aux, pos)])
        rel = np.linalg.norm(Sx - A) / np.linalg.norm(A)
        if eps == 0.0:
            assert rel <= 1e-12
        else:
            assert 0 < rel < 1e-1


# ---------------------------------------------------------------------------
# Krylov: exact preconditioner -> 1 CG
# iteration / <= 2 GMRES iterations; GMRES residual history monotone.
# ---------------------------------------------------------------------------
def test_krylov_exact_preconditioner():
    p = make_problem("cfg1", dims=(16, 16), depth=4)
    f = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 4, 0.0)
    mv = lambda v: O.spmv(p.row_ptr, p.col_idx, p.values, v)
    pc = lambda v: O.solve(f, v)
    r1 = O.pcg(mv, pc, p.b, tol=1e-10)
    assert r1.converged and r1.iters == 1 and r1.relres <= 1e-10
    r2 = O.gmres(mv, pc, p.b, tol=1e-10)
    assert r2.converged and r2.iters <= 2 and r2.relres <= 1e-10


def test_krylov_identity_and_monotone():
    n = 50
    I = lambda v: v.copy()
    b = np.linspace(-1, 1, n)
    assert O.pcg(I, I, b).iters == 1
    assert O.gmres(I, I, b).iters == 1
    p = make_problem("cfg1", dims=(24, 24), kind="upwind", depth=5)
    f = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 5, 1e-1)
    mv = lambda v: O.spmv(p.row_ptr, p.col_idx, p.values, v)
    res = O.gmres(mv, lambda v: O.solve(f, v), p.b, tol=1e-10)
    assert res.converged and res.relres <= 1e-9
    h = res.history
    assert all(h[k + 1] <= h[k] * (1 + 1e-12) for k in range(len(h) - 1))


def test_pcg_preconditioned_converges_cfg1():
    p = make_problem("cfg1")
    f = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, p.depth, 1e-2)
    mv = lambda v: O.spmv(p.row_ptr, p.col_idx, p.values, v)
    r = O.pcg(mv, lambda v: O.solve(f, v), p.b, tol=1e-10)
    assert r.converged and r.relres <= 1e-10 and r.iters < 20
