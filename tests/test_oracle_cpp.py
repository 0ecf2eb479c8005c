"""Pins of the C++17 LAPACK-free oracle (oracle/cpp/lorasp_oracle.cpp) against
what the paper and the mathematics fix, plus the pins the numpy oracle lacked
(SpMV / GMRES on a NONSYMMETRIC matrix, the paper's preconditioned residual,
P:l.603 "residual smaller than the error").

None of these compares an oracle with itself: each test checks a closed form, a
brute-force dense computation (numpy / scipy library routines as the special
case the method reduces to), a paper-printed value or trace, or an invariant
the paper states.  The last group cross-checks the two independently pinned
oracles (C++ plain loops vs numpy/LAPACK) on ranks and x = Ã b.
"""
import math
import os

import numpy as np
import pytest
import scipy.linalg as sla

from conftest import ring_problem
from oracle import cpp_oracle as CO
from oracle import lorasp_oracle as O
from synth import csr_to_dense, make_problem

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _dense(p):
    return csr_to_dense(p.n, p.row_ptr, p.col_idx, p.values)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


# ---------------------------------------------------------------------------
# Dense kernels against their textbook definitions
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("R,m,k,graded", [(40, 16, 16, False), (200, 32, 7, False), (5, 12, 5, False),
                                          (64, 24, 24, True), (3, 3, 1, False), (90, 40, 40, True)])
def test_svd_kernel_singular_values(R, m, k, graded):
    """One-sided Jacobi (+ QR when R > m): sigma equals LAPACK's SVD (the
    mathematical singular values), M V has orthogonal columns of norms sigma,
    V is orthogonal (Eq. lra, P:l.333-355)."""
    rng = np.random.default_rng(R * 100 + m)
    if graded:
        U, _ = np.linalg.qr(rng.standard_normal((R, min(R, m))))
        W, _ = np.linalg.qr(rng.standard_normal((m, m)))
        s = 10.0 ** -np.linspace(0, 9, min(R, m))
        M = U @ np.diag(s) @ W[:, :min(R, m)].T
    else:
        M = rng.standard_normal((R, k)) @ rng.standard_normal((k, m))
    sig, V = CO.svd_right(M)
    ref = np.zeros(m)
    sv = np.linalg.svd(M, compute_uv=False)
    ref[:sv.size] = sv
    # backward-stable SVDs agree to O(m u sigma_0) absolutely (Weyl)
    assert np.allclose(sig, ref, rtol=1e-12, atol=1e-13 * ref[0])
    assert np.all(np.diff(sig) <= 0)
    assert np.allclose(V.T @ V, np.eye(m), atol=1e-13)
    MV = M @ V
    assert np.allclose(np.linalg.norm(MV, axis=0), sig, rtol=1e-10, atol=1e-12 * ref[0])


def test_lu_kernel_and_singular_detection():
    """Partial-pivot LU solves (Eq. elimination's Mat(p->p)^{-1}, reading Z11)."""
    rng = np.random.default_rng(1)
    A = rng.standard_normal((30, 30))
    A[0, 0] = 0.0                                   # needs pivoting
    b = rng.standard_normal((30, 3))
    x = CO.lu_solve_dense(A, b)
    assert _rel(x, np.linalg.solve(A, b)) <= 1e-12
    S = np.ones((4, 4))                             # rank 1: singular (Z11)
    with pytest.raises(CO.OracleError):
        CO.lu_solve_dense(S, np.ones(4))


def test_qrcp_kernel_matches_businger_golub():
    """Column-pivoted QR (f1, reading F1): |R_kk| and the pivot order equal
    LAPACK's dgeqp3 on a tie-free matrix; |R_kk| non-increasing."""
    rng = np.random.default_rng(2)
    M = rng.standard_normal((40, 12)) * (1.0 + np.arange(12))
    d, perm = CO.qr_colpiv(M)
    Rq, piv = sla.qr(M, mode="r", pivoting=True)
    assert np.array_equal(perm, piv)
    assert np.allclose(d, np.abs(np.diag(Rq)), rtol=1e-12)
    assert np.all(np.diff(d) <= 1e-12 * d[0])


# ---------------------------------------------------------------------------
# eps = 0 is exact (BASELINE north_star; P:l.404): x equals a dense LU solve
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dims,kind,depth,kw", [
    ((16, 16), "poisson", 4, {}),
    ((16, 16), "poisson", 4, {"order": "natural"}),
    ((8, 8, 8), "poisson", 5, {}),
    ((8, 8, 8), "varcoef", 5, {}),
    ((16, 16), "upwind", 4, {}),
    ((24, 16), "poisson", 4, {}),
    ((32, 32), "poisson", 6, {}),
    ((16, 16), "poisson", 4, {"partition": "algebraic"}),
    ((16, 16), "upwind", 4, {"compressor": "rrqr"}),
    ((16, 16), "poisson", 4, {"truncation": "frobenius"}),
])
def test_eps0_matches_dense_lu(dims, kind, depth, kw):
    p = make_problem("cfg1", dims=dims, kind=kind, depth=depth)
    f = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, depth, 0.0, **kw)
    x = CO.solve(f, p.b)
    xd = np.linalg.solve(_dense(p), p.b)
    assert _rel(x, xd) <= 1e-10
    assert sum(f.rank.values()) > 0          # compression happened (not vacuous)
    assert f.max_edge_distance <= 2          # Theorem, P:l.515-521


def test_eps0_ring_exact_and_appendix_a_trace():
    """Appendix A (P:l.846-912): the 8-leaf periodic ring in natural order gives
    exactly the captions' step sequence; eps = 0 solves exactly."""
    rp, ci, va, xy = ring_problem(64)
    f = CO.factorize(64, rp, ci, va, xy, 3, 1e-8, order="natural", trace=True)
    want = [t.strip() for t in open(os.path.join(GOLDEN, "appendix_a_trace.txt"))
            if t.strip() and not t.startswith("#")]
    assert f.trace == want
    assert f.size[("r", 2, 0)] == 0 and f.size[("r", 2, 2)] == 0 and f.size[("s", 1, 0)] == 0
    f0 = CO.factorize(64, rp, ci, va, xy, 3, 0.0, order="natural")
    b = np.sin(np.arange(64.0))
    A = csr_to_dense(64, rp, ci, va)
    assert _rel(CO.solve(f0, b), np.linalg.solve(A, b)) <= 1e-12


def test_identity_matrix_solve_is_identity():
    n = 64
    rp = np.arange(n + 1, dtype=np.int64)
    ci = np.arange(n, dtype=np.int64)
    f = CO.factorize(n, rp, ci, np.ones(n), np.arange(n, dtype=float).reshape(-1, 1), 3, 0.5)
    b = np.arange(n, dtype=float)
    assert np.array_equal(CO.solve(f, b), b)


def test_solve_linearity():
    p = make_problem("cfg1", dims=(16, 16), depth=4)
    f = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 4, 1e-2)
    rng = np.random.default_rng(0)
    b1, b2 = rng.standard_normal(p.n), rng.standard_normal(p.n)
    lhs = CO.solve(f, 2.0 * b1 - 3.0 * b2)
    rhs = 2.0 * CO.solve(f, b1) - 3.0 * CO.solve(f, b2)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)


def test_symmetric_preconditioner_on_spd():
    """SPD input: the oracle's Ã is symmetric to rounding (u^T Ã v = v^T Ã u)."""
    p = make_problem("cfg1", dims=(8, 8, 8), kind="varcoef", depth=5)
    f = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 5, 1e-2)
    rng = np.random.default_rng(4)
    u, v = rng.standard_normal(p.n), rng.standard_normal(p.n)
    a, b = u @ CO.solve(f, v), v @ CO.solve(f, u)
    assert abs(a - b) <= 1e-12 * max(abs(a), 1.0)


# ---------------------------------------------------------------------------
# Compression: constructed spectrum (S:l.272) through a whole factorization
# ---------------------------------------------------------------------------
def test_first_compress_rank_one_fill_ring():
    """Ring of 4 level-3 supers: eliminating s_0 couples s_1 and s_3 through the
    rank-1 fill -A_{31} S_0^{-1} A_{01} (P:l.101-106), so the first compress (s_1,
    partner s_3) has exactly one nonzero singular value, equal (stack [A; B]) to
    sqrt(2) |fill|_F: rank 1 for every eps in (0, 1)."""
    rp, ci, va, xy = ring_problem(64)
    for eps in (1e-1, 1e-4, 1e-8):
        f = CO.factorize(64, rp, ci, va, xy, 3, eps, order="natural")
        assert f.rank[(3, 1)] == 1
    A = csr_to_dense(64, rp, ci, va)
    s0, s1, s3 = np.arange(0, 16), np.arange(16, 32), np.arange(48, 64)
    fill = A[np.ix_(s3, s0)] @ np.linalg.solve(A[np.ix_(s0, s0)], A[np.ix_(s0, s1)])
    sig = f.sigma[(3, 1)]
    assert sig[0] == pytest.approx(math.sqrt(2.0) * np.linalg.norm(fill), rel=1e-12)
    assert np.all(sig[1:] <= 1e-12 * sig[0])


def test_frobenius_rule_threshold_ring():
    """F2 (Eq. curOff6, P:l.756-761, reading F2): at the first level the
    denominator is the Frobenius norm of every super-node block after
    MergeRedNodes, i.e. ||A||_F (hand-computed: 64 * 2.1^2 + 128 * 1^2).  The
    rank-1 stack of s_1 is dropped iff sigma_0 < eps ||A||_F."""
    rp, ci, va, xy = ring_problem(64)
    D = math.sqrt(64 * 2.1 ** 2 + 128 * 1.0)
    A = csr_to_dense(64, rp, ci, va)
    assert np.linalg.norm(A) == pytest.approx(D, rel=1e-14)
    s0, s1, s3 = np.arange(0, 16), np.arange(16, 32), np.arange(48, 64)
    fill = A[np.ix_(s3, s0)] @ np.linalg.solve(A[np.ix_(s0, s0)], A[np.ix_(s0, s1)])
    sigma0 = math.sqrt(2.0) * np.linalg.norm(fill)
    thr = sigma0 / D
    lo = CO.factorize(64, rp, ci, va, xy, 3, thr * 0.999, order="natural", truncation="frobenius")
    hi = CO.factorize(64, rp, ci, va, xy, 3, thr * 1.001, order="natural", truncation="frobenius")
    assert lo.rank[(3, 1)] == 1 and hi.rank[(3, 1)] == 0


def test_frobenius_rule_more_truncation_than_relative_sigma():
    """The Frobenius rule's denominator (every block of every level so far) is at
    least the stack's own sigma_0, so at equal eps it never keeps more: per-level
    rank totals <= those of Eq. cutOff1, and both fall as eps grows."""
    p = make_problem("cfg1", dims=(32, 32), depth=6)
    tot = {}
    for tr in ("sigma", "frobenius"):
        for eps in (1e-2, 1e-4):
            f = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 6, eps, truncation=tr)
            tot[(tr, eps)] = sum(f.rank.values())
    assert tot[("frobenius", 1e-2)] <= tot[("sigma", 1e-2)]
    assert tot[("frobenius", 1e-4)] <= tot[("sigma", 1e-4)]
    assert tot[("frobenius", 1e-2)] <= tot[("frobenius", 1e-4)]


# ---------------------------------------------------------------------------
# eps behaviour (P:l.585-603)
# ---------------------------------------------------------------------------
def test_residual_below_error_3d_poisson():
    """P:l.603 (3D Poisson, eps sweep): "the error and residual decrease
    proportional to ... eps. Furthermore ... the residual is smaller than the
    error."  3D 7-point Poisson 32x32x16 (the paper's 64x64x32 at 1/8 size,
    64-dof leaves), seeded uniform[-1,1] RHS, stand-alone solve x = Ã b."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    p = make_problem("cfg3", dims=(32, 32, 16))
    A = sp.csr_matrix((p.values, p.col_idx, p.row_ptr), shape=(p.n, p.n))
    xs = spl.spsolve(A.tocsc(), p.b)
    errs, ress = [], []
    for eps in (1e-1, 1e-2, 1e-3, 1e-4):
        f = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, p.depth, eps)
        x = CO.solve(f, p.b)
        errs.append(_rel(x, xs))
        ress.append(float(np.linalg.norm(A @ x - p.b) / np.linalg.norm(p.b)))
        f.close()
    assert all(r < e for r, e in zip(ress, errs)), (ress, errs)
    assert all(errs[k + 1] < errs[k] for k in range(3)) and all(ress[k + 1] < ress[k] for k in range(3))


def test_paper_2d_eps1e4_accuracy():
    """P:l.641-647: 2D Poisson, eps = 1e-4, leaf super-node 64 -> relative error ~1e-4."""
    p = make_problem("cfg1", dims=(64, 64), depth=7)
    f = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 7, 1e-4)
    x = CO.solve(f, p.b)
    err = _rel(x, np.linalg.solve(_dense(p), p.b))
    assert 1e-5 < err < 5e-4


# ---------------------------------------------------------------------------
# SpMV and Krylov on a NONSYMMETRIC matrix (both oracles; P:l.651-669)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("spmv", [CO.spmv, O.spmv], ids=["cpp", "numpy"])
def test_spmv_nonsymmetric_matches_dense(spmv):
    """A transposed SpMV would fail here: the upwind matrix is nonsymmetric."""
    p = make_problem("cfg1", dims=(24, 20), kind="upwind", depth=4)
    A = _dense(p)
    assert np.abs(A - A.T).max() > 1e-2
    x = np.random.default_rng(5).standard_normal(p.n)
    assert np.allclose(spmv(p.row_ptr, p.col_idx, p.values, x), A @ x, rtol=0, atol=1e-13 * np.abs(A @ x).max())


def test_cpp_gmres_nonsymmetric_solves():
    p = make_problem("cfg1", dims=(24, 24), kind="upwind", depth=5)
    A = _dense(p)
    xs = np.linalg.solve(A, p.b)
    f = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 5, 1e-1)
    r = CO.krylov(f, p.row_ptr, p.col_idx, p.values, p.b, method="gmres", tol=1e-10, restart=5)
    assert r.converged and r.iters > 1
    assert np.linalg.norm(A @ r.x - p.b) / np.linalg.norm(p.b) <= 1e-10
    assert _rel(r.x, xs) <= 1e-8
    f0 = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 5, 0.0)    # exact preconditioner
    r0 = CO.krylov(f0, p.row_ptr, p.col_idx, p.values, p.b, method="gmres", tol=1e-10)
    assert r0.converged and r0.iters <= 2


def test_numpy_gmres_nonsymmetric_solves():
    p = make_problem("cfg1", dims=(24, 24), kind="upwind", depth=5)
    A = _dense(p)
    f = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 5, 1e-1)
    r = O.gmres(lambda v: A @ v, lambda v: O.solve(f, v), p.b, tol=1e-10, restart=5)
    assert r.converged and r.iters > 1
    assert _rel(r.x, np.linalg.solve(A, p.b)) <= 1e-8


def test_cpp_pcg_exact_and_spd():
    p = make_problem("cfg1", dims=(16, 16), depth=4)
    f0 = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 4, 0.0)
    r0 = CO.krylov(f0, p.row_ptr, p.col_idx, p.values, p.b, method="cg")
    assert r0.converged and r0.iters == 1 and r0.relres <= 1e-10
    p = make_problem("cfg1")
    f = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, p.depth, 1e-2)
    r = CO.krylov(f, p.row_ptr, p.col_idx, p.values, p.b, method="cg")
    assert r.converged and 1 < r.iters < 20
    assert np.linalg.norm(_dense(p) @ r.x - p.b) / np.linalg.norm(p.b) <= 1e-10


@pytest.mark.parametrize("which", ["cpp", "numpy"])
def test_paper_preconditioned_residual_definition(which):
    """Eq. GMRES_residual (P:l.665-669) ||Ã b - Ã A x|| / ||Ã b||: with the exact
    preconditioner (eps = 0, Ã = A^{-1}) it is the relative error of x."""
    p = make_problem("cfg1", dims=(16, 16), kind="upwind", depth=4)
    A = _dense(p)
    xs = np.linalg.solve(A, p.b)
    x = xs + 1e-3 * np.random.default_rng(6).standard_normal(p.n)
    if which == "cpp":
        f = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 4, 0.0)
        val = CO.paper_preconditioned_residual(f, p.row_ptr, p.col_idx, p.values, p.b, x)
        one = CO.paper_preconditioned_residual(f, p.row_ptr, p.col_idx, p.values, p.b, np.zeros(p.n))
    else:
        f = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, 4, 0.0)
        mv = lambda v: A @ v
        pc = lambda v: O.solve(f, v)
        val = O.paper_preconditioned_residual(mv, pc, p.b, x)
        one = O.paper_preconditioned_residual(mv, pc, p.b, np.zeros(p.n))
    assert val == pytest.approx(_rel(x, xs), rel=1e-9)
    assert one == pytest.approx(1.0, rel=1e-14)


# ---------------------------------------------------------------------------
# Wave parallelism is exact: any thread count gives the sequential result bit
# for bit (the wave footprints are checked disjoint inside the oracle)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dims,kind,depth,eps", [((32, 32), "poisson", 6, 1e-2), ((12, 12, 12), "varcoef", 6, 1e-2),
                                                 ((32, 32), "upwind", 6, 1e-3)])
def test_threads_bitwise_equal(dims, kind, depth, eps):
    p = make_problem("cfg1", dims=dims, kind=kind, depth=depth)
    f1 = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, depth, eps, threads=1)
    f8 = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, depth, eps, threads=8)
    assert f8.info()["waves_parallel"] > 0
    assert f1.rank == f8.rank
    assert np.array_equal(CO.solve(f1, p.b, threads=1), CO.solve(f8, p.b, threads=8))


# ---------------------------------------------------------------------------
# Cross-check of the two independently pinned oracles (C++ loops vs numpy/LAPACK)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dims,kind,depth,eps,kw", [
    ((32, 32), "poisson", 6, 1e-2, {}), ((12, 12, 12), "varcoef", 6, 1e-2, {}),
    ((32, 32), "upwind", 6, 1e-3, {}), ((40, 24), "poisson", 5, 1e-3, {}),
    ((16, 16), "poisson", 4, 1e-2, {"order": "natural"}),
    ((16, 16), "poisson", 4, 1e-2, {"partition": "algebraic"}),
    ((12, 12, 12), "varcoef", 6, 1e-2, {"compressor": "rrqr"}),
])
def test_cpp_matches_numpy_oracle(dims, kind, depth, eps, kw):
    p = make_problem("cfg1", dims=dims, kind=kind, depth=depth)
    fc = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, depth, eps, **kw)
    fo = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, depth, eps, **kw)
    for i in range(1, depth + 1):
        seq_c, _ = fc.level_order(i)
        assert list(seq_c) == list(fo.level_order[i])
    bad = [k for k in fc.rank if fc.rank[k] != fo.rank.get(k, 0)]
    assert not bad
    assert _rel(CO.solve(fc, p.b), O.solve(fo, p.b)) <= 1e-11
