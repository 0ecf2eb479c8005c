"""Pins of the oracle's RRQR compressor (P:l.616, P:l.840):
column-pivoted QR  stack P = Q R,  keep the leading k with |R_kk| >= eps |R_00|
(reading F1), V = orthonormal basis of the rows of R[:r, :] P^T.

Pinned against facts that do not depend on the implementation:
  * orthogonal columns with known norms: Businger-Golub pivoting takes them in
    descending norm order, so |R_kk| are the sorted norms, r follows from them
    and V spans exactly the kept coordinate directions;
  * an exactly rank-k stack: r = k for any eps well above rounding;
  * the QR truncation bound ||M (I - V V^T)||_F <= ||R_22||_F (the rows of
    R[:r, :] P^T span the kept space; what is dropped is R_22);
  * eps = 0: nothing is truncated and the factorization is exact (dense LU).
"""
import numpy as np
import pytest
import scipy.linalg as sla

from oracle import lorasp_oracle as O
from synth import csr_to_dense, make_problem


def _fz():
    return O._Factorizer.__new__(O._Factorizer)


def _rrqr(M, eps):
    fz = _fz()
    fz.eps = eps
    return fz._rrqr(M, M.shape[1])


def test_orthogonal_columns_known_norms():
    rng = np.random.default_rng(1)
    m = 9
    norms = np.array([3.0, 0.5, 7.0, 1e-4, 2.0, 0.05, 1e-6, 1.0, 0.2])
    Q, _ = np.linalg.qr(rng.standard_normal((20, m)))
    M = Q * norms                                    # column j = norms[j] q_j
    for eps in (0.1, 0.01, 1e-3):
        r, sig, V = _rrqr(M, eps)
        srt = np.sort(norms)[::-1]
        assert np.allclose(sig[:m], srt, rtol=1e-12)
        want = int(np.sum(srt >= eps * srt[0]))     # prefix = count (norms distinct)
        assert r == want
        kept = np.argsort(-norms)[:r]
        P = np.zeros((m, m))
        P[kept, kept] = 1.0                          # projector on the kept coordinates
        assert np.allclose(V @ V.T, P, atol=1e-12)


@pytest.mark.parametrize("k", [1, 3, 6])
def test_exact_low_rank(k):
    rng = np.random.default_rng(k)
    M = rng.standard_normal((30, k)) @ rng.standard_normal((k, 12))
    for eps in (1e-2, 1e-8):
        r, sig, V = _rrqr(M, eps)
        assert r == k
        assert np.linalg.norm(M - M @ V @ V.T) <= 1e-12 * np.linalg.norm(M)


def test_truncation_bound_r22():
    rng = np.random.default_rng(5)
    m = 16
    M = rng.standard_normal((40, m)) @ np.diag(0.5 ** np.arange(m)) @ np.linalg.qr(rng.standard_normal((m, m)))[0]
    for eps in (0.3, 0.05, 0.01):
        r, sig, V = _rrqr(M, eps)
        R, piv = sla.qr(M, mode="r", pivoting=True)
        r22 = np.linalg.norm(R[r:, r:])
        assert np.allclose(V.T @ V, np.eye(r), atol=1e-12)
        assert np.linalg.norm(M - M @ V @ V.T) <= r22 * (1 + 1e-10) + 1e-14
        assert sig[r] < eps * sig[0] <= sig[r - 1]


def test_zero_stack_and_eps0():
    r, sig, V = _rrqr(np.zeros((5, 4)), 1e-2)
    assert r == 0 and V.shape == (4, 0)
    rng = np.random.default_rng(2)
    M = rng.standard_normal((3, 6))                  # fewer rows than columns
    r, sig, V = _rrqr(M, 0.0)
    assert r == 6 and np.allclose(V.T @ V, np.eye(6))


@pytest.mark.parametrize("name,dims", [("cfg1", (16, 16)), ("cfg3", (8, 8, 8)), ("cfg5", (16, 16))])
def test_rrqr_eps0_matches_dense_lu(name, dims):
    p = make_problem(name, dims=dims)
    f = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, p.depth, 0.0, compressor="rrqr")
    A = csr_to_dense(p.n, p.row_ptr, p.col_idx, p.values)
    x = O.solve(f, p.b)
    xe = np.linalg.solve(A, p.b)
    assert np.linalg.norm(x - xe) <= 1e-10 * np.linalg.norm(xe)


def test_rrqr_preconditioner_quality_tracks_eps():
    """Smaller eps -> a closer approximate inverse, of the same quality as the
    SVD compressor at the same eps (both keep the dominant row space)."""
    p = make_problem("cfg1", dims=(16, 16), kind="varcoef")
    A = csr_to_dense(p.n, p.row_ptr, p.col_idx, p.values)
    xe = np.linalg.solve(A, p.b)
    err = {}
    for comp in ("rrqr", "svd"):
        for eps in (1e-1, 1e-3):
            f = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, p.depth, eps, compressor=comp)
            err[comp, eps] = np.linalg.norm(O.solve(f, p.b) - xe) / np.linalg.norm(xe)
    assert err["rrqr", 1e-3] < 0.1 * err["rrqr", 1e-1]
    for eps in (1e-1, 1e-3):
        assert 0.5 < err["rrqr", eps] / err["svd", eps] < 2.0
