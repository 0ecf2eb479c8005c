"""GPU unit parity of the fused (s, b) pivot (P:l.396-399, P:l.101-106)
through the C-ABI hook `lorasp_test_pivot`, for both kernels the sweep uses:
k_pivot_blk (n <= 160, blocked, shared memory) and k_pivot (n > 160).

K = [[S, V], [V^T, 0]] with S SPD factors as K = L diag(I_m, -I_r) L^T; the
hook returns L^{-1} (lower triangle, strict upper zero).  Checks against the
definition, not against another implementation:
  * L^{-1} is lower triangular with a positive diagonal;
  * (L^{-1}) K (L^{-1})^T = diag(I_m, -I_r) within 1e-11 (cond(K) here <= ~1e3);
  * the leading m x m block of L^{-1} is the inverse Cholesky factor of S
    (unique): compared with numpy's Cholesky within 1e-11 relative.
A non-positive pivot is reported as LORASP_E_SINGULAR_PIVOT (-3)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1510_07363_b200 import build, lorasp
    build.build()
    return lorasp


def fused(m, r, seed):
    rng = np.random.default_rng(seed)
    B = rng.standard_normal((m, m))
    S = B @ B.T / m + np.eye(m)
    V = np.linalg.qr(rng.standard_normal((m, max(r, 1))))[0][:, :r] if r else np.zeros((m, 0))
    K = np.zeros((m + r, m + r))
    K[:m, :m] = S
    K[:m, m:] = V
    K[m:, :m] = V.T
    return K, S


@pytest.mark.parametrize("m,r", [(1, 0), (1, 1), (5, 3), (20, 0), (25, 7), (31, 1), (32, 32), (40, 24),
                                 (50, 14), (63, 1), (64, 0), (45, 20), (100, 30), (128, 20), (150, 10),
                                 (170, 40)])
def test_pivot_signed_cholesky_inverse(L, m, r):
    K, S = fused(m, r, seed=m * 100 + r)
    n = m + r
    X, st = L.test_pivot(K, m, r)
    assert st == 0
    assert np.array_equal(np.triu(X, 1), np.zeros((n, n)))
    assert np.all(np.diag(X) > 0)
    D = np.diag(np.r_[np.ones(m), -np.ones(r)])
    assert np.max(np.abs(X @ K @ X.T - D)) <= 1e-11 * max(1.0, np.linalg.cond(K) / 1e2)
    Ls = np.linalg.cholesky(S)
    assert np.allclose(X[:m, :m], np.linalg.inv(Ls), rtol=0, atol=1e-11 * np.abs(np.linalg.inv(Ls)).max())


@pytest.mark.parametrize("m", [8, 40, 100])
def test_pivot_indefinite_s_fails(L, m):
    K, S = fused(m, 0, seed=m)
    K[m // 2, m // 2] = -5.0          # S no longer positive definite
    _, st = L.test_pivot(K, m, 0)
    assert st == -3
