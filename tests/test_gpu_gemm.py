"""The two FP64 tile-GEMM kernels (k_gemm2 on the FMA pipe, k_gemm2_dmma on the
FP64 tensor cores) against numpy on ragged shapes, every transpose combination
and both tile widths (N <= 32 narrow tiles), through lorasp_test_gemm."""
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


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("M,N,K,ta,tb", [(70, 130, 37, 0, 0), (64, 64, 16, 1, 0), (129, 31, 200, 0, 1),
                                         (5, 3, 2, 1, 1), (200, 24, 1, 0, 0), (160, 160, 168, 1, 0)])
def test_tile_gemm_matches_numpy(L, variant, M, N, K, ta, tb):
    rng = np.random.default_rng(M * 1000 + N * 10 + K)
    A = rng.standard_normal((K, M) if ta else (M, K))
    B = rng.standard_normal((N, K) if tb else (K, N))
    C, ms = L.test_gemm(A, B, variant, ta, tb, reps=3)
    ref = (A.T if ta else A) @ (B.T if tb else B)
    # FP64 with K-term sums: |error| <= K u max|a| max|b| (both accumulate in FP64)
    assert np.abs(C - ref).max() <= 4 * K * 2.2e-16 * np.abs(A).max() * np.abs(B).max()
    assert ms > 0
