"""DMMA (FP64 tensor cores) vs DFMA tile GEMM on the sweep's block shapes
(north_star item 3), through the C-ABI hook lorasp_test_gemm.  Prints one JSON
object: per shape the launch time of each variant, the achieved TFLOP/s and the
max relative difference of C to numpy.   python tools/gemm_dmma_vs_dfma.py"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_07363_b200 import lorasp as L  # noqa: E402

# (name, M, N, K, ta, tb, reps): reps = equal GEMMs in one launch (a wave)
SHAPES = [
    ("schur_2d_leaf", 160, 160, 168, 1, 0, 100),     # T_ab -= Z_a^T D Z_b, cfg2 leaf wave
    ("schur_3d_leaf", 384, 384, 180, 1, 0, 64),      # cfg4 leaf (W ~ 2.8 x 128 + 2 r)
    ("trsm_3d_leaf", 180, 420, 180, 0, 0, 128),      # Z = L^{-1} C
    ("gram_leaf", 128, 128, 800, 1, 0, 128),         # G = M^T M over the partner stack
    ("project_narrow", 800, 32, 128, 0, 0, 128),     # R_k = A_k V_r (N <= 32: 64 x 32 tiles)
    ("upper_512", 512, 512, 512, 0, 0, 8),           # upper-level node
]

out = {}
rng = np.random.default_rng(0)
for name, M, N, K, ta, tb, reps in SHAPES:
    A = rng.standard_normal((K, M) if ta else (M, K))
    B = rng.standard_normal((N, K) if tb else (K, N))
    ref = (A.T if ta else A) @ (B.T if tb else B)
    rec = {"M": M, "N": N, "K": K, "ta": ta, "tb": tb, "reps": reps}
    for v, lab in ((0, "dfma"), (1, "dmma")):
        C, ms = L.test_gemm(A, B, v, ta, tb, reps)
        rec[lab + "_ms"] = ms
        rec[lab + "_tflops"] = 2.0 * M * N * K * reps / (ms / 1e3) / 1e12
        rec[lab + "_relerr"] = float(np.abs(C - ref).max() / np.abs(ref).max())
    rec["dmma_speedup"] = rec["dfma_ms"] / rec["dmma_ms"]
    out[name] = rec
print(json.dumps(out, indent=1))
