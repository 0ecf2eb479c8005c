import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer CPU test")


def ring_problem(n=64, diag=2.1):
    """1D periodic ring tridiag(-1, diag, -1) (SPD for diag > 2), coords x_i = i."""
    import numpy as np
    rows, cols, vals = [], [], []
    for i in range(n):
        for j, v in sorted({i: diag, (i - 1) % n: -1.0, (i + 1) % n: -1.0}.items()):
            rows.append(i); cols.append(j); vals.append(v)
    rows = np.array(rows); cols = np.array(cols, dtype=np.int64); vals = np.array(vals)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    coords = np.arange(n, dtype=np.float64).reshape(-1, 1)
    return row_ptr, cols, vals, coords
