"""ORACLE (C++17, LAPACK-free) for the LoRaSp level sweep -- TEST INFRASTRUCTURE ONLY.

Python front end of `oracle/cpp/lorasp_oracle.cpp` (plain loops, no BLAS/LAPACK,
OpenMP across the nodes of one colour wave; BASELINE north_star "dense
LAPACK-free loops").  Only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s cpu_baseline / `--impl reference` leg may import this module.
It shares no code with the CUDA path (`paper_1510_07363_b200/`): it builds its
own shared library with g++ and loads it with ctypes; inputs come from `synth/`.

The numpy transcription `oracle/lorasp_oracle.py` is the second oracle; the two
are cross-checked in tests/test_oracle_cpp.py.  Functions mirror its API:

  factorize(...) -> CFactorization (rank / sigma dicts, level_order, trace, size)
  solve(f, b)                         Alg. 2-4 (P:l.401-500)
  krylov(f, row_ptr, col_idx, values, b, method, ...)   PCG / GMRES(restart) (P:l.651-669)
  paper_preconditioned_residual(...)  Eq. GMRES_residual (P:l.665-669)
  spmv(...)                           y = A x (CSR, row by row)
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import subprocess
import threading
from typing import Dict, List, Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cpp", "lorasp_oracle.cpp")
LIB = os.path.join(HERE, "cpp", "liblorasp_oracle.so")
CXX = os.environ.get("ORACLE_CXX", "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++")
FLAGS = ["-O3", "-march=x86-64-v3", "-fopenmp", "-std=c++17", "-shared", "-fPIC"]

F_NATURAL, F_SYMSTACK, F_RRQR, F_ALGEBRAIC, F_TRACE, F_FROBENIUS = 1, 2, 4, 8, 16, 32

_lib = None
_lock = threading.Lock()


def build(force: bool = False) -> str:
    """Compile the oracle library in-tree (g++; building the checker is not using it)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".{os.getpid()}.tmp"
        res = subprocess.run([CXX] + FLAGS + ["-o", tmp, SRC], capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("g++ failed building the oracle:\n" + res.stdout + res.stderr)
        os.replace(tmp, LIB)
    return LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = C.CDLL(LIB)
            P = C.c_void_p
            i64p, dp, ip = C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_int)
            lib.orc_factorize.argtypes = [C.c_int64, i64p, i64p, dp, C.c_int, dp, C.c_int, C.c_double, C.c_int,
                                          C.c_int, C.POINTER(P)]
            lib.orc_free.argtypes = [P]
            lib.orc_solve.argtypes = [P, dp, dp, C.c_int]
            lib.orc_ranks.argtypes = [P, C.c_int, ip]
            lib.orc_sigma.argtypes = [P, C.c_int, C.c_int64, dp, C.c_int]
            lib.orc_level_order.argtypes = [P, C.c_int, i64p, ip]
            lib.orc_node_counts.argtypes = [P, C.c_int, ip, ip]
            lib.orc_trace.argtypes = [P, C.c_char_p, C.c_int64]
            lib.orc_trace.restype = C.c_int64
            lib.orc_info.argtypes = [P, i64p]
            lib.orc_size.argtypes = [P, C.c_int, C.c_int, C.c_int64]
            lib.orc_frob_d2.argtypes = [P, C.c_int]
            lib.orc_frob_d2.restype = C.c_double
            lib.orc_spmv.argtypes = [C.c_int64, i64p, i64p, dp, dp, dp]
            lib.orc_krylov.argtypes = [P, C.c_int64, i64p, i64p, dp, dp, dp, C.c_double, C.c_int, C.c_int, C.c_int,
                                       C.c_int, ip, ip, ip, dp]
            lib.orc_paper_residual.argtypes = [P, C.c_int64, i64p, i64p, dp, dp, dp, C.c_int]
            lib.orc_paper_residual.restype = C.c_double
            lib.orc_test_svd.argtypes = [dp, C.c_int, C.c_int, dp, dp]
            lib.orc_test_lu_solve.argtypes = [dp, C.c_int, dp, C.c_int]
            lib.orc_test_qrcp.argtypes = [dp, C.c_int, C.c_int, dp, ip]
            lib.orc_last_error.restype = C.c_char_p
            _lib = lib
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def default_threads() -> int:
    return int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1))


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


KIND = {"s": 0, "b": 1, "r": 2}


class _Size(dict):
    """f.size[(kind, level, c)] looked up in the C++ store."""

    def __init__(self, f):
        super().__init__()
        self._f = f

    def __getitem__(self, key):
        k, i, c = key
        return int(_load().orc_size(self._f._h, KIND[k], int(i), int(c)))

    def get(self, key, default=0):
        return self[key]


class CFactorization:
    """Handle of one oracle factorization (frees the C++ store on close / GC)."""

    def __init__(self, h, n, depth, eps, threads):
        self._h = h
        self.n, self.depth, self.eps, self.threads = n, depth, eps, threads
        self._rank = None
        self._sigma = {}
        self.size = _Size(self)

    def close(self):
        if self._h:
            _load().orc_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:   # noqa: BLE001 - interpreter shutdown
            pass

    def ranks(self, level: int) -> np.ndarray:
        out = np.zeros(2 ** (level - 1), dtype=np.int32)
        _load().orc_ranks(self._h, level, _p(out, C.c_int))
        return out

    @property
    def rank(self) -> Dict[Tuple[int, int], int]:
        if self._rank is None:
            d = {}
            for i in range(1, self.depth + 1):
                for c, r in enumerate(self.ranks(i)):
                    d[(i, c)] = int(r)
            self._rank = d
        return self._rank

    def sigma_of(self, level: int, c: int) -> np.ndarray:
        key = (level, c)
        if key not in self._sigma:
            lib = _load()
            k = lib.orc_sigma(self._h, level, c, None, 0)
            buf = np.zeros(max(k, 1))
            lib.orc_sigma(self._h, level, c, _p(buf, C.c_double), k)
            self._sigma[key] = buf[:k]
        return self._sigma[key]

    @property
    def sigma(self):
        f = self

        class _S:
            def get(self, key, default=None):
                s = f.sigma_of(*key)
                return s if s.size or default is None else default

            def __getitem__(self, key):
                return f.sigma_of(*key)
        return _S()

    def level_order(self, level: int) -> Tuple[np.ndarray, np.ndarray]:
        seq = np.zeros(2 ** (level - 1), dtype=np.int64)
        wave = np.zeros(2 ** (level - 1), dtype=np.int32)
        _load().orc_level_order(self._h, level, _p(seq, C.c_int64), _p(wave, C.c_int))
        return seq, wave

    def node_counts(self, level: int):
        a = np.zeros(2 ** (level - 1), dtype=np.int32)
        b = np.zeros_like(a)
        _load().orc_node_counts(self._h, level, _p(a, C.c_int), _p(b, C.c_int))
        return a, b

    @property
    def trace(self) -> List[str]:
        lib = _load()
        k = lib.orc_trace(self._h, None, 0)
        buf = C.create_string_buffer(int(k) + 1)
        lib.orc_trace(self._h, buf, k + 1)
        return [t for t in buf.value.decode().split("\n") if t]

    def info(self) -> Dict[str, int]:
        a = np.zeros(5, dtype=np.int64)
        _load().orc_info(self._h, _p(a, C.c_int64))
        return {"max_edge_distance": int(a[0]), "waves_parallel": int(a[1]), "waves_total": int(a[2]),
                "blocks": int(a[3]), "doubles": int(a[4])}

    def frob_d2(self, level: int) -> float:
        """Frobenius rule (F2): ||all levels below||_F^2 used at `level`."""
        return float(_load().orc_frob_d2(self._h, level))

    @property
    def max_edge_distance(self) -> int:
        return self.info()["max_edge_distance"]


def factorize(n, row_ptr, col_idx, values, coords, depth, eps, order="coloured", symmetric_stack=False,
              trace=False, compressor="svd", partition="coordinates", truncation="sigma",
              threads: Optional[int] = None) -> CFactorization:
    """Alg. 1 (P:l.265-289) on the CSR matrix A.  compressor "svd" (Eq. lra,
    one-sided Jacobi) or "rrqr" (f1); truncation "sigma" (Eq. cutOff1) or
    "frobenius" (Eq. curOff6, reading F2)."""
    lib = _load()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int64)
    va = np.ascontiguousarray(values, dtype=np.float64)
    xy = np.ascontiguousarray(np.asarray(coords, dtype=np.float64).reshape(n, -1))
    flags = 0
    flags |= F_NATURAL if order == "natural" else 0
    flags |= F_SYMSTACK if symmetric_stack else 0
    flags |= F_RRQR if compressor == "rrqr" else 0
    flags |= F_ALGEBRAIC if partition == "algebraic" else 0
    flags |= F_TRACE if trace else 0
    flags |= F_FROBENIUS if truncation == "frobenius" else 0
    th = default_threads() if threads is None else int(threads)
    h = C.c_void_p()
    rc = lib.orc_factorize(int(n), _p(rp, C.c_int64), _p(ci, C.c_int64), _p(va, C.c_double), xy.shape[1],
                           _p(xy, C.c_double), int(depth), float(eps), flags, th, C.byref(h))
    if rc != 0:
        raise OracleError(rc, lib.orc_last_error().decode())
    return CFactorization(h, int(n), int(depth), float(eps), th)


def solve(f: CFactorization, b: np.ndarray, threads: Optional[int] = None) -> np.ndarray:
    """x ~= A^{-1} b by Alg. 2-4 (P:l.401-500)."""
    lib = _load()
    bb = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(f.n)
    rc = lib.orc_solve(f._h, _p(bb, C.c_double), _p(x, C.c_double), f.threads if threads is None else threads)
    if rc != 0:
        raise OracleError(rc, lib.orc_last_error().decode())
    return x


def spmv(row_ptr, col_idx, values, x) -> np.ndarray:
    lib = _load()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int64)
    va = np.ascontiguousarray(values, dtype=np.float64)
    xx = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(rp.size - 1)
    lib.orc_spmv(rp.size - 1, _p(rp, C.c_int64), _p(ci, C.c_int64), _p(va, C.c_double), _p(xx, C.c_double),
                 _p(y, C.c_double))
    return y


@dataclasses.dataclass
class KrylovResult:
    x: np.ndarray
    iters: int
    relres: float
    converged: bool
    breakdown: bool = False


def krylov(f: CFactorization, row_ptr, col_idx, values, b, method="cg", tol=1e-10, restart=50,
           maxit=500) -> KrylovResult:
    """PCG (method "cg") or right-preconditioned GMRES(restart) (method "gmres"),
    x0 = 0, tolerance on ||b - A x|| / ||b|| (readings Z21/Z24/Z27)."""
    lib = _load()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int64)
    va = np.ascontiguousarray(values, dtype=np.float64)
    bb = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(f.n)
    it, cv, bd = C.c_int(), C.c_int(), C.c_int()
    rr = C.c_double()
    rc = lib.orc_krylov(f._h, f.n, _p(rp, C.c_int64), _p(ci, C.c_int64), _p(va, C.c_double), _p(bb, C.c_double),
                        _p(x, C.c_double), float(tol), 0 if method == "cg" else 1, int(restart), int(maxit),
                        f.threads, C.byref(it), C.byref(cv), C.byref(bd), C.byref(rr))
    if rc != 0:
        raise OracleError(rc, lib.orc_last_error().decode())
    return KrylovResult(x, it.value, rr.value, bool(cv.value), bool(bd.value))


def paper_preconditioned_residual(f: CFactorization, row_ptr, col_idx, values, b, x) -> float:
    """Eq. GMRES_residual (P:l.665-669): ||Ã b - Ã A x|| / ||Ã b||."""
    lib = _load()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int64)
    va = np.ascontiguousarray(values, dtype=np.float64)
    bb = np.ascontiguousarray(b, dtype=np.float64)
    xx = np.ascontiguousarray(x, dtype=np.float64)
    return float(lib.orc_paper_residual(f._h, f.n, _p(rp, C.c_int64), _p(ci, C.c_int64), _p(va, C.c_double),
                                        _p(bb, C.c_double), _p(xx, C.c_double), f.threads))


# kernel-level entry points for the pins ------------------------------------
def svd_right(M: np.ndarray):
    """(sigma descending, V) of M by Householder QR + one-sided Jacobi."""
    lib = _load()
    R, m = M.shape
    Mc = np.asfortranarray(M, dtype=np.float64)
    s = np.zeros(m)
    V = np.zeros((m, m), order="F")
    rc = lib.orc_test_svd(_p(Mc, C.c_double), R, m, _p(s, C.c_double), _p(V, C.c_double))
    if rc != 0:
        raise OracleError(rc, lib.orc_last_error().decode())
    return s, V


def lu_solve_dense(A: np.ndarray, b: np.ndarray) -> np.ndarray:
    lib = _load()
    n = A.shape[0]
    Ac = np.asfortranarray(A, dtype=np.float64)
    x = np.asfortranarray(np.array(b, dtype=np.float64).reshape(n, -1))
    rc = lib.orc_test_lu_solve(_p(Ac, C.c_double), n, _p(x, C.c_double), x.shape[1])
    if rc != 0:
        raise OracleError(rc, lib.orc_last_error().decode())
    return x.reshape(np.shape(b))


def qr_colpiv(M: np.ndarray):
    lib = _load()
    R, m = M.shape
    Mc = np.asfortranarray(M, dtype=np.float64)
    d = np.zeros(min(R, m))
    perm = np.zeros(m, dtype=np.int32)
    lib.orc_test_qrcp(_p(Mc, C.c_double), R, m, _p(d, C.c_double), _p(perm, C.c_int))
    return d, perm
