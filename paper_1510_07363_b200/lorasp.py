"""Thin ctypes binding of liblorasp (include/lorasp.h) — argument marshalling only.

Every step of the factorization, the apply and the Krylov solvers runs in the
library's sm_100a kernels.  There is no Python or CPU fallback: if the shared
library is missing or fails to load, `load()` raises.

Arrays may be numpy arrays (host) or CUDA tensors (anything with
`data_ptr()` and `is_cuda`); the library detects host vs device pointers
itself.
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblorasp.so")

LORASP_OK = 0
LORASP_NOT_CONVERGED = 1
LORASP_SPD = 0x1
LORASP_ORDER_NATURAL = 0x2
LORASP_RRQR = 0x4          # f1: column-pivoted QR compressor (include/lorasp.h)
LORASP_ALGEBRAIC = 0x10    # f4: partition from the graph of A (include/lorasp.h)
LORASP_FROBENIUS = 0x20    # f2: Frobenius truncation rule Eq. curOff6 (include/lorasp.h)
LORASP_CG = 0
LORASP_GMRES = 1

STATUS = {0: "OK", 1: "NOT_CONVERGED", -1: "E_ARG", -2: "E_PATTERN", -3: "E_SINGULAR_PIVOT",
          -4: "E_EIG_NOCONV", -5: "E_CUDA", -6: "E_OOM", -7: "E_NCCL", -8: "E_STATE"}

# every symbol include/lorasp.h declares
SYMBOLS = ["lorasp_analyze", "lorasp_factor", "lorasp_apply", "lorasp_gmres", "lorasp_krylov_ex",
           "lorasp_set_stream", "lorasp_set_timing", "lorasp_get_depth", "lorasp_get_level_order", "lorasp_get_node_counts",
           "lorasp_get_ranks",
           "lorasp_get_sizes", "lorasp_get_stats", "lorasp_get_launch_count", "lorasp_test_eig",
           "lorasp_test_pivot", "lorasp_test_gemm", "lorasp_last_error", "lorasp_destroy", "lorasp_set_dist",
           "lorasp_set_dist_buffers", "lorasp_dist_owner", "lorasp_paper_residual", "lorasp_nccl_unique_id",
           "lorasp_set_dist_nccl", "lorasp_test_nccl", "lorasp_dist_counts"]

LORASP_COLL_ALLGATHER = 0
LORASP_COLL_MAXINT = 1
LORASP_COLL_RESERVE = 2
LORASP_COLL_ALLTOALLV = 3
# int (*lorasp_coll_fn)(void *user, int kind, int64_t nbytes)
COLL_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64)

_lib = None


class LoraspError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


def load(path: Optional[str] = None) -> ctypes.CDLL:
    """Load liblorasp.so (raises if absent: the product path has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(f"liblorasp.so not built at {path}: run `python -m paper_1510_07363_b200.build`")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    i64p = ctypes.POINTER(ctypes.c_int64)
    lib.lorasp_analyze.argtypes = [ctypes.c_int64, P, P, ctypes.c_int, P, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_double, ctypes.c_uint, ctypes.c_int, ctypes.POINTER(P)]
    lib.lorasp_factor.argtypes = [P, P]
    lib.lorasp_apply.argtypes = [P, P, P]
    lib.lorasp_gmres.argtypes = [P, P, P, ctypes.c_double]
    lib.lorasp_krylov_ex.argtypes = [P, P, P, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)]
    lib.lorasp_paper_residual.argtypes = [P, P, P, ctypes.POINTER(ctypes.c_double)]
    lib.lorasp_set_stream.argtypes = [P, P]
    lib.lorasp_set_timing.argtypes = [P, ctypes.c_int]
    lib.lorasp_get_depth.argtypes = [P, ctypes.POINTER(ctypes.c_int)]
    lib.lorasp_get_level_order.argtypes = [P, ctypes.c_int, P, P, ctypes.c_int]
    lib.lorasp_get_ranks.argtypes = [P, ctypes.c_int, P, ctypes.c_int]
    lib.lorasp_get_sizes.argtypes = [P, ctypes.c_int, P, ctypes.c_int]
    lib.lorasp_get_stats.argtypes = [P, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
    lib.lorasp_get_launch_count.argtypes = [P, i64p, i64p, i64p]
    lib.lorasp_test_eig.argtypes = [ctypes.c_int, P, ctypes.c_int, ctypes.c_double, P, P,
                                    ctypes.POINTER(ctypes.c_int)]
    lib.lorasp_test_pivot.argtypes = [ctypes.c_int, P, ctypes.c_int, ctypes.c_int]
    lib.lorasp_test_gemm.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P, ctypes.POINTER(ctypes.c_double)]
    lib.lorasp_last_error.argtypes = [P]
    lib.lorasp_last_error.restype = ctypes.c_char_p
    lib.lorasp_destroy.argtypes = [P]
    lib.lorasp_destroy.restype = None
    lib.lorasp_set_dist.argtypes = [P, ctypes.c_int, ctypes.c_int, COLL_FN, P]
    lib.lorasp_set_dist_buffers.argtypes = [P, P, ctypes.c_int64, P, ctypes.c_int64]
    lib.lorasp_dist_owner.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
    lib.lorasp_nccl_unique_id.argtypes = [P]
    lib.lorasp_set_dist_nccl.argtypes = [P, ctypes.c_int, ctypes.c_int, P]
    lib.lorasp_test_nccl.argtypes = [ctypes.c_int, ctypes.c_int]
    lib.lorasp_dist_counts.argtypes = [P, P, ctypes.c_int]
    for s in SYMBOLS:
        if s not in ("lorasp_last_error", "lorasp_destroy"):
            getattr(lib, s).restype = ctypes.c_int
    _lib = lib
    return lib


def _ptr(a):
    """Raw pointer of a numpy array (host) or a CUDA tensor (device)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return ctypes.c_void_p(a.data_ptr())
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return ctypes.c_void_p(a.ctypes.data)
    raise TypeError(f"unsupported buffer type {type(a)}")


class Handle:
    """lorasp_analyze(...) -> handle; factor / apply / krylov through the C ABI."""

    def __init__(self, n, row_ptr, col_idx, coords, depth=0, leaf_size=64, eps=1e-2,
                 flags=LORASP_SPD, device=0):
        lib = load()
        self._lib = lib
        self.n = int(n)
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int64)
        xy = np.ascontiguousarray(coords, dtype=np.float64)
        dim = 1 if xy.ndim == 1 else xy.shape[1]
        h = ctypes.c_void_p()
        rc = lib.lorasp_analyze(self.n, _ptr(rp), _ptr(ci), dim, _ptr(xy), int(leaf_size), int(depth),
                                float(eps), int(flags), int(device), ctypes.byref(h))
        if rc != LORASP_OK:
            raise LoraspError(rc, "lorasp_analyze failed")
        self.h = h
        self.nnz = int(rp[-1])
        d = ctypes.c_int()
        lib.lorasp_get_depth(self.h, ctypes.byref(d))
        self.depth = d.value

    def _check(self, rc, what):
        if rc < 0:
            raise LoraspError(rc, f"{what}: {self._lib.lorasp_last_error(self.h).decode()}")
        return rc

    def factor(self, values):
        return self._check(self._lib.lorasp_factor(self.h, _ptr(values)), "lorasp_factor")

    def apply(self, b, x):
        return self._check(self._lib.lorasp_apply(self.h, _ptr(b), _ptr(x)), "lorasp_apply")

    def gmres(self, b, x, tol=1e-10):
        return self._check(self._lib.lorasp_gmres(self.h, _ptr(b), _ptr(x), float(tol)), "lorasp_gmres")

    def krylov(self, b, x, tol=1e-10, method=LORASP_CG, restart=50, max_it=500):
        it = ctypes.c_int()
        rr = ctypes.c_double()
        rc = self._check(self._lib.lorasp_krylov_ex(self.h, _ptr(b), _ptr(x), float(tol), int(method),
                                                    int(restart), int(max_it), ctypes.byref(it),
                                                    ctypes.byref(rr)), "lorasp_krylov_ex")
        return rc, it.value, rr.value

    def paper_residual(self, b, x) -> float:
        """Eq. GMRES_residual (P:l.665-669): ||Ã b - Ã A x|| / ||Ã b|| (on the device)."""
        out = ctypes.c_double()
        self._check(self._lib.lorasp_paper_residual(self.h, _ptr(b), _ptr(x), ctypes.byref(out)),
                    "lorasp_paper_residual")
        return out.value

    def set_stream(self, stream_ptr: int):
        return self._check(self._lib.lorasp_set_stream(self.h, ctypes.c_void_p(stream_ptr)), "set_stream")

    def set_dist(self, rank, world, comm=None):
        """Distributed factorization (include/lorasp.h, lorasp_set_dist): `comm`
        provides reserve(nbytes) -> (send, recv) device tensors, allgather(nbytes)
        and allmax_int(nbytes) (paper_1510_07363_b200.dist).  world = 1 resets."""
        lib = self._lib
        if world == 1 or comm is None:
            self._coll = None
            return self._check(lib.lorasp_set_dist(self.h, 0, 1, COLL_FN(), None), "set_dist")

        def cb(_user, kind, nbytes):
            try:
                if kind == LORASP_COLL_RESERVE:
                    send, recv = comm.reserve(int(nbytes))
                    lib.lorasp_set_dist_buffers(self.h, _ptr(send), send.numel() * send.element_size(),
                                                _ptr(recv), recv.numel() * recv.element_size())
                elif kind == LORASP_COLL_ALLGATHER:
                    comm.allgather(int(nbytes))
                elif kind == LORASP_COLL_MAXINT:
                    comm.allmax_int(int(nbytes))
                elif kind == LORASP_COLL_ALLTOALLV:
                    cnt = np.zeros(world * world, dtype=np.int64)
                    lib.lorasp_dist_counts(self.h, ctypes.c_void_p(cnt.ctypes.data), cnt.size)
                    comm.alltoallv(cnt.reshape(world, world))
                else:
                    return 1
                return 0
            except Exception:   # reported to the engine, which aborts with E_CUDA
                import traceback
                traceback.print_exc()
                return 1

        self._coll = COLL_FN(cb)   # the handle keeps the callback alive
        return self._check(lib.lorasp_set_dist(self.h, int(rank), int(world), self._coll, None), "set_dist")

    def set_dist_nccl(self, rank, world, unique_id: bytes):
        """Distributed mode over a library-owned NCCL communicator (include/lorasp.h)."""
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        return self._check(self._lib.lorasp_set_dist_nccl(self.h, int(rank), int(world), buf), "set_dist_nccl")

    def set_timing(self, mask):
        """mask: True = all kernel classes, False = off, or an int bitmask of classes."""
        m = -1 if mask is True else (0 if mask is False else int(mask))
        return self._check(self._lib.lorasp_set_timing(self.h, m), "set_timing")

    def level_order(self, level):
        K = 2 ** (level - 1)
        order = np.zeros(K, dtype=np.int32)
        wave = np.zeros(K, dtype=np.int32)
        self._check(self._lib.lorasp_get_level_order(self.h, level, _ptr(order), _ptr(wave), K), "order")
        return order, wave

    def ranks(self, level):
        K = 2 ** (level - 1)
        out = np.zeros(K, dtype=np.int32)
        self._check(self._lib.lorasp_get_ranks(self.h, level, _ptr(out), K), "ranks")
        return out

    def node_counts(self, level):
        """(partners, n1) per level-`level` super-node: the kappa_2 / kappa_1 edges
        of the symbolic Alg. 1 replay (lorasp_get_node_counts)."""
        K = 2 ** (level - 1)
        a = np.zeros(K, dtype=np.int32)
        b = np.zeros(K, dtype=np.int32)
        self._check(self._lib.lorasp_get_node_counts(self.h, level, _ptr(a), _ptr(b), K), "node_counts")
        return a, b

    def sizes(self, level):
        K = 2 ** (level - 1)
        out = np.zeros(K, dtype=np.int32)
        self._check(self._lib.lorasp_get_sizes(self.h, level, _ptr(out), K), "sizes")
        return out

    def stats(self) -> dict:
        ln = ctypes.c_size_t()
        self._lib.lorasp_get_stats(self.h, None, 0, ctypes.byref(ln))
        buf = ctypes.create_string_buffer(ln.value + 16)
        self._lib.lorasp_get_stats(self.h, buf, len(buf), None)
        return json.loads(buf.value.decode())

    def launch_counts(self):
        f, a, k = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        self._lib.lorasp_get_launch_count(self.h, ctypes.byref(f), ctypes.byref(a), ctypes.byref(k))
        return f.value, a.value, k.value

    def close(self):
        if getattr(self, "h", None):
            self._lib.lorasp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for lorasp_set_dist_nccl (call on one rank, share it)."""
    buf = ctypes.create_string_buffer(128)
    rc = load().lorasp_nccl_unique_id(buf)
    if rc != LORASP_OK:
        raise LoraspError(rc, "lorasp_nccl_unique_id")
    return buf.raw


def test_nccl(n=1000, device=0):
    """NCCL plumbing hook (1-rank communicator): status code."""
    return load().lorasp_test_nccl(int(device), int(n))


def dist_owner(level, c, world):
    """Owner rank of level-`level` super-node c (lorasp_dist_owner)."""
    return load().lorasp_dist_owner(int(level), int(c), int(world))


def test_eig(G, eps, device=0):
    """Kernel hook: Jacobi eigen-solver on one Gram matrix -> (sigma, V_r, r, status)."""
    lib = load()
    G = np.asfortranarray(G, dtype=np.float64)
    m = G.shape[0]
    V = np.zeros((m, m), order="F")
    sig = np.zeros(m)
    r = ctypes.c_int()
    st = lib.lorasp_test_eig(device, ctypes.c_void_p(G.ctypes.data), m, float(eps),
                             ctypes.c_void_p(V.ctypes.data), ctypes.c_void_p(sig.ctypes.data), ctypes.byref(r))
    # the library writes V as m x r column-major: reinterpret the first m*r entries
    Vr = V.reshape(-1, order="F")[: m * r.value].reshape((m, r.value), order="F")
    return sig, Vr.copy(), r.value, st


def test_gemm(A, B, variant, ta=0, tb=0, reps=1, device=0):
    """Kernel hook: C = op(A) op(B) through k_gemm2 (variant 0, DFMA) or
    k_gemm2_dmma (1, DMMA) on `reps` copies -> (C, ms per launch)."""
    lib = load()
    A = np.asfortranarray(A, dtype=np.float64)
    B = np.asfortranarray(B, dtype=np.float64)
    M = A.shape[1] if ta else A.shape[0]
    K = A.shape[0] if ta else A.shape[1]
    N = B.shape[0] if tb else B.shape[1]
    C = np.zeros((M, N), order="F")
    ms = ctypes.c_double()
    st = lib.lorasp_test_gemm(device, variant, M, N, K, ta, tb, reps, ctypes.c_void_p(A.ctypes.data),
                              ctypes.c_void_p(B.ctypes.data), ctypes.c_void_p(C.ctypes.data), ctypes.byref(ms))
    if st != 0:
        raise LoraspError(st, "lorasp_test_gemm")
    return C, ms.value


def test_pivot(K, m, r, device=0):
    """Kernel hook: signed Cholesky + inverse of the fused pivot -> (L^{-1}, status)."""
    lib = load()
    A = np.asfortranarray(K, dtype=np.float64).copy(order="F")
    st = lib.lorasp_test_pivot(device, ctypes.c_void_p(A.ctypes.data), int(m), int(r))
    return A, st


def analyze_problem(p, eps=None, flags=None, device=0, depth=None) -> Handle:
    """Convenience: analyze a synth.Problem (SPD path for symmetric problems,
    the general LU path otherwise, unless flags are given)."""
    if flags is None:
        flags = LORASP_SPD if getattr(p, "symmetric", True) else 0
    return Handle(p.n, p.row_ptr, p.col_idx, p.coords, depth=p.depth if depth is None else depth,
                  leaf_size=p.leaf, eps=p.eps if eps is None else eps, flags=flags, device=device)
