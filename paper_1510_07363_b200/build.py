"""Build liblorasp.so in-tree with nvcc for sm_100a (B200).

    python -m paper_1510_07363_b200.build [--force]

The shared library is the C-ABI boundary (include/lorasp.h); the Python
binding (paper_1510_07363_b200/lorasp.py) loads it with ctypes.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "liblorasp.so")
SOURCES = [os.path.join(CSRC, f) for f in ("lorasp.cu", "analyze.cpp")]
HEADERS = [os.path.join(CSRC, f) for f in ("internal.h", "kernels.cuh")] + [os.path.join(ROOT, "include", "lorasp.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "-shared", "-Xptxas", "-v",
         "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    cmd = [NVCC] + FLAGS + ["-o", LIB + ".tmp"] + SOURCES + ["-lcudart", "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building liblorasp.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
