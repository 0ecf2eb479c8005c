"""B200-native (sm_100a) LoRaSp level sweep (arxiv 1510.07363).

The product is the C-ABI shared library `liblorasp.so` (include/lorasp.h,
sources in csrc/); `lorasp.py` is its ctypes binding.
"""
from .lorasp import Handle, LoraspError, analyze_problem, load  # noqa: F401
