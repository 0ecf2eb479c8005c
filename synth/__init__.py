"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This package holds NONE of the method's arithmetic (no tree, no elimination,
no compression): only the PDE stencil generators of the BASELINE.json configs
and the splitmix64 right-hand sides.  It is the one module both `oracle/` and
the CUDA path's harness may import.
"""
from .problems import (CONFIGS, Problem, make_problem, grid_poisson, grid_varcoef,
                       grid_upwind, splitmix64_uniform, rhs_uniform, csr_to_dense,
                       csr_matvec)

__all__ = ["CONFIGS", "Problem", "make_problem", "grid_poisson", "grid_varcoef",
           "grid_upwind", "splitmix64_uniform", "rhs_uniform", "csr_to_dense",
           "csr_matvec"]
