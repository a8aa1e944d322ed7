"""paper_2303_06742_b200 — B200-native (sm_100a, fp64) space-time GMRES–GMG slab solver of arXiv:2303.06742.

The product is libstgmg.so (C ABI: include/stgmg.h, CUDA sources: csrc/).  ``Solver`` is a thin ctypes binding;
PyTorch is only used for device memory and streams.  There is no CPU fallback.
"""
from .build import build, LIB
from .stgmg import Solver, LShapeSolver, StgmgError, load_library, SIGNATURES, TOL_REL, TOL_ABS

__all__ = ["build", "LIB", "Solver", "LShapeSolver", "StgmgError", "load_library", "SIGNATURES", "TOL_REL", "TOL_ABS"]
