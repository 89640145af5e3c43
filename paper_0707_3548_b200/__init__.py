"""B200-native (sm_100a) fp64 tiled QR factorization (arXiv 0707.3548).

The compute path is libtqr.so (CUDA kernels + C ABI, include/tqr.h); this package is a
thin ctypes binding over it.  No CPU fallback exists: importing a function whose library
is missing raises.
"""
from .tqr import (Plan, TqrError, colmajor, flops_standard, flops_tiled, from_colmajor, lib, schedule_inspect,
                  supported)
from .tlu import LUPlan  # the tiled LU (include/tlu.h)

__all__ = ["LUPlan", "Plan", "TqrError", "colmajor", "flops_standard", "flops_tiled", "from_colmajor", "lib",
           "schedule_inspect", "supported"]
