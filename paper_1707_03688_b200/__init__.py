"""B200-native 2D nonseparable discrete LCT (arxiv 1707.03688).

The product is libnslct.so (C ABI in include/nslct.h, CUDA kernels for sm_100a, C++
host planner); `nslct` is its thin ctypes binding.  There is no CPU fallback.
"""
from .nslct import (Plan, SlabPlan, NslctError, lib, nslct_plan_describe, nsdlct, nsdlct_inverse,  # noqa: F401
                    inverse_matrix, EXPORTS, LIB_PATH)
