"""B200-native LeanAttention decode (arXiv 2405.10480): C-ABI library + thin binding.

The hot path lives in ``csrc/`` (CUDA kernels for sm_100a + host planner + C ABI, built
into ``lib/libleanattn.so``); :mod:`.leanattn` marshals torch tensors into it.  There is no
CPU or library fallback on the product path.
"""
from .leanattn import (Plan, la_plan, la_combine, launch_count, lib, LaError, LIB_PATH, EXPORTS)

__all__ = ["Plan", "la_plan", "la_combine", "launch_count", "lib", "LaError", "LIB_PATH", "EXPORTS"]
