"""B200-native LeanAttention decode (arXiv 2405.10480): C-ABI library + thin binding.

The hot path lives in ``csrc/`` (CUDA kernels for sm_100a + host planner + C ABI, built
into ``lib/libleanattn.so``); :mod:`.leanattn` marshals torch tensors into it.  There is no
CPU or library fallback on the product path.
"""
from .leanattn import (Plan, la_plan, la_combine, launch_count, lib, LaError, LIB_PATH, EXPORTS,
                       LA_OK, LA_ERR_INVALID, LA_ERR_UNSUPPORTED, LA_ERR_CUDA, LA_ERR_NOMEM, LA_ERR_STATE,
                       LA_ERR_TIMEOUT)

__all__ = ["Plan", "la_plan", "la_combine", "launch_count", "lib", "LaError", "LIB_PATH", "EXPORTS",
           "LA_OK", "LA_ERR_INVALID", "LA_ERR_UNSUPPORTED", "LA_ERR_CUDA", "LA_ERR_NOMEM", "LA_ERR_STATE",
           "LA_ERR_TIMEOUT"]
