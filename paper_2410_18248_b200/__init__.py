"""B200-native LAMPS scheduling pass (arXiv 2410.18248).

The pass itself is CUDA (sm_100a) behind the C ABI in include/lamps.h; this
package holds those sources (csrc/), the in-tree build and a ctypes binding.
"""
from .lamps import (  # noqa: F401
    LampsError, Scheduler, lib, lamps_init, lamps_submit, lamps_api_return, lamps_schedule_step,
    lamps_free, lamps_last_error, LAMPS_DEBUG_OUT, LAMPS_TIMING, LAMPS_MULTI_KERNEL, LAMPS_FORCE_FALLBACK,
    LAMPS_TRACE, LAMPS_MERGE, LAMPS_HEAD_ONLY,
)

__all__ = ["Scheduler", "LampsError", "lib", "lamps_init", "lamps_submit", "lamps_api_return",
           "lamps_schedule_step", "lamps_free", "lamps_last_error"]
