"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

Holds no method arithmetic (see pools.py / trace.py docstrings)."""
from .configs import CONFIGS, PROFILES, API_CLASSES, lib_config  # noqa: F401
from .pools import snapshot, requests, truths  # noqa: F401
from .trace import ClosedLoop, seg_row  # noqa: F401
