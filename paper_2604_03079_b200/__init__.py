"""B200-native evaluate+stamp hot path of EEspice (arxiv 2604.03079).

``Context`` wraps the C ABI of ``include/ees.h`` (libees.so, sm_100a).
"""
from .api import Context, EESError, RULES, VARIANTS  # noqa: F401

__all__ = ["Context", "EESError", "VARIANTS", "RULES"]
