"""B200-native evaluate+stamp hot path of EEspice (arxiv 2604.03079).

``Context`` wraps the C ABI of ``include/ees.h`` (libees.so, sm_100a).  The
binding is imported lazily so ``python -m paper_2604_03079_b200.build`` works
before the library exists.
"""
__all__ = ["Context", "EESError", "VARIANTS", "RULES", "fp64_peak", "red_throughput", "stream_probe", "Solver"]


def __getattr__(name):
    if name in __all__:
        from . import api
        return getattr(api, name)
    raise AttributeError(name)
