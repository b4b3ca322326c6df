"""B200-native CoMoE MoE-layer hot path (arXiv 2508.09208).

Host API mirrors the reference package `comoe` (pkg/src/comoe) for routing,
aggregation and offload policy; every tensor computation runs in the
sm_100a kernels of libcomoe_b200.so (loaded by _lib, no CPU fallback).
"""

__version__ = "0.1.0"

from .errors import CoMoEError, ConfigError, InfeasibleError, TraceError  # noqa: F401

_LAZY = {
    "MoELayer": ("layer", "MoELayer"),
    "ExpertPool": ("pool", "ExpertPool"),
}


def __getattr__(name):
    if name in _LAZY:
        import importlib
        mod, attr = _LAZY[name]
        return getattr(importlib.import_module(f".{mod}", __name__), attr)
    raise AttributeError(name)
