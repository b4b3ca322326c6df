"""ctypes binding of libcomoe_b200.so (the C ABI in include/comoe_b200.h).

There is no fallback: if the library is missing or fails to load, every
compute entry point raises. Domain errors from the C side (bad sizes,
unsupported shapes) become ValueError, CUDA failures RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libcomoe_b200.so"
ABI_VERSION = 2

_c_int, _c_long, _c_double = ctypes.c_int, ctypes.c_long, ctypes.c_double
_p = ctypes.c_void_p

# name -> argtypes (all return int unless listed in _RESTYPES)
_SIGNATURES = {
    "comoe_version": [],
    "comoe_last_error": [],
    "comoe_num_sms": [_c_int],
    "comoe_gate_padded_experts": [_c_int],
    "comoe_gate_num_tiles": [_c_int],
    "comoe_gate_prepare": [_p, _c_int, _c_int, _p, _p],
    "comoe_gate_topk": [_p, _c_int, _c_int, _p, _c_int, _c_int, _c_int, _p, _c_int, _p,
                        _p, _p, _p, _p, _p, _p],
    "comoe_gate_route_workspace_bytes": [_c_int, _c_int, _c_int],
    "comoe_gate_route": [_p, _c_int, _c_int, _p, _c_int, _c_int, _c_int, _p, _c_int, _c_int,
                         _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p],
    "comoe_route_from_indices": [_p, _p, _c_int, _c_int, _c_int, _p, _c_int, _p, _p, _p, _p, _p],
    "comoe_route_scan": [_p, _c_int, _c_int, _c_int, _c_int, _p, _p, _p, _p, _p],
    "comoe_expert_histogram": [_p, _c_long, _c_int, _p, _p],
    "comoe_permute": [_p, _c_int, _c_int, _c_int, _p, _p, _p, _p, _p, _c_int, _c_int, _p,
                      _p, _p, _p, _p, _p],
    "comoe_grouped_gemm": [_p, _c_long, _p, _c_int, _c_long, _c_long, _c_int, _c_int, _p, _p,
                           _p, _c_int, _c_int, _p, _c_int, _p, _p, _p, _p],
    "comoe_grouped_ffn": [_p, _c_long, _c_int, _c_int, _c_int, _p, _c_int, _c_long, _p, _p,
                          _p, _c_int, _p, _p, _c_int, _p, _p, _p],
    "comoe_fused_ffn": [_p, _c_long, _p, _c_int, _c_int, _p, _c_int, _c_long, _p, _p, _p, _c_int,
                        _p, _c_int, _p, _p, _p],
    "comoe_fused_ffn_supported": [_c_int, _c_int, _c_int, _c_int],
    "comoe_fused_ffn_enabled": [],
    "comoe_debug_fused_prof": [_p],
    "comoe_combine": [_p, _p, _p, _c_int, _c_int, _c_int, _p, _p],
    "comoe_debug_gemm_clock": [_p],
    "comoe_debug_set_gemm": [_c_int],
    "comoe_debug_gate_timeline": [_p, _p],
    "comoe_debug_set_gate_tm": [_c_int],
    "comoe_permute_peers": [_p, _c_int, _c_int, _c_int, _p, _p, _p, _p, _p, _c_int, _c_int, _p,
                            _c_int, _c_long, _c_int, _p, _p, _p, _p],
    "comoe_combine_peers": [_p, _c_int, _c_long, _c_int, _p, _p, _c_int, _c_int, _c_int, _p, _p],
    "comoe_peer_scatter_counts": [_p, _c_int, _c_int, _c_int, _p, _p],
    "comoe_peer_barrier": [_p, _c_int, _c_int, _c_int, ctypes.c_longlong, _p, _p],
    "comoe_ipc_handle_size": [],
    "comoe_ipc_get_handle": [_p, _p, _p],
    "comoe_ipc_open": [_p, _c_long, _p],
    "comoe_ipc_close": [_p, _c_long],
    "comoe_merge": [_c_int, _p, _p, _p, _p, _p, _c_int, _c_int, _c_long, _p],
    "comoe_sim_workspace_bytes": [_c_int, _c_int, _c_int, _c_long],
    "comoe_sim_contract": [_c_int, _p, _c_int, _c_long, _p, _c_int, _p, _c_int, _p, _p, _p,
                           _p],
    "comoe_sim_tc_supported": [_c_int, _c_long],
    "comoe_sim_gram_strided": [_p, _c_long, _c_int, _c_long, _p, _p, _p],
    "comoe_sim_finalize": [_p, _p, _c_int, _c_int, _c_int, _c_double, _p, _p],
    "comoe_predictor_workspace_bytes": [_c_int, _c_int],
    "comoe_predictor_mlp": [_p, _c_int, _c_int, _p, _c_int, _p, _c_int, _p, _p, _c_int, _p,
                            _p, _c_int, _p, _p, _c_int, _p, _p],
}
_RESTYPES = {"comoe_last_error": ctypes.c_char_p, "comoe_sim_workspace_bytes": _c_long,
             "comoe_ipc_handle_size": _c_int,
             "comoe_predictor_workspace_bytes": _c_long,
             "comoe_gate_route_workspace_bytes": _c_long}

EXPORTED = tuple(_SIGNATURES)

STATUS_BADARG, STATUS_UNSUPPORTED, STATUS_CUDA, STATUS_NODRIVER = -1, -2, -3, -4

_lock = threading.Lock()
_lib = None


class ExtensionMissing(RuntimeError):
    """libcomoe_b200.so is absent or unloadable; there is no CPU path."""


def library_path() -> Path:
    return Path(os.environ.get("COMOE_B200_LIB", _LIB_PATH))


def load():
    """Load (once) and return the ctypes library; raise ExtensionMissing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = library_path()
        if not path.exists():
            raise ExtensionMissing(
                f"{path} not found: build it with `python -m paper_2508_09208_b200.build` "
                "(or __graft_entry__.build()); this package has no CPU fallback")
        try:
            lib = ctypes.CDLL(str(path))
        except OSError as exc:
            raise ExtensionMissing(f"cannot load {path}: {exc}") from exc
        for name, args in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, _c_int)
        ver = lib.comoe_version()
        if ver != ABI_VERSION:
            raise ExtensionMissing(f"ABI version {ver} != expected {ABI_VERSION}; rebuild")
        _lib = lib
    return _lib


def last_error() -> str:
    msg = load().comoe_last_error()
    return msg.decode() if msg else ""


def call(name: str, *args) -> int:
    """Invoke a status-returning entry point and raise on failure."""
    rc = getattr(load(), name)(*args)
    if rc == 0:
        return rc
    msg = last_error()
    if rc in (STATUS_BADARG, STATUS_UNSUPPORTED):
        raise ValueError(f"{name}: {msg}")
    raise RuntimeError(f"{name} failed ({rc}): {msg}")
