"""The C-ABI library loads without a GPU and exports every symbol that
include/comoe_b200.h declares; the product path has no CPU fallback."""

import re
from pathlib import Path

import pytest

from conftest import ROOT


def _declared():
    text = (ROOT / "include" / "comoe_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|long|const char\*)\s+(comoe_\w+)\s*\(", text, re.M)))


def test_header_declares_expected_entry_points():
    names = _declared()
    for n in ("comoe_gate_topk", "comoe_permute", "comoe_grouped_ffn", "comoe_combine",
              "comoe_merge", "comoe_sim_contract", "comoe_predictor_mlp", "comoe_version"):
        assert n in names


def test_library_exports_all_declared_symbols():
    from paper_2508_09208_b200 import _lib
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(_lib.EXPORTED)
    assert lib.comoe_version() == _lib.ABI_VERSION == 2
    # fused FFN shape gate (host-side; no device needed)
    assert lib.comoe_fused_ffn_supported(768, 3072, 0, 128) == 1
    assert lib.comoe_fused_ffn_supported(1024, 3072, 0, 128) == 0   # Y + H exceed TMEM
    assert lib.comoe_fused_ffn_supported(4096, 14336, 1, 8) == 0    # SwiGLU: two launches
    assert lib.comoe_fused_ffn_enabled() in (0, 1)                  # opt-in: COMOE_FUSED_FFN=1
    assert lib.comoe_gate_padded_experts(8) == 16
    assert lib.comoe_gate_padded_experts(128) == 128
    assert lib.comoe_gate_padded_experts(129) == -1
    assert lib.comoe_gate_num_tiles(129) == 2


def test_library_rejects_bad_arguments_without_device():
    import ctypes
    from paper_2508_09208_b200 import _lib
    with pytest.raises(ValueError, match="null"):
        _lib.call("comoe_merge", 0, None, None, None, None, None, 1, 1, 8, None)
    with pytest.raises(ValueError, match="top_k"):
        _lib.call("comoe_gate_topk", ctypes.c_void_p(16), 128, 64, ctypes.c_void_p(16), 8, 3, 0,
                  None, 8, None, ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.c_void_p(16),
                  ctypes.c_void_p(16), ctypes.c_void_p(16), None)


def test_no_cpu_fallback():
    import torch
    from paper_2508_09208_b200 import kernels
    with pytest.raises(ValueError, match="CUDA"):
        kernels.gate_prepare(torch.zeros(64, 8))


def test_product_never_imports_the_oracle():
    for p in (ROOT / "paper_2508_09208_b200").rglob("*.py"):
        src = p.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), p


def test_similarity_row_layout_detection():
    """kernels._shared_stride picks the tcgen05 Gram only for consecutive
    rows of one 16-byte-multiple stride (pool slots, rows of a matrix)."""
    import torch
    from paper_2508_09208_b200 import kernels
    P = torch.zeros(6, 1024, dtype=torch.bfloat16)
    base, stride = kernels._shared_stride([P[i] for i in range(6)])
    assert base == P.data_ptr() and stride == 1024
    pool = torch.zeros(8, 1536, dtype=torch.bfloat16)  # slot stride > row length
    assert kernels._shared_stride([pool[i, :1024] for i in range(2, 6)])[1] == 1536
    assert kernels._shared_stride([P[i] for i in (0, 2, 1)]) is None   # out of order
    assert kernels._shared_stride([P[i] for i in (0, 2, 4)])[1] == 2048  # every other row
    Q = torch.zeros(4, 1028, dtype=torch.bfloat16)  # 2056-byte stride: not 16-byte aligned
    assert kernels._shared_stride([Q[i] for i in range(4)]) is None
