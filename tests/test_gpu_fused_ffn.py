"""K3F fused expert FFN (GEMM1 -> ReLU -> GEMM2, H on chip) against the
oracle's per-expert FFN (oracle/switch_layer.expert_ffn, fp64 math with H
rounded to bf16 like the device) and against the two-launch FFN.

Ragged group sizes cover the tile edges of the kernel: empty groups, 1 row,
the 16-row MMA granularity, the 128-token tile boundary and multi-tile
groups; both token sources (the permuted copy and the TMA gather from the
unpermuted rows) and both epilogues (in-place rows, and the top-1 scale +
scatter to the token's row).
"""

import numpy as np
import pytest
import torch

from oracle import switch_layer as O

pytestmark = pytest.mark.gpu

NORMWISE_TOL = 5e-3   # bf16 H and Y
ROW_TOL = 2e-2        # per-row normwise (rows with few accumulations)


def _setup(d, d_ff, sizes, seed=0, n_tokens=None):
    from paper_2508_09208_b200 import ExpertPool, kernels
    g = torch.Generator().manual_seed(seed)
    G = len(sizes)
    rows = int(sum(sizes))
    T = n_tokens or rows + 37
    x = torch.randn(T, d, generator=g).to(torch.bfloat16)
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
    # pool slots in a shuffled order: group g uses slot perm[g]
    n_slots = G + 2
    w = (torch.randn(n_slots, numel, generator=g) * 0.02).to(torch.bfloat16)
    pool = ExpertPool(n_slots, numel)
    pool.data[:, :numel].copy_(w.cuda())
    slot = torch.randperm(n_slots, generator=g)[:G].to(torch.int32)
    # the permuted order: a random subset of token ids (distinct)
    row_token = torch.randperm(T, generator=g)[:rows].to(torch.int32)
    base = torch.tensor(np.concatenate([[0], np.cumsum(sizes)[:-1]]), dtype=torch.int32)
    prob = torch.rand(rows, generator=g) * 0.9 + 0.1
    return dict(x=x, w=w, pool=pool, slot=slot, row_token=row_token, base=base,
                sizes=torch.tensor(sizes, dtype=torch.int32), prob=prob, T=T, G=G, rows=rows)


def _oracle_rows(s, d, d_ff):
    xs = s["x"].float().numpy()[s["row_token"].numpy()]
    ref = np.zeros((s["rows"], d))
    for g in range(s["G"]):
        lo, n = int(s["base"][g]), int(s["sizes"][g])
        if n == 0:
            continue
        w_in, w_out = O.split_expert(s["w"][int(s["slot"][g])].float().numpy(), d, d_ff, "relu")
        ref[lo:lo + n] = O.expert_ffn(xs[lo:lo + n], w_in, w_out, "relu", round_h=True)
    return ref


SIZES = [0, 1, 15, 16, 17, 64, 127, 128, 129, 255, 300, 513, 8, 0, 96]


@pytest.mark.parametrize("d,d_ff", [(768, 3072), (256, 512), (512, 768)])
@pytest.mark.parametrize("gather", [False, True])
def test_fused_ffn_rows_match_oracle(d, d_ff, gather):
    from paper_2508_09208_b200 import kernels
    if not kernels.fused_ffn_supported(d, d_ff, kernels.ACT_RELU, len(SIZES)):
        pytest.skip("shape not supported by the fused FFN")
    s = _setup(d, d_ff, SIZES, seed=d + d_ff)
    dev = "cuda"
    x = s["x"].to(dev)
    rt = s["row_token"].to(dev)
    src = x if gather else x[rt.long()].contiguous()
    out = torch.full((s["rows"], d), float("nan"), dtype=torch.bfloat16, device=dev)
    kernels.fused_ffn(src, s["pool"].data, d_ff, s["sizes"].to(dev), s["base"].to(dev),
                      s["slot"].to(dev), out, gather_rows=rt if gather else None)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    ref = _oracle_rows(s, d, d_ff)
    assert np.isfinite(got).all()
    assert O.normwise_error(got, ref) < NORMWISE_TOL
    for r in range(0, s["rows"], 7):  # spot rows: every row's own error is small too
        assert O.normwise_error(got[r], ref[r]) < ROW_TOL


def test_fused_ffn_scatter_epilogue_and_untouched_rows():
    """Top-1 fused combine: out[row_token[r]] = prob[r] * FFN(row r); token
    rows nobody routes to are left untouched."""
    from paper_2508_09208_b200 import kernels
    d, d_ff = 768, 3072
    if not kernels.fused_ffn_supported(d, d_ff, kernels.ACT_RELU, len(SIZES)):
        pytest.skip("shape not supported by the fused FFN")
    s = _setup(d, d_ff, SIZES, seed=7)
    dev = "cuda"
    x, rt, pr = s["x"].to(dev), s["row_token"].to(dev), s["prob"].to(dev)
    out = torch.full((s["T"], d), 3.0, dtype=torch.bfloat16, device=dev)
    kernels.fused_ffn(x, s["pool"].data, d_ff, s["sizes"].to(dev), s["base"].to(dev),
                      s["slot"].to(dev), out, gather_rows=rt, row_token=rt, row_prob=pr)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    ref_rows = _oracle_rows(s, d, d_ff) * s["prob"].numpy()[:, None]
    tok = s["row_token"].numpy()
    assert O.normwise_error(got[tok], ref_rows) < NORMWISE_TOL
    untouched = np.setdiff1d(np.arange(s["T"]), tok)
    assert (got[untouched] == 3.0).all()


def test_fused_matches_two_launch_ffn():
    """The fused kernel and GEMM1 -> HBM -> GEMM2 accumulate in the same k
    order; their outputs agree to bf16 rounding."""
    from paper_2508_09208_b200 import kernels
    d, d_ff = 768, 3072
    sizes = [200, 0, 640, 17, 128, 333]
    if not kernels.fused_ffn_supported(d, d_ff, kernels.ACT_RELU, len(sizes)):
        pytest.skip("shape not supported by the fused FFN")
    s = _setup(d, d_ff, sizes, seed=3)
    dev = "cuda"
    xp = s["x"].to(dev)[s["row_token"].to(dev).long()].contiguous()
    args = (s["sizes"].to(dev), s["base"].to(dev), s["slot"].to(dev))
    y1 = torch.empty((s["rows"], d), dtype=torch.bfloat16, device=dev)
    kernels.fused_ffn(xp, s["pool"].data, d_ff, *args, y1)
    h = torch.empty((s["rows"], d_ff), dtype=torch.bfloat16, device=dev)
    y2 = torch.empty_like(y1)
    kernels.grouped_gemm(xp, s["pool"].data, 0, d_ff, *args, kernels.EPI_RELU, h)
    kernels.grouped_gemm(h, s["pool"].data, d_ff * d, d, *args, kernels.EPI_STORE, y2)
    torch.cuda.synchronize()
    a, b = y1.float().cpu().numpy(), y2.float().cpu().numpy()
    assert O.normwise_error(a, b) < 1e-3
    frac_equal = float((a == b).mean())
    assert frac_equal > 0.9, frac_equal


def test_fused_ffn_rejects_unsupported_shapes():
    from paper_2508_09208_b200 import kernels
    assert not kernels.fused_ffn_supported(1024, 3072, kernels.ACT_RELU, 8)   # TMEM: d <= 768
    assert not kernels.fused_ffn_supported(768, 3072, kernels.ACT_SWIGLU, 8)  # ReLU only
    assert not kernels.fused_ffn_supported(768, 3000, kernels.ACT_RELU, 8)
    assert not kernels.fused_ffn_supported(768, 3072, kernels.ACT_RELU, 257)
    s = _setup(256, 512, [4, 4])
    out = torch.empty((8, 1024), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        kernels.fused_ffn(torch.zeros((8, 1024), dtype=torch.bfloat16, device="cuda"),
                          s["pool"].data, 512, s["sizes"].cuda(), s["base"].cuda(),
                          s["slot"].cuda(), out)
