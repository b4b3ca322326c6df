"""Edge cases of the device layer against the oracle: ragged and tiny token
counts, empty input, every token on one expert (massive drops), capacity 1,
empty groups, a single expert, and shape errors raised before any launch."""

import math

import numpy as np
import pytest
import torch

from oracle import switch_layer as O

pytestmark = pytest.mark.gpu


def _make(T, d, d_ff, E, cf, seed=0, bias=None, top_k=1):
    from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(max(T, 1), d, generator=g).to(torch.bfloat16)[:T]
    wg = torch.randn(d, E, generator=g) / math.sqrt(d)
    if bias is not None:
        x = x.clone()
        x[:, 0] = 1.0
        wg[0, :] = torch.as_tensor(bias, dtype=torch.float32)
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
    w = (torch.randn(E, numel, generator=g) * 0.02).to(torch.bfloat16)
    pool = ExpertPool(E, numel)
    pool.data[:, :numel].copy_(w.cuda())
    layer = MoELayer(wg.cuda(), pool, d_ff, top_k=top_k, capacity_factor=cf)
    return layer, x.cuda(), wg, w


def _check(layer, x, wg, w, cf, top_k=1):
    T = x.shape[0]
    E = wg.shape[1]
    y = layer.forward(x, want_logits=True)
    torch.cuda.synchronize()
    logits = layer.last.gate.logits.cpu().numpy()
    ref, info = O.layer_forward(x.float().cpu().numpy(), wg.numpy(),
                                [w[e].float().numpy() for e in range(E)], top_k=top_k,
                                norm_topk=top_k == 2, capacity_factor=cf, act="relu",
                                d_ff=layer.d_ff, logits=logits)
    np.testing.assert_array_equal(layer.last.gate.expert_idx.cpu().numpy(), info["expert_idx"])
    np.testing.assert_array_equal(layer.last.perm.token_pos.cpu().numpy(), info["pos"])
    np.testing.assert_array_equal(layer.last.scan.group_kept.cpu().numpy(), info["kept"])
    if np.abs(ref).max() > 0:
        assert O.normwise_error(y.float().cpu().numpy(), ref) < 5e-3
    dropped = np.nonzero((info["pos"] < 0).all(axis=1))[0]
    if len(dropped):
        assert torch.all(y[torch.as_tensor(dropped).cuda()] == 0)
    return info


@pytest.mark.parametrize("T", [1, 2, 127, 128, 129, 255, 257])
def test_tiny_and_ragged_token_counts(T):
    layer, x, wg, w = _make(T, 256, 256, 8, 1.25, seed=T)
    _check(layer, x, wg, w, 1.25)


def test_empty_input():
    layer, x, wg, w = _make(0, 256, 256, 8, 1.25)
    y = layer.forward(torch.empty((0, 256), dtype=torch.bfloat16, device="cuda"))
    assert y.shape == (0, 256)


def test_all_tokens_on_one_expert_massive_drops():
    bias = np.full(16, -30.0)
    bias[5] = 30.0
    layer, x, wg, w = _make(3000, 256, 256, 16, 1.25, seed=2, bias=bias)
    info = _check(layer, x, wg, w, 1.25)
    kept = info["kept"]
    assert kept[5] == O.capacity(3000, 16, 1, 1.25) and kept.sum() == kept[5]
    assert (info["pos"] < 0).sum() == 3000 - kept[5]


def test_capacity_one_and_empty_groups():
    layer, x, wg, w = _make(500, 256, 256, 64, 0.05, seed=3)  # C = ceil(0.05*500/64) = 1
    assert layer.capacity(500) == 1
    info = _check(layer, x, wg, w, 0.05)
    assert (info["kept"] <= 1).all()


def test_top2_capacity_and_single_expert():
    layer, x, wg, w = _make(600, 256, 256, 4, 0.5, seed=4, top_k=2)
    _check(layer, x, wg, w, 0.5, top_k=2)
    layer1, x1, wg1, w1 = _make(300, 256, 256, 1, None, seed=5)
    info = _check(layer1, x1, wg1, w1, None)
    assert (info["expert_idx"] == 0).all()


def test_shape_errors_raise_before_launch():
    from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
    pool = ExpertPool(4, kernels.expert_numel(96, 256, kernels.ACT_RELU))
    with pytest.raises(ValueError):  # d = 96 is not a multiple of 64
        MoELayer(torch.randn(96, 4, device="cuda"), pool, 256)
    layer, x, wg, w = _make(64, 256, 256, 8, 1.25)
    with pytest.raises(ValueError):
        layer.forward(torch.zeros(64, 128, dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(ValueError):
        kernels.gate_padded_experts(129)


@pytest.mark.parametrize("top_k,E", [(1, 16), (2, 16), (1, 64), (2, 64)])
def test_logit_ties_pick_lowest_expert(top_k, E):
    """Exactly equal logits (duplicate router columns; all-zero tokens) go to
    the lowest expert id, the reference's tie rule (aggregation.py:165,193),
    including ties between even and odd expert columns and (E = 64, the
    split epilogue) between the two halves of the experts."""
    layer, x, wg, w = _make(700, 256, 256, E, 2.0, seed=6, top_k=top_k)
    wg = wg.clone()
    x = x.clone()
    x[:, 0] = 1.0
    far = 12 if E == 16 else 40  # E = 64: a duplicate in the other half
    wg[:, far] = wg[:, 5]
    wg[:, 2] = wg[:, 5]
    wg[0, 5] = wg[0, 2] = wg[0, far] = 40.0  # three columns win with equal logits
    x[600:] = 0                               # all-zero tokens: every logit is 0
    from paper_2508_09208_b200 import MoELayer
    layer = MoELayer(wg.cuda(), layer.pool, 256, top_k=top_k, capacity_factor=2.0)
    info = _check(layer, x, wg, w, 2.0, top_k=top_k)  # parity with the oracle on device logits
    idx = info["expert_idx"]
    lg = layer.last.gate.logits.cpu().numpy()
    tied = (lg[:600, 2] == lg[:600, 5]) & (lg[:600, 5] == lg[:600, far])
    assert tied.mean() > 0.9  # identical columns give identical MMA sums
    assert (idx[:600][tied, 0] == 2).all() and (idx[600:, 0] == 0).all()
    if top_k == 2:
        assert (idx[:600][tied, 1] == 5).all() and (idx[600:, 1] == 1).all()
        p = layer.last.gate.gate_prob.cpu().numpy()
        np.testing.assert_allclose(p[:600][tied], 0.5, atol=1e-6)
