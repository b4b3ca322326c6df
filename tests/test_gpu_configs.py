"""BASELINE configs other than C2 at their full shapes, against the oracle.

C1: Switch-Base-8 layer (d 768, d_ff 3072, E 8, top-1) on 4,096 tokens,
    merged 8 -> 4 by the device fuse_model (similarity, grouping, K5 merge
    into pool slots): merged weights within the bf16 merge bar of the fp64
    reference merge (oracle/merge.py, bit-exact to the reference's
    merge_group), routing through the slot map bit-exact given the device
    logits, output within the bf16 bar of the oracle forward.
C5: Mixtral-8x7B layer (d 4096, d_ff 14336, E 8, top-2 SwiGLU,
    renormalised) on 512 tokens, original and merged 8 -> 4.
"""

import math

import numpy as np
import pytest
import torch

from oracle import merge as M
from oracle import switch_layer as O

pytestmark = pytest.mark.gpu

NORMWISE_TOL = 5e-3


def _np(t):
    return t.detach().float().cpu().numpy()


def _setup(T, d, d_ff, E, act, extra_slots, seed):
    from paper_2508_09208_b200 import ExpertPool, kernels
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(seed)
    x = torch.randn(T, d, device=dev, generator=g).to(torch.bfloat16)
    wg = torch.randn(d, E, device=dev, generator=g) / math.sqrt(d)
    a = kernels.ACT_SWIGLU if act == "swiglu" else kernels.ACT_RELU
    numel = kernels.expert_numel(d, d_ff, a)
    pool = ExpertPool(E + extra_slots, numel, device=dev)
    for s in range(E):
        pool.view(s).normal_(0.0, 0.02, generator=g)
    for s in range(E):  # shared structure: grouping is non-trivial
        pool.view(s).add_(pool.view(s % max(1, E // 2)), alpha=0.5)
    for _ in range(E):
        pool.alloc()
    return x, wg, pool, numel


def _fuse(layer, pool, x, E, numel, ratio, calib_kind):
    from paper_2508_09208_b200 import aggregation as A
    from paper_2508_09208_b200.moe import (Expert, MoeModel, MoeModelSpec, make_calibration,
                                           stats_from_routing)
    r = layer.route(x)
    stats = stats_from_routing({1: r.gate.expert_idx}, E)
    spec = MoeModelSpec(total_layers=1, encoder_moe_layers=(1,), decoder_moe_layers=(),
                        experts_per_layer=E, expert_size_bytes=float(pool.slot_bytes),
                        top_k=layer.top_k, expert_param_dim=numel)
    model = MoeModel(spec, {(1, s): Expert(1, s, pool.view(s), float(pool.slot_bytes))
                            for s in range(E)})
    if calib_kind == "cosine":
        from paper_2508_09208_b200.moe import cosine_only_calibration
        calib, alpha = cosine_only_calibration(), 1.0
    else:
        calib, alpha = make_calibration(numel, 8, 7, 8), 0.5
    var = A.fuse_model(model, stats, A.FusionConfig(mode="fixed", r=ratio), alpha, calib,
                       pool=pool)
    return var, stats


def _check_merged(var, stats, pool, E):
    """Every merged expert vs bf16(fp64 merge_group of the bf16 members)."""
    freqs = stats.freqs(1)
    groups = {}
    for s, p in var.slot_map[1].items():
        groups.setdefault(p, []).append(s)
    for p, members in groups.items():
        got = var.retained[1][p].params
        if len(members) == 1:
            assert got.data_ptr() == pool.view(p).data_ptr()  # singleton aliases its principal
            continue
        slots = [p] + sorted(m for m in members if m != p)
        V = [pool.view(s).double().cpu().numpy() for s in slots]
        ref = M.merge_params(V, np.asarray([freqs[s] for s in slots]))
        refb = O.bf16_round(ref.astype(np.float32)).astype(np.float64)
        g64 = got.double().cpu().numpy()
        bound = np.abs(refb) * 2.0 ** -7 + 2.0 ** -24 * max(np.abs(v).max() for v in V)
        assert np.all(np.abs(g64 - refb) <= bound + 1e-30)


def _oracle_forward(layer, x, wg, d, d_ff, act, top_k, norm, cf, logits):
    """Oracle forward over the layer's current groups (fp32 BLAS, bf16 H),
    per-group weights read back from the pool slots the device uses."""
    slots = layer.group_slot.cpu().tolist()
    n1 = 2 * d_ff if act == "swiglu" else d_ff
    w_in, w_out = [], []
    for s in slots:
        v = layer.pool.view(s).float().cpu().numpy()
        w_in.append(v[:n1 * d].reshape(n1, d))
        w_out.append(v[n1 * d:n1 * d + d * d_ff].reshape(d, d_ff))
    return O.layer_forward_fast(_np(x), _np(wg), w_in, w_out, top_k, norm, cf,
                                slot_map=layer.slot_map.cpu().numpy(), act=act, logits=logits,
                                round_h=True)


def _check(layer, x, wg, d, d_ff, act, top_k, norm, cf):
    y = layer.forward(x, want_logits=True)
    torch.cuda.synchronize()
    logits = layer.last.gate.logits.cpu().numpy()
    ref, info = _oracle_forward(layer, x, wg, d, d_ff, act, top_k, norm, cf, logits)
    r = layer.last
    np.testing.assert_array_equal(r.gate.expert_idx.cpu().numpy(), info["expert_idx"])
    np.testing.assert_array_equal(r.gate.group_idx.cpu().numpy(), info["group_idx"])
    np.testing.assert_array_equal(r.scan.group_kept.cpu().numpy(), info["kept"])
    np.testing.assert_array_equal(r.perm.token_pos.cpu().numpy(), info["pos"])
    assert O.normwise_error(_np(y), ref) < NORMWISE_TOL


def test_c1_sb8_merged_8_to_4_full_shape():
    T, d, d_ff, E = 4096, 768, 3072, 8
    from paper_2508_09208_b200 import MoELayer
    x, wg, pool, numel = _setup(T, d, d_ff, E, "relu", 4, seed=11)
    layer = MoELayer(wg, pool, d_ff, act="relu", top_k=1, capacity_factor=1.25)
    _check(layer, x, wg, d, d_ff, "relu", 1, False, 1.25)           # original 8
    var, stats = _fuse(layer, pool, x, E, numel, 0.5, "probes")
    assert len(var.retained[1]) == 4
    _check_merged(var, stats, pool, E)
    layer.use_variant(var, 1)
    assert layer.G == 4
    _check(layer, x, wg, d, d_ff, "relu", 1, False, 1.25)           # merged 4


def test_c5_mixtral_full_shape_top2_swiglu():
    T, d, d_ff, E = 512, 4096, 14336, 8
    from paper_2508_09208_b200 import MoELayer
    x, wg, pool, numel = _setup(T, d, d_ff, E, "swiglu", 4, seed=12)
    layer = MoELayer(wg, pool, d_ff, act="swiglu", top_k=2, capacity_factor=1.25)
    assert layer.norm_topk
    _check(layer, x, wg, d, d_ff, "swiglu", 2, True, 1.25)          # original 8
    var, stats = _fuse(layer, pool, x, E, numel, 0.5, "cosine")
    _check_merged(var, stats, pool, E)
    layer.use_variant(var, 1)
    _check(layer, x, wg, d, d_ff, "swiglu", 2, True, 1.25)          # merged 4
