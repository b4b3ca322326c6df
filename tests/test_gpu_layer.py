"""Device parity of the MoE-layer hot path against the CPU oracle.

Routing (indices, group remap, tile ranks, histograms, capacity scan,
permutation order) must be bit-exact given the device's fp32 logits; logits
within fp32 accumulation error of the fp64 oracle; layer outputs within the
bf16 normwise tolerance below.
"""

import math

import numpy as np
import pytest
import torch

from oracle import switch_layer as O

pytestmark = pytest.mark.gpu

NORMWISE_TOL = 5e-3       # bf16 storage of H and Y
LOGIT_ABS_TOL = 2e-5      # fp32-faithful split router vs fp64 oracle, |logit| ~ 1..5
PROB_TOL = 2e-6


def _layer_inputs(T, d, d_ff, E, act, seed=0, dev="cuda"):
    from paper_2508_09208_b200 import kernels
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(T, d, generator=g).to(torch.bfloat16)
    wg = torch.randn(d, E, generator=g) / math.sqrt(d)
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_SWIGLU if act == "swiglu" else kernels.ACT_RELU)
    w = (torch.randn(E, numel, generator=g) * 0.02).to(torch.bfloat16)
    return x.to(dev), wg.to(dev), w


def _build(T, d, d_ff, E, act, top_k, cf, seed=0):
    from paper_2508_09208_b200 import ExpertPool, MoELayer
    x, wg, w = _layer_inputs(T, d, d_ff, E, act, seed)
    pool = ExpertPool(E, w.shape[1])
    for s in range(E):
        pool.view(s).copy_(w[s].cuda())
    layer = MoELayer(wg, pool, d_ff, act=act, top_k=top_k, capacity_factor=cf)
    return layer, x, wg, w


def _np(t):
    return t.detach().float().cpu().numpy() if t.dtype == torch.bfloat16 else t.detach().cpu().numpy()


def _check_routing(layer, x, wg, info, T):
    r = layer.last
    g = r.gate
    # logits vs fp64 oracle
    ref_logits = O.gate_logits(_np(x), _np(wg)).astype(np.float64)
    got_logits = g.logits.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(got_logits - ref_logits)) < LOGIT_ABS_TOL
    # bit-exact routing given identical logits
    np.testing.assert_array_equal(g.expert_idx.cpu().numpy(), info["expert_idx"])
    np.testing.assert_array_equal(g.group_idx.cpu().numpy(), info["group_idx"])
    gp = g.gate_prob.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(gp - info["prob"])) < PROB_TOL
    np.testing.assert_array_equal(g.local_rank.cpu().numpy(), info["local_rank"])
    s = r.scan
    # stream-order tile prefixes (first choices in token order, then second
    # choices): written by the gate's folded look-back, or by the scan kernel
    # from the histograms (COMOE_GATE_FOLD=0)
    hist = info["tile_hist"].reshape(-1, info["tile_hist"].shape[-1])
    np.testing.assert_array_equal(s.tile_offset.cpu().numpy().reshape(hist.shape),
                                  np.cumsum(hist, axis=0) - hist)
    from paper_2508_09208_b200.layer import _gate_fold
    if not _gate_fold():
        np.testing.assert_array_equal(g.tile_hist.cpu().numpy(), info["tile_hist"])
    np.testing.assert_array_equal(s.group_count.cpu().numpy(), info["count"])
    np.testing.assert_array_equal(s.group_kept.cpu().numpy(), info["kept"])
    np.testing.assert_array_equal(s.group_base.cpu().numpy(), info["base"])
    np.testing.assert_array_equal(r.perm.token_pos.cpu().numpy(), info["pos"])
    rows = int(info["kept"].sum())
    np.testing.assert_array_equal(r.perm.row_token[:rows].cpu().numpy(), info["row_token"])
    # the permuted rows are exact copies of the token rows (when materialised;
    # the ReLU 2-SM path gathers token rows inside the GEMM instead)
    from paper_2508_09208_b200.layer import _gather_enabled
    if not _gather_enabled(layer.act):
        xp = r.perm.x_perm[:rows].cpu()
        assert torch.equal(xp, x.cpu()[torch.as_tensor(info["row_token"])])


@pytest.mark.parametrize("T,d,d_ff,E,cf", [
    (1000, 256, 512, 8, 1.25),      # ragged last tile
    (4096, 256, 512, 16, 1.0),      # drops
    (2048, 768, 3072, 8, 1.25),     # Switch FFN shape (sb8 slice)
    (3000, 256, 256, 128, 1.25),    # E = 128 gate
    (777, 512, 1024, 32, None),     # no capacity limit
])
def test_switch_layer_top1(T, d, d_ff, E, cf):
    layer, x, wg, w = _build(T, d, d_ff, E, "relu", 1, cf)
    y = layer.forward(x, want_logits=True)
    torch.cuda.synchronize()
    logits = layer.last.gate.logits.cpu().numpy()
    ref, info = O.layer_forward(_np(x), _np(wg), [_np(w[e]) for e in range(E)], top_k=1,
                                capacity_factor=cf, act="relu", d_ff=d_ff, logits=logits)
    _check_routing(layer, x, wg, info, T)
    err = O.normwise_error(_np(y), ref)
    assert err < NORMWISE_TOL, err
    dropped = (info["pos"][:, 0] < 0)
    if dropped.any():
        assert torch.all(y[torch.as_tensor(np.nonzero(dropped)[0]).cuda()] == 0)


@pytest.mark.parametrize("T,d,d_ff,E,norm", [
    (1024, 256, 512, 8, True),     # Mixtral semantics (renormalised top-2)
    (1500, 256, 256, 8, False),
])
def test_swiglu_layer_top2(T, d, d_ff, E, norm):
    from paper_2508_09208_b200 import ExpertPool, MoELayer
    x, wg, w = _layer_inputs(T, d, d_ff, E, "swiglu", seed=3)
    pool = ExpertPool(E, w.shape[1])
    pool.data[:, : w.shape[1]].copy_(w.cuda())
    layer = MoELayer(wg, pool, d_ff, act="swiglu", top_k=2, norm_topk=norm, capacity_factor=1.25)
    y = layer.forward(x, want_logits=True)
    torch.cuda.synchronize()
    logits = layer.last.gate.logits.cpu().numpy()
    ref, info = O.layer_forward(_np(x), _np(wg), [_np(w[e]) for e in range(E)], top_k=2,
                                norm_topk=norm, capacity_factor=1.25, act="swiglu", d_ff=d_ff,
                                logits=logits)
    _check_routing(layer, x, wg, info, T)
    assert O.normwise_error(_np(y), ref) < NORMWISE_TOL


def test_swiglu_large_experts_feature_major_order():
    """Experts whose W_in block exceeds 32 MB (d 1024, d_ff 8192: 33.5 MB)
    take the feature-tile-major tile order of the 1-SM GEMM (the Mixtral
    fix); outputs must not change."""
    from paper_2508_09208_b200 import ExpertPool, MoELayer
    T, d, d_ff, E = 512, 1024, 8192, 2
    x, wg, w = _layer_inputs(T, d, d_ff, E, "swiglu", seed=5)
    pool = ExpertPool(E, w.shape[1])
    pool.data[:, : w.shape[1]].copy_(w.cuda())
    layer = MoELayer(wg, pool, d_ff, act="swiglu", top_k=2, norm_topk=True, capacity_factor=1.25)
    y = layer.forward(x, want_logits=True)
    torch.cuda.synchronize()
    logits = layer.last.gate.logits.cpu().numpy()
    ref, info = O.layer_forward(_np(x), _np(wg), [_np(w[e]) for e in range(E)], top_k=2,
                                norm_topk=True, capacity_factor=1.25, act="swiglu", d_ff=d_ff,
                                logits=logits)
    _check_routing(layer, x, wg, info, T)
    assert O.normwise_error(_np(y), ref) < NORMWISE_TOL


def test_relu_large_experts_feature_major_order():
    """2-SM ReLU GEMMs with weight blocks above 32 MB (d 1024, d_ff 16384:
    33.5 MB) take the feature-tile-major order; outputs must not change."""
    T, d, d_ff, E = 640, 1024, 16384, 2
    layer, x, wg, w = _build(T, d, d_ff, E, "relu", 1, 1.25, seed=6)
    y = layer.forward(x, want_logits=True)
    torch.cuda.synchronize()
    logits = layer.last.gate.logits.cpu().numpy()
    ref, info = O.layer_forward(_np(x), _np(wg), [_np(w[e]) for e in range(E)], top_k=1,
                                capacity_factor=1.25, act="relu", d_ff=d_ff, logits=logits)
    _check_routing(layer, x, wg, info, T)
    assert O.normwise_error(_np(y), ref) < NORMWISE_TOL


def test_merged_variant_routing_and_output():
    """8 experts merged into 4 groups: slot remap in the gate, capacity on
    the merged count, FFN on merged pool slots."""
    T, d, d_ff, E = 2048, 256, 512, 8
    layer, x, wg, w = _build(T, d, d_ff, E, "relu", 1, 1.25)
    slot_map = [0, 1, 2, 3, 0, 1, 2, 3]
    merged = torch.stack([(w[g].float() + w[g + 4].float()) * 0.5 for g in range(4)]).to(torch.bfloat16)
    for g in range(4):
        layer.pool.view(g).copy_(merged[g].cuda())
    layer.set_variant(slot_map, [0, 1, 2, 3])
    y = layer.forward(x, want_logits=True)
    torch.cuda.synchronize()
    logits = layer.last.gate.logits.cpu().numpy()
    ref, info = O.layer_forward(_np(x), _np(wg), [_np(merged[g]) for g in range(4)], top_k=1,
                                capacity_factor=1.25, slot_map=slot_map, act="relu", d_ff=d_ff,
                                logits=logits)
    _check_routing(layer, x, wg, info, T)
    assert O.normwise_error(_np(y), ref) < NORMWISE_TOL


def test_forward_is_deterministic():
    layer, x, wg, w = _build(4096, 256, 512, 16, "relu", 1, 1.0)
    y1 = layer.forward(x).clone()
    r1 = layer.last.perm.row_token.clone()
    y2 = layer.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    assert torch.equal(r1, layer.last.perm.row_token)


def test_full_size_c2_sb128():
    """C2 shape (T=65536, E=128, cf=1.25), compared whole:
    * logits within 2e-5 of the fp64 oracle for every token;
    * expert choice, per-group counts / kept / bases, every token's row and
      the full row -> token permutation bit-exact against the oracle's
      vectorised dispatch on the device logits;
    * the whole output within the bf16 bar of the oracle forward (fp32 BLAS,
      H rounded to bf16 like the device), dropped tokens exactly 0."""
    T, d, d_ff, E = 65536, 768, 3072, 128
    from paper_2508_09208_b200 import ExpertPool, MoELayer
    torch.manual_seed(0)
    x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
    wg = torch.randn(d, E, device="cuda") / math.sqrt(d)
    pool = ExpertPool(E, 2 * d * d_ff)
    pool.data.normal_(0, 0.02)
    layer = MoELayer(wg, pool, d_ff, capacity_factor=1.25)
    y = layer.forward(x, want_logits=True)
    torch.cuda.synchronize()
    r = layer.last
    assert r.capacity == 640
    xs, wgs = _np(x), _np(wg)
    logits = r.gate.logits.cpu().numpy()
    ref_logits = O.gate_logits(xs, wgs).astype(np.float64)
    assert np.max(np.abs(logits.astype(np.float64) - ref_logits)) < LOGIT_ABS_TOL
    idx, grp, prob = O.topk_route(logits, 1, False)
    np.testing.assert_array_equal(r.gate.expert_idx.cpu().numpy(), idx)
    assert np.max(np.abs(r.gate.gate_prob.cpu().numpy() - prob)) < PROB_TOL
    disp = O.dispatch_fast(grp, E, 640)
    np.testing.assert_array_equal(r.scan.group_count.cpu().numpy(), disp["count"])
    np.testing.assert_array_equal(r.scan.group_kept.cpu().numpy(), disp["kept"])
    np.testing.assert_array_equal(r.scan.group_base.cpu().numpy(), disp["base"])
    np.testing.assert_array_equal(r.perm.token_pos.cpu().numpy(), disp["pos"])
    rows = int(disp["kept"].sum())
    np.testing.assert_array_equal(r.perm.row_token[:rows].cpu().numpy(), disp["row_token"])
    w = pool.data[:, :2 * d * d_ff].float().cpu().numpy()
    w_in = w[:, :d_ff * d].reshape(E, d_ff, d)
    w_out = w[:, d_ff * d:].reshape(E, d, d_ff)
    del w
    ref, _ = O.layer_forward_fast(xs, wgs, w_in, w_out, 1, False, 1.25, logits=logits,
                                  round_h=True)
    got = _np(y)
    assert O.normwise_error(got, ref) < NORMWISE_TOL
    dropped = disp["pos"][:, 0] < 0
    assert dropped.any() and (got[dropped] == 0).all()


def test_replayed_trace_routing_matches_oracle():
    """A reference-style RoutingTrace replayed through the device layer
    (comoe_route_from_indices): tables and outputs equal the oracle given the
    same expert choices (top-2, with a merge that folds pairs)."""
    from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
    from paper_2508_09208_b200.moe import MoeModelSpec, RoutingGeneratorSpec, generate_routing
    T, d, d_ff, E = 700, 256, 512, 8
    spec = MoeModelSpec(total_layers=2, encoder_moe_layers=(1,), decoder_moe_layers=(),
                        experts_per_layer=E, expert_size_bytes=1.0, top_k=2)
    tr = generate_routing(RoutingGeneratorSpec(skew=1.0, seed=3), spec, T)
    idx = tr.expert_indices(1)
    x, wg, w = _layer_inputs(T, d, d_ff, E, "relu", seed=5)
    pool = ExpertPool(E, w.shape[1])
    pool.data[:, : w.shape[1]].copy_(w.cuda())
    layer = MoELayer(wg, pool, d_ff, act="relu", top_k=2, capacity_factor=1.0)
    slot_map = [0, 1, 2, 3, 0, 1, 2, 3]
    layer.set_variant(slot_map, [0, 1, 2, 3])
    probs = np.full((T, 2), 0.5, np.float32)
    y = layer.forward(x, routing=(torch.as_tensor(idx).cuda(), torch.as_tensor(probs).cuda()))
    torch.cuda.synchronize()
    g = layer.last.gate
    group = np.asarray(slot_map)[idx]
    pr = probs.astype(np.float64).copy()
    same = group[:, 1] == group[:, 0]
    pr[same, 0] += pr[same, 1]
    pr[same, 1] = 0
    group[same, 1] = -1
    C = O.capacity(T, 4, 2, 1.0)
    disp = O.dispatch(group, 4, C)
    np.testing.assert_array_equal(g.group_idx.cpu().numpy(), group)
    np.testing.assert_array_equal(g.local_rank.cpu().numpy(), disp["local_rank"])
    np.testing.assert_array_equal(layer.last.perm.token_pos.cpu().numpy(), disp["pos"])
    xs = _np(x)
    ref = np.zeros((T, d))
    for t in range(T):
        for j in range(2):
            p_ = disp["pos"][t, j]
            if p_ >= 0:
                w_in, w_out = O.split_expert(_np(w[group[t, j]]), d, d_ff, "relu")
                ref[t] += pr[t, j] * O.expert_ffn(xs[t:t + 1], w_in, w_out, "relu")[0]
    assert O.normwise_error(_np(y), ref) < NORMWISE_TOL


def test_gather_gemm1_matches_permuted_copy():
    """The opt-in GEMM1 that gathers token rows with TMA gather4 (index-only
    permute, a_gather = row_token) computes exactly what the permuted-copy
    path computes."""
    from paper_2508_09208_b200 import kernels
    T, d, d_ff, E = 2048, 256, 512, 8
    layer, x, wg, w = _build(T, d, d_ff, E, "relu", 1, 1.25)
    layer.forward(x)
    r = layer.last
    ws = layer._workspace(T)
    h_copy = torch.empty_like(ws["h"])
    h_gather = torch.empty_like(ws["h"])
    kernels.grouped_gemm(r.perm.x_perm, layer.pool.data, 0, d_ff, r.scan.group_kept,
                         r.scan.group_base, layer.group_slot, kernels.EPI_RELU, h_copy)
    kernels.grouped_gemm(x, layer.pool.data, 0, d_ff, r.scan.group_kept, r.scan.group_base,
                         layer.group_slot, kernels.EPI_RELU, h_gather, a_gather=r.perm.row_token)
    torch.cuda.synchronize()
    rows = int(r.scan.group_kept.sum())
    assert torch.equal(h_copy[:rows], h_gather[:rows])
