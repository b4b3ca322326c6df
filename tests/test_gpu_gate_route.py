"""The folded router (comoe_gate_route: gate + capacity scan in one launch,
decoupled look-back over per-tile group histograms) against the two-launch
path (comoe_gate_topk + comoe_route_scan) and the oracle's stream-order
dispatch: every table bit-identical, across ragged token counts, top-1 and
top-2, merged variants, capacity drops, repeated launches (the device-side
epoch advances per launch) and CUDA-graph replays of new inputs."""

import math

import numpy as np
import pytest
import torch

from oracle import switch_layer as O

pytestmark = pytest.mark.gpu


def _inputs(T, d, E, seed, skew=0.0):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(T, d, generator=g).to(torch.bfloat16)
    wg = torch.randn(d, E, generator=g) / math.sqrt(d)
    if skew:
        x[:, 0] = 1.0
        wg[0, :] = -skew * torch.arange(E, dtype=torch.float32) / E
    return x.cuda(), wg.cuda()


def _both(x, wg, E, top_k, cf, slot_map=None, G=None):
    from paper_2508_09208_b200 import kernels
    T = x.shape[0]
    G = E if G is None else G
    split = kernels.gate_prepare(wg)
    C = kernels.capacity_for(T, G, top_k, cf)
    sm = None if slot_map is None else torch.tensor(slot_map, dtype=torch.int32, device="cuda")
    g2 = kernels.gate_topk(x, split, E, top_k, top_k == 2, slot_map=sm, n_groups=G)
    s2 = kernels.route_scan(g2.tile_hist, C)
    ws = kernels.gate_route_workspace(T, top_k, G, x.device)
    g1, s1 = kernels.gate_route(x, split, E, top_k, top_k == 2, C, ws, slot_map=sm, n_groups=G)
    torch.cuda.synchronize()
    return (g1, s1), (g2, s2), C, ws, split, sm


def _same(a, b):
    (g1, s1), (g2, s2) = a, b
    for f in ("expert_idx", "group_idx", "gate_prob", "local_rank"):
        assert torch.equal(getattr(g1, f), getattr(g2, f)), f
    for f in ("tile_offset", "group_count", "group_kept", "group_base"):
        assert torch.equal(getattr(s1, f), getattr(s2, f)), f


@pytest.mark.parametrize("T,E,top_k,cf", [
    (1, 8, 1, 1.25), (129, 8, 1, 1.25), (1000, 16, 1, 1.0), (4096, 64, 1, 1.25),
    (3000, 128, 1, 1.25), (65536, 128, 1, 1.25), (777, 32, 2, 1.25), (8192, 8, 2, 1.0),
    (5000, 128, 2, 2.0),
])
def test_folded_route_matches_two_launch(T, E, top_k, cf):
    x, wg = _inputs(T, 256 if T < 65536 else 768, E, seed=T + E)
    a, b, C, *_ = _both(x, wg, E, top_k, cf)
    _same(a, b)
    # and the oracle's stream-order dispatch on the same groups
    g = a[0].group_idx.cpu().numpy()
    disp = O.dispatch_fast(g, E, C)
    np.testing.assert_array_equal(a[1].group_count.cpu().numpy(), disp["count"])
    np.testing.assert_array_equal(a[1].group_kept.cpu().numpy(), disp["kept"])
    np.testing.assert_array_equal(a[1].group_base.cpu().numpy(), disp["base"])


def test_folded_route_merged_variant_and_drops():
    E, G = 64, 20
    rng = np.random.default_rng(3)
    slot_map = rng.integers(0, G, size=E).tolist()
    slot_map[:G] = list(range(G))
    x, wg = _inputs(6000, 256, E, seed=9, skew=4.0)
    a, b, C, *_ = _both(x, wg, E, 2, 0.5, slot_map=slot_map, G=G)
    _same(a, b)
    assert (a[1].group_count > a[1].group_kept).any()  # capacity drops happened


def test_folded_route_epochs_and_graph_replay():
    """The workspace is reused launch after launch (eager, then as a CUDA
    graph over new inputs) without a reset."""
    from paper_2508_09208_b200 import kernels
    E, T, top_k = 128, 20000, 1
    x, wg = _inputs(T, 256, E, seed=1)
    a, b, C, ws, split, sm = _both(x, wg, E, top_k, 1.25)
    _same(a, b)
    g1, s1 = a
    for it in range(3):
        x.copy_(_inputs(T, 256, E, seed=100 + it, skew=float(it))[0])
        kernels.gate_route(x, split, E, top_k, False, C, ws, out=g1, scan=s1)
        g2 = kernels.gate_topk(x, split, E, top_k, False)
        s2 = kernels.route_scan(g2.tile_hist, C)
        torch.cuda.synchronize()
        _same((g1, s1), (g2, s2))
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph):
            kernels.gate_route(x, split, E, top_k, False, C, ws, out=g1, scan=s1)
    torch.cuda.current_stream().wait_stream(side)
    for it in range(4):
        x.copy_(_inputs(T, 256, E, seed=200 + it, skew=2.0 * it)[0])
        graph.replay()
        g2 = kernels.gate_topk(x, split, E, top_k, False)
        s2 = kernels.route_scan(g2.tile_hist, C)
        torch.cuda.synchronize()
        _same((g1, s1), (g2, s2))


def test_gate_route_workspace_checked():
    from paper_2508_09208_b200 import kernels
    x, wg = _inputs(1024, 256, 8, seed=0)
    split = kernels.gate_prepare(wg)
    small = torch.zeros(4, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError):
        kernels.gate_route(x, split, 8, 1, False, 160, small)


@pytest.mark.parametrize("T,top_k,d,cf", [(65536, 1, 768, 1.25), (3000, 1, 512, 1.25),
                                          (5000, 2, 768, 2.0), (1, 1, 768, 1.25)])
def test_router_in_tmem_gate(T, top_k, d, cf):
    """The opt-in router-in-TMEM gate (gate_tm.cuh, E = 128) against the
    oracle on its own device logits (routing, probabilities, stream-order
    dispatch), and its logits against the default pair gate's (the two
    kernels accumulate x.hi and x.mid in transposed MMA shapes)."""
    from paper_2508_09208_b200 import _lib, kernels
    E = 128
    x, wg = _inputs(T, d, E, seed=T + d)
    split = kernels.gate_prepare(wg)
    C = kernels.capacity_for(T, E, top_k, cf)
    out = []
    try:
        for tm in (0, 1):
            _lib.call("comoe_debug_set_gate_tm", tm)
            ws = kernels.gate_route_workspace(T, top_k, E, x.device)
            g, s = kernels.gate_route(x, split, E, top_k, top_k == 2, C, ws, n_groups=E,
                                      want_logits=True)
            torch.cuda.synchronize()
            out.append((g, s))
    finally:
        _lib.call("comoe_debug_set_gate_tm", -1)
    (g0, _), (g1, s1) = out
    torch.testing.assert_close(g1.logits, g0.logits, rtol=0, atol=2e-6)
    idx, group, prob = O.topk_route(g1.logits.cpu().numpy(), top_k, top_k == 2)
    np.testing.assert_array_equal(g1.expert_idx.cpu().numpy(), idx)
    np.testing.assert_array_equal(g1.group_idx.cpu().numpy(), group)
    np.testing.assert_allclose(g1.gate_prob.cpu().numpy(), prob, rtol=2e-5, atol=1e-7)
    disp = O.dispatch_fast(group, E, C)
    np.testing.assert_array_equal(s1.group_count.cpu().numpy(), disp["count"])
    np.testing.assert_array_equal(s1.group_kept.cpu().numpy(), disp["kept"])
    np.testing.assert_array_equal(s1.group_base.cpu().numpy(), disp["base"])
    # stream-order rank = the tile's offset for the group + the in-tile rank
    lr = g1.local_rank.cpu().numpy()
    to = s1.tile_offset.cpu().numpy()  # [k][tiles][G]
    tok = np.arange(T)
    for j in range(top_k):
        m = group[:, j] >= 0
        got = to[j, tok[m] // 128, group[m, j]] + lr[m, j]
        np.testing.assert_array_equal(got, disp["rank"][m, j])
