"""Device checks of SURVEY §8(a) rows that round 1 left untested:
a3  the device activation histogram (comoe_expert_histogram ->
    moe.stats_from_routing) equals the reference's collect_stats
    (moe.py:250-262) on reference-identical traces (tests/golden/traces.json);
a21 the device substitution path: a miss served from the most similar
    resident expert's slot (correct_misprediction, offload.py:525-546 ->
    ExpertCache.serve) computes exactly the forward whose group uses the
    substitute's weights;
K3  comoe_grouped_ffn (the two-launch FFN entry point) equals its two
    comoe_grouped_gemm launches bit for bit.
"""

import json
import math

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

TRACES = json.loads((GOLDEN / "traces.json").read_text())


@pytest.mark.parametrize("c", TRACES, ids=lambda c: f"E{c['E']}k{c['K']}")
def test_device_histogram_matches_reference_collect_stats(c):
    from paper_2508_09208_b200 import kernels
    from paper_2508_09208_b200.moe import stats_from_routing
    E, K = c["E"], c["K"]
    layers = [1, 3, 5]   # the fixture spec's MoE layers (encoder 1, 3; decoder 5)
    idx = {l: torch.tensor([tok[i] for tok in c["experts"]], dtype=torch.int32).reshape(-1, K)
           .cuda() for i, l in enumerate(layers)}
    st = stats_from_routing(idx, E)
    for l in layers:
        ref = np.asarray(c["collect_stats"]["counts"][str(l)])
        np.testing.assert_array_equal(st.counts[l], ref)
        assert st.totals[l] == c["collect_stats"]["totals"][str(l)]
        h = kernels.expert_histogram(idx[l], E).cpu().numpy()
        np.testing.assert_array_equal(h, ref)


def test_substitution_serves_misses_from_the_substitute_slot():
    from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
    from paper_2508_09208_b200.cache import CachedMoELayer, ExpertCache
    from paper_2508_09208_b200.offload import OffloadPolicy
    T, d, d_ff, E = 96, 256, 512, 16
    g = torch.Generator().manual_seed(8)
    x = torch.randn(T, d, generator=g).to(torch.bfloat16).cuda()
    wg = torch.randn(d, E, generator=g) / math.sqrt(d)
    x[:, 0] = 1.0
    wg[0, :] = torch.as_tensor(-1.0 * np.log(np.arange(1, E + 1)), dtype=torch.float32)
    wg = wg.cuda()
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
    w = (torch.randn(E, numel, generator=g) * 0.02).to(torch.bfloat16)
    sim = lambda a, b: 1.0 - abs(a[1] - b[1]) / E            # nearest id = most similar
    cache = ExpertCache(w.contiguous().pin_memory(), layer=1, n_slots=6, workspace_slots=2,
                        policy=OffloadPolicy(substitution_sim_min=0.5), substitution=True,
                        similarity=sim, priorities={}, priority_threshold=1.0)
    layer = CachedMoELayer(wg, cache, d_ff, capacity_factor=2.0)
    y = layer.forward(x)
    torch.cuda.synchronize()
    subs = {e[1][1]: e[2][1] for e in cache.stats.events if e[0] == "substitute"}
    assert subs and cache.stats.substitutions == len(subs)
    assert all(abs(a - b) <= E // 2 for a, b in subs.items())
    # reference: every expert resident; substituted groups use the substitute's weights
    pool = ExpertPool(E, numel)
    pool.data[:, :numel].copy_(w.cuda())
    ref = MoELayer(wg, pool, d_ff, capacity_factor=2.0)
    ref.set_variant(list(range(E)), [subs.get(e, e) for e in range(E)])
    assert torch.equal(y, ref.forward(x))
    cache.check()


def test_grouped_ffn_entry_point_equals_its_two_gemms():
    from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
    T, d, d_ff, E = 2048, 256, 512, 8
    g = torch.Generator().manual_seed(2)
    x = torch.randn(T, d, generator=g).to(torch.bfloat16).cuda()
    wg = (torch.randn(d, E, generator=g) / math.sqrt(d)).cuda()
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
    pool = ExpertPool(E, numel)
    pool.data[:, :numel].copy_((torch.randn(E, numel, generator=g) * 0.02).to(torch.bfloat16).cuda())
    layer = MoELayer(wg, pool, d_ff, capacity_factor=1.25)
    y_layer = layer.forward(x).clone()
    r = layer.last
    rows = r.perm.x_perm.shape[0]
    h = torch.empty((rows, d_ff), dtype=torch.bfloat16, device="cuda")
    args = (r.scan.group_kept, r.scan.group_base, layer.group_slot)
    y1 = torch.zeros((T, d), dtype=torch.bfloat16, device="cuda")
    kernels.grouped_ffn(r.perm.x_perm, pool.data, d_ff, kernels.ACT_RELU, *args, h, y1,
                        row_token=r.perm.row_token, row_prob=r.perm.row_prob)
    y2 = torch.zeros_like(y1)
    h2 = torch.empty_like(h)
    kernels.grouped_gemm(r.perm.x_perm, pool.data, 0, d_ff, *args, kernels.EPI_RELU, h2)
    kernels.grouped_gemm(h2, pool.data, d_ff * d, d, *args, kernels.EPI_SCALE_SCATTER, y2,
                         row_token=r.perm.row_token, row_prob=r.perm.row_prob)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    kept = r.perm.token_pos[:, 0] >= 0
    assert torch.equal(y1[kept], y_layer[kept])
