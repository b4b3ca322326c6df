"""HBM-budgeted expert cache: outputs bit-identical to the all-resident
layer, policy invariants after every forward, prefetch/hit accounting."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _setup(T, d, d_ff, E, n_slots, seed=0, bias=None):
    from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
    from paper_2508_09208_b200.cache import CachedMoELayer, ExpertCache
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(T, d, generator=g).to(torch.bfloat16).cuda()
    wg = (torch.randn(d, E, generator=g) / math.sqrt(d))
    if bias is not None:  # skew routing: add a per-expert logit offset through a constant feature
        x[:, 0] = 1.0
        wg[0, :] = torch.as_tensor(bias, dtype=torch.float32)
    wg = wg.cuda()
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
    w = (torch.randn(E, numel, generator=g) * 0.02).to(torch.bfloat16)
    pool = ExpertPool(E, numel)
    pool.data[:, :numel].copy_(w.cuda())
    ref_layer = MoELayer(wg, pool, d_ff, capacity_factor=1.25)
    cache = ExpertCache(w.contiguous().pin_memory(), layer=1, n_slots=n_slots, workspace_slots=2)
    layer = CachedMoELayer(wg, cache, d_ff, capacity_factor=1.25)
    return layer, ref_layer, cache, x


def test_cached_layer_bit_identical_30pct_cache_waves():
    layer, ref, cache, x = _setup(4096, 256, 512, 32, n_slots=10)
    y_ref = ref.forward(x)
    for _ in range(3):
        y = layer.forward(x)
        torch.cuda.synchronize()
        assert torch.equal(y, y_ref)
    assert cache.stats.waves >= 3 * 4
    assert cache.stats.fetches > 0
    cache.check()


def test_cached_layer_skewed_small_batches_hit_and_prefetch():
    E = 32
    bias = -1.5 * np.log(np.arange(1, E + 1))  # Zipf-like s=1.5 over expert rank
    layer, ref, cache, x = _setup(64, 256, 512, E, n_slots=10, bias=bias)
    y_ref = ref.forward(x)
    y = layer.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref)
    h0 = cache.stats.hits
    y = layer.forward(x)  # same demand again: all hits now
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref)
    assert cache.stats.hits > h0
    # prefetch the next-most-likely experts, then demand them
    probs = np.zeros(E)
    probs[[20, 21]] = 0.9
    chosen = cache.prefetch(probs, theta=0.5)
    assert chosen and all(cache.state.resident(e) for e in chosen)
    assert cache.stats.prefetch_issued == len(chosen)
    cache.check()


def test_cached_stack_predictive_prefetch():
    """Two-layer stack: the K8 predictor on layer 1's routing drives
    prefetches into layer 2's cache; outputs equal the all-resident stack."""
    from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
    from paper_2508_09208_b200.cache import CachedMoELayer, ExpertCache
    from paper_2508_09208_b200.offload import OffloadPolicy, PredictorMLP
    from paper_2508_09208_b200.stack import CachedMoEStack, StackLayer
    T, d, d_ff, E = 256, 256, 512, 16
    g = torch.Generator().manual_seed(9)
    x = torch.randn(T, d, generator=g).to(torch.bfloat16).cuda()
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
    layers, refs = [], []
    for l in range(2):
        wg = (torch.randn(d, E, generator=g) / math.sqrt(d)).cuda()
        w = (torch.randn(E, numel, generator=g) * 0.02).to(torch.bfloat16)
        pool = ExpertPool(E, numel)
        pool.data[:, :numel].copy_(w.cuda())
        refs.append(MoELayer(wg, pool, d_ff, capacity_factor=2.0))
        cache = ExpertCache(w.contiguous().pin_memory(), layer=l + 1, n_slots=6, workspace_slots=1)
        layers.append(StackLayer(l + 1, CachedMoELayer(wg, cache, d_ff, capacity_factor=2.0)))
    rng = np.random.default_rng(0)
    mlp = PredictorMLP(w1=rng.normal(scale=0.5, size=(32, E + 4 + 2)), b1=np.zeros(32),
                       w2=rng.normal(scale=2.0, size=(E, 32)), b2=np.zeros(E),
                       experts_per_layer=E, embed_dim=4, context_dim=2)
    emb = torch.randn(T, 4, dtype=torch.float64, generator=g).cuda()
    ctx = torch.randn(T, 2, dtype=torch.float64, generator=g).cuda()
    stack = CachedMoEStack(layers, predictor=mlp,
                           policy=OffloadPolicy(threshold_mode="constant", theta_base=0.05))
    y = stack.forward(x, emb, ctx)
    h = x
    for ref in refs:
        h = (ref.forward(h).float() + h.float()).to(torch.bfloat16)
    torch.cuda.synchronize()
    assert torch.equal(y, h)
    assert len(stack.prefetch_log) == 1
    for sl in layers:
        sl.layer.cache.check()


def test_activate_variant_cache_for_fused_layer():
    """_activate_variant-style cache for a fused (8 -> 4) variant: the cached
    layer reproduces the all-resident merged layer bit for bit."""
    from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
    from paper_2508_09208_b200 import aggregation as A
    from paper_2508_09208_b200.cache import CachedMoELayer, activate_variant
    from paper_2508_09208_b200.moe import (Expert, MoeModel, MoeModelSpec,
                                           cosine_only_calibration, stats_from_routing)
    T, d, d_ff, E = 2048, 256, 512, 8
    g = torch.Generator().manual_seed(21)
    x = torch.randn(T, d, generator=g).to(torch.bfloat16).cuda()
    wg = (torch.randn(d, E, generator=g) / math.sqrt(d)).cuda()
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
    pool = ExpertPool(E + 4, numel)
    for s in range(E):
        pool.view(pool.alloc()).copy_((torch.randn(numel, generator=g) * 0.02).to(torch.bfloat16).cuda())
    layer = MoELayer(wg, pool, d_ff, capacity_factor=1.25)
    stats = stats_from_routing({1: layer.route(x).gate.expert_idx}, E)
    spec = MoeModelSpec(1, (1,), (), E, float(pool.slot_bytes), 1, numel)
    model = MoeModel(spec, {(1, s): Expert(1, s, pool.view(s), float(pool.slot_bytes)) for s in range(E)})
    var = A.fuse_model(model, stats, A.FusionConfig(mode="fixed", r=0.5), 1.0,
                       cosine_only_calibration(), pool=pool)
    layer.use_variant(var, 1)
    y_ref = layer.forward(x).clone()
    lut, principals = var.group_table(1, E)
    host = torch.stack([var.retained[1][p].params.cpu() for p in principals]).contiguous().pin_memory()
    cache = activate_variant(var, 1, stats, host, budget_bytes=3 * pool.slot_bytes, workspace_slots=1)
    cl = CachedMoELayer(wg, cache, d_ff, capacity_factor=1.25)
    cl.set_groups(lut)
    y = cl.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref)
    assert cache.prio_threshold <= 1.0 and len(cache.priorities) == len(principals)


def test_variant_controller_switches_under_memory_trace():
    """Live variant switching (simulator.py:624-680): a memory trace drops
    below the original model's requirement (forced switch to a fused
    variant) and recovers (hysteresis, then switch back). After every switch
    the cached layer reproduces the all-resident forward of the active
    variant bit for bit."""
    from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
    from paper_2508_09208_b200 import aggregation as A
    from paper_2508_09208_b200.moe import (Expert, MoeModel, MoeModelSpec,
                                           cosine_only_calibration, stats_from_routing)
    from paper_2508_09208_b200.switching import VariantController
    T, d, d_ff, E = 1024, 256, 512, 8
    g = torch.Generator().manual_seed(31)
    x = torch.randn(T, d, generator=g).to(torch.bfloat16).cuda()
    wg = (torch.randn(d, E, generator=g) / math.sqrt(d)).cuda()
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
    pool = ExpertPool(E + 8, numel)
    for s in range(E):
        pool.view(pool.alloc()).copy_((torch.randn(numel, generator=g) * 0.02).to(torch.bfloat16).cuda())
    ref_layer = MoELayer(wg, pool, d_ff, capacity_factor=1.25)
    stats = stats_from_routing({1: ref_layer.route(x).gate.expert_idx}, E)
    eb = float(pool.slot_bytes)
    spec = MoeModelSpec(1, (1,), (), E, eb, 1, numel)
    model = MoeModel(spec, {(1, s): Expert(1, s, pool.view(s), eb) for s in range(E)})
    lib = A.build_library(model, stats, [A.FusionConfig(mode="fixed", r=0.5),
                                         A.FusionConfig(mode="fixed", r=0.25)],
                          1.0, cosine_only_calibration(), pool=pool)
    stores = {}
    for v in lib.variants:
        _, principals = v.group_table(1, E)
        stores[v.variant_id] = {1: torch.stack([v.retained[1][p].params.cpu() for p in principals])
                                .contiguous().pin_memory()}
    ctl = VariantController(lib, stats, stores, {1: (wg, d_ff)}, d_ff,
                            policy=A.SwitchPolicy(lambda_switch=0.5, switch_cost=0.05,
                                                  t_threshold=2.0),
                            reeval_interval=2, required_bytes=lambda v: v.expert_bytes,
                            workspace_slots=1)

    def check():
        ref_layer.use_variant(ctl.variant, 1)
        y_ref = ref_layer.forward(x)
        y = ctl.forward(x, 1)
        torch.cuda.synchronize()
        assert torch.equal(y, y_ref), ctl.variant.variant_id

    big = 10 * eb
    ctl.start(big)
    assert ctl.variant.perf_estimate == max(v.perf_estimate for v in lib.variants)
    check()
    top = ctl.variant.variant_id
    trace = [big, big, 4.5 * eb, 4.5 * eb, 4.5 * eb, 2.5 * eb, 2.5 * eb, big, big, big, big, big]
    switches = []
    for t, m in enumerate(trace, start=1):
        e = ctl.tick(t, m)
        if e is not None:
            switches.append(e)
            check()
    assert any(e.forced for e in switches)  # memory dropped below the active variant
    assert ctl.variant.variant_id == top      # recovered after the hysteresis window
    assert all(e.migrated_bytes > 0 and e.seconds > 0 for e in switches)


def test_activate_variant_pool_never_exceeds_variant_plus_workspace():
    """activate_variant caps the HBM slots at the variant's experts of the
    layer plus the workspace (_resident_budget never exceeds the variant,
    simulator.py:275-286), however large the memory budget."""
    from paper_2508_09208_b200 import aggregation as A
    from paper_2508_09208_b200.cache import activate_variant
    from paper_2508_09208_b200.moe import (ActivationStats, Expert, MoeModel, MoeModelSpec)
    E, numel = 8, 4096
    spec = MoeModelSpec(1, (1,), (), E, float(numel * 2), 1, numel)
    ex = {(1, s): Expert(1, s, torch.zeros(numel, dtype=torch.bfloat16, device="cuda"),
                         float(numel * 2)) for s in range(E)}
    var = A.original_variant(MoeModel(spec, ex), 0.0)
    stats = ActivationStats(counts={1: np.arange(1, E + 1, dtype=float)}, totals={1: 36},
                            experts_per_layer=E)
    host = torch.zeros(E, numel, dtype=torch.bfloat16).pin_memory()
    cache = activate_variant(var, 1, stats, host, budget_bytes=1000.0 * numel * 2,
                             workspace_slots=2)
    assert cache.pool.n_slots <= E + 2
    cache.check()


def test_hits_are_served_in_one_wave():
    """All-hit forwards need no copies: one wave, whatever the free slots."""
    layer, ref, cache, x = _setup(64, 256, 512, 32, n_slots=10,
                                  bias=-2.0 * np.log(np.arange(1, 33)))
    layer.forward(x)                       # warm: demanded experts become resident
    torch.cuda.synchronize()
    w0, f0 = cache.stats.waves, cache.stats.fetches
    y = layer.forward(x)
    torch.cuda.synchronize()
    if cache.stats.fetches == f0:          # every demanded expert was a hit
        assert cache.stats.waves - w0 == 1
    assert torch.equal(y, ref.forward(x))


def test_stack_prefetch_folds_demand_into_a_fused_next_layer():
    """The predictor's per-expert demand for the next layer is folded into
    that layer's group space (fused variant: ids (layer, group)) before
    decide_prefetch; outputs still equal the all-resident stack."""
    from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
    from paper_2508_09208_b200.cache import CachedMoELayer, ExpertCache
    from paper_2508_09208_b200.offload import OffloadPolicy, PredictorMLP
    from paper_2508_09208_b200.stack import CachedMoEStack, StackLayer
    T, d, d_ff, E, G = 256, 256, 512, 16, 8
    g = torch.Generator().manual_seed(19)
    x = torch.randn(T, d, generator=g).to(torch.bfloat16).cuda()
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
    lut = [e % G for e in range(E)]           # next layer: a fused 16 -> 8 variant
    layers, refs = [], []
    for l in range(2):
        wg = (torch.randn(d, E, generator=g) / math.sqrt(d)).cuda()
        n = E if l == 0 else G
        w = (torch.randn(n, numel, generator=g) * 0.02).to(torch.bfloat16)
        pool = ExpertPool(n, numel)
        pool.data[:, :numel].copy_(w.cuda())
        ref = MoELayer(wg, pool, d_ff, capacity_factor=2.0, expert_slots=[0] * E)
        if l == 0:
            ref.set_variant(list(range(E)), list(range(E)))
        cache = ExpertCache(w.contiguous().pin_memory(), layer=l + 1, n_slots=5,
                            workspace_slots=1)
        cl = CachedMoELayer(wg, cache, d_ff, capacity_factor=2.0)
        if l == 1:
            ref.set_variant(lut, list(range(G)))
            cl.set_groups(lut)
        refs.append(ref)
        layers.append(StackLayer(l + 1, cl))
    rng = np.random.default_rng(1)
    mlp = PredictorMLP(w1=rng.normal(scale=0.5, size=(32, E + 4 + 2)), b1=np.zeros(32),
                       w2=rng.normal(scale=2.0, size=(E, 32)), b2=np.zeros(E),
                       experts_per_layer=E, embed_dim=4, context_dim=2)
    emb = torch.randn(T, 4, dtype=torch.float64, generator=g).cuda()
    ctx = torch.randn(T, 2, dtype=torch.float64, generator=g).cuda()
    stack = CachedMoEStack(layers, predictor=mlp,
                           policy=OffloadPolicy(threshold_mode="constant", theta_base=0.05))
    y = stack.forward(x, emb, ctx)
    h = x
    for ref in refs:
        h = (ref.forward(h).float() + h.float()).to(torch.bfloat16)
    torch.cuda.synchronize()
    assert torch.equal(y, h)
    (_, _, chosen), = stack.prefetch_log
    assert all(e[0] == 2 and 0 <= e[1] < G for e in chosen)
    for sl in layers:
        sl.layer.cache.check()


def test_merge_outputs_never_alias_members_and_slots_are_released():
    """A pool filled through .data (no alloc) still gets merge outputs in
    slots that hold no member; a dropped variant returns its slots."""
    from paper_2508_09208_b200 import ExpertPool, kernels
    from paper_2508_09208_b200 import aggregation as A
    from paper_2508_09208_b200.moe import (ActivationStats, Expert, MoeModel, MoeModelSpec,
                                           cosine_only_calibration)
    from oracle import merge as M
    from oracle.switch_layer import bf16_round
    E, numel = 8, 8192
    pool = ExpertPool(E + 4, numel)
    g = torch.Generator(device="cuda").manual_seed(4)
    pool.data.normal_(0, 0.02, generator=g)       # members written without alloc()
    orig = pool.data[:E, :numel].clone()
    spec = MoeModelSpec(1, (1,), (), E, float(numel * 2), 1, numel)
    model = MoeModel(spec, {(1, s): Expert(1, s, pool.view(s), float(numel * 2))
                            for s in range(E)})
    counts = np.arange(1, E + 1, dtype=float)
    stats = ActivationStats(counts={1: counts}, totals={1: int(counts.sum())},
                            experts_per_layer=E)
    free0 = pool.free_slots()
    var = A.fuse_model(model, stats, A.FusionConfig(mode="fixed", r=0.5), 1.0,
                       cosine_only_calibration(), pool=pool)
    assert var.pool_slots and all(s >= E for s in var.pool_slots)
    assert torch.equal(pool.data[:E, :numel], orig)   # no member was overwritten
    freqs = stats.freqs(1)
    for grp in var.groups[1]:
        if not grp.member_slots:
            continue
        slots = (grp.principal_slot,) + tuple(grp.member_slots)
        ref = M.merge_params([orig[s].double().cpu().numpy() for s in slots],
                             [freqs[s] for s in slots])
        got = var.retained[1][grp.principal_slot].params.double().cpu().numpy()
        refb = bf16_round(ref.astype(np.float32)).astype(np.float64)
        assert np.all(np.abs(got - refb) <= np.abs(refb) * 2.0 ** -7 + 2.0 ** -24 * 0.2)
    var.release_slots(pool)
    assert pool.free_slots() == free0 - E            # members got reserved, merges returned
    for _ in range(3):                                # rebuilding does not leak slots
        v = A.fuse_model(model, stats, A.FusionConfig(mode="fixed", r=0.5), 1.0,
                         cosine_only_calibration(), pool=pool)
        v.release_slots(pool)
    assert pool.free_slots() == free0 - E
