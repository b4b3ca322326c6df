"""Generate golden fixtures from the UNMODIFIED reference package.

Run in the build container (where /root/reference exists):
    python oracle/gen_golden.py
It imports comoe from /root/reference/pkg/src (read-only; nothing is copied)
and writes small JSON fixtures to tests/golden/. The GPU box never runs this;
tests there read the committed fixtures only.

Fixtures
  fusion_cases.json    per-layer fusion pipeline cases: inputs (freqs, params,
                       calibration) and the reference's similarity matrix,
                       principals, grouping, merged params, slot_map, score
  merge_hand.json      the reference unit-test hand cases for merge_group
  merge_bigsum.json    seeded large merges (D up to 4,718,592): sha256 of the
                       reference merge_group output bytes (fp64), for the
                       device fp64 bit-exactness check
  policy_cases.json    cache-policy decisions: prefetch_threshold, eviction
                       scores, evict victims / infeasible, decide_prefetch,
                       plan_initial_placement, correct_misprediction
  priority_cases.json  offload_priority values and error cases
  cache_parity.json    the reference runtime's per-token cache decision
                       stream (hit / fetch / substitute / prefetch /
                       demote / evict) on a small scenario + its inputs
  traces.json          generate_routing traces (+ the reference's
                       collect_stats of each) and a trained predictor
  library_cases.json   build_library over two-layer models: every variant's
                       groups / slot map / sizes / score, variant_freqs,
                       library_manifest, select_variant at several memory
                       levels, plus should_switch and granularity_decision
                       cases (values and error cases)
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def _ref():
    sys.path.insert(0, str(REF))
    import comoe  # noqa: F401
    from comoe import aggregation, moe, offload
    return moe, aggregation, offload


def fusion_cases(moe, agg, n_cases=40):
    rng = np.random.default_rng(20260901)
    cases = []
    for i in range(n_cases):
        E = int(rng.integers(2, 17))
        dim = int(rng.choice([6, 16, 64]))
        spec = moe.MoeModelSpec(total_layers=2, encoder_moe_layers=(1,), decoder_moe_layers=(),
                                experts_per_layer=E, expert_size_bytes=1e6, top_k=1,
                                expert_param_dim=dim)
        model = moe.synthesize_model(spec, int(rng.integers(0, 2 ** 31)))
        counts = rng.integers(0, 50, size=E).astype(float)
        if i % 7 == 3:
            counts[:] = 0.0
            counts[0] = 1.0   # one active expert -> zero-frequency groups
        if counts.sum() == 0:
            counts[0] = 1.0
        if i % 5 == 2:
            counts[1 % E] = counts[0]  # frequency ties
        stats = moe.ActivationStats(counts={1: counts}, totals={1: int(counts.sum())},
                                    experts_per_layer=E)
        calib = moe.make_calibration(dim, n_probes=int(rng.integers(1, 9)),
                                     seed=int(rng.integers(0, 1000)),
                                     buckets=int(rng.integers(2, 9)))
        alpha = float(rng.choice([0.0, 0.5, 1.0, 0.3]))
        r = float(rng.choice([0.25, 0.5, 0.75]))
        theta = float(rng.choice([0.0, 0.0, 0.1, 0.3]))
        cfg = agg.FusionConfig(mode="fixed", r=r, theta_act=theta)
        experts = model.layer_experts(1)
        S = moe.similarity_matrix(experts, alpha, calib)
        target = agg.fixed_retention(E, r)
        princ = agg.identify_principals(stats, 1, target, theta)
        groups = agg.group_experts(experts, princ, S)
        by_slot = {e.slot: e for e in experts}
        merged = {g.principal_slot: agg.merge_group(g, by_slot, stats, 1).params.tolist()
                  for g in groups}
        var = agg.fuse_model(model, stats, cfg, alpha, calib)
        h, hbar = agg.layer_entropy(stats, 1)
        cases.append(dict(
            E=E, dim=dim, counts=counts.tolist(), alpha=alpha, r=r, theta_act=theta,
            params=[e.params.tolist() for e in experts],
            probes=calib.probes.tolist(), projection=calib.projection.tolist(),
            sim=S.tolist(), target=target, principals=princ,
            groups={str(g.principal_slot): list(g.member_slots) for g in groups},
            merged={str(k): v for k, v in merged.items()},
            slot_map={str(k): v for k, v in var.slot_map[1].items()},
            perf_estimate=var.perf_estimate, entropy=h, hbar=hbar,
            adaptive=agg.adaptive_retention(E, 0.25, 0.3, hbar, 1)))
    return cases


def merge_hand(moe, agg):
    Ex = moe.Expert
    out = []
    by = {0: Ex(1, 0, np.array([2.0, 0.0]), 3.0), 1: Ex(1, 1, np.array([0.0, 4.0]), 3.0)}
    st = moe.ActivationStats(counts={1: np.array([3.0, 1.0])}, totals={1: 4},
                             experts_per_layer=2)
    m = agg.merge_group(agg.ExpertGroup(0, (1,)), by, st, 1)
    out.append(dict(vectors=[[2.0, 0.0], [0.0, 4.0]], freqs=[0.75, 0.25], expected=m.params.tolist()))
    st0 = moe.ActivationStats(counts={1: np.zeros(2)}, totals={1: 10}, experts_per_layer=2)
    m0 = agg.merge_group(agg.ExpertGroup(0, (1,)), by, st0, 1)
    out.append(dict(vectors=[[2.0, 0.0], [0.0, 4.0]], freqs=[0.0, 0.0], expected=m0.params.tolist()))
    return out


def merge_bigsum(moe, agg):
    """Seeded large groups; the device must reproduce the bytes exactly."""
    out = []
    for seed, n, D in ((11, 2, 4_718_592), (12, 4, 1_000_003), (13, 9, 262_144), (14, 3, 65_537)):
        rng = np.random.default_rng(seed)
        V = rng.normal(size=(n, D)) * 0.02
        f = rng.integers(0, 100, size=n).astype(float)
        if seed == 14:
            f[:] = 0.0
        total = float(f.sum()) if f.sum() > 0 else 1.0
        experts = {s: moe.Expert(1, s, V[s], 1.0) for s in range(n)}
        st = moe.ActivationStats(counts={1: f}, totals={1: max(int(f.sum()), 1)},
                                 experts_per_layer=n)
        g = agg.ExpertGroup(0, tuple(range(1, n)))
        m = agg.merge_group(g, experts, st, 1).params
        out.append(dict(seed=seed, n=n, D=D, counts=f.tolist(), total=total,
                        sha256=hashlib.sha256(np.ascontiguousarray(m).tobytes()).hexdigest(),
                        head=m[:4].tolist()))
    return out


def policy_cases(off, n_cases=60):
    rng = np.random.default_rng(777)
    cases = []
    for i in range(n_cases):
        E = int(rng.integers(3, 12))
        layers = int(rng.integers(1, 3))
        experts = [(l, s) for l in range(layers) for s in range(E)]
        sizes = {e: float(rng.choice([1.0, 1.5, 2.0])) for e in experts}
        ws_cap = float(rng.choice([2.0, 3.0, 4.0]))
        ca_cap = float(rng.choice([3.0, 5.0, 8.0]))
        freqs = {e: float(rng.random()) for e in experts}
        if i % 4 == 0:
            for e in experts[:3]:
                freqs[e] = 0.5  # ties
        pinned = set()
        if i % 3 == 0:
            pinned = {experts[int(rng.integers(0, len(experts)))]}
        try:
            plan = off.plan_initial_placement(sizes, freqs, ws_cap, ca_cap, pinned=frozenset(pinned),
                                              working_set_bytes=1.0)
            placement = {f"{e[0]},{e[1]}": t for e, t in plan.assignment.items()}
            order = [list(e) for e in plan.order]
            eta = plan.eta_gs
            state = off.build_cache_state(plan, sizes, ws_cap, ca_cap, pinned=pinned)
            infeasible_place = False
        except Exception as exc:  # InfeasibleError
            placement, order, eta, state = None, None, None, None
            infeasible_place = type(exc).__name__
        case = dict(sizes={f"{e[0]},{e[1]}": v for e, v in sizes.items()},
                    freqs={f"{e[0]},{e[1]}": v for e, v in freqs.items()},
                    ws_cap=ws_cap, ca_cap=ca_cap, pinned=[list(e) for e in pinned],
                    placement=placement, order=order, eta_gs=eta,
                    placement_error=infeasible_place)
        if state is not None:
            scores = {e: float(rng.uniform(0, 3)) for e in state.cache}
            need = float(rng.uniform(0, ca_cap * 1.2))
            try:
                vict = off.evict(state, need, scores)
                ev = [list(e) for e in vict]
                ev_err = False
            except Exception as exc:
                ev, ev_err = None, type(exc).__name__
            probs = rng.random(E)
            if i % 5 == 1:
                probs[1] = probs[0]
            theta = float(rng.choice([0.0, 0.2, 0.5, 0.8]))
            layer = int(rng.integers(0, layers))
            budget = None if i % 2 else float(rng.uniform(0, 6))
            pre = off.decide_prefetch(probs, theta, state, layer, lambda e: sizes[e],
                                      budget_bytes=budget)
            case.update(cache={f"{e[0]},{e[1]}": v for e, v in state.cache.items()},
                        workspace={f"{e[0]},{e[1]}": v for e, v in state.workspace.items()},
                        scores={f"{e[0]},{e[1]}": v for e, v in scores.items()},
                        bytes_needed=need, evict=ev, evict_error=ev_err,
                        probs=probs.tolist(), theta=theta, layer=layer, budget=budget,
                        prefetch=[list(e) for e in pre])
            # substitution
            host = sorted(state.host)
            if host:
                needed = host[int(rng.integers(0, len(host)))]
                simv = {e: float(rng.uniform(0.5, 1.0)) for e in experts}
                pol = off.OffloadPolicy(substitution_sim_min=float(rng.choice([0.7, 0.8, 0.95])))
                prio = float(rng.random())
                dec = off.correct_misprediction(needed, state, lambda a, b: simv[b], pol,
                                                priority=prio, priority_threshold=0.8)
                case.update(subst=dict(needed=list(needed), sim={f"{e[0]},{e[1]}": v for e, v in simv.items()},
                                       sim_min=pol.substitution_sim_min, priority=prio,
                                       action=dec.action, expert=list(dec.expert),
                                       penalty=dec.penalty))
        # threshold + score grid
        pol = off.OffloadPolicy(theta_base=float(rng.uniform(0, 1)), delta_pref=float(rng.random()),
                                gamma_cachethr=float(rng.random()),
                                threshold_mode=str(rng.choice(["resource-aware", "storage-fraction", "constant"])),
                                conservative_stability=bool(i % 2))
        s_b, m_av, m_tot = float(rng.random()), float(rng.uniform(0, 8e9)), 8e9
        case["threshold"] = dict(mode=pol.threshold_mode, theta_base=pol.theta_base,
                                 delta_pref=pol.delta_pref, gamma_cachethr=pol.gamma_cachethr,
                                 conservative=pol.conservative_stability, s_b=s_b, m_avail=m_av,
                                 m_total=m_tot, value=off.prefetch_threshold(pol, s_b, m_av, m_tot))
        args = (float(rng.random()), float(rng.choice([0.0, 1e-9, rng.random() * 4])),
                float(rng.choice([0.0, rng.random()])), float(rng.random()), float(rng.random()))
        case["score"] = dict(args=list(args), value=off.eviction_score(*args))
        cases.append(case)
    return cases


def traces_and_predictor(moe, off):
    out = []
    for i, (E, K, skew, rho, n) in enumerate(((8, 1, 1.0, 0.9, 40), (16, 2, {"default": 0.5, 3: 2.0}, 0.5, 30),
                                              (128, 1, 1.2, 1.0, 20))):
        spec = moe.MoeModelSpec(total_layers=6, encoder_moe_layers=(1, 3), decoder_moe_layers=(5,),
                                experts_per_layer=E, expert_size_bytes=1e6, top_k=K)
        g = moe.RoutingGeneratorSpec(skew=skew, rho=rho, seed=10 + i, structure_seed=3 + i)
        tr = moe.generate_routing(g, spec, n)
        rec = dict(E=E, K=K, skew={str(k): v for k, v in skew.items()} if isinstance(skew, dict) else skew,
                   rho=rho, seed=10 + i, structure_seed=3 + i, n=n,
                   experts=[[list(tok.layer_experts[l]) for l in spec.moe_layer_indices] for tok in tr.tokens],
                   emb_sum=float(sum(float(t.embedding.sum()) for t in tr.tokens)),
                   ctx_sum=float(sum(float(t.context.sum()) for t in tr.tokens)))
        st = moe.collect_stats(tr)  # the reference's ActivationStats of this trace
        rec["collect_stats"] = dict(counts={str(l): st.counts[l].tolist() for l in st.counts},
                                    totals={str(l): int(st.totals[l]) for l in st.totals})
        if i == 0:
            big = moe.generate_routing(g, spec, 300)
            mlp, metrics = off.train_predictor(big, hidden_dim=8, lr=0.05, epochs=2, seed=5)
            rec["predictor"] = dict(n=300, hidden=8, epochs=2, seed=5, w1=mlp.w1.tolist(),
                                    b1=mlp.b1.tolist(), w2=mlp.w2.tolist(), b2=mlp.b2.tolist(),
                                    metrics=metrics)
        out.append(rec)
    return out


def priority_cases(off, n_cases=40):
    """offload_priority (offload.py:430-438) on seeded inputs, including the
    simulator's uniform-size use (normalizer = size / estimate,
    simulator.py:423-431) and the error cases."""
    rng = np.random.default_rng(20261017)
    cases = []
    for i in range(n_cases):
        f = float(rng.random()) if i % 5 else 0.0
        size = float(rng.choice([9437184.0, 352321536.0, rng.random() * 1e9 + 1]))
        est = float(rng.random() * 1e-2 + 1e-6)
        gamma = float(rng.choice([0.0, 1.0, rng.random()]))
        norm = size / est if i % 2 else float(rng.random() * 1e11 + 1.0)
        cases.append(dict(args=[f, size, est, gamma, norm],
                          value=off.offload_priority(f, size, est, gamma, norm)))
    for bad in ([0.5, 1.0, 0.0, 0.5, 1.0], [0.5, 1.0, 1.0, 0.5, 0.0]):
        try:
            off.offload_priority(*bad)
            raise AssertionError("expected ValueError")
        except ValueError as e:
            cases.append(dict(args=bad, error=str(e)))
    return cases


PARITY_SCENARIO = {
    # small geometry on one device: 3 MoE layers x 8 experts, 1 MB experts;
    # an absolute 13-expert HBM budget (1 workspace + 12 cache slots, the
    # decoder layer's 8 experts pinned), MLP predictor with a constant
    # prefetch threshold, substitution on, and a host link fast enough that
    # every prefetch lands before its next use (no late-prefetch timing).
    # 192 tokens exercise every decision kind: hit, fetch, substitute,
    # prefetch, demote, evict
    "model": {"preset": None, "total_layers": 4, "encoder_moe_layers": [1, 2],
              "decoder_moe_layers": [3], "experts_per_layer": 8, "top_k": 1,
              "expert_size_bytes": 1.0e6, "expert_param_dim": 64},
    "fusion": {"enabled": False},
    "offload": {"enabled": True, "cache_mode": "absolute", "cache_bytes": 13.0e6,
                "workspace_slots": 1, "predictor": "mlp", "predictor_hidden": 16,
                "predictor_epochs": 3, "prefetch": True, "threshold_mode": "constant",
                "theta_base": 0.1, "substitution": True, "substitution_sim_min": 0.5,
                "pin_decoder": True},
    "resources": {"devices": [{"device_id": "parity",
                               "base": {"gpu_mem_total": 8.0e9, "bw_gpu_cpu": 1.0e15}}]},
    "workload": {"sequence_length": 64, "sequences": 3,
                 "routing": {"mode": "generate", "skew": 1.2, "rho": 0.9, "seed": 77,
                             "structure_seed": 5}},
}


def cache_parity(moe):
    """The reference runtime's per-token cache loop (simulator.py:684-724,
    _serve_demand / _predict_and_prefetch / eviction) on PARITY_SCENARIO:
    its decision event stream plus every input needed to replay the same
    decisions through the B200 cache (trace, predictor weights, merged
    frequencies, similarities, offload priorities, initial placement)."""
    import copy
    from comoe import scenario as scen
    from comoe import simulator as sim
    captured = []

    class _Captured(sim._Run):  # records the run object (no behaviour change)
        def __init__(self, *a, **k):
            super().__init__(*a, **k)
            captured.append(self)

        def _activate_variant(self, variant, tick):
            super()._activate_variant(variant, tick)
            self._initial_cache = copy.deepcopy(self.cache)

    orig = sim._Run
    sim._Run = _Captured
    try:
        report = sim.run_inference(copy.deepcopy(PARITY_SCENARIO))
    finally:
        sim._Run = orig
    run = captured[0]
    cfg = scen.normalize(copy.deepcopy(PARITY_SCENARIO))
    spec = scen.build_model_spec(cfg)
    trace = moe.generate_routing(scen.build_routing_spec(cfg), spec, report.tokens)
    layers = list(spec.moe_layer_indices)
    key = lambda e: f"{e[0]},{e[1]}"
    ic = run._initial_cache
    sims = {str(l): [[run._similarity((l, a), (l, b)) for b in range(8)] for a in range(8)]
            for l in layers}
    kinds = {"hit", "fetch", "substitute", "prefetch", "demote", "evict"}
    return dict(
        scenario=PARITY_SCENARIO, layers=layers, encoder_layers=list(spec.encoder_moe_layers),
        tokens=[dict(experts={str(l): list(t.layer_experts[l]) for l in layers},
                     embedding=t.embedding.tolist(), context=t.context.tolist())
                for t in trace.tokens],
        predictor=dict(w1=run.mlp.w1.tolist(), b1=run.mlp.b1.tolist(), w2=run.mlp.w2.tolist(),
                       b2=run.mlp.b2.tolist(), embed_dim=run.mlp.embed_dim,
                       context_dim=run.mlp.context_dim),
        freqs={key(e): f for e, f in run.freqs.items()},
        priorities={key(e): p for e, p in run.priorities.items()},
        prio_threshold=run.prio_threshold, hard_pinned=sorted(key(e) for e in run.hard_pinned),
        similarity=sims,
        policy=dict(theta_base=run.policy.theta_base, delta_evict=run.policy.delta_evict,
                    lambda_evict=run.policy.lambda_evict,
                    substitution_sim_min=run.policy.substitution_sim_min,
                    half_life=ic.half_life),
        initial=dict(workspace=[key(e) for e in ic.workspace], cache=[key(e) for e in ic.cache]),
        capacities=dict(workspace=ic.workspace_capacity, cache=ic.cache_capacity),
        events=[r for r in report.events if r["event"] in kinds],
        report=dict(demand_count=report.demand_count, hit_count=report.hit_count,
                    hit_rate=report.hit_rate, prefetch_issued=report.prefetch_issued,
                    prefetch_hit_count=report.prefetch_hit_count,
                    substitution_count=report.substitution_count,
                    late_prefetch_count=report.late_prefetch_count))


def library_cases(moe, agg, n_cases=12):
    rng = np.random.default_rng(20261017)
    cases = []
    for i in range(n_cases):
        E = int(rng.integers(3, 13))
        dim = 16
        scope = "both" if i % 3 == 2 else "encoder"
        spec = moe.MoeModelSpec(total_layers=4, encoder_moe_layers=(1,), decoder_moe_layers=(3,),
                                experts_per_layer=E, expert_size_bytes=float(rng.choice([1e6, 2.5e6])),
                                top_k=1, expert_param_dim=dim)
        model = moe.synthesize_model(spec, int(rng.integers(0, 2 ** 31)))
        counts = {}
        for layer in (1, 3):
            c = rng.integers(0, 40, size=E).astype(float)
            if c.sum() == 0:
                c[0] = 1.0
            if i % 4 == 1:
                c[1 % E] = c[0]  # frequency ties
            counts[layer] = c
        stats = moe.ActivationStats(counts=counts, totals={l: int(c.sum()) for l, c in counts.items()},
                                    experts_per_layer=E)
        calib = moe.make_calibration(dim, n_probes=4, seed=int(rng.integers(0, 1000)), buckets=4)
        alpha = float(rng.choice([0.0, 0.5, 1.0]))
        m_other = float(rng.choice([0.0, 3e6]))
        configs = [agg.FusionConfig(mode="fixed", r=0.5, scope=scope),
                   agg.FusionConfig(mode="fixed", r=0.25, theta_act=0.05, scope=scope),
                   agg.FusionConfig(mode="adaptive", r_base=0.5, delta_r=0.25, e_min=1, scope=scope)]
        lib = agg.build_library(model, stats, configs, alpha, calib, m_other)
        variants = []
        for v in lib.variants:
            variants.append(dict(
                id=v.variant_id, mem_required=v.mem_required, expert_bytes=v.expert_bytes,
                perf_estimate=v.perf_estimate,
                slot_map={str(l): {str(k): int(x) for k, x in m.items()} for l, m in v.slot_map.items()},
                groups={str(l): [[g.principal_slot, list(g.member_slots)] for g in gs]
                        for l, gs in v.groups.items()},
                freqs=[[int(l), int(sl), float(f)] for (l, sl), f in
                       sorted(agg.variant_freqs(v, stats).items())]))
        mems = sorted({v.mem_required for v in lib.variants})
        levels = [mems[0] * 0.5] + mems + [0.5 * (a + b) for a, b in zip(mems, mems[1:])] + [mems[-1] * 2]
        selects = []
        for m in levels:
            try:
                selects.append([m, agg.select_variant(lib, m).variant_id])
            except Exception as exc:  # infeasible
                selects.append([m, type(exc).__name__])
        cases.append(dict(E=E, scope=scope, alpha=alpha, m_other=m_other,
                          params={str(l): [e.params.tolist() for e in model.layer_experts(l)]
                                  for l in (1, 3)},
                          sizes={str(l): [e.size for e in model.layer_experts(l)] for l in (1, 3)},
                          counts={str(l): c.tolist() for l, c in counts.items()},
                          probes=calib.probes.tolist(), projection=calib.projection.tolist(),
                          variants=variants, manifest=agg.library_manifest(lib), selects=selects))
    switch = []
    for _ in range(40):
        a = agg.ModelVariant(variant_id=str(rng.choice(["a", "b"])), retained={}, slot_map={},
                             groups={}, mem_required=1.0, perf_estimate=0.5)
        b = agg.ModelVariant(variant_id=str(rng.choice(["a", "b", "c"])), retained={}, slot_map={},
                             groups={}, mem_required=1.0, perf_estimate=0.5)
        pol = agg.SwitchPolicy(lambda_switch=float(rng.choice([0.0, 0.5, 1.0])),
                               switch_cost=float(rng.choice([0.0, 0.05, 0.2])),
                               t_threshold=float(rng.choice([0.0, 4.0, 8.0])))
        dp = float(rng.choice([0.0, 0.01, 0.025, 0.1, 0.5]))
        ts = float(rng.choice([-1.0, 0.0, 4.0, 8.0, 9.0]))
        try:
            out = bool(agg.should_switch(a, b, dp, pol, ts))
        except ValueError:
            out = "ValueError"
        switch.append(dict(cur=a.variant_id, cand=b.variant_id, delta_p=dp, lambda_switch=pol.lambda_switch,
                           switch_cost=pol.switch_cost, t_threshold=pol.t_threshold, t_stable=ts, out=out))
    gran = []
    for _ in range(40):
        args = (float(rng.choice([0.0, 0.3, 0.7, 0.95, 1.0])), float(rng.choice([1e9, 8e9, 80e9])),
                float(rng.choice([0.0, 9.4e6, 4.7e8])), float(rng.choice([0.0, 0.5, 2.0])),
                float(rng.choice([-0.1, 0.0, 0.4, 1.0])), int(rng.choice([8, 64, 128])))
        try:
            out = int(agg.granularity_decision(*args))
        except ValueError:
            out = "ValueError"
        gran.append(dict(args=list(args), out=out))
    return dict(cases=cases, should_switch=switch, granularity=gran)


def main():
    moe, agg, off = _ref()
    (OUT / "cache_parity.json").write_text(json.dumps(cache_parity(moe)))
    (OUT / "priority_cases.json").write_text(json.dumps(priority_cases(off), indent=1))
    (OUT / "traces.json").write_text(json.dumps(traces_and_predictor(moe, off)))
    OUT.mkdir(parents=True, exist_ok=True)
    (OUT / "fusion_cases.json").write_text(json.dumps(fusion_cases(moe, agg)))
    (OUT / "merge_hand.json").write_text(json.dumps(merge_hand(moe, agg), indent=1))
    (OUT / "merge_bigsum.json").write_text(json.dumps(merge_bigsum(moe, agg), indent=1))
    (OUT / "policy_cases.json").write_text(json.dumps(policy_cases(off)))
    (OUT / "library_cases.json").write_text(json.dumps(library_cases(moe, agg)))
    for p in sorted(OUT.glob("*.json")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
