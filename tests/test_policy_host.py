"""The package's host policy (offload.py / aggregation.py decisions) against
reference-generated golden decisions and the naive oracle (CPU only)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import merge as M
from oracle import policy as P
from paper_2508_09208_b200 import aggregation as A
from paper_2508_09208_b200 import offload as off
from paper_2508_09208_b200.errors import ConfigError, InfeasibleError
from paper_2508_09208_b200.moe import ActivationStats, Expert

POLICY = json.loads((GOLDEN / "policy_cases.json").read_text())
FUSION = json.loads((GOLDEN / "fusion_cases.json").read_text())
key = lambda s: tuple(int(v) for v in s.split(","))


@pytest.mark.parametrize("case", POLICY, ids=lambda c: str(len(c["sizes"])))
def test_policy_decisions_match_reference(case):
    th = case["threshold"]
    pol = off.OffloadPolicy(theta_base=th["theta_base"], delta_pref=th["delta_pref"],
                            gamma_cachethr=th["gamma_cachethr"], threshold_mode=th["mode"],
                            conservative_stability=th["conservative"])
    assert off.prefetch_threshold(pol, th["s_b"], th["m_avail"], th["m_total"]) == th["value"]
    assert off.eviction_score(*case["score"]["args"]) == case["score"]["value"]
    sizes = {key(k): v for k, v in case["sizes"].items()}
    freqs = {key(k): v for k, v in case["freqs"].items()}
    pinned = {tuple(e) for e in case["pinned"]}
    if case["placement_error"]:
        with pytest.raises(InfeasibleError):
            off.plan_initial_placement(sizes, freqs, case["ws_cap"], case["ca_cap"],
                                       pinned=frozenset(pinned), working_set_bytes=1.0)
        return
    plan = off.plan_initial_placement(sizes, freqs, case["ws_cap"], case["ca_cap"],
                                      pinned=frozenset(pinned), working_set_bytes=1.0)
    assert {f"{e[0]},{e[1]}": t for e, t in plan.assignment.items()} == case["placement"]
    assert [list(e) for e in plan.order] == case["order"]
    assert plan.eta_gs == case["eta_gs"]
    st = off.build_cache_state(plan, sizes, case["ws_cap"], case["ca_cap"], pinned=pinned)
    scores = {key(k): v for k, v in case["scores"].items()}
    before = (dict(st.workspace), dict(st.cache), dict(st.host))
    if case["evict_error"]:
        with pytest.raises(InfeasibleError):
            off.evict(st, case["bytes_needed"], scores)
    else:
        assert off.evict(st, case["bytes_needed"], scores) == [tuple(e) for e in case["evict"]]
    assert (dict(st.workspace), dict(st.cache), dict(st.host)) == before  # no mutation
    got = off.decide_prefetch(np.asarray(case["probs"]), case["theta"], st, case["layer"],
                              lambda e: sizes[e], budget_bytes=case["budget"])
    assert got == [tuple(e) for e in case["prefetch"]]
    if "subst" in case:
        s = case["subst"]
        simv = {key(k): v for k, v in s["sim"].items()}
        dec = off.correct_misprediction(tuple(s["needed"]), st, lambda a, b: simv[b],
                                        off.OffloadPolicy(substitution_sim_min=s["sim_min"]),
                                        priority=s["priority"], priority_threshold=0.8)
        assert (dec.action, list(dec.expert), dec.penalty) == (s["action"], s["expert"], s["penalty"])


def test_evict_matches_exhaustive_oracle_fuzz():
    rng = np.random.default_rng(5)
    for _ in range(300):
        n = int(rng.integers(1, 9))
        ids = [(0, i) for i in range(n)]
        st = off.CacheState(workspace_capacity=1.0, cache_capacity=float(rng.uniform(2, 8)))
        used = 0.0
        for e in ids:
            b = float(rng.uniform(0.2, 1.5))
            if used + b <= st.cache_capacity:
                st.cache[e] = b
                used += b
            else:
                st.host[e] = b
        st.pinned = {e for e in st.cache if rng.random() < 0.3}
        scores = {e: float(rng.choice([0.5, 1.0, rng.random()])) for e in st.cache}
        need = float(rng.uniform(0, st.cache_capacity * 1.2))
        ref = P.victims(st.cache, st.pinned, st.cache_capacity, need, scores)
        if ref is None:
            with pytest.raises(InfeasibleError):
                off.evict(st, need, scores)
        else:
            assert off.evict(st, need, scores) == ref


def test_cache_state_invariants_and_errors():
    st = off.CacheState(workspace_capacity=2.0, cache_capacity=3.0)
    st.host.update({(0, 0): 1.0, (0, 1): 2.0})
    st.move((0, 0), off.HOST, off.WORKSPACE)
    assert st.tier_of((0, 0)) == off.WORKSPACE and st.free_bytes(off.WORKSPACE) == 1.0
    with pytest.raises(KeyError):
        st.move((0, 0), off.HOST, off.CACHE)
    st.pinned.add((0, 1))
    with pytest.raises(AssertionError):
        st.check_invariants()
    st.record_access((0, 0), 0)
    st.record_access((0, 0), 256)
    assert st.recent_value((0, 0), 256) == pytest.approx(1.5)
    with pytest.raises(ConfigError):
        off.OffloadPolicy(theta_base=-1).validate()


def _stats(counts):
    c = np.asarray(counts, float)
    return ActivationStats(counts={1: c}, totals={1: max(int(c.sum()), 1)}, experts_per_layer=len(c))


@pytest.mark.parametrize("case", FUSION[:20], ids=lambda c: f"E{c['E']}")
def test_fusion_decisions_match_reference(case):
    E = case["E"]
    st = _stats(case["counts"])
    assert A.fixed_retention(E, case["r"]) == case["target"]
    h, hbar = A.layer_entropy(st, 1)
    assert h == pytest.approx(case["entropy"], rel=1e-12, abs=1e-15)
    assert A.adaptive_retention(E, 0.25, 0.3, hbar, 1) == case["adaptive"]
    ps = A.identify_principals(st, 1, case["target"], case["theta_act"])
    assert ps == case["principals"]
    experts = [Expert(1, s, None, 1.0) for s in range(E)]
    groups = A.group_experts(experts, ps, np.asarray(case["sim"]))
    assert {str(g.principal_slot): list(g.member_slots) for g in groups} == case["groups"]


def test_fusion_config_validation_and_selection():
    assert A.FusionConfig(mode="fixed", r=0.25).config_id == "fixed-0.25"
    assert A.FusionConfig(mode="adaptive", r_base=0.6, delta_r=0.3).config_id == "adaptive-0.6-0.3"
    for bad in (dict(mode="magic", r=0.5), dict(mode="fixed", r=0.0),
                dict(mode="adaptive", r_base=0.5, delta_r=-1.0),
                dict(mode="fixed", r=0.5, theta_act=1.0), dict(mode="fixed", r=0.5, scope="x")):
        with pytest.raises(ConfigError):
            A.FusionConfig(**bad).validate()
    mk = lambda vid, mem, perf: A.ModelVariant(vid, {}, {}, {}, mem, perf)
    lib = A.VariantLibrary([mk("a", 10, 0.9), mk("b", 5, 0.9), mk("c", 20, 1.0)])
    assert A.select_variant(lib, 12).variant_id == "b"
    assert A.select_variant(lib, 25).variant_id == "c"
    with pytest.raises(InfeasibleError):
        A.select_variant(lib, 1)
    with pytest.raises(ConfigError):
        A.VariantLibrary([mk("a", 1, 1), mk("a", 2, 1)])


def test_resident_budget_modes_match_simulator_rules():
    """_resident_budget / _required_fn (simulator.py:275-293), hand cases."""
    from paper_2508_09208_b200.cache import required_bytes_fn, resident_budget
    assert resident_budget(10.0, "fraction_of_variant", 0.5, 100.0) == 5.0
    assert resident_budget(10.0, "fraction_of_model", 0.3, 100.0) == 10.0   # capped by the variant
    assert resident_budget(50.0, "fraction_of_model", 0.3, 100.0) == 30.0
    assert resident_budget(50.0, "absolute", 0.0, 100.0, cache_bytes=7.0) == 7.0
    assert resident_budget(50.0, "absolute", 0.0, 100.0, cache_bytes=70.0, offload=False) == 50.0
    with pytest.raises(ValueError):
        resident_budget(1.0, "bogus", 0.5, 1.0)
    v = A.ModelVariant("x", {}, {}, {}, 0.0, 1.0, expert_bytes=40.0)
    req = required_bytes_fn("fraction_of_variant", 0.5, 100.0, m_other=3.0, workspace_bytes=2.0)
    assert req(v) == 25.0


def test_fold_demand_into_group_space():
    """stack.fold_demand: P(group demanded) = 1 - prod over its members."""
    from paper_2508_09208_b200.stack import fold_demand
    p = np.array([0.5, 0.2, 0.0, 1.0, 0.3])
    lut = [0, 0, 1, 2, 1]
    out = fold_demand(p, lut, 3)
    np.testing.assert_allclose(out, [1 - 0.5 * 0.8, 1 - 1.0 * 0.7, 1.0])
    np.testing.assert_allclose(fold_demand(p, range(5), 5), p)  # identity variant: unchanged


def test_pool_alloc_skips_excluded_slots_and_reserves_them():
    from paper_2508_09208_b200.pool import ExpertPool
    pool = ExpertPool(6, 64, device="cpu")
    a = pool.alloc(exclude={0, 1})
    assert a not in (0, 1)
    assert pool.free_slots() == 3                    # 0 and 1 reserved, a taken
    assert all(pool.alloc() not in (0, 1, a) for _ in range(3))
    pool.reserve(0)                                  # already reserved: no-op
    with pytest.raises(RuntimeError):
        pool.alloc()


def test_offload_priority_matches_reference():
    """a19: offload_priority (offload.py:430-438) on reference-generated
    cases (oracle/gen_golden.py -> priority_cases.json), bit for bit."""
    from paper_2508_09208_b200.offload import offload_priority
    cases = json.loads((GOLDEN / "priority_cases.json").read_text())
    assert len(cases) > 40
    for c in cases:
        if "error" in c:
            with pytest.raises(ValueError, match=c["error"]):
                offload_priority(*c["args"])
        else:
            assert offload_priority(*c["args"]) == c["value"]


def test_prefetch_governor_keeps_the_faster_setting():
    """PrefetchGovernor (stack.py): probe `window` forwards with prefetch on,
    `window` off, hold the faster for `hold` steps, probe again; state is
    kept per batch size."""
    from paper_2508_09208_b200.stack import PrefetchGovernor
    g = PrefetchGovernor(window=2, hold=3)
    seq = []
    for step in range(9):
        on = g.enabled(64)
        seq.append(on)
        g.record(64, on, 10.0 if on else 7.0)   # prefetch costs time at 64 tokens
    # on, on (probe), off, off (probe), off x3 (hold the faster), on, on (re-probe)
    assert seq == [True, True, False, False, False, False, False, True, True]
    assert g._state(64)["last"] == (10.0, 7.0)
    g2 = PrefetchGovernor(window=1, hold=2)
    seq = []
    for step in range(4):
        on = g2.enabled(16)
        seq.append(on)
        g2.record(16, on, 3.0 if on else 5.0)   # prefetch pays at 16 tokens
    assert seq == [True, False, True, True]
    assert g2.enabled(1024)  # a new batch size starts probing with prefetch on
