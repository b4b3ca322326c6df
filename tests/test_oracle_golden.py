"""Pin the CPU oracle against vectors produced by the reference itself
(oracle/gen_golden.py ran /root/reference/pkg/src/comoe unmodified)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import merge as M
from oracle import policy as P

FUSION = json.loads((GOLDEN / "fusion_cases.json").read_text())
POLICY = json.loads((GOLDEN / "policy_cases.json").read_text())


def test_merge_hand_cases():
    for case in json.loads((GOLDEN / "merge_hand.json").read_text()):
        got = M.merge_params(case["vectors"], case["freqs"])
        np.testing.assert_array_equal(got, case["expected"])


@pytest.mark.parametrize("case", FUSION, ids=lambda c: f"E{c['E']}d{c['dim']}")
def test_fusion_oracle_matches_reference(case):
    E = case["E"]
    P_ = np.asarray(case["params"])
    counts = np.asarray(case["counts"])
    freqs = counts / max(int(counts.sum()), 1)
    h, hbar = M.entropy(freqs)
    assert h == pytest.approx(case["entropy"], rel=1e-12, abs=1e-15)
    assert M.retention_adaptive(E, 0.25, 0.3, hbar, 1) == case["adaptive"]
    assert M.retention_fixed(E, case["r"]) == case["target"]
    S = M.similarity(P_, case["probes"], case["projection"], case["alpha"])
    np.testing.assert_allclose(S, case["sim"], rtol=1e-9, atol=1e-10)
    ps = M.principals(freqs, case["target"], case["theta_act"])
    assert ps == case["principals"]
    # grouping given the reference's own S is exact
    ps2, members, merged, smap = M.fuse_layer(P_, freqs, case["target"], np.asarray(case["sim"]),
                                              case["theta_act"])
    assert {str(k): v for k, v in smap.items()} == case["slot_map"]
    assert {str(k): v for k, v in members.items()} == case["groups"]
    for p, ref in case["merged"].items():
        np.testing.assert_array_equal(merged[int(p)], np.asarray(ref))


@pytest.mark.parametrize("case", POLICY, ids=lambda c: str(len(c["sizes"])))
def test_policy_oracle_matches_reference(case):
    th = case["threshold"]
    assert P.threshold(th["mode"], th["theta_base"], th["delta_pref"], th["gamma_cachethr"],
                       th["conservative"], th["s_b"], th["m_avail"], th["m_total"]) == th["value"]
    assert P.score(*case["score"]["args"]) == case["score"]["value"]
    if "cache" not in case:
        return
    key = lambda s: tuple(int(v) for v in s.split(","))
    cache = {key(k): v for k, v in case["cache"].items()}
    pinned = {tuple(e) for e in case["pinned"]}
    scores = {key(k): v for k, v in case["scores"].items()}
    got = P.victims(cache, pinned, case["ca_cap"], case["bytes_needed"], scores)
    if case["evict_error"]:
        assert got is None
    else:
        assert got == [tuple(e) for e in case["evict"]]
    sizes = {key(k): v for k, v in case["sizes"].items()}
    resident = set(cache) | {key(k) for k in case["workspace"]}
    budget = case["budget"]
    if budget is None:
        budget = case["ca_cap"] - sum(cache.values()) + sum(v for e, v in cache.items() if e not in pinned)
    pre = P.prefetch_choice(case["probs"], case["theta"], case["layer"], resident, sizes, budget)
    assert pre == [tuple(e) for e in case["prefetch"]]
