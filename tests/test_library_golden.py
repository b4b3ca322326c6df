"""Variant-library rows against fixtures the unmodified reference produced
(oracle/gen_golden.py -> tests/golden/library_cases.json): build_library
over two-layer models (fixed and adaptive configs, encoder-only and both
scopes), variant_freqs, library_manifest, select_variant at memory levels
around every variant's requirement, should_switch and granularity_decision
(values and error cases). Reference: aggregation.py:319-404."""

import json

import numpy as np
import pytest

from conftest import GOLDEN

CASES = json.loads((GOLDEN / "library_cases.json").read_text())


def _stats(case):
    from paper_2508_09208_b200.moe import ActivationStats
    counts = {int(l): np.asarray(c, float) for l, c in case["counts"].items()}
    return ActivationStats(counts=counts, totals={l: int(c.sum()) for l, c in counts.items()},
                           experts_per_layer=case["E"])


def _host_variants(case):
    """Our ModelVariant objects carrying the reference variants' decisions."""
    from paper_2508_09208_b200.aggregation import ExpertGroup, ModelVariant
    out = []
    for v in case["variants"]:
        groups = {int(l): [ExpertGroup(p, tuple(m)) for p, m in gs] for l, gs in v["groups"].items()}
        out.append(ModelVariant(
            variant_id=v["id"], retained={l: {g.principal_slot: None for g in gs} for l, gs in groups.items()},
            slot_map={int(l): {int(k): x for k, x in m.items()} for l, m in v["slot_map"].items()},
            groups=groups, mem_required=v["mem_required"], perf_estimate=v["perf_estimate"],
            expert_bytes=v["expert_bytes"]))
    return out


@pytest.mark.parametrize("i", range(len(CASES["cases"])))
def test_variant_freqs_manifest_and_selection(i):
    from paper_2508_09208_b200 import aggregation as A
    from paper_2508_09208_b200.errors import InfeasibleError
    case = CASES["cases"][i]
    st = _stats(case)
    variants = _host_variants(case)
    for v, ref in zip(variants, case["variants"]):
        got = [[l, s, f] for (l, s), f in sorted(A.variant_freqs(v, st).items())]
        assert got == ref["freqs"]  # same summation order: bit-identical
    lib = A.VariantLibrary(variants=variants)
    assert [v.variant_id for v in lib.variants] == [v["id"] for v in case["variants"]]
    assert json.loads(json.dumps(A.library_manifest(lib))) == case["manifest"]
    for mem, want in case["selects"]:
        if want == "InfeasibleError":
            with pytest.raises(InfeasibleError):
                A.select_variant(lib, mem)
        else:
            assert A.select_variant(lib, mem).variant_id == want


def test_should_switch_cases():
    from paper_2508_09208_b200 import aggregation as A
    for c in CASES["should_switch"]:
        cur = A.ModelVariant(c["cur"], {}, {}, {}, 1.0, 0.5)
        cand = A.ModelVariant(c["cand"], {}, {}, {}, 1.0, 0.5)
        pol = A.SwitchPolicy(c["lambda_switch"], c["switch_cost"], c["t_threshold"])
        if c["out"] == "ValueError":
            with pytest.raises(ValueError):
                A.should_switch(cur, cand, c["delta_p"], pol, c["t_stable"])
        else:
            assert A.should_switch(cur, cand, c["delta_p"], pol, c["t_stable"]) is c["out"]


def test_granularity_decision_cases():
    from paper_2508_09208_b200 import aggregation as A
    for c in CASES["granularity"]:
        if c["out"] == "ValueError":
            with pytest.raises(ValueError):
                A.granularity_decision(*c["args"])
        else:
            assert A.granularity_decision(*c["args"]) == c["out"]


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(CASES["cases"])))
def test_build_library_on_device_matches_reference(i):
    """build_library with the device similarity (K6) and merge (K5) kernels
    builds the reference's variants: groups, slot maps, byte counts and
    scores, hence the same manifest, frequencies and selections."""
    import torch

    from paper_2508_09208_b200 import aggregation as A
    from paper_2508_09208_b200.moe import Calibration, Expert, MoeModel, MoeModelSpec
    case = CASES["cases"][i]
    E = case["E"]
    experts = {}
    for l, P in case["params"].items():
        for s, p in enumerate(P):
            experts[(int(l), s)] = Expert(int(l), s, torch.as_tensor(np.asarray(p), dtype=torch.float64,
                                                                     device="cuda"),
                                          case["sizes"][l][s])
    spec = MoeModelSpec(4, (1,), (3,), E, case["sizes"]["1"][0], 1, len(case["params"]["1"][0]))
    model = MoeModel(spec, experts)
    st = _stats(case)
    calib = Calibration(np.asarray(case["probes"]), np.asarray(case["projection"]))
    scope = case["scope"]
    configs = [A.FusionConfig(mode="fixed", r=0.5, scope=scope),
               A.FusionConfig(mode="fixed", r=0.25, theta_act=0.05, scope=scope),
               A.FusionConfig(mode="adaptive", r_base=0.5, delta_r=0.25, e_min=1, scope=scope)]
    lib = A.build_library(model, st, configs, case["alpha"], calib, case["m_other"])
    assert [v.variant_id for v in lib.variants] == [v["id"] for v in case["variants"]]
    for v, ref in zip(lib.variants, case["variants"]):
        assert {str(l): {str(k): x for k, x in m.items()} for l, m in v.slot_map.items()} == ref["slot_map"]
        assert {str(l): [[g.principal_slot, list(g.member_slots)] for g in gs]
                for l, gs in v.groups.items()} == ref["groups"]
        assert v.mem_required == ref["mem_required"] and v.expert_bytes == ref["expert_bytes"]
        assert v.perf_estimate == pytest.approx(ref["perf_estimate"], rel=1e-9, abs=1e-12)
        got = [[l, s, f] for (l, s), f in sorted(A.variant_freqs(v, st).items())]
        assert got == ref["freqs"]
    for mem, want in case["selects"]:
        if want != "InfeasibleError":
            assert A.select_variant(lib, mem).variant_id == want
