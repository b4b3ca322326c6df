"""Routing traces and predictor training vs reference-generated fixtures
(tests/golden/traces.json, oracle/gen_golden.py). CPU only."""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2508_09208_b200 import offload as off
from paper_2508_09208_b200 import presets
from paper_2508_09208_b200.moe import (MoeModelSpec, RoutingGeneratorSpec, collect_stats,
                                       generate_routing, trace_from_jsonl, trace_to_jsonl)

CASES = json.loads((GOLDEN / "traces.json").read_text())


def _spec(c):
    return MoeModelSpec(total_layers=6, encoder_moe_layers=(1, 3), decoder_moe_layers=(5,),
                        experts_per_layer=c["E"], expert_size_bytes=1e6, top_k=c["K"])


def _gspec(c):
    skew = c["skew"]
    if isinstance(skew, dict):
        skew = {("default" if k == "default" else int(k)): v for k, v in skew.items()}
    return RoutingGeneratorSpec(skew=skew, rho=c["rho"], seed=c["seed"],
                                structure_seed=c["structure_seed"])


@pytest.mark.parametrize("c", CASES, ids=lambda c: f"E{c['E']}k{c['K']}")
def test_generate_routing_matches_reference(c):
    spec = _spec(c)
    tr = generate_routing(_gspec(c), spec, c["n"])
    got = [[list(tok.layer_experts[l]) for l in spec.moe_layer_indices] for tok in tr.tokens]
    assert got == c["experts"]
    assert sum(float(t.embedding.sum()) for t in tr.tokens) == pytest.approx(c["emb_sum"], rel=1e-12)
    assert sum(float(t.context.sum()) for t in tr.tokens) == pytest.approx(c["ctx_sum"], rel=1e-12)


def test_train_predictor_matches_reference():
    c = CASES[0]
    p = c["predictor"]
    tr = generate_routing(_gspec(c), _spec(c), p["n"])
    mlp, metrics = off.train_predictor(tr, hidden_dim=p["hidden"], lr=0.05, epochs=p["epochs"],
                                       seed=p["seed"])
    for name in ("w1", "b1", "w2", "b2"):
        np.testing.assert_allclose(getattr(mlp, name), np.asarray(p[name]), rtol=1e-12, atol=1e-14)
    for k in ("samples", "train_top1", "val_top1", "val_top3"):
        assert metrics[k] == pytest.approx(p["metrics"][k], rel=1e-12)


def test_trace_jsonl_roundtrip_and_stats(tmp_path):
    c = CASES[1]
    tr = generate_routing(_gspec(c), _spec(c), 25)
    path = tmp_path / "t.jsonl"
    trace_to_jsonl(tr, str(path))
    back = trace_from_jsonl(str(path), experts_per_layer=c["E"])
    assert [t.layer_experts for t in back.tokens] == [t.layer_experts for t in tr.tokens]
    assert back.top_k == c["K"]
    st = collect_stats(back)
    for l in back.moe_layer_indices:
        assert st.totals[l] == 25 * c["K"]
        assert st.counts[l].sum() == 25 * c["K"]
    assert tr.expert_indices(1).shape == (25, c["K"])


def test_presets():
    g = presets.preset_geometry("sb128")
    assert g["experts_per_layer"] == 128 and g["top_k"] == 1
    b = presets.expert_size_bytes(g["total_params"], 2.0, 12, 128)
    assert abs(b - 9_635_416.67) < 1
    with pytest.raises(Exception):
        presets.preset_geometry("sb7")


@pytest.mark.parametrize("c", CASES, ids=lambda c: f"E{c['E']}k{c['K']}")
def test_collect_stats_matches_reference(c):
    """a3: collect_stats (moe.py:250-262) of the reference-identical trace
    equals the reference's own ActivationStats (traces.json)."""
    tr = generate_routing(_gspec(c), _spec(c), c["n"])
    st = collect_stats(tr)
    ref = c["collect_stats"]
    for l in tr.moe_layer_indices:
        np.testing.assert_array_equal(st.counts[l], np.asarray(ref["counts"][str(l)]))
        assert st.totals[l] == ref["totals"][str(l)]
