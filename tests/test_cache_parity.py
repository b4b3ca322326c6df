"""Cache-policy decision parity with the reference runtime (SURVEY §8a
a14-a24, §8f rank 3).

tests/golden/cache_parity.json holds the reference simulator's own
per-token decision stream (simulator.py:684-724: _serve_demand,
_predict_and_prefetch, _room_in_workspace, _evict_from_cache) on a small
scenario (3 MoE layers x 8 experts, 13-expert HBM budget, decoder layer
pinned, MLP predictor, substitution), recorded by oracle/gen_golden.py from
the unmodified reference, together with every input of those decisions.

Here the same token stream runs through the B200 runtime at one token per
step: a CachedMoEStack of CachedMoELayers sharing ONE ExpertCache (the
reference's single CacheState over all layers), routing replayed from the
trace, the K8 device predictor on the token's choices, real H2D copies. The
cache's JSONL event log must equal the reference's hit / fetch / substitute
/ prefetch / demote / evict records one for one (tick, kind, expert, tiers,
substitute used), and so must the hit / prefetch / substitution counts.
"""

import json
import math

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

CASE = json.loads((GOLDEN / "cache_parity.json").read_text())


def _eid(k):
    a, b = k.split(",")
    return int(a), int(b)


def _run_case(d=256, d_ff=256):
    from paper_2508_09208_b200 import kernels
    from paper_2508_09208_b200.cache import CachedMoELayer, ExpertCache
    from paper_2508_09208_b200.offload import OffloadPolicy, PredictorMLP
    from paper_2508_09208_b200.stack import CachedMoEStack, StackLayer
    c = CASE
    E = 8
    layers = c["layers"]
    g = torch.Generator().manual_seed(0)
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
    hosts = {l: (torch.randn(E, numel, generator=g) * 0.02).to(torch.bfloat16).pin_memory()
             for l in layers}
    pol = c["policy"]
    policy = OffloadPolicy(threshold_mode="constant", theta_base=pol["theta_base"],
                           delta_evict=pol["delta_evict"], lambda_evict=pol["lambda_evict"],
                           substitution_sim_min=pol["substitution_sim_min"])
    sims = {int(l): np.asarray(m) for l, m in c["similarity"].items()}
    cap = c["capacities"]
    ws_slots = int(round(cap["workspace"] / 1e6))
    n_slots = ws_slots + int(round(cap["cache"] / 1e6))
    cache = ExpertCache(hosts, n_slots=n_slots, workspace_slots=ws_slots, policy=policy,
                        freqs={_eid(k): v for k, v in c["freqs"].items()},
                        pinned={_eid(k) for k in c["hard_pinned"]}, substitution=True,
                        similarity=lambda a, b: float(sims[a[0]][a[1], b[1]]),
                        priorities={_eid(k): v for k, v in c["priorities"].items()},
                        priority_threshold=c["prio_threshold"], half_life=pol["half_life"])
    # the reference's initial placement (plan_initial_placement + build_cache_state)
    assert [list(e) for e in cache.state.workspace] == [list(_eid(k)) for k in c["initial"]["workspace"]]
    assert sorted(cache.state.cache) == sorted(_eid(k) for k in c["initial"]["cache"])
    enc = set(c["encoder_layers"])
    stack_layers = []
    for l in layers:
        wg = (torch.randn(d, E, generator=g) / math.sqrt(d)).cuda()
        cl = CachedMoELayer(wg, cache, d_ff, capacity_factor=1.0, layer=l)
        stack_layers.append(StackLayer(l, cl, encoder=l in enc))
    p = c["predictor"]
    mlp = PredictorMLP(w1=np.asarray(p["w1"]), b1=np.asarray(p["b1"]), w2=np.asarray(p["w2"]),
                       b2=np.asarray(p["b2"]), experts_per_layer=E, embed_dim=p["embed_dim"],
                       context_dim=p["context_dim"])
    stack = CachedMoEStack(stack_layers, predictor=mlp, policy=policy, theta=pol["theta_base"])
    one = torch.ones((1, 1), dtype=torch.float32, device="cuda")
    for t, tok in enumerate(c["tokens"]):
        x = torch.randn(1, d, generator=g).to(torch.bfloat16).cuda()
        routings = [(torch.tensor([tok["experts"][str(l)]], dtype=torch.int32, device="cuda"), one)
                    for l in layers]
        emb = torch.tensor([tok["embedding"]], dtype=torch.float64, device="cuda")
        ctx = torch.tensor([tok["context"]], dtype=torch.float64, device="cuda")
        stack.forward(x, emb, ctx, routings=routings, tick=t)
    torch.cuda.synchronize()
    cache.check()
    return cache


def _decision(rec):
    return (rec["tick"], rec["event"], tuple(rec["expert"]), rec["tier_from"], rec["tier_to"],
            tuple(rec["used"]) if "used" in rec else None)


def test_cache_decisions_match_reference_runtime(tmp_path):
    cache = _run_case()
    ours = [_decision(r) for r in cache.log.records]
    ref = [_decision(r) for r in CASE["events"]]
    first = next((i for i, (a, b) in enumerate(zip(ours, ref)) if a != b), None)
    assert first is None and len(ours) == len(ref), \
        f"first difference at {first}: ours {ours[first] if first is not None else None} " \
        f"ref {ref[first] if first is not None else None}; {len(ours)} vs {len(ref)} events"
    rep = CASE["report"]
    st = cache.stats
    assert (st.demand, st.hits, st.prefetch_issued, st.prefetch_hits, st.substitutions) == \
        (rep["demand_count"], rep["hit_count"], rep["prefetch_issued"],
         rep["prefetch_hit_count"], rep["substitution_count"])
    assert st.hit_rate() == pytest.approx(rep["hit_rate"], abs=0)
    # the JSONL log round-trips through the reference's reader format
    path = tmp_path / "events.jsonl"
    cache.log.write_jsonl(str(path))
    back = [json.loads(line) for line in path.read_text().splitlines()]
    assert back == cache.log.records
    assert all(list(r) == ["tick", "event", "seq"] + sorted(set(r) - {"tick", "event", "seq"})
               for r in back)
