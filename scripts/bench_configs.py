"""BASELINE.json configs other than the bench.py headline (C2):

C1  Switch-Base-8 layer (d 768, d_ff 3072, 8 experts, top-1) on 4096 tokens
    with CoMoE merging 8 -> 4 (device similarity + one merge launch).
C5  Mixtral-8x7B-shaped layer (d 4096, d_ff 14336, 8 experts, top-2,
    SwiGLU) with the merge sweep 8 -> 4 -> 2 (cosine-only similarity: the
    reference's n x D fp64 calibration is 11 GB per matrix at D = 176M).

Per config: similarity time (device; the first call also uploads the
calibration), merge kernel time and achieved GB/s over the
algorithmic bytes sum_{|g|>=2} (|g|+1)*expert_bytes (vs measured HBM peak),
and layer tokens/s for every variant. Prints one JSON line per measurement.
"""
import json
import math
import sys
import time

sys.path.insert(0, __file__.rsplit("/scripts", 1)[0])
import numpy as np
import torch

from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
from paper_2508_09208_b200 import aggregation as A
from paper_2508_09208_b200.moe import (Expert, MoeModel, MoeModelSpec, cosine_only_calibration,
                                       make_calibration, similarity_matrix, stats_from_routing)

HBM = json.load(open(__file__.rsplit("/scripts", 1)[0] + "/MEASURED_PEAKS.json")).get("hbm_gbs", 6549.4) \
    if __import__("os").path.exists(__file__.rsplit("/scripts", 1)[0] + "/MEASURED_PEAKS.json") else 6549.4


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def run_config(name, d, d_ff, E, top_k, act, T, ratios, calib_kind):
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(T, d, device=dev, generator=g).to(torch.bfloat16)
    wg = torch.randn(d, E, device=dev, generator=g) / math.sqrt(d)
    a = kernels.ACT_SWIGLU if act == "swiglu" else kernels.ACT_RELU
    numel = kernels.expert_numel(d, d_ff, a)
    n_slots = E + sum(max(1, int(E * r)) for r in ratios)
    pool = ExpertPool(n_slots, numel, device=dev)
    for s in range(E):
        pool.view(s).normal_(0.0, 0.02, generator=g)
    for s in range(E):  # experts share structure so grouping is non-trivial
        pool.view(s).add_(pool.view(s % max(1, E // 2)), alpha=0.5)
    for _ in range(E):
        pool.alloc()  # slots 0..E-1 hold the originals
    layer = MoELayer(wg, pool, d_ff, act=act, top_k=top_k, capacity_factor=1.25)
    ebytes = pool.slot_bytes
    out = []
    ms = timed(lambda: layer.forward(x))
    flops = 2.0 * T * top_k * (numel)
    # device time: the same forward as one CUDA-graph replay (no per-launch
    # host overhead, which dominates the eager small-batch C1 figure)
    y = torch.empty_like(x)
    cap = layer.capture(x, y)
    ms_g = timed(cap.replay, reps=20)
    out.append({"config": name, "variant": f"original-{E}", "tokens": T, "ms": ms,
                "tokens_per_s": T / ms * 1e3, "expert_tflops": flops / ms / 1e9,
                "graph_ms": ms_g, "graph_tokens_per_s": T / ms_g * 1e3,
                "graph_expert_tflops": flops / ms_g / 1e9})
    # activation statistics from the device router
    r = layer.route(x)
    stats = stats_from_routing({1: r.gate.expert_idx}, E)
    spec = MoeModelSpec(total_layers=1, encoder_moe_layers=(1,), decoder_moe_layers=(),
                        experts_per_layer=E, expert_size_bytes=float(ebytes), top_k=top_k,
                        expert_param_dim=numel)
    model = MoeModel(spec, {(1, s): Expert(1, s, pool.view(s), float(ebytes)) for s in range(E)})
    calib = cosine_only_calibration() if calib_kind == "cosine" else make_calibration(numel, 8, 7, 8)
    alpha = 1.0 if calib_kind == "cosine" else 0.5
    experts = model.layer_experts(1)
    t0 = time.perf_counter()
    sim = similarity_matrix(experts, alpha, calib)  # first call: uploads the calibration
    sim_first_ms = (time.perf_counter() - t0) * 1e3
    sim_ms = timed(lambda: similarity_matrix(experts, alpha, calib), reps=3)
    for ratio in ratios:
        cfg = A.FusionConfig(mode="fixed", r=ratio)
        target = A.fixed_retention(E, ratio)
        principals = A.identify_principals(stats, 1, target)
        groups = A.group_experts(experts, principals, sim)
        by_slot = {e.slot: e for e in experts}
        multi = [gr for gr in groups if gr.member_slots]
        mbytes = sum((1 + len(gr.member_slots) + 1) * ebytes for gr in multi)
        # time the one-launch merge of this layer (outputs into scratch slots)
        scratch = [pool.view(pool.alloc()) for _ in multi]
        freqs = stats.freqs(1)
        mem = [[by_slot[s].params for s in gr.slots] for gr in multi]
        wts, divs = [], []
        for gr in multi:
            w, dv = A._merge_weights(freqs, gr.slots)
            wts.append(w)
            divs.append(dv)
        plan = kernels.MergePlan(mem, wts, divs, scratch, torch.bfloat16)
        merge_ms = timed(plan.run) if multi else 0.0
        for s_ in scratch:
            pool.release(pool.slot_of(s_))
        var = A.fuse_model(model, stats, cfg, alpha, calib, pool=pool)
        layer.use_variant(var, 1)
        ms_v = timed(lambda: layer.forward(x))
        cap_v = layer.capture(x, y)
        ms_vg = timed(cap_v.replay, reps=20)
        out.append({"config": name, "variant": var.variant_id, "experts_after": target,
                    "graph_ms": ms_vg, "graph_tokens_per_s": T / ms_vg * 1e3,
                    "groups": {g_.principal_slot: list(g_.member_slots) for g_ in groups},
                    "similarity_ms": sim_ms, "similarity_first_call_ms": sim_first_ms,
                    "merge_ms": merge_ms, "merge_bytes": mbytes,
                    "merge_GBps": mbytes / (merge_ms * 1e-3) / 1e9 if merge_ms else None,
                    "merge_frac_of_hbm": (mbytes / (merge_ms * 1e-3) / 1e9) / HBM if merge_ms else None,
                    "tokens": T, "ms": ms_v, "tokens_per_s": T / ms_v * 1e3,
                    "perf_estimate": var.perf_estimate})
        layer.set_variant(list(range(E)), list(range(E)))
    return out


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c5"]
    res = []
    if "c1" in which:
        res += run_config("C1 sb8", 768, 3072, 8, 1, "relu", 4096, [0.5], "probes")
    if "c5" in which:
        res += run_config("C5 mixtral", 4096, 14336, 8, 2, "swiglu", 8192, [0.5, 0.25], "cosine")
    for r in res:
        print(json.dumps(r))
