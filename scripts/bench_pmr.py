"""Measured performance-memory ratio (the reference's headline metric,
compute_pmr, pkg/src/comoe/simulator.py:207-214: tokens per millisecond per
GB of peak memory) of the Switch-Base-128 layer on one B200, under the three
memory regimes CoMoE trades between:
  original   all 128 experts HBM-resident;
  variant    CoMoE merge 128 -> 64 and 128 -> 32 (device similarity + merges,
             fuse_model), the retained experts resident;
  cached     the original experts over a pinned-host store with 38 of 128
             HBM slots (30%), demand/prefetch copies inside the timed forward.
Memory = expert bytes resident in HBM (what the reference's peak_mem_bytes
counts: pool slots, cache + workspace slots). Time = wall time per forward (synchronised). Skewed routing (Zipf
s = 1 gate bias) so small batches touch few experts. Prints one
JSON line per (regime, tokens)."""
import json
import math
import sys
import time

sys.path.insert(0, __file__.rsplit("/scripts", 1)[0])
import numpy as np
import torch

from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
from paper_2508_09208_b200 import aggregation as A
from paper_2508_09208_b200.cache import CachedMoELayer, ExpertCache
from paper_2508_09208_b200.moe import (Expert, MoeModel, MoeModelSpec, cosine_only_calibration,
                                       stats_from_routing)

D, D_FF, E, SLOTS = 768, 3072, 128, 38
TOKENS = (64, 1024, 65536)


def inputs(T, wg_base=None):
    g = torch.Generator(device="cuda").manual_seed(T)
    x = torch.randn(T, D, device="cuda", generator=g).to(torch.bfloat16)
    x[:, 0] = 1.0
    return x


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


SKEW = 0.0


def line(regime, T, sec, expert_bytes, extra=None):
    tpm = T / (sec * 1e3)
    r = {"skew": SKEW, "regime": regime, "tokens": T, "ms_per_forward": sec * 1e3, "tokens_per_ms": tpm,
         "expert_bytes_resident": expert_bytes, "pmr": tpm / (expert_bytes / 1e9)}
    r.update(extra or {})
    print(json.dumps(r), flush=True)


def main(skew):
    global SKEW
    SKEW = skew
    numel = kernels.expert_numel(D, D_FF, kernels.ACT_RELU)
    ebytes = numel * 2
    g = torch.Generator(device="cuda").manual_seed(1)
    wg = torch.randn(D, E, device="cuda", generator=g) / math.sqrt(D)
    perm = np.random.default_rng(0).permutation(E)
    bias = np.empty(E)
    bias[perm] = -skew * np.log(np.arange(1, E + 1))
    wg[0, :] = torch.as_tensor(bias, dtype=torch.float32, device="cuda")
    host = torch.empty((E, numel), dtype=torch.bfloat16).pin_memory()
    host.normal_(0, 0.02, generator=torch.Generator().manual_seed(2))

    # original, all resident (+ slots for the merged experts of the variants)
    pool = ExpertPool(E + 96, numel, device="cuda")
    pool.data[:E].copy_(host.cuda())
    for _ in range(E):
        pool.alloc()
    layer = MoELayer(wg, pool, D_FF, capacity_factor=1.25)
    for T in TOKENS:
        x = inputs(T, wg)
        sec = timed(lambda: layer.forward(x), 10)
        line("original", T, sec, E * ebytes)

    # CoMoE variants from the layer's own routing statistics (device similarity
    # and merges, fuse_model), retained experts resident
    x = inputs(65536, wg)
    r = layer.route(x)
    stats = stats_from_routing({1: r.gate.expert_idx}, E)
    spec = MoeModelSpec(total_layers=1, encoder_moe_layers=(1,), decoder_moe_layers=(),
                        experts_per_layer=E, expert_size_bytes=float(ebytes), top_k=1,
                        expert_param_dim=numel)
    model = MoeModel(spec, {(1, s): Expert(1, s, pool.view(s), float(ebytes)) for s in range(E)})
    for ratio in (0.5, 0.25):
        var = A.fuse_model(model, stats, A.FusionConfig(mode="fixed", r=ratio), 1.0,
                           cosine_only_calibration(), pool=pool)
        layer.use_variant(var, 1)
        kept = A.fixed_retention(E, ratio)
        for T in TOKENS:
            xt = inputs(T, wg)
            sec = timed(lambda: layer.forward(xt), 10)
            line(f"variant-{kept}", T, sec, kept * ebytes, {"perf_estimate": var.perf_estimate})
        layer.set_variant(list(range(E)), list(range(E)))

    # cached original: 38 HBM slots over the pinned host store
    for T in TOKENS:
        cache = ExpertCache(host, layer=1, n_slots=SLOTS, workspace_slots=2)
        cl = CachedMoELayer(wg, cache, D_FF, capacity_factor=1.25)
        xt = inputs(T, wg)
        sec = timed(lambda: cl.forward(xt), 5)
        line("cached-30pct", T, sec, (SLOTS + 2) * ebytes, {"hit_rate": cache.stats.hit_rate()})


if __name__ == "__main__":
    for s_ in (0.0, 1.0):
        main(s_)
