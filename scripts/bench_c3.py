"""C3: Switch-Base-128 layer with an HBM expert cache at 30% of experts
(38 of 128 slots, pinned-host master copies), random-init weights.

Reports per batch size: layer tokens/s (compute stream, includes demand
copies and the demand-set host sync), achieved H2D GB/s while streaming,
hit rate and waves. T=65536 is the pure-bandwidth point (every expert is
demanded); small batches with Zipf-skewed routing are where the policy
matters."""
import json, math, sys, time
sys.path.insert(0, __file__.rsplit("/scripts", 1)[0])
import numpy as np
import torch
from paper_2508_09208_b200 import kernels
from paper_2508_09208_b200.cache import CachedMoELayer, ExpertCache

D, D_FF, E, SLOTS = 768, 3072, 128, 38


def run(T, skew, reps=5):
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(T, D, device="cuda", generator=g).to(torch.bfloat16)
    wg = torch.randn(D, E, device="cuda", generator=g) / math.sqrt(D)
    if skew:
        perm = np.random.default_rng(0).permutation(E)
        bias = np.empty(E); bias[perm] = -skew * np.log(np.arange(1, E + 1))
        x[:, 0] = 1.0
        wg[0, :] = torch.as_tensor(bias, dtype=torch.float32, device="cuda")
    numel = kernels.expert_numel(D, D_FF, kernels.ACT_RELU)
    host = torch.empty((E, numel), dtype=torch.bfloat16).pin_memory()
    host.normal_(0, 0.02)
    cache = ExpertCache(host, layer=1, n_slots=SLOTS, workspace_slots=2)
    layer = CachedMoELayer(wg, cache, D_FF, capacity_factor=1.25)
    layer.forward(x); torch.cuda.synchronize()
    b0, t0, h0, d0 = cache.stats.h2d_bytes, time.perf_counter(), cache.stats.hits, cache.stats.demand
    for _ in range(reps):
        layer.forward(x)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    nb = (cache.stats.h2d_bytes - b0) / reps
    return {"tokens": T, "zipf_s": skew, "ms_per_forward": dt * 1e3, "tokens_per_s": T / dt,
            "h2d_MB_per_forward": nb / 1e6, "h2d_GBps": nb / dt / 1e9 if nb else 0.0,
            "hit_rate": (cache.stats.hits - h0) / max(1, cache.stats.demand - d0),
            "waves_total": cache.stats.waves}


if __name__ == "__main__":
    out = [run(65536, 0.0, reps=3)]
    for s in (1.0, 2.0):
        for T in (64, 256, 1024):
            out.append(run(T, s))
    for r in out:
        print(json.dumps(r))
