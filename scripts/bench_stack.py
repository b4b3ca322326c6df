"""C3 policy sweep on a multi-layer stack:
four Switch-Base-128 MoE layers, each with an HBM expert cache of 38 of 128
slots (30%) over a pinned-host store, routing replayed from a reference-
identical rho-correlated Zipf trace (traces.generate_routing, rho = 0.9).
For every batch size T and skew s: hit rate, demand fetches, prefetches and
ms per stack forward, without and with the K8 predictor (trained on a
separate trace with the reference's SGD, offload.train_predictor) driving
the resource-aware prefetch of layer l+1 while layer l computes."""
import json
import math
import sys
import time

sys.path.insert(0, __file__.rsplit("/scripts", 1)[0])
import numpy as np
import torch

from paper_2508_09208_b200 import kernels
from paper_2508_09208_b200.cache import CachedMoELayer, ExpertCache
from paper_2508_09208_b200.moe import MoeModelSpec
from paper_2508_09208_b200.offload import OffloadPolicy, train_predictor
from paper_2508_09208_b200.stack import CachedMoEStack, PrefetchGovernor, StackLayer
from paper_2508_09208_b200.traces import RoutingGeneratorSpec, generate_routing

D, D_FF, E, SLOTS, LAYERS = 768, 3072, 128, 38, 4


def main():
    numel = kernels.expert_numel(D, D_FF, kernels.ACT_RELU)
    g = torch.Generator().manual_seed(0)
    hosts = []
    for _ in range(LAYERS):
        h = torch.empty((E, numel), dtype=torch.bfloat16).pin_memory()
        h.normal_(0, 0.02, generator=g)
        hosts.append(h)
    wgs = [(torch.randn(D, E, generator=g) / math.sqrt(D)).cuda() for _ in range(LAYERS)]
    spec = MoeModelSpec(total_layers=LAYERS, encoder_moe_layers=tuple(range(1, LAYERS + 1)),
                        decoder_moe_layers=(), experts_per_layer=E,
                        expert_size_bytes=float(numel * 2), top_k=1, expert_param_dim=numel)
    out = []
    for s in (1.0, 2.0):
        train = generate_routing(RoutingGeneratorSpec(skew=s, rho=0.9, seed=1), spec, 2048)
        mlp, metrics = train_predictor(train, hidden_dim=32, epochs=4)
        for T in (16, 64, 256, 1024):
            n_batches = max(48, min(96, 16384 // T))
            trace = generate_routing(RoutingGeneratorSpec(skew=s, rho=0.9, seed=2), spec,
                                     T * n_batches)
            idx = [torch.as_tensor(trace.expert_indices(l + 1)).cuda() for l in range(LAYERS)]
            emb = torch.as_tensor(np.stack([t.embedding for t in trace.tokens])).cuda()
            ctx = torch.as_tensor(np.stack([t.context for t in trace.tokens])).cuda()
            x = torch.randn(T, D, generator=g).to(torch.bfloat16).cuda()
            for mode in ("off", "on", "governed"):
                predictive = mode != "off"
                layers = []
                for l in range(LAYERS):
                    cache = ExpertCache(hosts[l], layer=l + 1, n_slots=SLOTS, workspace_slots=2)
                    layers.append(StackLayer(l + 1, CachedMoELayer(wgs[l], cache, D_FF,
                                                                   capacity_factor=None)))
                stack = CachedMoEStack(layers, predictor=mlp if predictive else None,
                                       policy=OffloadPolicy(), s_b=1.0, mem_avail=0.3,
                                       mem_total=1.0,
                                       governor=PrefetchGovernor() if mode == "governed" else None)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for b in range(n_batches):
                    sl = slice(b * T, (b + 1) * T)
                    stack.forward(x, emb[sl], ctx[sl],
                                  routings=[(idx[l][sl], None) for l in range(LAYERS)])
                torch.cuda.synchronize()
                dt = (time.perf_counter() - t0) / n_batches
                st = [sl_.layer.cache.stats for sl_ in layers]
                dem, hits = sum(x_.demand for x_ in st), sum(x_.hits for x_ in st)
                out.append({"zipf_s": s, "tokens": T, "batches": n_batches,
                            "predictor": predictive, "mode": mode,
                            "predictor_val_top1": metrics["val_top1"],
                            "hit_rate": hits / max(1, dem),
                            "demand_fetches": sum(x_.fetches for x_ in st),
                            "prefetch_issued": sum(x_.prefetch_issued for x_ in st),
                            "prefetch_hits": sum(x_.prefetch_hits for x_ in st),
                            "h2d_MB_per_batch": sum(x_.h2d_bytes for x_ in st) / n_batches / 1e6,
                            "ms_per_stack_forward": dt * 1e3})
                print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
