"""Live variant switching at Switch-Base-128 scale: one
MoE layer (128 experts, d 768, d_ff 3072), a library of the original model
and two CoMoE-fused variants (128 -> 64 -> 32, cosine grouping, merged on
the device with K5), and a memory trace that forces a switch down and then
allows one back up. Reports, per switch, the bytes copied host -> HBM for
the new variant's resident experts and the rebuild time (policy + copies,
synchronised), plus the layer forward time after each switch. The trace is
replayed twice; the second (warm) pass is reported."""
import json
import math
import sys
import time

sys.path.insert(0, __file__.rsplit("/scripts", 1)[0])
import torch

from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
from paper_2508_09208_b200 import aggregation as A
from paper_2508_09208_b200.cache import required_bytes_fn
from paper_2508_09208_b200.moe import (Expert, MoeModel, MoeModelSpec, cosine_only_calibration,
                                       stats_from_routing)
from paper_2508_09208_b200.switching import VariantController

T, D, D_FF, E = 4096, 768, 3072, 128


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(T, D, device="cuda", generator=g).to(torch.bfloat16)
    wg = torch.randn(D, E, device="cuda", generator=g) / math.sqrt(D)
    numel = kernels.expert_numel(D, D_FF, kernels.ACT_RELU)
    pool = ExpertPool(E + 96, numel)
    for s in range(E):
        v = pool.view(pool.alloc())
        v.normal_(0.0, 0.02, generator=g)
    for s in range(E):
        pool.view(s).add_(pool.view(s % 16), alpha=0.5)
    ref = MoELayer(wg, pool, D_FF, capacity_factor=1.25)
    stats = stats_from_routing({1: ref.route(x).gate.expert_idx}, E)
    eb = float(pool.slot_bytes)
    spec = MoeModelSpec(1, (1,), (), E, eb, 1, numel)
    model = MoeModel(spec, {(1, s): Expert(1, s, pool.view(s), eb) for s in range(E)})
    t0 = time.perf_counter()
    lib = A.build_library(model, stats, [A.FusionConfig(mode="fixed", r=0.5),
                                         A.FusionConfig(mode="fixed", r=0.25)],
                          1.0, cosine_only_calibration(), pool=pool)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    stores = {}
    for v in lib.variants:
        _, principals = v.group_table(1, E)
        stores[v.variant_id] = {1: torch.stack([v.retained[1][p].params.cpu() for p in principals])
                                .contiguous().pin_memory()}
    total = E * eb
    req = required_bytes_fn("fraction_of_variant", 0.3, total, 0.0, 2 * eb)
    ctl = VariantController(lib, stats, stores, {1: (wg, D_FF)}, D_FF,
                            policy=A.SwitchPolicy(lambda_switch=0.5, switch_cost=0.05,
                                                  t_threshold=2.0),
                            reeval_interval=2, required_bytes=req)

    def fwd_ms():
        ctl.forward(x, 1)
        torch.cuda.synchronize()
        a = time.perf_counter()
        for _ in range(5):
            ctl.forward(x, 1)
        torch.cuda.synchronize()
        return (time.perf_counter() - a) / 5 * 1e3

    out = {"library_build_s": build_s,
           "variants": [{"id": v.variant_id, "experts": len(v.retained[1]),
                         "perf_estimate": v.perf_estimate, "resident_bytes_required": req(v)}
                        for v in lib.variants]}
    ev = ctl.start(req(max(lib.variants, key=lambda v: req(v))))
    out["start"] = {"variant": ev.variant_to, "h2d_MB": ev.migrated_bytes / 1e6,
                    "rebuild_ms": ev.seconds * 1e3, "forward_ms": fwd_ms()}
    high = req(max(lib.variants, key=lambda v: req(v)))
    mid = sorted(req(v) for v in lib.variants)[1] * 1.01
    low = min(req(v) for v in lib.variants) * 1.01
    trace = [high, low, low, low, mid, mid, mid, mid, mid, high, high, high, high, high]
    # pass 1 warms allocator pools, events and kernels; pass 2 is reported
    for rep in range(2):
        switches = []
        for t, m in enumerate(trace, start=1 + rep * 100):
            e = ctl.tick(t, m)
            if e is not None:
                switches.append({"tick": t, "from": e.variant_from, "to": e.variant_to,
                                 "forced": e.forced, "h2d_MB": e.migrated_bytes / 1e6,
                                 "rebuild_ms": e.seconds * 1e3,
                                 "h2d_GBps": e.migrated_bytes / e.seconds / 1e9,
                                 "forward_ms_after": fwd_ms()})
    out["switches"] = switches
    print(json.dumps(out))


if __name__ == "__main__":
    main()
