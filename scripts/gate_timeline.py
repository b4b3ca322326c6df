"""Gate (K1, folded route) timeline at the C2 shape (dev probe): with
COMOE_GATE_DEBUG=256 CTAs 0 and 1 (one CTA pair) stamp clock64 at their
producer, MMA and epilogue progress points per unit (plain stores, no
atomics); this prints [name, unit iteration, cycles since the CTA's entry].
One JSON line per CTA and launch."""
import ctypes
import json
import math
import os
import sys

os.environ["COMOE_GATE_DEBUG"] = "256"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_09208_b200 import ExpertPool, MoELayer, _lib, kernels

T, d, d_ff, E = 65536, 768, 3072, 128
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(T, d, device=dev, generator=g).to(torch.bfloat16)
wg = torch.randn(d, E, device=dev, generator=g) / math.sqrt(d)
pool = ExpertPool(E, kernels.expert_numel(d, d_ff, kernels.ACT_RELU), device=dev)
for _ in range(E):
    pool.alloc()
layer = MoELayer(wg, pool, d_ff, act="relu", top_k=1, capacity_factor=1.25)
ws = layer._workspace(T)
lbw = kernels.gate_route_workspace(T, 1, E, dev)
run = lambda: kernels.gate_route(x, layer.wg_split, E, 1, False, ws["C"], lbw,
                                 slot_map=layer.slot_map, n_groups=E, out=ws["gate"],
                                 scan=ws["scan"])
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
NAMES = {1: "prologue_done", 2: "prod_kb0", 3: "prod_kblast", 4: "mma_tempty", 5: "mma_full0",
         6: "mma_commit", 7: "epi0_tfull", 8: "epi0_release", 9: "epi0_done", 15: "epi1_tfull",
         16: "epi1_release", 17: "epi1_done", 13: "stash_full", 14: "tok_read", 15: "tok_partial",
         18: "xch_got", 19: "ranks_bar", 10: "loop_end", 11: "cluster_sync", 12: "scan_done"}
buf = (ctypes.c_ulonglong * 2048)()
cnt = (ctypes.c_uint * 2)()
for rep in range(3):
    flush.fill_(1)
    torch.cuda._sleep(400_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _lib.call("comoe_debug_gate_timeline", buf, cnt)  # reset
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3
    _lib.call("comoe_debug_gate_timeline", buf, cnt)
    for c in range(2):
        recs = []
        for idx in range(1024):
            v = buf[c * 1024 + idx]
            if v:
                recs.append((v - 1, idx // 32, idx % 32))
        recs.sort()
        end = max(r[0] for r in recs) if recs else 1
        print(json.dumps({"rep": rep, "cta": c, "event_us": round(us, 1), "cycles_total": end,
                          "events": [[NAMES.get(k, k), it, t] for t, k, it in recs]}))
