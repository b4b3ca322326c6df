"""Gate (K1) alone at the C2 shape: CUDA-event time with an L2 flush before
each launch, for A/B of gate variants (env COMOE_GATE_*) and as the target
of `ncu -k regex:gate_kernel`. Prints one JSON line."""
import json
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels

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
mode = os.environ.get("MODE", "topk")  # topk | scan (topk + route_scan) | route (folded)
lbw = kernels.gate_route_workspace(T, 1, E, dev)
C = ws["C"]
if mode == "route":
    run = lambda: kernels.gate_route(x, layer.wg_split, E, 1, False, C, lbw,
                                     slot_map=layer.slot_map, n_groups=E, out=ws["gate"],
                                     scan=ws["scan"])
elif mode == "scan":
    def run():
        kernels.gate_topk(x, layer.wg_split, E, 1, False, slot_map=layer.slot_map, n_groups=E,
                          out=ws["gate"])
        kernels.route_scan(ws["gate"].tile_hist, C, out=ws["scan"])
else:
    run = lambda: kernels.gate_topk(x, layer.wg_split, E, 1, False, slot_map=layer.slot_map,
                                    n_groups=E, out=ws["gate"])
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
reps = int(os.environ.get("REPS", "30"))
run()
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    flush.fill_(1)
    torch.cuda._sleep(400_000)  # keep the GPU busy while the host prepares the launch
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = statistics.median(ts)
ref = kernels.gate_topk(x, layer.wg_split, E, 1, False, slot_map=layer.slot_map, n_groups=E)
print(json.dumps({"kernel": "gate", "mode": mode, "min_us": min(ts) * 1e3, "us": ms * 1e3, "GBps": T * d * 2 / (ms * 1e-3) / 1e9,
                  "env": {k: v for k, v in os.environ.items() if k.startswith("COMOE_")}}))
