"""C2 layer: one CUDA-graph replay of the forward against the sum of its
kernels, each timed alone back to back (dev probe): the difference is what
kernel boundaries cost inside the graph (launch latency, prologue, ramp-up /
tail). Run once per COMOE_PDL setting; env T / E pick the batch and the
expert count (default the C2 shape; T=4096 E=8 is C1). One JSON line, µs."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels

T = int(os.environ.get("T", "65536"))
E = int(os.environ.get("E", "128"))
D, F = 768, 3072
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(T, D, device=dev, generator=g).to(torch.bfloat16)
wg = torch.randn(D, E, device=dev, generator=g) / math.sqrt(D)
pool = ExpertPool(E, 2 * D * F, device=dev)
pool.data.normal_(0, 0.02, generator=g)
layer = MoELayer(wg, pool, F, capacity_factor=1.25)
y = torch.empty_like(x)
layer.forward(x, out=y)
torch.cuda.synchronize()
ws = layer._workspace(T)
r = layer.last


def timed(fn, n=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


cap = layer.capture(x, y)
out = {"graph_us": timed(cap.replay)}
out["route_us"] = timed(lambda: layer.route(x))
out["permute_us"] = timed(lambda: kernels.permute(x, r.gate, r.scan, r.capacity, r.rows,
                                                  y_zero=y, out=r.perm))
out["ffn1_us"] = timed(lambda: kernels.grouped_gemm(r.perm.x_perm, pool.data, 0, F, r.scan.group_kept,
                                                    r.scan.group_base, layer.group_slot,
                                                    kernels.EPI_RELU, ws["h"]))
out["ffn2_us"] = timed(lambda: kernels.grouped_gemm(ws["h"], pool.data, F * D, D, r.scan.group_kept,
                                                    r.scan.group_base, layer.group_slot,
                                                    kernels.EPI_SCALE_SCATTER, y,
                                                    row_token=r.perm.row_token,
                                                    row_prob=r.perm.row_prob))
out["sum_us"] = out["route_us"] + out["permute_us"] + out["ffn1_us"] + out["ffn2_us"]
out["graph_minus_sum_us"] = out["graph_us"] - out["sum_us"]
out["env"] = {k: v for k, v in os.environ.items() if k.startswith("COMOE_")}
out["T"], out["E"] = T, E
print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in out.items()}))
