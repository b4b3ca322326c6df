"""Receiver-side grouped FFN of expert parallelism at the C4 shape, one GPU
standing in for one rank of world = 8 (16 local experts, 8 source blocks of
C = 640 rows each, ~512 kept): expert-major group order (ep.DeviceOps) vs
source-major (dev tool)."""
import json
import math
import sys

sys.path.insert(0, __file__.rsplit("/scripts", 1)[0])
import torch

from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
from paper_2508_09208_b200.ep import DeviceOps

world, E, d, d_ff, C = 8, 128, 768, 3072, 640
El = E // world
numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
pool = ExpertPool(El, numel)
pool.data.normal_(0, 0.02)
wg = torch.randn(d, E, device="cuda") / math.sqrt(d)
ops = DeviceOps(MoELayer(wg, pool, d_ff, capacity_factor=1.0, expert_slots=[0] * E))
recv = torch.randn(world * El * C, d, device="cuda").to(torch.bfloat16)
counts = torch.randint(480, 545, (world * El,), dtype=torch.int32, device="cuda")
rows = int(counts.sum())
G = world * El
base = torch.arange(G, dtype=torch.int32, device="cuda") * C
slot = (torch.arange(G, dtype=torch.int32, device="cuda") % El).contiguous()
h = torch.empty((recv.shape[0], d_ff), dtype=torch.bfloat16, device="cuda")
y = torch.empty_like(recv)


def source_major():
    kernels.grouped_gemm(recv, pool.data, 0, d_ff, counts, base, slot, kernels.EPI_RELU, h)
    kernels.grouped_gemm(h, pool.data, d_ff * d, d, counts, base, slot, kernels.EPI_STORE, y)


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


out = {"rows": rows}
for name, fn in (("source_major", source_major),
                 ("expert_major", lambda: ops.expert_ffn(recv, counts, El, C, world))):
    ms = timed(fn)
    out[name] = {"ms": round(ms, 4), "TFLOPs": round(2 * 2 * rows * d * d_ff / ms / 1e9, 1)}
print(json.dumps(out))
