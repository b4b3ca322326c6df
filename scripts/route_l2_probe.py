"""Gate -> permute L2 reuse of x (dev probe): the C2 layer's route and
permute stages timed back to back with CUDA events (eager forward, no
flush between the two kernels), under the env variants COMOE_GATE_XPOL
(L2 policy of the gate's x loads) and COMOE_PERMUTE_REV (permute walks
the tokens last-to-first, i.e. most recently loaded rows first). One JSON
line: median µs per stage over REPS forwards."""
import json
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_09208_b200 import ExpertPool, MoELayer

T, D, F, E = 65536, 768, 3072, 128
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(T, D, device=dev, generator=g).to(torch.bfloat16)
wg = torch.randn(D, E, device=dev, generator=g) / math.sqrt(D)
pool = ExpertPool(E, 2 * D * F, device=dev)
pool.data.normal_(0, 0.02, generator=g)
layer = MoELayer(wg, pool, F, capacity_factor=1.25)
y = torch.empty_like(x)
ev = {}


class Stage:
    def __init__(self, name):
        self.name = name

    def __enter__(self):
        self.a = torch.cuda.Event(enable_timing=True)
        self.a.record()

    def __exit__(self, *exc):
        b = torch.cuda.Event(enable_timing=True)
        b.record()
        ev.setdefault(self.name, []).append((self.a, b))


for _ in range(3):
    layer.forward(x, out=y)
torch.cuda.synchronize()
reps = int(os.environ.get("REPS", "30"))
for _ in range(reps):
    layer.forward(x, out=y, timer=Stage)
torch.cuda.synchronize()
out = {k: round(statistics.median(a.elapsed_time(b) for a, b in v) * 1e3, 1) for k, v in ev.items()}
out["env"] = {k: v for k, v in os.environ.items() if k.startswith("COMOE_")}
print(json.dumps(out))
