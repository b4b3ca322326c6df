"""Layer latency at small token counts (decode-like batches) on the C2
layer (E=128, all experts resident): eager forward vs one CUDA-graph replay,
per-stage eager times. Prints one JSON line per token count."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_09208_b200 import ExpertPool, MoELayer

d, d_ff, E = 768, 3072, 128
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
wg = torch.randn(d, E, device=dev, generator=g) / math.sqrt(d)
pool = ExpertPool(E, 2 * d * d_ff, device=dev)
pool.data.normal_(0.0, 0.02, generator=g)
for _ in range(E):
    pool.alloc()
layer = MoELayer(wg, pool, d_ff, capacity_factor=1.25)


def timed(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


for T in (16, 64, 256, 1024, 4096, 16384):
    x = torch.randn(T, d, device=dev, generator=g).to(torch.bfloat16)
    y = torch.empty_like(x)
    eager = timed(lambda: layer.forward(x, out=y))
    cap = layer.capture(x, y)
    graph = timed(cap.replay)
    ev = {}

    class St:
        def __init__(self, name):
            self.name = name

        def __enter__(self):
            self.a = torch.cuda.Event(enable_timing=True)
            self.a.record()

        def __exit__(self, *e):
            b = torch.cuda.Event(enable_timing=True)
            b.record()
            ev.setdefault(self.name, []).append((self.a, b))

    for _ in range(10):
        layer.forward(x, out=y, timer=St)
    torch.cuda.synchronize()
    stages = {k: sum(a.elapsed_time(b) for a, b in v) / len(v) * 1e3 for k, v in ev.items()}
    experts = int((layer.last.scan.group_kept > 0).sum())
    print(json.dumps({"tokens": T, "eager_us": eager, "graph_us": graph, "stages_us": stages,
                      "experts_touched": experts,
                      "weight_MB_streamed": experts * 2 * d * d_ff * 2 / 1e6}), flush=True)
