"""Host-to-host pipeline sweep at the bench workload (C2 layer, 65,536
tokens): CUDA-event ms per step of HostPipeline for pipeline depth, copy
chunks and copy streams per direction. Prints one JSON line per setting."""
import itertools
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_09208_b200 import ExpertPool, MoELayer
from paper_2508_09208_b200.stream import HostPipeline

T, d, d_ff, E = 65536, 768, 3072, 128
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(T, d, device=dev, generator=g).to(torch.bfloat16)
wg = torch.randn(d, E, device=dev, generator=g) / math.sqrt(d)
pool = ExpertPool(E, 2 * d * d_ff, device=dev)
pool.data.normal_(0.0, 0.02, generator=g)
for _ in range(E):
    pool.alloc()
layer = MoELayer(wg, pool, d_ff, capacity_factor=1.25)
xh = x.cpu().pin_memory()
yhs = [torch.empty_like(xh).pin_memory() for _ in range(3)]
steps = int(os.environ.get("STEPS", "20"))
grid = os.environ.get("GRID")  # e.g. "2:1:1,2:4:2" = depth:chunks:streams
combos = ([tuple(int(v) for v in c.split(":")) for c in grid.split(",")] if grid else
          itertools.product((2, 3), (1, 2, 4, 8, 16), (1, 2, 4)))
for depth, chunks, cs in combos:
    pipe = HostPipeline(layer, T, d, depth=depth, device=dev, chunks=chunks, copy_streams=cs,
                        graphs=os.environ.get("GRAPHS", "1") == "1")
    pipe.run([xh] * 3, [yhs[i % 3] for i in range(3)])
    pipe.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pipe.run([xh] * steps, [yhs[i % 3] for i in range(steps)], start_event=s, end_event=e)
    pipe.synchronize()
    print(json.dumps({"depth": depth, "chunks": chunks, "copy_streams": cs, "steps": steps,
                      "ms_per_step": s.elapsed_time(e) / steps}), flush=True)
