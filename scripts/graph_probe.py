"""C2 layer forward: eager stream launches vs one CUDA graph replay (dev tool)."""
import math, sys, json
sys.path.insert(0, __file__.rsplit("/scripts", 1)[0])
import torch
from paper_2508_09208_b200 import ExpertPool, MoELayer

T, d, d_ff, E = 65536, 768, 3072, 128
torch.manual_seed(0)
x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
wg = torch.randn(d, E, device="cuda") / math.sqrt(d)
pool = ExpertPool(E, 2 * d * d_ff); pool.data.normal_(0, 0.02)
layer = MoELayer(wg, pool, d_ff, capacity_factor=1.25)
y = torch.empty_like(x)
def t(fn, n=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
eager = t(lambda: layer.forward(x, out=y))
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    layer.forward(x, out=y)
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    layer.forward(x, out=y)
graph = t(lambda: g.replay())
y_ref = y.clone(); g.replay(); torch.cuda.synchronize()
print(json.dumps({"eager_ms": eager, "graph_ms": graph, "graph_matches": bool(torch.equal(y, y_ref))}))
