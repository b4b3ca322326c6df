"""SwiGLU MoE layer at the C2 shape (d 768, d_ff 3072, 128 experts), top-1 and top-2 (dev tool)."""
import math, sys, torch
sys.path.insert(0, __file__.rsplit("/scripts", 1)[0])
from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
T, d, d_ff, E = 65536, 768, 3072, 128
x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
wg = torch.randn(d, E, device="cuda") / math.sqrt(d)
pool = ExpertPool(E, kernels.expert_numel(d, d_ff, kernels.ACT_SWIGLU))
pool.data.normal_(0, 0.02)
for k in (1, 2):
    layer = MoELayer(wg, pool, d_ff, act="swiglu", top_k=k, capacity_factor=1.25)
    for _ in range(3): layer.forward(x)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): layer.forward(x)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"top{k} swiglu C2-shape: {ms:.3f} ms, {3 * 2 * T * k * d * d_ff / ms / 1e9:.0f} TF/s")
