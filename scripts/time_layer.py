"""Quick per-kernel timing of the C2 layer (dev tool; bench.py is the contract)."""
import math, sys, time
sys.path.insert(0, __file__.rsplit("/scripts", 1)[0])
import torch
from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels

T, d, d_ff, E = 65536, 768, 3072, 128
torch.manual_seed(0)
x = torch.randn(T, d, device="cuda").to(torch.bfloat16)
wg = torch.randn(d, E, device="cuda") / math.sqrt(d)
pool = ExpertPool(E, 2 * d * d_ff)
pool.data.normal_(0, 0.02)
layer = MoELayer(wg, pool, d_ff, capacity_factor=1.25)
for _ in range(3):
    layer.forward(x)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
n = 20
ev[0].record()
for _ in range(n):
    layer.forward(x)
ev[1].record()
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / n
print(f"layer forward: {ms:.3f} ms  -> {T/ms*1e3:.3e} tok/s")
r = layer.last
ws = layer._ws[T]
# per stage timing
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
tg = t(lambda: kernels.gate_topk(x, layer.wg_split, E, 1, False, slot_map=layer.slot_map, n_groups=E, out=r.gate))
ts = t(lambda: kernels.route_scan(r.gate.tile_hist, r.capacity, out=r.scan))
y = torch.empty_like(x)
tp = t(lambda: kernels.permute(x, r.gate, r.scan, r.capacity, r.rows, y_zero=y, out=r.perm))
rows = int(r.scan.group_kept.sum())
def g1(): kernels.grouped_gemm(r.perm.x_perm, pool.data, 0, d_ff, r.scan.group_kept, r.scan.group_base, layer.group_slot, kernels.EPI_RELU, ws["h"])
def g2(): kernels.grouped_gemm(ws["h"], pool.data, d_ff * d, d, r.scan.group_kept, r.scan.group_base, layer.group_slot, kernels.EPI_SCALE_SCATTER, y, r.perm.row_token, r.perm.row_prob)
t1 = t(g1); t2 = t(g2)
fl = 2 * rows * d * d_ff
print(f"gate {tg*1e3:.1f} us ({(T*d*2)/tg/1e6:.0f} GB/s)  scan {ts*1e3:.1f} us  permute {tp*1e3:.1f} us ({(T*d*2 + rows*d*2)/tp/1e6:.0f} GB/s)")
print(f"gemm1 {t1*1e3:.1f} us ({fl/t1/1e9:.0f} TF/s)  gemm2 {t2*1e3:.1f} us ({fl/t2/1e9:.0f} TF/s)  rows={rows}")
