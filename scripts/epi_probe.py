"""Grouped-GEMM epilogue attribution at the C2 layer shape (dev tool): the
real routing of a C2 batch, GEMM1 (ReLU, TMA bulk stores of H) and GEMM2
(gate-probability scale + scatter to token rows, the fused top-1 combine)
timed with CUDA events; run once per COMOE_GEMM_DEBUG setting (1: TMEM reads
only; 1024: + epilogue math; 512: + staging, no global stores)."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels

T, D, F, E = 65536, 768, 3072, 128
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
f1 = lambda: kernels.grouped_gemm(r.perm.x_perm, pool.data, 0, F, r.scan.group_kept, r.scan.group_base,
                                  layer.group_slot, kernels.EPI_RELU, ws["h"])
f2 = lambda: kernels.grouped_gemm(ws["h"], pool.data, F * D, D, r.scan.group_kept, r.scan.group_base,
                                  layer.group_slot, kernels.EPI_SCALE_SCATTER, y,
                                  row_token=r.perm.row_token, row_prob=r.perm.row_prob)
f3 = lambda: kernels.grouped_gemm(ws["h"], pool.data, F * D, D, r.scan.group_kept, r.scan.group_base,
                                  layer.group_slot, kernels.EPI_STORE, ws["y_perm_probe"])
ws["y_perm_probe"] = torch.empty_like(x)
out = {"debug": os.environ.get("COMOE_GEMM_DEBUG", "0")}
only = os.environ.get("EPI_ONLY")  # one GEMM only (for ncu: EPI_ONLY=gemm2_scatter REPS=1)
reps = int(os.environ.get("REPS", "10"))
for name, f in (("gemm1_relu_tma", f1), ("gemm2_scatter", f2), ("gemm2_store_tma", f3)):
    if only and name != only:
        continue
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    out[name] = round(a.elapsed_time(b) / reps * 1e3, 1)
print(json.dumps(out))
