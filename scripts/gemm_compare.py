"""C2 expert GEMMs: this repo's grouped tcgen05 GEMM vs library GEMMs on the
same ragged groups (dev tool; library numbers are the comparison, never the
product path):
  * torch._grouped_mm (PyTorch's CUTLASS grouped GEMM, sm_100)
  * torch.matmul on one dense [rows, K] x [K, N] (cuBLAS; same FLOPs, no
    grouping) — an upper reference for what the library reaches on this shape.
Also sweeps back-to-back GEMM1+GEMM2 to see the clock under sustained load.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2508_09208_b200 import ExpertPool, kernels

D, F, G = 768, 3072, 128
rng = np.random.default_rng(0)
rows_l = list(np.minimum(rng.binomial(65536, 1 / 128, G), 640))
rows = torch.tensor(rows_l, dtype=torch.int32, device="cuda")
base = torch.zeros_like(rows)
base[1:] = torch.cumsum(rows, 0)[:-1].to(torch.int32)
R = int(rows.sum())
pool = ExpertPool(G, 2 * D * F)
pool.data.normal_(0, 0.02)
slot = torch.arange(G, dtype=torch.int32, device="cuda")
x = torch.randn(R + 256, D, device="cuda").to(torch.bfloat16)
h = torch.empty(R + 256, F, device="cuda", dtype=torch.bfloat16)
y = torch.empty(R + 256, D, device="cuda", dtype=torch.bfloat16)
flop = 2.0 * R * D * F


def tflops(f, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    return {"us": round(ms * 1e3, 1), "TFLOPs": round(flop / ms / 1e9, 1)}


res = {"rows": R}
res["ours_gemm1"] = tflops(lambda: kernels.grouped_gemm(x, pool.data, 0, F, rows, base, slot,
                                                        kernels.EPI_RELU, h))
res["ours_gemm2"] = tflops(lambda: kernels.grouped_gemm(h, pool.data, F * D, D, rows, base, slot,
                                                        kernels.EPI_STORE, y))
w1 = pool.data[:, :F * D].view(G, F, D)          # [G, N, K] K-major
w2 = pool.data[:, F * D:2 * F * D].view(G, D, F)
offs = torch.cumsum(rows, 0).to(torch.int32)
try:
    res["torch_grouped_mm_gemm1"] = tflops(lambda: torch._grouped_mm(
        x[:R], w1.transpose(1, 2), offs=offs, out_dtype=torch.bfloat16))
    res["torch_grouped_mm_gemm2"] = tflops(lambda: torch._grouped_mm(
        h[:R], w2.transpose(1, 2), offs=offs, out_dtype=torch.bfloat16))
except Exception as e:  # noqa: BLE001
    res["torch_grouped_mm"] = f"unavailable: {type(e).__name__}: {e}"[:200]
wd1 = w1[0].t()
wd2 = w2[0].t()
res["cublas_dense_gemm1"] = tflops(lambda: torch.matmul(x[:R], wd1, out=h[:R]))
res["cublas_dense_gemm2"] = tflops(lambda: torch.matmul(h[:R], wd2, out=y[:R]))


def both():
    kernels.grouped_gemm(x, pool.data, 0, F, rows, base, slot, kernels.EPI_RELU, h)
    kernels.grouped_gemm(h, pool.data, F * D, D, rows, base, slot, kernels.EPI_STORE, y)


flop *= 2
res["ours_both_x200"] = tflops(both, reps=200)
print(json.dumps(res))
