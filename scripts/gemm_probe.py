"""Grouped-GEMM probe: uniform vs ragged group sizes, both kernels (dev tool)."""
import os, sys, json
sys.path.insert(0, __file__.rsplit("/scripts", 1)[0])
import torch
from paper_2508_09208_b200 import kernels, ExpertPool

D, F, G = 768, 3072, 128
pool = ExpertPool(G, 2 * D * F)
pool.data.normal_(0, 0.02)
slot = torch.arange(G, dtype=torch.int32, device="cuda")

def run(rows_per_group, which):
    rows = torch.tensor(rows_per_group, dtype=torch.int32, device="cuda")
    base = torch.zeros_like(rows); base[1:] = torch.cumsum(rows, 0)[:-1].to(torch.int32)
    R = int(rows.sum())
    x = torch.randn(R + 256, D, device="cuda").to(torch.bfloat16)
    h = torch.empty(R + 256, F, device="cuda", dtype=torch.bfloat16)
    y = torch.empty(R + 256, D, device="cuda", dtype=torch.bfloat16)
    f1 = lambda: kernels.grouped_gemm(x, pool.data, 0, F, rows, base, slot, kernels.EPI_RELU, h)
    f2 = lambda: kernels.grouped_gemm(h, pool.data, F * D, D, rows, base, slot, kernels.EPI_STORE, y)
    out = {}
    for name, f in (("gemm1", f1), ("gemm2", f2)):
        for _ in range(3): f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10): f()
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        out[name] = round(2 * R * D * F / ms / 1e9, 1)
    return out

import numpy as np
rng = np.random.default_rng(0)
cases = {"uniform512": [512] * G, "uniform256": [256] * G, "uniform640": [640] * G,
         "ragged_c2": list(np.minimum(rng.binomial(65536, 1 / 128, G), 640))}
which = os.environ.get("COMOE_GEMM_1SM", "0")
for k, v in cases.items():
    print(json.dumps({"kernel": "1sm" if which == "1" else "2sm", "case": k, "TFLOPs": run(v, which)}))
