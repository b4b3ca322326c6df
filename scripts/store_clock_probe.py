"""Epilogue stores vs SM clock in the grouped GEMMs (dev probe): the C2
layer's real routing, each GEMM run in alternating blocks with and without
its global stores (COMOE_GEMM_DEBUG 512 = staged, not stored), the SM clock
of each block read from CTA 0's clock64 / globaltimer stamps (debug 256).
Prints one JSON line per block: mode, µs per launch (CUDA events), MHz."""
import ctypes
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_09208_b200 import ExpertPool, MoELayer, _lib, kernels

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


def mhz():
    buf = (ctypes.c_ulonglong * 4)()
    _lib.call("comoe_debug_gemm_clock", buf)
    return (buf[2] - buf[0]) / max(1, buf[3] - buf[1]) * 1e3


modes = [int(m) for m in os.environ.get("MODES", "256,768").split(",")]
reps = int(os.environ.get("REPS", "20"))
for rnd in range(int(os.environ.get("ROUNDS", "3"))):
    for name, f in (("gemm1", f1), ("gemm2", f2)):
        for m in modes:
            _lib.call("comoe_debug_set_gemm", m)
            f()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                f()
            b.record()
            torch.cuda.synchronize()
            us = a.elapsed_time(b) / reps * 1e3
            clk = mhz()
            print(json.dumps({"round": rnd, "gemm": name, "debug": m, "us": round(us, 1),
                              "mhz_last": round(clk, 0), "kcycles": round(us * clk / 1e3, 1)}),
                  flush=True)
_lib.call("comoe_debug_set_gemm", -1)
