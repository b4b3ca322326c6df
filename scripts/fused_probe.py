"""Time the fused expert FFN (K3F) alone on the C2 routing (dev tool).

    COMOE_FUSED_DEBUG=<bits> COMOE_FUSED_PF=<n> python scripts/fused_probe.py [--two]

Builds the bench's C2 layer (65,536 tokens, E=128, d=768, d_ff=3072), runs
one forward for the routing tables, then times kernels.fused_ffn (TMA gather
from the unpermuted tokens, top-1 scatter epilogue) with CUDA events; --two
also times the two-launch FFN (GEMM1 -> H -> GEMM2) on the same groups.
Prints one JSON line.
"""
import json
import math
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels  # noqa: E402

D, D_FF, E = 768, 3072, 128
T = next((int(a.split("=")[1]) for a in sys.argv if a.startswith("--tokens=")), 65536)


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(1234)
    x = torch.randn(T, D, device=dev, generator=g).to(torch.bfloat16)
    wg = torch.randn(D, E, device=dev, generator=torch.Generator(device=dev).manual_seed(1)) / math.sqrt(D)
    pool = ExpertPool(E, 2 * D * D_FF, device=dev)
    pool.data.normal_(0.0, 0.02, generator=torch.Generator(device=dev).manual_seed(2))
    layer = MoELayer(wg, pool, D_FF, act="relu", top_k=1, capacity_factor=1.25)
    y = torch.empty_like(x)
    layer.forward(x, out=y)
    r = layer.last
    kept = int(r.scan.group_kept.sum())
    args = (r.scan.group_kept, r.scan.group_base, layer.group_slot)

    gather = "--nogather" not in sys.argv
    xsrc = x if gather else x[r.perm.row_token.long()].contiguous()

    def fused():
        kernels.fused_ffn(xsrc, pool.data, D_FF, *args, y,
                          gather_rows=r.perm.row_token if gather else None,
                          row_token=r.perm.row_token, row_prob=r.perm.row_prob)

    def timeit(fn, n=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n * 1e3

    out = {"env": {k: v for k, v in os.environ.items() if k.startswith("COMOE_")}, "kept": kept}
    us = timeit(fused)
    out["fused_us"] = us
    out["fused_tflops"] = 4.0 * kept * D * D_FF / (us * 1e-6) / 1e12
    if int(os.environ.get("COMOE_FUSED_DEBUG", "0")) & 256:
        import ctypes
        import numpy as np
        from paper_2508_09208_b200 import _lib
        buf = (ctypes.c_ulonglong * (128 * 16))()
        fused()
        torch.cuda.synchronize()
        _lib.call("comoe_debug_fused_prof", ctypes.cast(buf, ctypes.c_void_p))
        a = np.array(buf, dtype=np.float64).reshape(128, 16)[:74]
        names = ["total", "x_full", "h_empty", "g1_full", "y_empty", "hs_full", "g2_full", "tiles",
                 "prod0_empty", "prod1_empty", "prod0_total", "prod1_total", "-", "-", "-", "-"]
        out["issuer_wait_frac"] = {n: round(float(a[:, i].sum() / a[:, 0].sum()), 4)
                                   for i, n in enumerate(names) if n not in ("total", "tiles", "-")}
        out["tiles_per_pair"] = [int(a[:, 7].min()), int(a[:, 7].max())]
        out["issuer_kcycles_per_pair"] = [round(a[:, 0].min() / 1e3), round(a[:, 0].max() / 1e3)]
    if "--two" in sys.argv:
        xp = x[r.perm.row_token.long()].contiguous()
        h = torch.empty((xp.shape[0], D_FF), dtype=torch.bfloat16, device=dev)

        def two():
            kernels.grouped_gemm(xp, pool.data, 0, D_FF, *args, kernels.EPI_RELU, h)
            kernels.grouped_gemm(h, pool.data, D_FF * D, D, *args, kernels.EPI_SCALE_SCATTER, y,
                                 row_token=r.perm.row_token, row_prob=r.perm.row_prob)
        out["two_launch_us"] = timeit(two)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
