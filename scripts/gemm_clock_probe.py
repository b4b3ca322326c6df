"""SM clock during the grouped GEMMs of the C2 layer (dev probe): with
COMOE_GEMM_DEBUG=256 the 2-SM GEMM stamps clock64 and the global ns timer
at the start and end of CTA 0; clock cycles / ns = MHz while it runs.
Cold (first forward after idle) and steady (after N back-to-back
forwards). Prints one JSON line."""
import ctypes
import json
import math
import os
import sys
import time

os.environ["COMOE_GEMM_DEBUG"] = "256"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_09208_b200 import ExpertPool, MoELayer, _lib

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
y = torch.empty_like(x)


def mhz():
    buf = (ctypes.c_ulonglong * 4)()
    _lib.call("comoe_debug_gemm_clock", buf)
    return (buf[2] - buf[0]) / max(1, buf[3] - buf[1]) * 1e3, (buf[3] - buf[1]) / 1e3


layer.forward(x, out=y)
torch.cuda.synchronize()
time.sleep(2.0)  # idle
layer.forward(x, out=y)
torch.cuda.synchronize()
cold = mhz()
res = {"cold_mhz": cold[0], "cold_gemm2_us": cold[1]}
for n in (20, 200):
    for _ in range(n):
        layer.forward(x, out=y)
    torch.cuda.synchronize()
    m = mhz()
    res[f"after_{n}_mhz"] = m[0]
    res[f"after_{n}_gemm2_us"] = m[1]
print(json.dumps(res))
