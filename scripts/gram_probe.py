"""K6 cosine Gram alone at E=128 (Switch-Base-128 pool slots, D=4,718,592
bf16): CUDA-event time after an L2 flush; the target of
`ncu -k regex:sim_gram_tc`. Prints one JSON line."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_09208_b200 import ExpertPool, kernels

E, d, d_ff = 128, 768, 3072
dev = torch.device("cuda")
numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
pad = int(os.environ.get("PAD", "0"))  # extra elements per row (channel-mapping experiment)
if pad:
    buf = torch.empty((E, numel + pad), dtype=torch.bfloat16, device=dev)
    buf.normal_(0.0, 0.02, generator=torch.Generator(device=dev).manual_seed(0))
    rows = [buf[s, :numel] for s in range(E)]
else:
    pool = ExpertPool(E, numel, device=dev)
    pool.data.normal_(0.0, 0.02, generator=torch.Generator(device=dev).manual_seed(0))
    rows = [pool.view(s) for s in range(E)]
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
reps = int(os.environ.get("REPS", "10"))
kernels.similarity(rows, None, None, 1.0)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    flush.fill_(1)
    torch.cuda._sleep(400_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    kernels.similarity(rows, None, None, 1.0)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = statistics.median(ts)
nbytes = E * numel * 2
print(json.dumps({"kernel": "similarity cosine E=128", "us": ms * 1e3, "min_us": min(ts) * 1e3,
                  "GBps": nbytes / (ms * 1e-3) / 1e9,
                  "pad": pad, "env": {k: v for k, v in os.environ.items() if k.startswith("COMOE_")}}))
