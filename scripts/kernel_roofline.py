"""Per-kernel roofline at the C2 shape (Switch-Base-128, 65,536 tokens) for
the memory-bound kernels of SURVEY §8(d): gate (K1), route scan, permute
(K2), combine (K4, top-2 tables at the same shape), merge (K5, 128 -> 64
with the reference grouping rule), cosine similarity (K6) and the
next-layer predictor (K8).

Each launch is timed alone with CUDA events on the launching stream after
an L2 flush (a 512 MB write), median of N. `GBps` uses the ALGORITHMIC
bytes stated per kernel (inputs read once + outputs written once), `frac`
divides by the measured HBM copy bandwidth in MEASURED_PEAKS.json.
Prints one JSON line per kernel.
"""
import json
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
from paper_2508_09208_b200 import aggregation as A
from paper_2508_09208_b200.moe import stats_from_routing

PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
HBM = PEAKS.get("hbm_gbs", 6549.4)
BF16 = PEAKS.get("bf16_tflops", 1590.0)
REPS = int(os.environ.get("REPS", "20"))

_flush = None


def timed(fn, reps=REPS):
    global _flush
    if _flush is None:
        _flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        _flush.fill_(1)
        # keep the GPU busy while the host prepares the launch, so the events
        # bracket device time only (no host gap before the kernel starts)
        torch.cuda._sleep(400_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def line(kernel, ms, nbytes, note, flops=None):
    gbs = nbytes / (ms * 1e-3) / 1e9
    d = {"kernel": kernel, "us": ms * 1e3, "alg_bytes": int(nbytes), "GBps": gbs,
         "hbm_peak_GBps": HBM, "frac": gbs / HBM, "bytes": note}
    if flops:
        d["TFLOPs"] = flops / (ms * 1e-3) / 1e12
    print(json.dumps(d), flush=True)


def main():
    torch.manual_seed(0)
    dev = torch.device("cuda")
    T, d, d_ff, E = 65536, 768, 3072, 128
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(T, d, device=dev, generator=g).to(torch.bfloat16)
    wg = torch.randn(d, E, device=dev, generator=g) / math.sqrt(d)
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
    pool = ExpertPool(E + 64, numel, device=dev)
    pool.data.normal_(0.0, 0.02, generator=g)
    for _ in range(E):
        pool.alloc()
    layer = MoELayer(wg, pool, d_ff, act="relu", top_k=1, capacity_factor=1.25)
    y = torch.empty_like(x)
    layer.forward(x, out=y)
    torch.cuda.synchronize()
    ws = layer._workspace(T)
    r = layer.last
    kept = int(r.scan.group_kept.sum())

    # K1 gate: x read once + router split (3*128*768 bf16) + 4 [T] int/fp outputs + hist
    nt = kernels.gate_num_tiles(T)
    gbytes = T * d * 2 + 3 * 128 * d * 2 + T * 4 * 4 + nt * E * 4
    ms = timed(lambda: kernels.gate_topk(x, layer.wg_split, E, 1, False, slot_map=layer.slot_map,
                                         n_groups=E, out=ws["gate"]))
    line("gate_kernel (K1)", ms, gbytes, "T*d*2 (x) + Wg split + T*16 (idx,group,prob,rank) + hist",
         flops=2 * 2 * T * d * 128)  # two bf16 split terms (gate_terms())

    # route scan: hist read + offsets written + [G] outputs
    sbytes = 2 * nt * E * 4 + 3 * E * 4
    ms = timed(lambda: kernels.route_scan(ws["gate"].tile_hist, ws["C"], out=ws["scan"]))
    line("route_scan", ms, sbytes, "tile_hist read + tile_offset write + 3*G")

    # the production router: gate + capacity scan in one launch (comoe_gate_route)
    lbw = kernels.gate_route_workspace(T, 1, E, dev)
    ms = timed(lambda: kernels.gate_route(x, layer.wg_split, E, 1, False, ws["C"], lbw,
                                          slot_map=layer.slot_map, n_groups=E, out=ws["gate"],
                                          scan=ws["scan"]))
    line("gate_route (K1 + folded scan)", ms, gbytes + sbytes,
         "gate bytes + histogram write/read + tile_offset write + 3*G", flops=2 * 2 * T * d * 128)

    # K2 permute (top-1: copies kept rows, zeroes y rows of dropped tokens)
    pbytes = T * d * 2 + kept * d * 2 + (T - kept) * d * 2 + T * 4 * 4 + kept * 8
    ms = timed(lambda: kernels.permute(x, r.gate, r.scan, r.capacity, r.rows, y_zero=y,
                                       out=r.perm))
    line("permute (K2)", ms, pbytes, f"T*d*2 read + kept*d*2 write (kept={kept}) + dropped y rows "
         "zeroed + tables")

    # K4 combine at the same shape with top-2 tables: y = p0*Y[pos0] + p1*Y[pos1]
    k = 2
    rows2 = T * k
    y_perm = torch.randn(rows2, d, device=dev, generator=g).to(torch.bfloat16)
    pos = torch.randperm(rows2, device=dev, generator=g).to(torch.int32).view(T, k)
    prob = torch.rand(T, k, device=dev, generator=g)
    cbytes = k * T * d * 2 + T * d * 2 + T * k * 8
    ms = timed(lambda: kernels.combine(y_perm, pos, prob, out=y))
    line("combine (K4, top-2)", ms, cbytes, "k*T*d*2 gather + T*d*2 write + T*k*(pos,prob)")

    # K5 merge 128 -> 64 with the reference rule (principals by frequency,
    # members by argmax cosine similarity); synthetic correlated experts so
    # groups are ragged as measured in SURVEY a10
    stats = stats_from_routing({1: r.gate.expert_idx}, E)
    sim = torch.nn.functional.cosine_similarity(
        pool.data[:E, :4096].float().unsqueeze(1), pool.data[:E, :4096].float().unsqueeze(0),
        dim=2).double().cpu().numpy()
    principals = A.identify_principals(stats, 1, 64)

    class _E:
        def __init__(self, s):
            self.slot = s
    groups = A.group_experts([_E(s) for s in range(E)], principals, sim)
    multi = [gr for gr in groups if gr.member_slots]
    freqs = stats.freqs(1)
    mem = [[pool.view(s) for s in gr.slots] for gr in multi]
    wts, divs = [], []
    for gr in multi:
        w, dv = A._merge_weights(freqs, gr.slots)
        wts.append(w)
        divs.append(dv)
    outs = [pool.view(pool.alloc()) for _ in multi]
    ebytes = pool.slot_bytes
    mbytes = sum((len(gr.slots) + 1) * ebytes for gr in multi)
    plan = kernels.MergePlan(mem, wts, divs, outs, torch.bfloat16)
    ms = timed(plan.run)
    sizes = sorted(len(gr.slots) for gr in multi)
    line("merge (K5, 128->64 bf16)", ms, mbytes,
         f"sum over {len(multi)} multi-member groups of (members+1)*{ebytes} B; sizes {sizes}")

    # K6 cosine Gram at E=128 (bf16 params, D=4,718,592): reads E*D*2 once per column tile
    rows = [pool.view(s) for s in range(E)]
    ms = timed(lambda: kernels.similarity(rows, None, None, 1.0), reps=3)
    sb = E * numel * 2
    line("similarity cosine (K6, E=128)", ms, sb, "E*D*2 (every expert read once)",
         flops=2 * E * E * numel)
    rows8 = rows[:8]
    ms = timed(lambda: kernels.similarity(rows8, None, None, 1.0))
    line("similarity cosine (K6, E=8)", ms, 8 * numel * 2, "E*D*2", flops=2 * 8 * 8 * numel)

    # K6 with the reference's functional surrogate at C1 (E=8, 8 probes x 8
    # buckets over D): bytes = rows (bf16) + probes + projection (fp64)
    probes = torch.randn(8, numel, device=dev, dtype=torch.float64, generator=g)
    proj = torch.randn(8, numel, device=dev, dtype=torch.float64, generator=g)
    ms = timed(lambda: kernels.similarity(rows8, probes, proj, 0.5), reps=5)
    line("similarity + surrogate (K6, E=8, 8x8 probes)", ms, 8 * numel * 2 + 16 * numel * 8,
         "E*D*2 + (n+B)*D*8", flops=2 * 8 * (8 + 64 + 8) * numel)
    del probes, proj

    # K8 predictor over 65,536 tokens (E=128, emb 16, ctx 8, hidden 32)
    hid = 32
    w1 = torch.randn(hid, E + 24, device=dev, dtype=torch.float64) * 0.1
    b1 = torch.zeros(hid, device=dev, dtype=torch.float64)
    w2 = torch.randn(E, hid, device=dev, dtype=torch.float64) * 0.1
    b2 = torch.zeros(E, device=dev, dtype=torch.float64)
    emb = torch.randn(T, 16, device=dev, dtype=torch.float64)
    ctx = torch.randn(T, 8, device=dev, dtype=torch.float64)
    slots = r.gate.expert_idx
    pb = T * (4 + 24 * 8 + E * 8)
    ms = timed(lambda: kernels.predictor_mlp(slots, emb, ctx, w1, b1, w2, b2))
    line("predictor_mlp (K8)", ms, pb, "T*(slot + emb/ctx f64 + E f64 probs)")


if __name__ == "__main__":
    main()
