"""Host-to-host pipeline and expert-parallel path on one GPU."""

import math
import os

import numpy as np
import pytest
import torch

from oracle import switch_layer as O

pytestmark = pytest.mark.gpu


def _layer(T, d, d_ff, E, seed=0):
    from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(T, d, generator=g).to(torch.bfloat16)
    wg = (torch.randn(d, E, generator=g) / math.sqrt(d)).cuda()
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
    w = (torch.randn(E, numel, generator=g) * 0.02).to(torch.bfloat16)
    pool = ExpertPool(E, numel)
    pool.data[:, :numel].copy_(w.cuda())
    return MoELayer(wg, pool, d_ff, capacity_factor=1.25), x, wg, w


def test_host_pipeline_matches_device_forward():
    from paper_2508_09208_b200.stream import HostPipeline
    layer, x, wg, w = _layer(4096, 256, 512, 16)
    xs = [(x + i).contiguous().pin_memory() for i in range(5)]
    ys = [torch.empty_like(v).pin_memory() for v in xs]
    pipe = HostPipeline(layer, 4096, 256)
    pipe.run(xs, ys)
    pipe.synchronize()
    for xh, yh in zip(xs, ys):
        ref = layer.forward(xh.cuda())
        torch.cuda.synchronize()
        assert torch.equal(yh, ref.cpu())


def test_expert_parallel_world1_matches_oracle():
    import torch.distributed as dist
    from paper_2508_09208_b200.ep import EPMoELayer
    from paper_2508_09208_b200.pool import ExpertPool
    from paper_2508_09208_b200 import kernels
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1)
    T, d, d_ff, E = 3000, 256, 512, 16
    g = torch.Generator().manual_seed(4)
    x = torch.randn(T, d, generator=g).to(torch.bfloat16)
    wg = (torch.randn(d, E, generator=g) / math.sqrt(d)).cuda()
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
    w = (torch.randn(E, numel, generator=g) * 0.02).to(torch.bfloat16)
    pool = ExpertPool(E, numel)
    pool.data[:, :numel].copy_(w.cuda())
    layer = EPMoELayer(wg, pool, d_ff, world=1, rank=0, capacity_factor=1.0)
    y = layer.forward(x.cuda())
    # the chunked exchange (async all-to-all per chunk of local experts,
    # FFN of chunk k while chunk k+1 is in flight) computes every row the same
    for chunks in (2, 4):
        layer_c = EPMoELayer(wg, pool, d_ff, world=1, rank=0, capacity_factor=1.0, chunks=chunks)
        yc = layer_c.forward(x.cuda())
        torch.cuda.synchronize()
        assert torch.equal(yc, y), chunks
        # out=: the combine writes the caller's buffer (no extra copy)
        yo = torch.full_like(y, float("nan"))
        assert layer_c.forward(x.cuda(), out=yo) is yo
        torch.cuda.synchronize()
        assert torch.equal(yo, y), chunks
    yo = torch.empty_like(y)
    assert layer.forward(x.cuda(), out=yo) is yo
    torch.cuda.synchronize()
    assert torch.equal(yo, y)
    torch.cuda.synchronize()
    logits = None
    wi = np.stack([O.split_expert(w[e].float().numpy(), d, d_ff, "relu")[0] for e in range(E)])
    wo = np.stack([O.split_expert(w[e].float().numpy(), d, d_ff, "relu")[1] for e in range(E)])
    ref, info = O.layer_forward_fast(x.float().numpy(), wg.cpu().numpy(), wi, wo, 1, False, 1.0,
                                     dtype=np.float64, round_h=True)
    assert (info["pos"] < 0).sum() > 0
    assert O.normwise_error(y.float().cpu().numpy(), ref) < 5e-3  # the bf16 bar
    dist.destroy_process_group()


def test_ep_expert_ffn_expert_major_groups_world4():
    """The receiver-side grouped FFN of expert parallelism with a simulated
    world of 4 on one GPU: groups enumerated expert-major over the
    [src][local expert][C] receive buffer must give every block the FFN of
    its own local expert (fp32 torch reference, bf16 tolerance)."""
    from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
    from paper_2508_09208_b200.ep import DeviceOps
    world, E, d, d_ff, C = 4, 16, 256, 512, 96
    El = E // world
    g = torch.Generator().manual_seed(7)
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
    w = (torch.randn(El, numel, generator=g) * 0.05).to(torch.bfloat16).cuda()
    pool = ExpertPool(El, numel)
    pool.data[:, :numel].copy_(w)
    wg = (torch.randn(d, E, generator=g) / math.sqrt(d)).cuda()
    ops = DeviceOps(MoELayer(wg, pool, d_ff, capacity_factor=1.0, expert_slots=[0] * E))
    recv = torch.randn(world * El * C, d, generator=g).to(torch.bfloat16).cuda()
    counts = torch.randint(0, C + 1, (world * El,), generator=g, dtype=torch.int32).cuda()
    y = ops.expert_ffn(recv, counts, El, C, world)
    torch.cuda.synchronize()
    for src in range(world):
        for le in range(El):
            blk = src * El + le
            n = int(counts[blk])
            if n == 0:
                continue
            xs = recv[blk * C: blk * C + n].float()
            wi = w[le, : d_ff * d].view(d_ff, d).float()
            wo = w[le, d_ff * d: 2 * d_ff * d].view(d, d_ff).float()
            ref = torch.relu(xs @ wi.t()).to(torch.bfloat16).float() @ wo.t()
            got = y[blk * C: blk * C + n].float()
            assert (got - ref).norm() / ref.norm() < 5e-3, (src, le)


def test_captured_forward_top2_swiglu():
    """Capture of the top-2 SwiGLU layer (separate combine kernel, y_perm
    workspace): replays equal the eager forward."""
    from paper_2508_09208_b200 import ExpertPool, MoELayer, kernels
    g = torch.Generator().manual_seed(9)
    T, d, d_ff, E = 3000, 256, 512, 8
    wg = (torch.randn(d, E, generator=g) / math.sqrt(d)).cuda()
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_SWIGLU)
    pool = ExpertPool(E, numel)
    pool.data[:, :numel].copy_((torch.randn(E, numel, generator=g) * 0.02).to(torch.bfloat16).cuda())
    layer = MoELayer(wg, pool, d_ff, act="swiglu", top_k=2, capacity_factor=1.0)
    xbuf = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    cap = layer.capture(xbuf)
    for i in range(2):
        xi = torch.randn(T, d, generator=g).to(torch.bfloat16).cuda()
        xbuf.copy_(xi)
        y = cap.replay().clone()
        ref = layer.forward(xi)
        torch.cuda.synchronize()
        assert torch.equal(y, ref)


def test_captured_forward_replays_match_eager():
    """MoELayer.capture: every replay is a complete forward of the current
    contents of the static input (different batches route differently), bit
    for bit the eager forward; the graphed host pipeline matches too."""
    from paper_2508_09208_b200.stream import HostPipeline
    layer, x, wg, w = _layer(4096, 256, 512, 16)
    xs = [(x * (1 + 0.5 * i) + i).cuda() for i in range(3)]
    xbuf = torch.empty_like(xs[0])
    cap = layer.capture(xbuf)
    for xi in xs:
        xbuf.copy_(xi)
        y = cap.replay().clone()
        ref = layer.forward(xi)
        torch.cuda.synchronize()
        assert torch.equal(y, ref)
    hx = [v.cpu().pin_memory() for v in xs]
    hy = [torch.empty_like(v) .pin_memory() for v in hx]
    pipe = HostPipeline(layer, 4096, 256, graphs=True)
    pipe.run(hx, hy)
    pipe.synchronize()
    for xh, yh in zip(hx, hy):
        assert torch.equal(yh, layer.forward(xh.cuda()).cpu())
