"""Expert parallelism over peer memory on one GPU: a simulated world whose
"peers" are buffers of the same process (PeerBuffers.simulated). The
peer-store permute, count scatter, grouped FFN and peer-load combine must
give every rank exactly the output of the NCCL schedule (all-to-alls
emulated by block transposition of the same kernels' buffers), and that
output must match the oracle's per-rank forward. The flag barrier is run
with every rank on its own stream (concurrent kernels) and with a missing
peer (timeout flag, no hang)."""

import math

import numpy as np
import pytest
import torch

from oracle import switch_layer as O

pytestmark = pytest.mark.gpu


def _world(world, T, d, d_ff, E, cf, seed=11):
    from paper_2508_09208_b200 import ExpertPool, kernels
    from paper_2508_09208_b200.ep import EPMoELayer
    g = torch.Generator().manual_seed(seed)
    wg = torch.randn(d, E, generator=g) / math.sqrt(d)
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
    w = (torch.randn(E, numel, generator=g) * 0.02).to(torch.bfloat16)
    El = E // world
    layers = []
    for r in range(world):
        pool = ExpertPool(El, numel)
        pool.data[:, :numel].copy_(w[r * El:(r + 1) * El].cuda())
        layers.append(EPMoELayer(wg.cuda(), pool, d_ff, world=world, rank=r, capacity_factor=cf,
                                 transport="peer"))
    xs = [torch.randn(T, d, generator=g).to(torch.bfloat16).cuda() for _ in range(world)]
    return layers, xs, wg, w


def _alltoall_emulation(layers, xs, world, E, C):
    """The NCCL schedule of ep_forward with each all_to_all_single done as a
    block transposition of the same device buffers (E: routing groups, the
    padded space of a merged variant included)."""
    El = E // world
    blk = El * C
    routes, sends, tps = [], [], []
    for L, x in zip(layers, xs):
        r = L.ops.route(x)
        send, tp = L.ops.dispatch(x, r, C)
        routes.append(r)
        sends.append(send.clone())
        tps.append(tp.clone())
    ys = []
    for q, L in enumerate(layers):
        recv = torch.cat([sends[s][q * blk:(q + 1) * blk] for s in range(world)])
        counts = torch.cat([routes[s].kept[q * El:(q + 1) * El] for s in range(world)])
        ys.append(L.ops.expert_ffn(recv, counts, El, C, world).clone())
    outs = []
    for r, L in enumerate(layers):
        back = torch.cat([ys[q][r * blk:(r + 1) * blk] for q in range(world)])
        outs.append(L.ops.combine(back, tps[r], routes[r]).clone())
    return outs


@pytest.mark.parametrize("world,T,E,cf", [(4, 1000, 16, 1.0), (2, 777, 8, 1.25), (1, 500, 8, 1.25)])
def test_peer_transport_matches_alltoall_schedule(world, T, E, cf):
    from paper_2508_09208_b200.ep import PeerBuffers
    d, d_ff = 256, 512
    layers, xs, wg, w = _world(world, T, d, d_ff, E, cf)
    C = layers[0].capacity(T)
    ref = _alltoall_emulation(layers, xs, world, E, C)
    bufs = PeerBuffers.simulated(world, E * C, d, E, torch.device("cuda"))
    El = E // world
    routes, tps = [], []
    for r, L in enumerate(layers):      # phase 1 on every rank: route, peer-store permute, counts
        routes.append(L.ops.route(xs[r]))
        tps.append(L.ops.dispatch_peers(xs[r], routes[-1], C, bufs[r]).clone())
    for q, L in enumerate(layers):      # phase 2: grouped FFN on my receive buffer
        L.ops.expert_ffn(bufs[q].recv, bufs[q].counts, El, C, world, y_out=bufs[q].y)
    outs = [L.ops.combine_peers(tps[r], routes[r], bufs[r])  # phase 3: peer-load combine
            for r, L in enumerate(layers)]
    torch.cuda.synchronize()
    for r in range(world):
        assert torch.equal(outs[r], ref[r]), f"rank {r}"
        # counts landed where the all-to-all would put them
        exp = torch.cat([routes[s].kept[r * El:(r + 1) * El] for s in range(world)])
        assert torch.equal(bufs[r].counts, exp)
    # against the oracle: rank r's forward = a single-device layer over its own
    # tokens with every expert and the per-rank capacity
    wi = np.stack([O.split_expert(w[e].float().numpy(), d, d_ff, "relu")[0] for e in range(E)])
    wo = np.stack([O.split_expert(w[e].float().numpy(), d, d_ff, "relu")[1] for e in range(E)])
    for r in range(world):
        y_ref, info = O.layer_forward_fast(xs[r].float().cpu().numpy(), wg.numpy(), wi, wo, 1,
                                           False, cf, dtype=np.float64, round_h=True)
        assert O.normwise_error(outs[r].float().cpu().numpy(), y_ref) < 5e-3  # bf16 bar


def test_peer_barrier_concurrent_ranks_and_timeout():
    from paper_2508_09208_b200 import kernels
    from paper_2508_09208_b200.ep import PeerBuffers
    world = 4
    bufs = PeerBuffers.simulated(world, world * 8, 64, 8, torch.device("cuda"))
    streams = [torch.cuda.Stream() for _ in range(world)]
    for rep in range(3):  # epochs 1..3, every rank on its own stream
        for b, s in zip(bufs, streams):
            with torch.cuda.stream(s):
                b.barrier(timeout_s=20.0)
        torch.cuda.synchronize()
    for b in bufs:
        b.check()
        assert b.epoch == 3 and torch.equal(b.pad.cpu(), torch.full((world,), 3, dtype=torch.int32))
    # rank 0 alone at epoch 4: every other rank is missing -> flag, no hang
    bufs[0].barrier(timeout_s=0.05)
    torch.cuda.synchronize()
    assert int(bufs[0].err.item()) in (2, 3, 4)
    with pytest.raises(RuntimeError):
        bufs[0].check()


def test_ep_layer_peer_transport_world1():
    """EPMoELayer(transport="peer") through its public forward at world 1
    (IPC handle of its own buffers, barriers with itself)."""
    layers, xs, wg, w = _world(1, 900, 256, 512, 8, 1.25, seed=5)
    L = layers[0]
    y = L.forward(xs[0])
    L.peers.check()
    nccl_ops_out = _alltoall_emulation(layers, xs, 1, 8, L.capacity(900))[0]
    torch.cuda.synchronize()
    assert torch.equal(y, nccl_ops_out)
    y2 = L.forward(xs[0])   # second forward: epochs 3, 4 on the same pads
    torch.cuda.synchronize()
    assert torch.equal(y2, y) and L.peers.epoch == 4


def _merged_world(world, T, d, d_ff, E, principals, lut, cf, seed=21):
    """Per-rank EPMoELayers of a merged variant: group g's weights live in
    the pool of its principal's rank (ep_placement)."""
    from paper_2508_09208_b200 import ExpertPool, kernels
    from paper_2508_09208_b200.ep import EPMoELayer, ep_placement
    g = torch.Generator().manual_seed(seed)
    wg = torch.randn(d, E, generator=g) / math.sqrt(d)
    numel = kernels.expert_numel(d, d_ff, kernels.ACT_RELU)
    G = len(principals)
    w = (torch.randn(G, numel, generator=g) * 0.02).to(torch.bfloat16)
    pl = ep_placement(lut, principals, E, world)
    layers = []
    for r in range(world):
        mine = pl.local_groups(r)
        pool = ExpertPool(max(1, len(mine)) + 1, numel)
        slots = list(range(1, len(mine) + 1))          # slot 0 left unused on purpose
        for s_, grp in zip(slots, mine):
            pool.data[s_, :numel].copy_(w[grp].cuda())
        layers.append(EPMoELayer(wg.cuda(), pool, d_ff, world=world, rank=r, capacity_factor=cf,
                                 transport="peer", variant_table=(lut, principals),
                                 local_slots=slots))
    xs = [torch.randn(T, d, generator=g).to(torch.bfloat16).cuda() for _ in range(world)]
    return layers, xs, wg, w, pl


@pytest.mark.parametrize("world", [1, 2, 4])
def test_merged_variant_ep_peer_and_alltoall(world):
    """A CoMoE 16 -> 7 variant under EP: principals unevenly spread over the
    ranks. Peer transport == the all-to-all schedule bit for bit, counts in
    place, and every rank's output == the single-device oracle forward of
    the merged layer over its tokens (capacity over the 7 real groups)."""
    from paper_2508_09208_b200.ep import PeerBuffers
    E, d, d_ff, T, cf = 16, 256, 512, 700, 1.0
    principals = [0, 1, 2, 5, 9, 12, 13]
    lut = [0, 1, 2, 2, 1, 3, 3, 0, 4, 4, 5, 4, 5, 6, 6, 3]
    layers, xs, wg, w, pl = _merged_world(world, T, d, d_ff, E, principals, lut, cf)
    Gp, L = pl.G_pad, pl.L
    C = layers[0].capacity(T)
    assert C == math.ceil(cf * T / len(principals))
    ref = _alltoall_emulation(layers, xs, world, Gp, C)
    bufs = PeerBuffers.simulated(world, Gp * C, d, Gp, torch.device("cuda"))
    routes, tps = [], []
    for r, Lr in enumerate(layers):
        routes.append(Lr.ops.route(xs[r]))
        tps.append(Lr.ops.dispatch_peers(xs[r], routes[-1], C, bufs[r]).clone())
    for q, Lr in enumerate(layers):
        Lr.ops.expert_ffn(bufs[q].recv, bufs[q].counts, L, C, world, y_out=bufs[q].y)
    outs = [Lr.ops.combine_peers(tps[r], routes[r], bufs[r]) for r, Lr in enumerate(layers)]
    torch.cuda.synchronize()
    wi = np.stack([O.split_expert(w[g].float().numpy(), d, d_ff, "relu")[0] for g in range(len(principals))])
    wo = np.stack([O.split_expert(w[g].float().numpy(), d, d_ff, "relu")[1] for g in range(len(principals))])
    for r in range(world):
        assert torch.equal(outs[r], ref[r]), f"rank {r}"
        exp = torch.cat([routes[s].kept[r * L:(r + 1) * L] for s in range(world)])
        assert torch.equal(bufs[r].counts, exp)
        y_ref, info = O.layer_forward_fast(xs[r].float().cpu().numpy(), wg.numpy(), wi, wo, 1,
                                           False, cf, slot_map=lut, dtype=np.float64,
                                           round_h=True)
        assert (info["pos"] < 0).any()        # capacity drops exercised
        assert O.normwise_error(outs[r].float().cpu().numpy(), y_ref) < 5e-3
    # and through the public forward (IPC transport) at world 1
    if world == 1:
        y = layers[0].forward(xs[0])
        torch.cuda.synchronize()
        assert torch.equal(y, ref[0])
