"""The peer-memory EP transport across a real process boundary: two
processes on the same GPU (the pool's boxes have one), each a rank of a
world-2 EPMoELayer(transport="peer"). Exercises what the in-process
simulated world cannot: the CUDA IPC handle exchange (all_gather_object over
gloo), cudaIpcOpenMemHandle of the peer's buffers, the peer-store permute
into another process's HBM, the flag barrier across contexts (time-sliced on
one GPU), and the peer-load combine. Each rank's output must match the
oracle's single-device forward of its own tokens; a merged variant with
groups on their principals' ranks is run too."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import switch_layer as O

pytestmark = pytest.mark.gpu

T, D, D_FF, E, CF = 600, 256, 512, 8, 1.0


def _worker(rank, world, port, merged, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2508_09208_b200 import ExpertPool, kernels
        from paper_2508_09208_b200.ep import EPMoELayer, ep_placement
        g = torch.Generator().manual_seed(7)
        wg = torch.randn(D, E, generator=g) / math.sqrt(D)
        numel = kernels.expert_numel(D, D_FF, kernels.ACT_RELU)
        if merged:
            principals, lut = [0, 1, 2, 6], [0, 1, 2, 2, 1, 3, 3, 0]
        else:
            principals, lut = list(range(E)), list(range(E))
        G = len(principals)
        w = (torch.randn(G, numel, generator=g) * 0.02).to(torch.bfloat16)
        xs = [torch.randn(T, D, generator=g).to(torch.bfloat16) for _ in range(world)]
        pl = ep_placement(lut, principals, E, world)
        mine = pl.local_groups(rank)
        pool = ExpertPool(max(1, len(mine)), numel)
        for s, grp in enumerate(mine):
            pool.data[s, :numel].copy_(w[grp].cuda())
        layer = EPMoELayer(wg.cuda(), pool, D_FF, world=world, rank=rank, capacity_factor=CF,
                           transport="peer", variant_table=(lut, principals),
                           local_slots=list(range(len(mine))))
        x = xs[rank].cuda()
        outs = [layer.forward(x).clone() for _ in range(3)]   # epochs 1..6
        torch.cuda.synchronize()
        layer.peers.check()
        wi = np.stack([O.split_expert(w[k].float().numpy(), D, D_FF, "relu")[0] for k in range(G)])
        wo = np.stack([O.split_expert(w[k].float().numpy(), D, D_FF, "relu")[1] for k in range(G)])
        y_ref, info = O.layer_forward_fast(xs[rank].float().numpy(), wg.numpy(), wi, wo, 1, False,
                                           CF, slot_map=lut, dtype=np.float64, round_h=True)
        err = O.normwise_error(outs[0].float().cpu().numpy(), y_ref)
        same = all(torch.equal(o, outs[0]) for o in outs[1:])
        dist.barrier()
        layer.peers.close()
        q.put((rank, err, same, int((info["pos"] < 0).sum()), layer.peers.epoch, None))
        dist.destroy_process_group()
    except Exception as exc:  # report instead of hanging the parent
        q.put((rank, None, None, None, None, repr(exc)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("merged", [False, True])
def test_peer_transport_two_processes(merged):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, merged, q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        res = [q.get(timeout=240) for _ in procs]
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for rank, err, same, dropped, epoch, exc in res:
        assert exc is None, (rank, exc)
        assert err < 5e-3, (rank, err)
        assert same and epoch == 6
        assert dropped > 0
