"""Expert-parallel schedule (paper_2508_09208_b200.ep.ep_forward) with the
gloo backend, world size 2, on CPU: the same all-to-all layout/count logic
the NCCL path runs, with a CPU test double for the per-rank kernels. Each
rank's output must equal the single-device oracle forward of its tokens
(capacity is per token group)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import switch_layer as O

T_G, D, D_FF, E, CF = 300, 64, 128, 8, 1.0


class OracleOps:
    """CPU double of ep.DeviceOps (test infrastructure)."""

    def __init__(self, wg, w_in, w_out, rank, world, top_k=1, placement=None):
        """placement: ep.EPPlacement of a merged variant (w_in / w_out are
        then indexed by the variant's group); None = one group per expert."""
        self.wg, self.w_in, self.w_out = wg, w_in, w_out
        self.rank, self.world, self.top_k = rank, world, top_k
        self.pl = placement
        self.El = E // world if placement is None else placement.L
        self.G_pad = E if placement is None else placement.G_pad
        self.G = E if placement is None else placement.G

    def route(self, x):
        xn = x.numpy()
        logits = O.gate_logits(xn, self.wg)
        sm = None if self.pl is None else self.pl.slot_map
        idx, grp, prob = O.topk_route(logits, self.top_k, self.top_k == 2, sm)
        C = O.capacity(xn.shape[0], self.G, self.top_k, CF)
        disp = O.dispatch_fast(grp, self.G_pad, C)

        class R:
            pass
        r = R()
        r.prob, r.disp, r.C = prob, disp, C
        r.rank_ = disp["rank"]
        r.group = grp
        r.kept = torch.tensor(disp["kept"], dtype=torch.int32)
        return r

    def dispatch(self, x, route, C, base=None):
        xn = x.numpy()
        base = np.arange(self.G_pad) * C if base is None else base.numpy()
        rows = np.zeros((self.G_pad * C, xn.shape[1]), np.float32)
        pos = np.full(route.group.shape, -1, np.int64)
        for t in range(xn.shape[0]):
            for j in range(self.top_k):
                g, rk = route.group[t, j], route.rank_[t, j]
                if g >= 0 and rk < C:
                    pos[t, j] = base[g] + rk
                    rows[pos[t, j]] = xn[t]
        return torch.from_numpy(rows), pos

    def expert_ffn(self, recv_rows, recv_counts, El, C, world, stage=None, y_out=None,
                   slot_offset=0):
        out = torch.zeros_like(recv_rows) if y_out is None else y_out.zero_()
        cnt = recv_counts.numpy()
        for src in range(world):
            for le in range(El):
                g = src * El + le
                n = int(cnt[g])
                if n == 0:
                    continue
                lg = slot_offset + le                    # local group slot
                e = self.rank * self.El + lg if self.pl is None else \
                    self.pl.local_groups(self.rank)[lg]
                if self.pl is not None and lg >= self.pl.n_local[self.rank]:
                    continue
                xs = recv_rows[g * C:g * C + n].numpy().astype(np.float64)
                y = O.expert_ffn(xs, self.w_in[e], self.w_out[e], "relu", round_h=False)
                out[g * C:g * C + n] = torch.from_numpy(y.astype(np.float32))
        return out

    def combine(self, y_back, token_pos, route, out=None):
        yb = y_back.numpy()
        T = token_pos.shape[0]
        y = np.zeros((T, yb.shape[1]), np.float64)
        for j in range(self.top_k):
            m = token_pos[:, j] >= 0
            y[m] += route.prob[m, j][:, None] * yb[token_pos[m, j]]
        if out is not None:
            out.copy_(torch.from_numpy(y))
            return out
        return torch.from_numpy(y)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2508_09208_b200.ep import ep_forward
        rng = np.random.default_rng(0)
        wg = (rng.normal(size=(D, E)) / 8).astype(np.float32)
        w_in = O.bf16_round(rng.normal(size=(E, D_FF, D)) * 0.05)
        w_out = O.bf16_round(rng.normal(size=(E, D, D_FF)) * 0.05)
        xs = [O.bf16_round(np.random.default_rng(10 + r).normal(size=(T_G, D))) for r in range(world)]
        ops = OracleOps(wg, w_in, w_out, rank, world)
        C = O.capacity(T_G, E, 1, CF)
        y = ep_forward(torch.from_numpy(xs[rank]), ops, world, E, C).numpy()
        ref, info = O.layer_forward_fast(xs[rank], wg, w_in, w_out, 1, False, CF,
                                         dtype=np.float64)
        q.put((rank, float(np.abs(y - ref).max()), int((info["pos"] < 0).sum())))
    finally:
        dist.destroy_process_group()


# a merged 8 -> 4 variant whose principals are unevenly spread over 2 ranks
# (rank 0 owns principals 0, 2, 3; rank 1 owns 5): L = 3 group slots per
# rank, a padded routing space of 6 groups, capacity over the real 4
MERGED_PRINCIPALS = [0, 2, 3, 5]
MERGED_LUT = [0, 0, 1, 2, 1, 3, 3, 2]


def _merged_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2508_09208_b200.ep import ep_forward, ep_placement
        pl = ep_placement(MERGED_LUT, MERGED_PRINCIPALS, E, world)
        rng = np.random.default_rng(1)
        wg = (rng.normal(size=(D, E)) / 8).astype(np.float32)
        G = len(MERGED_PRINCIPALS)
        w_in = O.bf16_round(rng.normal(size=(G, D_FF, D)) * 0.05)
        w_out = O.bf16_round(rng.normal(size=(G, D, D_FF)) * 0.05)
        xs = [O.bf16_round(np.random.default_rng(20 + r).normal(size=(T_G, D))) for r in range(world)]
        ops = OracleOps(wg, w_in, w_out, rank, world, placement=pl)
        C = O.capacity(T_G, G, 1, CF)
        y = ep_forward(torch.from_numpy(xs[rank]), ops, world, pl.G_pad, C).numpy()
        ref, info = O.layer_forward_fast(xs[rank], wg, w_in, w_out, 1, False, CF,
                                         slot_map=MERGED_LUT, dtype=np.float64)
        q.put((rank, float(np.abs(y - ref).max()), int((info["pos"] < 0).sum())))
    finally:
        dist.destroy_process_group()


def _chunked_worker(rank, world, port, chunks, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2508_09208_b200.ep import ep_forward
        rng = np.random.default_rng(0)
        wg = (rng.normal(size=(D, E)) / 8).astype(np.float32)
        w_in = O.bf16_round(rng.normal(size=(E, D_FF, D)) * 0.05)
        w_out = O.bf16_round(rng.normal(size=(E, D, D_FF)) * 0.05)
        xs = [O.bf16_round(np.random.default_rng(10 + r).normal(size=(T_G, D))) for r in range(world)]
        ops = OracleOps(wg, w_in, w_out, rank, world)
        C = O.capacity(T_G, E, 1, CF)
        y = ep_forward(torch.from_numpy(xs[rank]), ops, world, E, C, chunks=chunks).numpy()
        ref, info = O.layer_forward_fast(xs[rank], wg, w_in, w_out, 1, False, CF,
                                         dtype=np.float64)
        q.put((rank, float(np.abs(y - ref).max()), int((info["pos"] < 0).sum())))
    finally:
        dist.destroy_process_group()


def test_ep_chunk_base_layout():
    from paper_2508_09208_b200.ep import ep_chunk_base
    # 8 groups, 2 ranks (El = 4), 2 chunks (Lc = 2), C = 10: send layout
    # [chunk][dst][Lc][C]: chunk 0 = (d0: g0 g1 | d1: g4 g5), chunk 1 = (d0: g2 g3 | d1: g6 g7)
    assert ep_chunk_base(8, 2, 10, 2).tolist() == [0, 10, 40, 50, 20, 30, 60, 70]
    assert ep_chunk_base(8, 2, 10, 1).tolist() == [10 * g for g in range(8)]
    with pytest.raises(ValueError):
        ep_chunk_base(8, 2, 10, 3)


@pytest.mark.parametrize("chunks", [2, 4])
def test_ep_forward_chunked_world2_gloo(chunks):
    """The chunked exchange (async all-to-all per chunk of local experts,
    FFN of chunk k while chunk k+1 is in flight) gives every rank the same
    output as the single-device oracle forward of its tokens."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chunked_worker, args=(r, 2, port, chunks, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, dropped in res:
        assert err < 1e-5, (rank, err)
        assert dropped > 0


def test_ep_placement_tables():
    from paper_2508_09208_b200.ep import ep_placement
    pl = ep_placement(MERGED_LUT, MERGED_PRINCIPALS, E, 2)
    assert pl.owner == [0, 0, 0, 1] and pl.local == [0, 1, 2, 0]
    assert pl.n_local == [3, 1] and pl.L == 3 and pl.G_pad == 6
    # padded index owner*L + local; every expert follows its group
    assert pl.slot_map == [0, 0, 1, 2, 1, 3, 3, 2]
    assert pl.local_groups(0) == [0, 1, 2] and pl.local_groups(1) == [3]
    ident = ep_placement(list(range(E)), list(range(E)), E, 4)
    assert ident.slot_map == list(range(E)) and ident.L == 2 and ident.G_pad == E
    with pytest.raises(ValueError):
        ep_placement(MERGED_LUT, [2, 0, 3, 5], E, 2)


def test_ep_merged_variant_world2_gloo():
    """A merged variant under EP: groups on their principal's rank, padded
    routing space, capacity over the real groups; each rank's output equals
    the single-device oracle forward of the merged layer on its tokens."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_merged_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, dropped in res:
        assert err < 1e-5, (rank, err)
        assert dropped > 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_ep_forward_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, dropped in res:
        assert err < 1e-5, (rank, err)
        assert dropped > 0  # capacity factor 1.0 forces drops: the per-group rule is exercised


def _peer_worker(rank, world, port, q):
    """PeerBuffers' handle exchange over gloo with the IPC calls stubbed: the
    pointer tables must list every rank's buffers in rank order (own buffers
    by address, peers' through ipc_open of their handle + offset)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2508_09208_b200 import kernels
        from paper_2508_09208_b200.ep import PeerBuffers
        opened = []
        kernels.ipc_handle = lambda t: (f"r{rank}:{t.numel()}".encode(), 100 + rank)
        kernels.ipc_open = lambda h, off: opened.append((h, off)) or (1 << 40) + 1000 * int(h[1:2]) + off
        b = PeerBuffers(world * 6, 16, 4 * world, world, rank, torch.device("cpu"))
        res = {f: getattr(b, f + "_ptrs").tolist() for f in PeerBuffers._FIELDS}
        q.put((rank, res, {f: getattr(b, f).data_ptr() for f in PeerBuffers._FIELDS},
               sorted(opened), len(b._opened)))
    finally:
        dist.destroy_process_group()


def test_peer_buffers_handle_exchange_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 3
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ptrs, own, opened, n_open in res:
        assert n_open == 4 * (world - 1)
        for f, table in ptrs.items():
            assert len(table) == world
            for qr in range(world):
                if qr == rank:
                    assert table[qr] == own[f]
                else:  # the fake mapping of rank qr's handle at its offset
                    assert table[qr] == (1 << 40) + 1000 * qr + 100 + qr
