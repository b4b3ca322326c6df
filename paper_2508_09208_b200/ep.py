"""Expert parallelism: experts block-partitioned over ranks, tokens data-
parallel, one NCCL all-to-all each way.

Per rank (T_g tokens, E experts, E_l = E / world local experts):
  gate (local, replicated router) -> scan -> permute straight into the send
  buffer laid out [dst rank][local expert][C_g][d] (fixed per-(source, expert)
  capacity C_g = ceil(cf*T_g*k/E), so every all-to-all chunk has the same
  size and no host synchronisation is needed)
  -> all_to_all(counts), all_to_all(rows)
  -> grouped FFN over (source rank, local expert) groups of the receive buffer
  -> all_to_all(rows back) -> combine (token_pos addresses the fixed layout).

`ep_forward_peers` is the same schedule over NVLink peer memory: the permute
stores rows straight into the owners' receive buffers and the combine loads
the outputs from the owners' output buffers (CUDA IPC mappings, flag
barriers; `EPMoELayer(transport="peer")` or COMOE_EP_TRANSPORT=peer).

The collective schedule lives in `ep_forward`, written once against an `ops`
object: `DeviceOps` calls the sm_100a kernels; tests pass a CPU double so the
N>1 data movement is exercised with gloo on a CPU-only box. Capacity is per
token group (GShard/Switch), so rank r's outputs equal a single-device
forward over rank r's tokens.
"""

from __future__ import annotations

import functools
import os
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import kernels
from .pool import ExpertPool


def ep_capacity(tokens_per_rank: int, n_experts: int, top_k: int, capacity_factor) -> int:
    return kernels.capacity_for(tokens_per_rank, n_experts, top_k, capacity_factor)


@dataclass
class EPPlacement:
    """Where the groups of a (possibly merged) variant live under expert
    parallelism. A group is placed on the rank that owns its principal
    expert under the block partition of the original experts (expert e on
    rank e // (E / world)), so a merged expert is computed where its
    principal already was. Groups are numbered in ascending principal order
    (ModelVariant.group_table), so each rank's groups are consecutive.

    Every rank gets the same number L of group slots (the most any rank
    holds); group g is routed as padded index owner(g) * L + local(g). The
    padded routing space has world * L <= E groups, some permanently
    empty, which keeps every exchange block the same size (fixed-layout
    all-to-all chunks, uniform peer blocks) while capacity stays
    C = ceil(cf * T * k / G) over the variant's real G groups."""
    E: int
    world: int
    G: int
    L: int
    owner: list          # [G] rank of each group
    local: list          # [G] index among its rank's groups
    slot_map: list       # [E] original expert -> padded group index
    n_local: list        # [world] groups per rank

    @property
    def G_pad(self) -> int:
        return self.world * self.L

    def local_groups(self, rank: int) -> list:
        """Group indices (variant numbering) of `rank`, in local order."""
        return [g for g in range(self.G) if self.owner[g] == rank]


def ep_placement(lut, principals, E: int, world: int) -> EPPlacement:
    """lut[E] -> group index, principals[G] ascending (ModelVariant.group_table)."""
    if E % world:
        raise ValueError(f"{E} experts do not split over {world} ranks")
    El = E // world
    G = len(principals)
    if list(principals) != sorted(principals) or len(set(principals)) != G:
        raise ValueError("principals must be distinct and ascending")
    if len(lut) != E or any(not 0 <= g < G for g in lut):
        raise ValueError("lut must map every expert to a group")
    owner = [int(p) // El for p in principals]
    n_local = [owner.count(r) for r in range(world)]
    L = max(n_local)
    local, seen = [], [0] * world
    for g in range(G):
        local.append(seen[owner[g]])
        seen[owner[g]] += 1
    padded = [owner[g] * L + local[g] for g in range(G)]
    return EPPlacement(E, world, G, L, owner, local, [padded[g] for g in lut], n_local)


class _NoStage:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


@functools.lru_cache(maxsize=64)
def ep_chunk_base(n_groups: int, world: int, capacity: int, chunks: int, device="cpu"):
    """Send-layout row base of every routing group for a `chunks`-way
    exchange: group g = dst * El + le goes to block
    ((le // Lc) * world + dst) * Lc + le % Lc (Lc = El / chunks), so chunk k
    of the send buffer is one contiguous [dst][Lc][C] all-to-all. chunks = 1
    is the plain [dst][El][C] layout (base = g * C)."""
    El = n_groups // world
    if El % chunks:
        raise ValueError(f"{El} groups per rank do not split into {chunks} chunks")
    Lc = El // chunks
    g = torch.arange(n_groups)
    dst, le = g // El, g % El
    return ((((le // Lc) * world + dst) * Lc + le % Lc) * capacity).to(torch.int32).to(device)


def ep_forward(x, ops, world: int, n_experts: int, capacity: int, group=None, stage=None,
               chunks: int = 1, out=None):
    """One EP layer forward of this rank's tokens `x` [T_g, d]. `stage`:
    optional callable(name) -> context manager timing each step (bench.py).

    chunks > 1 pipelines the exchange over groups of local experts: the send
    buffer is laid out [chunk][dst][El/chunks][C] (ep_chunk_base), every
    chunk's dispatch all-to-all is issued asynchronously up front, and chunk
    k's grouped FFN runs as soon as its rows have arrived — while chunk
    k+1's rows are still in flight — and its outputs go back asynchronously
    while chunk k+1 computes. Each expert's weights are still read once per
    chunk it belongs to, i.e. once. `out`: optional [T_g, d] tensor the
    combine writes into (no extra copy)."""
    st = stage if stage is not None else (lambda name: _NoStage())
    E, C = n_experts, capacity
    El = E // world
    with st("route"):
        route = ops.route(x)                                # gate + scan (counts per global expert)
    if chunks == 1:
        with st("permute"):
            send_rows, token_pos = ops.dispatch(x, route, C)    # [E*C, d] fixed layout
        kept = route.kept                                       # [E] int32, rows per expert from me
        with st("a2a_dispatch"):
            recv_counts = torch.empty_like(kept)
            dist.all_to_all_single(recv_counts, kept, group=group)
            recv_rows = torch.empty_like(send_rows)
            dist.all_to_all_single(recv_rows, send_rows, group=group)
        # groups on the receiver: (src, local expert) -> rows recv_counts[src*El+le]
        y_recv = ops.expert_ffn(recv_rows, recv_counts, El, C, world, stage=st)
        with st("a2a_combine"):
            y_back = torch.empty_like(y_recv)
            dist.all_to_all_single(y_back, y_recv, group=group)
        with st("combine"):
            return ops.combine(y_back, token_pos, route, out=out)
    Lc = El // chunks
    base = ep_chunk_base(E, world, C, chunks, x.device)
    with st("permute"):
        send_rows, token_pos = ops.dispatch(x, route, C, base=base)
    kept = route.kept
    blk = world * Lc * C                                    # rows per chunk
    with st("a2a_dispatch"):
        recv_counts = torch.empty_like(kept)
        dist.all_to_all_single(recv_counts, kept, group=group)
        recv_rows = torch.empty_like(send_rows)
        sends = [dist.all_to_all_single(recv_rows[k * blk:(k + 1) * blk],
                                        send_rows[k * blk:(k + 1) * blk], group=group,
                                        async_op=True) for k in range(chunks)]
    counts = recv_counts.view(world, chunks, Lc)           # [src][chunk][Lc]
    y_recv = torch.empty_like(recv_rows)
    y_back = torch.empty_like(recv_rows)
    backs = []
    for k in range(chunks):
        sends[k].wait()
        ops.expert_ffn(recv_rows[k * blk:(k + 1) * blk], counts[:, k].reshape(-1).contiguous(),
                       Lc, C, world, stage=st, y_out=y_recv[k * blk:(k + 1) * blk],
                       slot_offset=k * Lc)
        backs.append(dist.all_to_all_single(y_back[k * blk:(k + 1) * blk],
                                            y_recv[k * blk:(k + 1) * blk], group=group,
                                            async_op=True))
    with st("a2a_combine"):
        for w in backs:
            w.wait()
    with st("combine"):
        return ops.combine(y_back, token_pos, route, out=out)


class PeerBuffers:
    """This rank's expert-parallel exchange buffers in HBM and the world's
    addresses of them (the peer-memory transport, include/comoe_b200.h "EP
    over NVLink peer memory").

    recv [E*C, d]: rows sent to my experts, laid out [src][local expert][C];
    y [E*C, d]: my experts' outputs in the same layout, read by the sources;
    counts [E]: rows received per (src, local expert); pad [world]: barrier
    flags. Peers' buffers are mapped with CUDA IPC (handles exchanged over
    `group` with all_gather_object), or — `simulated` — are buffers of other
    PeerBuffers in this process (a world on one GPU, for tests)."""

    def __init__(self, rows: int, d: int, E: int, world: int, rank: int, device, group=None,
                 exchange: bool = True):
        self.rows, self.d, self.E, self.world, self.rank = rows, d, E, world, rank
        self.block_rows = rows // world
        self.device = device
        self.recv = torch.zeros((rows, d), dtype=torch.bfloat16, device=device)
        self.y = torch.zeros_like(self.recv)
        self.counts = torch.zeros(E, dtype=torch.int32, device=device)
        self.pad = torch.zeros(world, dtype=torch.int32, device=device)
        self.err = torch.zeros(1, dtype=torch.int32, device=device)
        self.epoch = 0
        self._opened = []
        if exchange:
            self._link_ipc(group)

    _FIELDS = ("recv", "y", "counts", "pad")

    def _link(self, addrs):
        """addrs[field] = world addresses -> int64 device pointer tables."""
        for f in self._FIELDS:
            setattr(self, f + "_ptrs", torch.tensor(addrs[f], dtype=torch.int64, device=self.device))

    def _link_ipc(self, group):
        mine = {f: kernels.ipc_handle(getattr(self, f)) for f in self._FIELDS}
        if self.world == 1:
            allh = [mine]
        else:
            allh = [None] * self.world
            dist.all_gather_object(allh, mine, group=group)
        addrs = {f: [] for f in self._FIELDS}
        for q in range(self.world):
            for f in self._FIELDS:
                if q == self.rank:
                    addrs[f].append(getattr(self, f).data_ptr())
                else:
                    h, off = allh[q][f]
                    ptr = kernels.ipc_open(h, off)
                    self._opened.append((ptr, off))
                    addrs[f].append(ptr)
        self._link(addrs)

    @classmethod
    def simulated(cls, world: int, rows: int, d: int, E: int, device):
        bufs = [cls(rows, d, E, world, r, device, exchange=False) for r in range(world)]
        addrs = {f: [getattr(b, f).data_ptr() for b in bufs] for f in cls._FIELDS}
        for b in bufs:
            b._link(addrs)
        return bufs

    def barrier(self, timeout_s: float = 10.0):
        """Stream-ordered: every later op on this stream runs after every
        rank's earlier ops (their peer stores included) have completed."""
        self.epoch += 1
        kernels.peer_barrier(self.pad_ptrs, self.world, self.rank, self.epoch, self.err, timeout_s)

    def check(self):
        """Raise if a barrier timed out (synchronises)."""
        e = int(self.err.item())
        if e:
            raise RuntimeError(f"peer barrier: rank {e - 1} did not arrive (epoch {self.epoch})")

    def close(self):
        for ptr, off in self._opened:
            kernels.ipc_close(ptr, off)
        self._opened = []


def ep_forward_peers(x, ops, bufs: PeerBuffers, n_experts: int, capacity: int, stage=None,
                     out=None):
    """ep_forward with the all-to-alls replaced by peer-memory stores and
    loads: permute into the owners' receive buffers (+ counts), barrier,
    grouped FFN into my output buffer, barrier, combine from the owners'
    output buffers. Two barriers per forward suffice: a rank reaches the
    next forward's first barrier only after its combine, and peers write my
    receive buffer only after the barrier that follows my GEMMs."""
    st = stage if stage is not None else (lambda name: _NoStage())
    El = n_experts // bufs.world
    with st("route"):
        route = ops.route(x)
    with st("permute"):
        token_pos = ops.dispatch_peers(x, route, capacity, bufs)
    with st("a2a_dispatch"):
        bufs.barrier()
    ops.expert_ffn(bufs.recv, bufs.counts, El, capacity, bufs.world, stage=st, y_out=bufs.y)
    with st("a2a_combine"):
        bufs.barrier()
    with st("combine"):
        return ops.combine_peers(token_pos, route, bufs, out=out)


class DeviceOps:
    """ep_forward ops backed by the CUDA kernels; owns the EP buffers."""

    def __init__(self, layer):
        self.layer = layer
        self._bufs = {}

    def _buf(self, key, make):
        if key not in self._bufs:
            self._bufs[key] = make()
        return self._bufs[key]

    def route(self, x):
        r = self.layer.route(x)
        r.kept = r.scan.group_kept
        self.layer.last = r
        return r

    def dispatch(self, x, route, C, base=None):
        """Permute into the send buffer; `base` [E] (ep_chunk_base) gives each
        group's first row (default g * C)."""
        L = self.layer
        dev, T, E, d = x.device, x.shape[0], L.G, L.d  # E: routing groups
        rows = E * C
        if base is None:
            base = self._buf(("base", E, C),
                             lambda: torch.arange(E, dtype=torch.int32, device=dev) * C)

        perm = self._buf(("perm", T, rows), lambda: kernels.PermuteOutput(
            torch.zeros((rows, d), dtype=torch.bfloat16, device=dev),
            torch.empty(rows, dtype=torch.int32, device=dev),
            torch.empty(rows, dtype=torch.float32, device=dev),
            torch.empty((T, L.top_k), dtype=torch.int32, device=dev)))
        fixed = kernels.ScanOutput(route.scan.tile_offset, route.scan.group_count,
                                   route.scan.group_kept, base)
        kernels.permute(x, route.gate, fixed, C, rows, y_zero=None, out=perm)
        return perm.x_perm, perm.token_pos

    def dispatch_peers(self, x, route, C, bufs):
        """Permute straight into the owners' receive buffers and scatter the
        per-expert row counts; returns token_pos (send-layout rows)."""
        L = self.layer
        dev, T, E = x.device, x.shape[0], L.G  # E: routing groups
        rows = E * C
        if rows != bufs.rows:
            raise ValueError(f"peer buffers hold {bufs.rows} rows, this batch needs {rows}")
        base = self._buf(("base", E, C),
                         lambda: torch.arange(E, dtype=torch.int32, device=dev) * C)
        perm = self._buf(("perm_peers", T, rows), lambda: kernels.PermuteOutput(
            None, torch.empty(rows, dtype=torch.int32, device=dev),
            torch.empty(rows, dtype=torch.float32, device=dev),
            torch.empty((T, L.top_k), dtype=torch.int32, device=dev)))
        fixed = kernels.ScanOutput(route.scan.tile_offset, route.scan.group_count,
                                   route.scan.group_kept, base)
        kernels.permute_peers(x, route.gate, fixed, C, bufs.recv_ptrs, bufs.block_rows,
                              bufs.rank, out=perm)
        kernels.peer_scatter_counts(route.kept, bufs.world, bufs.rank, bufs.counts_ptrs)
        return perm.token_pos

    def combine_peers(self, token_pos, route, bufs, out=None):
        return kernels.combine_peers(bufs.y_ptrs, bufs.block_rows, bufs.rank, token_pos,
                                     route.gate.gate_prob, bufs.d, out=out)

    def expert_ffn(self, recv_rows, recv_counts, El, C, world, stage=None, y_out=None,
                   slot_offset: int = 0):
        """Grouped FFN over the receive buffer [src][local expert][C] rows.
        Groups are enumerated expert-major (j -> local expert j // world,
        source j % world), so the tiles of one expert's `world` source
        blocks run on neighbouring CTA pairs and share its weights in L2
        (source-major order re-streamed each expert's weights once per
        source)."""
        L = self.layer
        dev = recv_rows.device
        G = world * El
        # buffer block of group j: src * El + le
        block = self._buf(("gblock", world, El), lambda: (
            torch.arange(G, device=dev) % world * El + torch.arange(G, device=dev) // world
        ).to(torch.int64))
        base = self._buf(("gbase", world, El, C), lambda: (block * C).to(torch.int32))
        local_slots = getattr(self, "local_slots", None)
        slot = self._buf(("gslot", world, El, slot_offset), lambda: (
            torch.arange(G, device=dev) // world + slot_offset if local_slots is None else
            local_slots.to(dev)[torch.arange(G, device=dev) // world + slot_offset]
        ).to(torch.int32).contiguous())
        recv_counts = recv_counts.index_select(0, block).contiguous()
        # rows this rank computes (bench FLOP count; summed over the chunks)
        self.last_recv_counts = recv_counts if slot_offset == 0 else \
            torch.cat([self.last_recv_counts, recv_counts])
        rows = recv_rows.shape[0]
        y = y_out if y_out is not None else self._buf(("y", rows),
                                                       lambda: torch.empty_like(recv_rows))
        st = stage if stage is not None else (lambda name: _NoStage())
        if kernels.fused_ffn_enabled() and kernels.fused_ffn_supported(
                L.d, L.d_ff, kernels.ACT_RELU if L.act == "relu" else kernels.ACT_SWIGLU, G):
            with st("ffn"):  # K3F: one launch, H on chip
                kernels.fused_ffn(recv_rows, L.pool.data, L.d_ff, recv_counts, base, slot, y)
            return y
        h = self._buf(("h", rows), lambda: torch.empty((rows, L.d_ff), dtype=torch.bfloat16,
                                                       device=dev))
        n1 = 2 * L.d_ff if L.act == "swiglu" else L.d_ff
        with st("ffn1"):
            kernels.grouped_gemm(recv_rows, L.pool.data, 0, n1, recv_counts, base, slot,
                                 kernels.EPI_SWIGLU if L.act == "swiglu" else kernels.EPI_RELU, h)
        with st("ffn2"):
            kernels.grouped_gemm(h, L.pool.data, n1 * L.d, L.d, recv_counts, base, slot,
                                 kernels.EPI_STORE, y)
        return y

    def combine(self, y_back, token_pos, route, out=None):
        return kernels.combine(y_back, token_pos, route.gate.gate_prob, out=out)


class EPMoELayer:
    """MoE layer with experts sharded over the ranks of `group`.

    Holds the full router and this rank's groups in an ExpertPool. Without a
    variant every expert is its own group and rank r holds experts
    [r*E/world, (r+1)*E/world) in pool slots 0..E/world-1. With a merged
    variant (`variant_table` = ModelVariant.group_table(layer, E)) each group
    lives on its principal's rank (ep_placement) and `local_slots[i]` is the
    pool slot of this rank's i-th group."""

    def __init__(self, wg, pool: ExpertPool, d_ff: int, world: int, rank: int, act="relu",
                 top_k=1, norm_topk=None, capacity_factor=1.25, group=None, transport=None,
                 variant_table=None, local_slots=None, chunks: int = None):
        from .layer import MoELayer
        d, E = wg.shape
        if E % world:
            raise ValueError(f"{E} experts do not split over {world} ranks")
        lut, principals = variant_table if variant_table is not None else \
            (list(range(E)), list(range(E)))
        self.placement = ep_placement(lut, principals, E, world)
        n_mine = self.placement.n_local[rank]
        if local_slots is None:
            local_slots = list(range(n_mine))
        if len(local_slots) != n_mine or any(not 0 <= s < pool.n_slots for s in local_slots):
            raise ValueError(f"pool must hold this rank's {n_mine} groups (local_slots)")
        self.world, self.rank, self.E = world, rank, E
        self.G = self.placement.G
        self.El = self.placement.L          # group slots per rank (padded)
        self.G_pad = self.placement.G_pad   # routing groups (with empty placeholders)
        self.group = group
        self.capacity_factor = capacity_factor
        # gate/scan run over the padded group space; capacity uses the
        # variant's real group count (== E without a variant)
        self.local = MoELayer(wg, pool, d_ff, act=act, top_k=top_k, norm_topk=norm_topk,
                              capacity_factor=capacity_factor, expert_slots=[0] * E)
        self.local.set_variant(self.placement.slot_map, [0] * self.G_pad,
                               capacity_groups=self.G)
        self.ops = DeviceOps(self.local)
        self.ops.local_slots = torch.tensor(list(local_slots) + [local_slots[0] if local_slots
                                                                  else 0] * (self.El - n_mine),
                                            dtype=torch.int64)
        # "nccl": two ncclAllToAll per forward; "peer": stores / loads into the
        # peers' HBM over NVLink (CUDA IPC) with flag barriers
        self.transport = transport or os.environ.get("COMOE_EP_TRANSPORT", "nccl")
        # NCCL transport: the exchange pipelined over `chunks` groups of local
        # experts (ep_forward); default 2 when there are peers to overlap with
        if chunks is None:
            env = os.environ.get("COMOE_EP_CHUNKS")
            chunks = int(env) if env else (2 if world > 1 and self.El % 2 == 0 else 1)
        if chunks < 1 or self.El % chunks:
            raise ValueError(f"chunks={chunks} must divide the {self.El} group slots per rank")
        self.chunks = chunks
        if self.transport not in ("nccl", "peer"):
            raise ValueError(f"unknown EP transport {self.transport!r}")
        self.peers = None

    @classmethod
    def synthetic(cls, wg, d_ff, E, world, rank, capacity_factor=1.25, seed=2, act="relu"):
        d = wg.shape[0]
        numel = kernels.expert_numel(d, d_ff, kernels.ACT_SWIGLU if act == "swiglu" else kernels.ACT_RELU)
        pool = ExpertPool(E // world, numel, device=wg.device)
        pool.data.normal_(0.0, 0.02,
                          generator=torch.Generator(device=wg.device).manual_seed(seed + rank))
        return cls(wg, pool, d_ff, world, rank, act=act, capacity_factor=capacity_factor)

    def capacity(self, T: int) -> int:
        return ep_capacity(T, self.G, self.local.top_k, self.capacity_factor)

    @property
    def last(self):
        return self.local.last

    def peer_buffers(self, T: int) -> PeerBuffers:
        """The peer-transport buffers for T tokens per rank (collective on
        first use and whenever the capacity changes: every rank calls it
        with the same T)."""
        rows = self.G_pad * self.capacity(T)
        if self.peers is None or self.peers.rows != rows:
            if self.peers is not None:
                self.peers.close()
            self.peers = PeerBuffers(rows, self.local.d, self.G_pad, self.world, self.rank,
                                     self.local.wg.device, group=self.group)
        return self.peers

    # peer transport: a barrier that times out sets a sticky error flag
    # instead of hanging; forward() reads it (one host sync) every
    # `err_check_every` calls outside CUDA-graph capture and raises, so a
    # dead or late peer cannot leave partially written outputs unnoticed
    err_check_every = 8

    def forward(self, x, out=None, timer=None):
        C = self.capacity(x.shape[0])
        if self.transport == "peer":
            bufs = self.peer_buffers(x.shape[0])
            y = ep_forward_peers(x, self.ops, bufs, self.G_pad, C, stage=timer, out=out)
            self._calls = getattr(self, "_calls", 0) + 1
            if self._calls % self.err_check_every == 0 and \
                    not torch.cuda.is_current_stream_capturing():
                bufs.check()
        else:
            y = ep_forward(x, self.ops, self.world, self.G_pad, C, group=self.group, stage=timer,
                           chunks=self.chunks, out=out)
        return y

    __call__ = forward

    @property
    def kernels_per_forward(self) -> int:
        # gate (+ scan unless folded), permute, 2x GEMM, combine (NCCL's
        # all-to-all kernels not counted)
        from .layer import _gate_fold
        return 5 if _gate_fold() else 6
