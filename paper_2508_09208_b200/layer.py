"""MoELayer: the B200 MoE-layer forward (the new `MoELayer.forward(x)` of
SURVEY §8b). Replaces the reference's per-token analytic layer charge
(pkg/src/comoe/simulator.py:684-724, expert compute at :705) with

    K1 gate (tcgen05 fp32-faithful logits, softmax, top-k, slot remap, tile ranks)
    -> route scan (capacity in stream order, group bases)
    -> K2 permute (expert-sorted compact rows; zero rows of dropped tokens)
    -> K3 grouped FFN (tcgen05 GEMM1 + act -> H, GEMM2 -> fused top-1 combine)
    -> K4 combine (top-2 only)

all enqueued on the current stream, no host synchronisation. Expert weights
live in an ExpertPool; a merged variant only changes the slot_map LUT and
the per-group slot list, never the kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import kernels
from .pool import ExpertPool

import os

ACTS = {"relu": kernels.ACT_RELU, "swiglu": kernels.ACT_SWIGLU}


def _gather_enabled(act: str) -> bool:
    """Opt-in (COMOE_GATHER=1): GEMM1 gathers token rows with TMA gather4
    instead of reading the permuted copy. Correct, but measured 3.3x slower
    for GEMM1 at C2 (830 vs 255 us: 32 four-row gathers per k-block per CTA
    saturate the TMA unit), so the permute copy (42 us) stays the default."""
    return act == "relu" and os.environ.get("COMOE_GEMM_1SM", "0") != "1" and \
        os.environ.get("COMOE_GATHER", "0") == "1"


def _gate_fold() -> bool:
    """Gate and capacity scan as one launch (comoe_gate_route, default).
    COMOE_GATE_FOLD=0 runs comoe_gate_topk + comoe_route_scan (two
    launches, identical tables)."""
    return os.environ.get("COMOE_GATE_FOLD", "1") != "0" and \
        os.environ.get("COMOE_GATE_DEBUG", "0") == "0"


def _fused_gather() -> bool:
    """The fused FFN reads token rows straight from x with TMA gather4 (no
    permuted copy; default). COMOE_FUSED_GATHER=0 reads the permuted copy."""
    return os.environ.get("COMOE_FUSED_GATHER", "1") != "0"


class _NoTimer:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def _no_timer(name):
    return _NoTimer()


@dataclass
class LayerRouting:
    gate: kernels.GateOutput
    scan: kernels.ScanOutput
    perm: kernels.PermuteOutput
    capacity: int
    rows: int


class MoELayer:
    def __init__(self, wg: torch.Tensor, pool: ExpertPool, d_ff: int, act: str = "relu",
                 top_k: int = 1, norm_topk: bool = None, capacity_factor=1.25,
                 expert_slots=None):
        if act not in ACTS:
            raise ValueError(f"act must be one of {sorted(ACTS)}")
        if top_k not in (1, 2):
            raise ValueError("top_k must be 1 or 2")
        kernels._need(wg, "wg", torch.float32, 2)
        self.d, self.E = wg.shape
        self.d_ff = int(d_ff)
        self.act = act
        self.top_k = top_k
        self.norm_topk = (top_k > 1) if norm_topk is None else bool(norm_topk)
        self.capacity_factor = capacity_factor
        self.pool = pool
        if pool.numel < kernels.expert_numel(self.d, self.d_ff, ACTS[act]):
            raise ValueError("pool slots are too small for this expert shape")
        self.wg = wg
        self.wg_split = kernels.gate_prepare(wg)
        slots = list(range(self.E)) if expert_slots is None else list(expert_slots)
        self.set_variant(list(range(self.E)), slots)
        self._ws = {}
        self.last: LayerRouting = None

    # ------------------------------------------------------------ variants
    def set_variant(self, slot_map, group_slots, capacity_groups: int = None) -> None:
        """slot_map[E]: original expert -> group index; group_slots[G]: pool
        slot serving each group (ModelVariant.group_table gives both).
        `capacity_groups`: the G of the capacity formula when the routing
        groups include empty placeholders (expert parallelism pads every
        rank to the same number of group slots; ep.ep_placement)."""
        slot_map = [int(s) for s in slot_map]
        group_slots = [int(s) for s in group_slots]
        G = len(group_slots)
        if len(slot_map) != self.E or any(not 0 <= g < G for g in slot_map):
            raise ValueError("slot_map must map every expert to a group index")
        if any(not 0 <= s < self.pool.n_slots for s in group_slots):
            raise ValueError("group slot outside the pool")
        dev = self.wg.device
        self.G = G
        self.capacity_groups = G if capacity_groups is None else int(capacity_groups)
        self.slot_map_host = list(slot_map)
        self.slot_map = torch.tensor(slot_map, dtype=torch.int32, device=dev)
        self.group_slot = torch.tensor(group_slots, dtype=torch.int32, device=dev)
        self._ws = {}

    def use_variant(self, variant, layer: int) -> None:
        """Point the layer at a ModelVariant whose retained experts live in
        this layer's pool (aggregation.fuse_model(..., pool=...))."""
        lut, principals = variant.group_table(layer, self.E)
        slots = []
        for p in principals:
            s = self.pool.slot_of(variant.retained[layer][p].params)
            if s is None:
                raise ValueError(f"expert ({layer},{p}) is not a slot of this layer's pool")
            slots.append(s)
        self.set_variant(lut, slots)

    # ------------------------------------------------------------ workspace
    def capacity(self, T: int) -> int:
        return kernels.capacity_for(T, self.capacity_groups, self.top_k, self.capacity_factor)

    @property
    def fused(self) -> bool:
        """Whether the forward runs the fused FFN (K3F: one launch, H on chip)."""
        return kernels.fused_ffn_enabled() and \
            kernels.fused_ffn_supported(self.d, self.d_ff, ACTS[self.act], self.G)

    def _workspace(self, T: int):
        ws = self._ws.get(T)
        if ws is not None:
            return ws
        dev = self.wg.device
        C = self.capacity(T)
        rows = max(1, min(T * self.top_k, self.G * C))
        k, nt = self.top_k, kernels.gate_num_tiles(T)
        fused = self.fused
        gather = fused and _fused_gather()
        ws = dict(
            C=C, rows=rows, fused=fused, gather=gather,
            gate=kernels.GateOutput(
                torch.empty((T, k), dtype=torch.int32, device=dev),
                torch.empty((T, k), dtype=torch.int32, device=dev),
                torch.empty((T, k), dtype=torch.float32, device=dev),
                torch.empty((T, k), dtype=torch.int32, device=dev),
                torch.empty((k, nt, self.G), dtype=torch.int32, device=dev)),
            scan=kernels.ScanOutput(torch.empty((k, nt, self.G), dtype=torch.int32, device=dev),
                                    *(torch.empty(self.G, dtype=torch.int32, device=dev)
                                      for _ in range(3))),
            perm=kernels.PermuteOutput(torch.empty((1 if gather else rows, self.d),
                                                   dtype=torch.bfloat16, device=dev),
                                       torch.empty(rows, dtype=torch.int32, device=dev),
                                       torch.empty(rows, dtype=torch.float32, device=dev),
                                       torch.empty((T, k), dtype=torch.int32, device=dev)),
            lb=kernels.gate_route_workspace(T, k, self.G, dev) if _gate_fold() else None,
            h=None if fused else torch.empty((rows, self.d_ff), dtype=torch.bfloat16, device=dev),
            y_perm=torch.empty((rows, self.d), dtype=torch.bfloat16, device=dev) if k > 1 else None,
        )
        self._ws[T] = ws
        return ws

    # ------------------------------------------------------------ forward
    def route(self, x: torch.Tensor, want_logits: bool = False, routing=None) -> LayerRouting:
        """Gate + capacity scan. `routing` = (expert_idx [T,k] int32, probs
        [T,k] float32 or None) replays given choices (e.g. a reference
        RoutingTrace) instead of running the router."""
        kernels._need(x, "x", torch.bfloat16, 2)
        T = x.shape[0]
        ws = self._workspace(T)
        gate = ws["gate"]
        if routing is not None:
            idx, probs = routing
            if tuple(idx.shape) != (T, self.top_k):
                raise ValueError(f"routing must be [T, {self.top_k}]")
            kernels.route_from_indices(idx.to(torch.int32).contiguous(), self.E, probs=probs,
                                       slot_map=self.slot_map, n_groups=self.G, out=gate)
            kernels.route_scan(gate.tile_hist, ws["C"], out=ws["scan"])
            return LayerRouting(gate, ws["scan"], ws["perm"], ws["C"], ws["rows"])
        if want_logits:
            gate = kernels.GateOutput(gate.expert_idx, gate.group_idx, gate.gate_prob,
                                      gate.local_rank, gate.tile_hist,
                                      torch.empty((T, self.E), dtype=torch.float32, device=x.device))
        if ws["lb"] is not None:
            kernels.gate_route(x, self.wg_split, self.E, self.top_k, self.norm_topk, ws["C"],
                               ws["lb"], slot_map=self.slot_map, n_groups=self.G, out=gate,
                               scan=ws["scan"])
        else:
            kernels.gate_topk(x, self.wg_split, self.E, self.top_k, self.norm_topk,
                              slot_map=self.slot_map, n_groups=self.G, out=gate)
            kernels.route_scan(gate.tile_hist, ws["C"], out=ws["scan"])
        return LayerRouting(gate, ws["scan"], ws["perm"], ws["C"], ws["rows"])

    def forward(self, x: torch.Tensor, out: torch.Tensor = None,
                want_logits: bool = False, timer=None, routing=None) -> torch.Tensor:
        """`timer`: optional callable(name) -> context manager recording
        CUDA events around each stage on the current stream (bench.py)."""
        if x.shape[1] != self.d:
            raise ValueError(f"x must be [T, {self.d}]")
        T = x.shape[0]
        if out is None:
            out = torch.empty((T, self.d), dtype=torch.bfloat16, device=x.device)
        if T == 0:
            return out
        ws = self._workspace(T)
        stage = timer if timer is not None else _no_timer
        with stage("route"):
            r = self.route(x, want_logits, routing=routing)
        k1 = self.top_k == 1
        dst = out if k1 else ws["y_perm"]
        if ws["fused"]:
            gather = ws["gather"]
            with stage("permute"):  # (index tables only when the FFN gathers the rows)
                kernels.permute(x, r.gate, r.scan, r.capacity, r.rows,
                                y_zero=out if k1 else None, out=r.perm, copy_rows=not gather)
            with stage("ffn"):
                kernels.fused_ffn(x if gather else r.perm.x_perm, self.pool.data, self.d_ff,
                                  r.scan.group_kept, r.scan.group_base, self.group_slot, dst,
                                  gather_rows=r.perm.row_token if gather else None,
                                  row_token=r.perm.row_token if k1 else None,
                                  row_prob=r.perm.row_prob if k1 else None)
            if not k1:
                with stage("combine"):
                    kernels.combine(ws["y_perm"], r.perm.token_pos, r.gate.gate_prob, out=out)
            self.last = r
            return out
        gather = _gather_enabled(self.act)
        with stage("permute"):
            kernels.permute(x, r.gate, r.scan, r.capacity, r.rows, y_zero=out if k1 else None,
                            out=r.perm, copy_rows=not gather)
        n1 = 2 * self.d_ff if self.act == "swiglu" else self.d_ff
        with stage("ffn1"):
            kernels.grouped_gemm(x if gather else r.perm.x_perm, self.pool.data, 0, n1,
                                 r.scan.group_kept, r.scan.group_base, self.group_slot,
                                 kernels.EPI_SWIGLU if self.act == "swiglu" else kernels.EPI_RELU,
                                 ws["h"], a_gather=r.perm.row_token if gather else None)
        with stage("ffn2"):
            kernels.grouped_gemm(ws["h"], self.pool.data, n1 * self.d, self.d, r.scan.group_kept,
                                 r.scan.group_base, self.group_slot,
                                 kernels.EPI_SCALE_SCATTER if k1 else kernels.EPI_STORE, dst,
                                 row_token=r.perm.row_token if k1 else None,
                                 row_prob=r.perm.row_prob if k1 else None)
        if not k1:
            with stage("combine"):
                kernels.combine(ws["y_perm"], r.perm.token_pos, r.gate.gate_prob, out=out)
        self.last = r
        return out

    __call__ = forward

    @property
    def kernels_per_forward(self) -> int:
        """Device kernels one forward launches: gate (+ scan unless folded),
        permute, FFN (one fused launch or two GEMMs) [, combine]."""
        return (3 if self.fused else 4) + (0 if _gate_fold() else 1) + \
            (0 if self.top_k == 1 else 1)

    def capture(self, x: torch.Tensor, out: torch.Tensor = None) -> "CapturedForward":
        """Record one forward over the static buffers `x` (and `out`) as a
        CUDA graph: `replay()` re-runs gate -> scan -> permute -> GEMMs on
        whatever `x` holds (routing and capacity are computed on the
        device, so every replay is a complete forward of the current
        contents) without per-kernel launch overhead."""
        return CapturedForward(self, x, out)


class CapturedForward:
    """A MoELayer forward recorded as a CUDA graph on static device buffers.

    Write the batch into `.x` (e.g. the destination of an H2D copy), call
    `replay()` on the stream that should run it, read `.y`. The layer's
    workspace for this token count is shared with its eager forward (do not
    run both concurrently). Measured at C2: 0.647 ms eager vs 0.627 ms per
    replay (the five launches' gaps and host overhead)."""

    def __init__(self, layer: MoELayer, x: torch.Tensor, out: torch.Tensor = None):
        self.layer = layer
        self.x = x
        self.y = out if out is not None else torch.empty_like(x)
        dev = x.device
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):  # workspace and tensor maps outside the capture
            layer.forward(self.x, out=self.y)
        torch.cuda.current_stream(dev).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            layer.forward(self.x, out=self.y)

    def replay(self) -> torch.Tensor:
        self.graph.replay()
        return self.y
