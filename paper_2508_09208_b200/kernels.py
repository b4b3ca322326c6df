"""Thin PyTorch-facing wrappers over the C ABI (one function per kernel).

PyTorch only provides device memory and the current stream here; every
computation below runs in libcomoe_b200.so. Arguments are validated on the
host (device, dtype, contiguity, alignment) before the C call, which
validates sizes again and reports through comoe_last_error().
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import torch

from . import _lib

ACT_RELU, ACT_SWIGLU = 0, 1
EPI_RELU, EPI_SWIGLU, EPI_SCALE_SCATTER, EPI_STORE = 0, 1, 2, 3
DTYPE_BF16, DTYPE_F64 = 0, 1
GEMM_BM = 128


def _ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _need(t: torch.Tensor, name: str, dtype=None, dims=None, align=16):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must live on a CUDA device (no CPU path)")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if dims is not None and t.dim() != dims:
        raise ValueError(f"{name} must be {dims}-D, got shape {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.data_ptr() % align:
        raise ValueError(f"{name} must be {align}-byte aligned")
    return t


def _need_out(out: torch.Tensor, shape, device):
    """An output tensor handed in by the caller: bf16, `shape`, on `device`."""
    _need(out, "out", torch.bfloat16, len(shape))
    if tuple(out.shape) != tuple(shape):
        raise ValueError(f"out must have shape {tuple(shape)}, got {tuple(out.shape)}")
    if out.device != device:
        raise ValueError(f"out must live on {device}, got {out.device}")


def num_sms(device=None) -> int:
    dev = torch.cuda.current_device() if device is None else device
    return _lib.load().comoe_num_sms(int(dev))


# ---------------------------------------------------------------- K1 gate

def gate_padded_experts(E: int) -> int:
    ep = _lib.load().comoe_gate_padded_experts(int(E))
    if ep < 0:
        raise ValueError(f"gate supports 1..128 experts, got {E}")
    return ep


def gate_num_tiles(T: int) -> int:
    return (int(T) + GEMM_BM - 1) // GEMM_BM


def gate_prepare(wg: torch.Tensor) -> torch.Tensor:
    """fp32 router Wg[d, E] -> bf16 split terms [3, EP, d] (hi, mid, lo)."""
    _need(wg, "wg", torch.float32, 2)
    d, E = wg.shape
    ep = gate_padded_experts(E)
    out = torch.empty((3, ep, d), dtype=torch.bfloat16, device=wg.device)
    _lib.call("comoe_gate_prepare", _ptr(wg), d, E, _ptr(out), _stream())
    return out


@dataclass
class GateOutput:
    expert_idx: torch.Tensor   # [T, k] int32 original expert
    group_idx: torch.Tensor    # [T, k] int32 group after slot remap, -1 = none
    gate_prob: torch.Tensor    # [T, k] float32
    local_rank: torch.Tensor   # [T, k] int32 rank inside the 128-token tile
    tile_hist: torch.Tensor    # [k, ntiles, G] int32
    logits: torch.Tensor = None  # [T, E] float32 (optional)


def gate_topk(x, wg_split, E, top_k, norm_topk, slot_map=None, n_groups=None,
              want_logits=False, out: GateOutput = None) -> GateOutput:
    _need(x, "x", torch.bfloat16, 2)
    _need(wg_split, "wg_split", torch.bfloat16, 3)
    T, d = x.shape
    G = E if n_groups is None else int(n_groups)
    if slot_map is not None:
        _need(slot_map, "slot_map", torch.int32, 1)
    nt = gate_num_tiles(T)
    dev = x.device
    if out is None:
        out = GateOutput(
            expert_idx=torch.empty((T, top_k), dtype=torch.int32, device=dev),
            group_idx=torch.empty((T, top_k), dtype=torch.int32, device=dev),
            gate_prob=torch.empty((T, top_k), dtype=torch.float32, device=dev),
            local_rank=torch.empty((T, top_k), dtype=torch.int32, device=dev),
            tile_hist=torch.empty((top_k, nt, G), dtype=torch.int32, device=dev),
            logits=torch.empty((T, E), dtype=torch.float32, device=dev) if want_logits else None)
    _lib.call("comoe_gate_topk", _ptr(x), T, d, _ptr(wg_split), E, top_k, int(norm_topk),
              _ptr(slot_map), G, _ptr(out.logits), _ptr(out.expert_idx), _ptr(out.group_idx),
              _ptr(out.gate_prob), _ptr(out.local_rank), _ptr(out.tile_hist), _stream())
    return out


def gate_route_workspace(T: int, top_k: int, n_groups: int, device) -> torch.Tensor:
    """Zero-filled look-back workspace of comoe_gate_route (status words +
    a device-side epoch; self-maintaining after the zero fill)."""
    n = int(_lib.load().comoe_gate_route_workspace_bytes(int(T), int(top_k), int(n_groups)))
    return torch.zeros((n + 7) // 8, dtype=torch.int64, device=device)


def gate_route(x, wg_split, E, top_k, norm_topk, capacity: int, workspace: torch.Tensor,
               slot_map=None, n_groups=None, want_logits=False, out: GateOutput = None,
               scan: "ScanOutput" = None):
    """Gate + capacity scan in one launch (comoe_gate_route): the same
    tables as gate_topk followed by route_scan, except tile_hist (unused)."""
    _need(x, "x", torch.bfloat16, 2)
    _need(wg_split, "wg_split", torch.bfloat16, 3)
    T, d = x.shape
    G = E if n_groups is None else int(n_groups)
    if slot_map is not None:
        _need(slot_map, "slot_map", torch.int32, 1)
    nt = gate_num_tiles(T)
    dev = x.device
    need = int(_lib.load().comoe_gate_route_workspace_bytes(T, int(top_k), G))
    if workspace.device != dev or workspace.numel() * workspace.element_size() < need:
        raise ValueError(f"gate_route: workspace must hold {need} bytes on {dev}")
    if out is None:
        out = GateOutput(
            expert_idx=torch.empty((T, top_k), dtype=torch.int32, device=dev),
            group_idx=torch.empty((T, top_k), dtype=torch.int32, device=dev),
            gate_prob=torch.empty((T, top_k), dtype=torch.float32, device=dev),
            local_rank=torch.empty((T, top_k), dtype=torch.int32, device=dev),
            tile_hist=None,
            logits=torch.empty((T, E), dtype=torch.float32, device=dev) if want_logits else None)
    if scan is None:
        scan = ScanOutput(torch.empty((top_k, nt, G), dtype=torch.int32, device=dev),
                          *(torch.empty(G, dtype=torch.int32, device=dev) for _ in range(3)))
    _lib.call("comoe_gate_route", _ptr(x), T, d, _ptr(wg_split), E, top_k, int(norm_topk),
              _ptr(slot_map), G, int(capacity), _ptr(out.logits), _ptr(out.expert_idx),
              _ptr(out.group_idx), _ptr(out.gate_prob), _ptr(out.local_rank),
              _ptr(scan.tile_offset), _ptr(scan.group_count), _ptr(scan.group_kept),
              _ptr(scan.group_base), _ptr(workspace), _stream())
    return out, scan


def route_from_indices(expert_idx, E, probs=None, slot_map=None, n_groups=None,
                       out: GateOutput = None) -> GateOutput:
    """Routing tables from given expert choices (trace replay)."""
    _need(expert_idx, "expert_idx", torch.int32, 2)
    T, k = expert_idx.shape
    G = E if n_groups is None else int(n_groups)
    if probs is not None:
        _need(probs, "probs", torch.float32, 2)
    if slot_map is not None:
        _need(slot_map, "slot_map", torch.int32, 1)
    nt = gate_num_tiles(T)
    dev = expert_idx.device
    if out is None:
        out = GateOutput(expert_idx, torch.empty((T, k), dtype=torch.int32, device=dev),
                         torch.empty((T, k), dtype=torch.float32, device=dev),
                         torch.empty((T, k), dtype=torch.int32, device=dev),
                         torch.empty((k, nt, G), dtype=torch.int32, device=dev))
    else:
        out.expert_idx.copy_(expert_idx)
    _lib.call("comoe_route_from_indices", _ptr(expert_idx), _ptr(probs), T, E, k,
              _ptr(slot_map), G, _ptr(out.group_idx), _ptr(out.gate_prob), _ptr(out.local_rank),
              _ptr(out.tile_hist), _stream())
    return out


@dataclass
class ScanOutput:
    tile_offset: torch.Tensor  # [k, ntiles, G]
    group_count: torch.Tensor  # [G] assignments before capacity
    group_kept: torch.Tensor   # [G]
    group_base: torch.Tensor   # [G]


def route_scan(tile_hist, capacity: int, out: ScanOutput = None) -> ScanOutput:
    _need(tile_hist, "tile_hist", torch.int32, 3)
    k, nt, G = tile_hist.shape
    dev = tile_hist.device
    if out is None:
        out = ScanOutput(torch.empty_like(tile_hist),
                         *(torch.empty(G, dtype=torch.int32, device=dev) for _ in range(3)))
    _lib.call("comoe_route_scan", _ptr(tile_hist), k, nt, G, int(capacity), _ptr(out.tile_offset),
              _ptr(out.group_count), _ptr(out.group_kept), _ptr(out.group_base), _stream())
    return out


def expert_histogram(expert_idx: torch.Tensor, E: int, out=None) -> torch.Tensor:
    _need(expert_idx, "expert_idx", torch.int32)
    if out is None:
        out = torch.empty(E, dtype=torch.int32, device=expert_idx.device)
    _lib.call("comoe_expert_histogram", _ptr(expert_idx), expert_idx.numel(), E, _ptr(out),
              _stream())
    return out


# ---------------------------------------------------------------- K2 / K4

@dataclass
class PermuteOutput:
    x_perm: torch.Tensor     # [rows, d] bf16
    row_token: torch.Tensor  # [rows] int32
    row_prob: torch.Tensor   # [rows] float32
    token_pos: torch.Tensor  # [T, k] int32


def permute(x, gate: GateOutput, scan: ScanOutput, capacity: int, rows: int,
            y_zero=None, out: PermuteOutput = None, copy_rows: bool = True) -> PermuteOutput:
    _need(x, "x", torch.bfloat16, 2)
    T, d = x.shape
    k = gate.group_idx.shape[1]
    G = scan.group_base.numel()
    dev = x.device
    if out is None:
        out = PermuteOutput(torch.empty((max(rows, 1), d), dtype=torch.bfloat16, device=dev),
                            torch.empty(max(rows, 1), dtype=torch.int32, device=dev),
                            torch.empty(max(rows, 1), dtype=torch.float32, device=dev),
                            torch.empty((T, k), dtype=torch.int32, device=dev))
    if y_zero is not None:
        _need(y_zero, "y_zero", torch.bfloat16, 2)
    _lib.call("comoe_permute", _ptr(x), T, d, k, _ptr(gate.group_idx), _ptr(gate.gate_prob),
              _ptr(gate.local_rank), _ptr(scan.tile_offset), _ptr(scan.group_base), G,
              int(capacity), _ptr(out.x_perm) if copy_rows else None, _ptr(out.row_token),
              _ptr(out.row_prob), _ptr(out.token_pos), _ptr(y_zero), _stream())
    return out


def combine(y_perm, token_pos, gate_prob, out=None) -> torch.Tensor:
    _need(y_perm, "y_perm", torch.bfloat16, 2)
    _need(token_pos, "token_pos", torch.int32, 2)
    _need(gate_prob, "gate_prob", torch.float32, 2)
    T, k = token_pos.shape
    d = y_perm.shape[1]
    if out is None:
        out = torch.empty((T, d), dtype=torch.bfloat16, device=y_perm.device)
    _need_out(out, (T, d), y_perm.device)
    _lib.call("comoe_combine", _ptr(y_perm), _ptr(token_pos), _ptr(gate_prob), T, d, k,
              _ptr(out), _stream())
    return out


# ---------------------------------------------------------------- EP over peer memory

def permute_peers(x, gate: GateOutput, scan: ScanOutput, capacity: int, peer_rows,
                  block_rows: int, src_rank: int, out: PermuteOutput):
    """K2 with every kept row stored into its owner's receive buffer:
    `peer_rows` is an int64 device tensor of the world's receive-buffer
    addresses (see include/comoe_b200.h, EP over NVLink peer memory).
    `out.x_perm` is unused; row_token / row_prob / token_pos are local."""
    _need(x, "x", torch.bfloat16, 2)
    _need(peer_rows, "peer_rows", torch.int64, 1)
    T, d = x.shape
    k = gate.group_idx.shape[1]
    G = scan.group_base.numel()
    _lib.call("comoe_permute_peers", _ptr(x), T, d, k, _ptr(gate.group_idx), _ptr(gate.gate_prob),
              _ptr(gate.local_rank), _ptr(scan.tile_offset), _ptr(scan.group_base), G,
              int(capacity), _ptr(peer_rows), peer_rows.numel(), int(block_rows), int(src_rank),
              _ptr(out.row_token), _ptr(out.row_prob), _ptr(out.token_pos), _stream())
    return out


def combine_peers(peer_rows, block_rows: int, src_rank: int, token_pos, gate_prob, d: int,
                  out=None) -> torch.Tensor:
    """K4 reading each kept row from its owner's output buffer."""
    _need(peer_rows, "peer_rows", torch.int64, 1)
    _need(token_pos, "token_pos", torch.int32, 2)
    _need(gate_prob, "gate_prob", torch.float32, 2)
    T, k = token_pos.shape
    if out is None:
        out = torch.empty((T, d), dtype=torch.bfloat16, device=token_pos.device)
    _need_out(out, (T, d), token_pos.device)
    _lib.call("comoe_combine_peers", _ptr(peer_rows), peer_rows.numel(), int(block_rows),
              int(src_rank), _ptr(token_pos), _ptr(gate_prob), T, d, k, _ptr(out), _stream())
    return out


def peer_scatter_counts(counts, world: int, src_rank: int, peer_counts) -> None:
    _need(counts, "counts", torch.int32, 1)
    _need(peer_counts, "peer_counts", torch.int64, 1)
    _lib.call("comoe_peer_scatter_counts", _ptr(counts), counts.numel(), int(world),
              int(src_rank), _ptr(peer_counts), _stream())


def peer_barrier(pads, world: int, rank: int, epoch: int, err, timeout_s: float = 10.0) -> None:
    """Stream-ordered flag barrier over peer memory; a peer that does not
    arrive within `timeout_s` sets err[0] = 1 + peer instead of hanging."""
    _need(pads, "pads", torch.int64, 1)
    _need(err, "err", torch.int32, 1)
    _lib.call("comoe_peer_barrier", _ptr(pads), int(world), int(rank), int(epoch),
              int(timeout_s * 1e9), _ptr(err), _stream())


def ipc_handle(t: torch.Tensor):
    """(handle bytes, offset) naming the allocation that holds `t`."""
    n = _lib.load().comoe_ipc_handle_size()
    buf = ctypes.create_string_buffer(n)
    off = ctypes.c_long(0)
    _lib.call("comoe_ipc_get_handle", _ptr(t), buf, ctypes.byref(off))
    return bytes(buf.raw), int(off.value)


def ipc_open(handle: bytes, offset: int) -> int:
    ptr = ctypes.c_void_p(0)
    _lib.call("comoe_ipc_open", handle, int(offset), ctypes.byref(ptr))
    return int(ptr.value)


def ipc_close(ptr: int, offset: int) -> None:
    _lib.call("comoe_ipc_close", int(ptr), int(offset))


# ---------------------------------------------------------------- K3

def expert_numel(d: int, d_ff: int, act: int) -> int:
    n1 = 2 * d_ff if act == ACT_SWIGLU else d_ff
    return n1 * d + d * d_ff


def grouped_ffn(x_perm, pool, d_ff, act, group_rows, group_row_base, group_slot, h_work, out,
                row_token=None, row_prob=None):
    _need(x_perm, "x_perm", torch.bfloat16, 2)
    _need(pool, "pool", torch.bfloat16, 2)
    _need(h_work, "h_work", torch.bfloat16, 2)
    _need(out, "out", torch.bfloat16, 2)
    for name, t in (("group_rows", group_rows), ("group_row_base", group_row_base),
                    ("group_slot", group_slot)):
        _need(t, name, torch.int32, 1)
    rows, d = x_perm.shape
    if h_work.shape[0] < rows or h_work.shape[1] != d_ff:
        raise ValueError("h_work must be [rows, d_ff]")
    if pool.shape[1] < expert_numel(d, d_ff, act):
        raise ValueError("pool slot too small for the expert shape")
    _lib.call("comoe_grouped_ffn", _ptr(x_perm), rows, d, d_ff, act, _ptr(pool), pool.shape[0],
              pool.shape[1], _ptr(group_rows), _ptr(group_row_base), _ptr(group_slot),
              group_rows.numel(), _ptr(h_work), _ptr(out), out.shape[1], _ptr(row_token),
              _ptr(row_prob), _stream())
    return out


def fused_ffn_supported(d: int, d_ff: int, act: int, n_groups: int) -> bool:
    """Whether comoe_fused_ffn takes this shape."""
    return bool(_lib.load().comoe_fused_ffn_supported(int(d), int(d_ff), int(act), int(n_groups)))


def fused_ffn_enabled() -> bool:
    """The layer forward uses the fused FFN only when opted in
    (COMOE_FUSED_FFN=1): it measured slower than the two-launch FFN."""
    return bool(_lib.load().comoe_fused_ffn_enabled())


def fused_ffn(x, pool, d_ff, group_rows, group_row_base, group_slot, out, gather_rows=None,
              row_token=None, row_prob=None):
    """K3F: relu(X Wi^T) Wo^T per group in one launch, H on chip. `x` is the
    permuted copy, or (with `gather_rows` = the permute's row_token) the
    unpermuted tokens, gathered by TMA."""
    _need(x, "x", torch.bfloat16, 2)
    _need(pool, "pool", torch.bfloat16, 2)
    _need(out, "out", torch.bfloat16, 2)
    for name, t in (("group_rows", group_rows), ("group_row_base", group_row_base),
                    ("group_slot", group_slot)):
        _need(t, name, torch.int32, 1)
    if gather_rows is not None:
        _need(gather_rows, "gather_rows", torch.int32, 1)
    rows, d = x.shape
    if pool.shape[1] < expert_numel(d, d_ff, ACT_RELU):
        raise ValueError("pool slot too small for the expert shape")
    _lib.call("comoe_fused_ffn", _ptr(x), rows, _ptr(gather_rows), d, int(d_ff), _ptr(pool),
              pool.shape[0], pool.shape[1], _ptr(group_rows), _ptr(group_row_base),
              _ptr(group_slot), group_rows.numel(), _ptr(out), out.shape[1], _ptr(row_token),
              _ptr(row_prob), _stream())
    return out


def grouped_gemm(a, pool, b_offset, N, group_rows, group_row_base, group_slot, epi_mode, out,
                 row_token=None, row_prob=None, a_gather=None):
    _need(a, "a", torch.bfloat16, 2)
    _need(pool, "pool", torch.bfloat16, 2)
    _need(out, "out", torch.bfloat16, 2)
    rows, K = a.shape
    _lib.call("comoe_grouped_gemm", _ptr(a), rows, _ptr(pool), pool.shape[0], pool.shape[1],
              int(b_offset), int(N), K, _ptr(group_rows), _ptr(group_row_base),
              _ptr(group_slot), group_rows.numel(), int(epi_mode), _ptr(out), out.shape[1],
              _ptr(row_token), _ptr(row_prob), _ptr(a_gather), _stream())
    return out


# ---------------------------------------------------------------- K5 merge

class MergePlan:
    """Device group table for one K5 launch over a layer's multi-member
    groups: groups_members = per group, the member tensors (flat, same
    numel); weights = per-member floats; divisors = per-group floats; outs =
    per-group output tensors. Built once (one pinned async upload), run any
    number of times — a variant rebuild re-merges from the same table."""

    def __init__(self, groups_members, weights, divisors, outs, dtype):
        self.n_groups = len(outs)
        if not groups_members:
            return
        dev = outs[0].device
        D = outs[0].numel()
        if dtype not in (torch.bfloat16, torch.float64):
            raise ValueError("merge supports bf16 and float64 parameters")
        self.code = DTYPE_BF16 if dtype == torch.bfloat16 else DTYPE_F64
        ptrs, offs, ws = [], [0], []
        for members, wlist in zip(groups_members, weights):
            if len(members) != len(wlist):
                raise ValueError("one weight per member")
            for m in members:
                _need(m, "member", dtype, align=16 if dtype == torch.bfloat16 else 8)
                if m.numel() != D:
                    raise ValueError("member size mismatch")
                ptrs.append(m.data_ptr())
            ws.extend(float(w) for w in wlist)
            offs.append(len(ptrs))
        for o in outs:
            _need(o, "out", dtype, align=16 if dtype == torch.bfloat16 else 8)
            if o.numel() != D:
                raise ValueError("output size mismatch")
        self.D = D
        self.max_members = max(offs[i + 1] - offs[i] for i in range(len(outs)))
        # one pinned staging buffer, one async H2D: [ptrs | outs | offs | weights | divisors]
        nm, ng = len(ptrs), len(outs)
        host = torch.empty(nm + ng + (ng + 2) // 2 + nm + ng, dtype=torch.int64).pin_memory()
        host[:nm] = torch.tensor(ptrs, dtype=torch.int64)
        host[nm:nm + ng] = torch.tensor([o.data_ptr() for o in outs], dtype=torch.int64)
        o_off = nm + ng
        n_off_words = (ng + 2) // 2
        host[o_off:o_off + n_off_words].view(torch.int32)[:ng + 1] = torch.tensor(offs, dtype=torch.int32)
        w_off = o_off + n_off_words
        host[w_off:w_off + nm].view(torch.float64)[:] = torch.tensor(ws, dtype=torch.float64)
        host[w_off + nm:].view(torch.float64)[:] = torch.tensor([float(x) for x in divisors],
                                                               dtype=torch.float64)
        # PyTorch's pinned-host allocator records the async copy on the
        # stream before reusing `host`
        self.table = host.to(dev, non_blocking=True)
        self.t_ptrs, self.t_out = self.table[:nm], self.table[nm:nm + ng]
        self.t_offs = self.table[o_off:o_off + n_off_words].view(torch.int32)
        self.t_w = self.table[w_off:w_off + nm].view(torch.float64)
        self.t_div = self.table[w_off + nm:].view(torch.float64)

    def run(self) -> None:
        if not self.n_groups:
            return
        _lib.call("comoe_merge", self.code, _ptr(self.t_ptrs), _ptr(self.t_offs), _ptr(self.t_w),
                  _ptr(self.t_div), _ptr(self.t_out), self.n_groups, self.max_members, self.D,
                  _stream())


def merge_groups(groups_members, weights, divisors, outs, dtype) -> None:
    """One K5 launch for all groups (see MergePlan)."""
    MergePlan(groups_members, weights, divisors, outs, dtype).run()


# ---------------------------------------------------------------- K6 similarity

def _shared_stride(rows):
    """(base address, row stride in elements) when the bf16 rows are
    consecutive rows of one 16-byte-multiple stride no shorter than a row
    (a layer's pool slots, the rows of a matrix); else None."""
    ptrs = [r.data_ptr() for r in rows]
    D = rows[0].numel()
    stride = ptrs[1] - ptrs[0] if len(ptrs) > 1 else 2 * D
    if stride % 16 or stride < 2 * D or ptrs[0] % 16:
        return None
    if any(p != ptrs[0] + i * stride for i, p in enumerate(ptrs)):
        return None
    return ptrs[0], stride // 2


def similarity(rows, probes, proj, alpha):
    """rows: list of E flat expert tensors (bf16 or float64, same numel);
    probes [n, D], proj [B, D] float64 on the device. Returns (S, gram,
    logits) float64 device tensors."""
    E = len(rows)
    D = rows[0].numel()
    dt = rows[0].dtype
    if dt not in (torch.bfloat16, torch.float64):
        raise ValueError("similarity supports bf16 and float64 parameters")
    # the bf16 kernels for D % 8 == 0 move rows in 16-byte vectors / bulk copies
    row_align = 16 if (dt == torch.bfloat16 and D % 8 == 0) else rows[0].element_size()
    for r in rows:
        _need(r, "row", dt, align=row_align)
        if r.numel() != D:
            raise ValueError("parameter dimension mismatch")
    n = 0 if probes is None else probes.shape[0]
    B = 0 if proj is None else proj.shape[0]
    if n:
        _need(probes, "probes", torch.float64, 2)
        _need(proj, "proj", torch.float64, 2)
        if probes.shape[1] != D or proj.shape[1] != D:
            raise ValueError("calibration dimension mismatch")
    else:
        probes = proj = None
    dev = rows[0].device
    ws = _lib.load().comoe_sim_workspace_bytes(E, n, B, D)
    work = torch.empty(max(ws, 8), dtype=torch.uint8, device=dev)
    gram = torch.empty((E, E), dtype=torch.float64, device=dev)
    logits = torch.empty((E, n, B), dtype=torch.float64, device=dev) if n else None
    sim = torch.empty((E, E), dtype=torch.float64, device=dev)
    strided = _shared_stride(rows) if (dt == torch.bfloat16 and n == 0 and
                                       _lib.load().comoe_sim_tc_supported(E, D)) else None
    if strided is not None:  # tcgen05 Gram over a tensor map of the consecutive rows
        base, stride = strided
        _lib.call("comoe_sim_gram_strided", ctypes.c_void_p(base), stride, E, D, _ptr(gram),
                  _ptr(work), _stream())
    else:
        t_rows = torch.tensor([r.data_ptr() for r in rows], dtype=torch.int64).to(dev)
        code = DTYPE_BF16 if dt == torch.bfloat16 else DTYPE_F64
        _lib.call("comoe_sim_contract", code, _ptr(t_rows), E, D, _ptr(probes), n, _ptr(proj), B,
                  _ptr(gram), _ptr(logits), _ptr(work), _stream())
    _lib.call("comoe_sim_finalize", _ptr(gram), _ptr(logits), E, n, B, float(alpha), _ptr(sim),
              _stream())
    return sim, gram, logits


# ---------------------------------------------------------------- K8 predictor

def predictor_mlp(slots, emb, ctx, w1, b1, w2, b2, want_demand=False, demand_mode="sum"):
    """K8. demand_mode: "sum" = expected picks per expert over the batch,
    "any" = probability that at least one token of the batch picks it."""
    _need(slots, "slots", torch.int32, 2)
    B, K = slots.shape
    for name, t in (("w1", w1), ("b1", b1), ("w2", w2), ("b2", b2)):
        _need(t, name, torch.float64)
    E, hidden = w2.shape
    emb_dim = 0 if emb is None else emb.shape[1]
    ctx_dim = 0 if ctx is None else ctx.shape[1]
    if emb is not None:
        _need(emb, "emb", torch.float64, 2)
    if ctx is not None:
        _need(ctx, "ctx", torch.float64, 2)
    if w1.shape[1] != E + emb_dim + ctx_dim:
        raise ValueError("embedding/context dims do not match the predictor")
    probs = torch.empty((B, E), dtype=torch.float64, device=slots.device)
    demand = work = None
    if want_demand:
        demand = torch.empty(E, dtype=torch.float64, device=slots.device)
        nbytes = _lib.load().comoe_predictor_workspace_bytes(B, E)
        work = torch.empty(max(nbytes, 8), dtype=torch.uint8, device=slots.device)
    _lib.call("comoe_predictor_mlp", _ptr(slots), B, K, _ptr(emb), emb_dim, _ptr(ctx), ctx_dim,
              _ptr(w1), _ptr(b1), hidden, _ptr(w2), _ptr(b2), E, _ptr(probs), _ptr(demand),
              {"sum": 0, "any": 1}[demand_mode], _ptr(work), _stream())
    return (probs, demand) if want_demand else probs


def capacity_for(T: int, n_groups: int, top_k: int, capacity_factor) -> int:
    """C = ceil(cf * T * k / G) (GShard/Switch); None -> no drops."""
    if capacity_factor is None:
        return int(T) * int(top_k)
    return int(math.ceil(float(capacity_factor) * int(T) * int(top_k) / int(n_groups)))
