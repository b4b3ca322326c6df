"""NumPy oracle of one MoE layer forward (TEST INFRASTRUCTURE ONLY).

The reference has no router, capacity, permutation, expert FFN or combine
(routing is the synthetic generator pkg/src/comoe/moe.py:186-230
and expert compute an analytic charge, pkg/src/comoe/simulator.py:692-707).
This module states the Switch/GShard semantics the B200 path implements, in
plain loops/NumPy with fp64 math, so every choice is inspectable:

  * router: logits = x @ Wg (fp64 accumulate of the bf16 inputs, rounded to
    fp32 — the fp32 router of Switch);
  * top-k on the fp32 LOGITS, ties -> lowest expert index (reference tie
    rule, aggregation.py:165,193; oracles.py:48-62);
  * probabilities: norm_topk=0 -> softmax over all E at the picked experts
    (Switch); norm_topk=1 -> softmax over the k picked logits (Mixtral);
  * slot remap: group = slot_map[expert] (ModelVariant.resolve,
    aggregation.py:101-103); if both top-2 picks land in one group the
    second folds into the first (probabilities add) — the dedup that
    simulator.py:696-702 applies to resolved ids;
  * capacity C = ceil(cf * T * k / G) per group; priority = stream order:
    every first choice in token order, then every second choice;
  * kept assignments are laid out group-major, rank order inside a group;
  * FFN: ReLU (Switch) or SiLU-gated (Mixtral, gate/up rows interleaved in
    128-row blocks); H optionally rounded to bf16 like the device
    intermediate; combine y_t = sum_j p_tj * Y[pos_tj], dropped -> 0.
"""

from __future__ import annotations

import math

import numpy as np

GATE_TILE = 128
SWIGLU_BLOCK = 128


def bf16_round(a) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as float32 values."""
    f = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    out = r.astype(np.uint32).view(np.float32)
    nan = np.isnan(f)
    if nan.any():
        out = out.copy()
        out[nan] = np.nan
    return out


def det_uniform(shape, seed: int, scale: float) -> np.ndarray:
    """Deterministic test inputs: a counter-based splitmix64 stream mapped to
    uniform(-1, 1) * scale * sqrt(3) (unit variance before `scale`), float32.
    Bit-identical on every numpy version (no library RNG), so golden
    fixtures store seeds instead of tensors (oracle/gen_layer_golden.py)."""
    n = int(np.prod(shape))
    with np.errstate(over="ignore"):
        z = np.arange(n, dtype=np.uint64) + np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 2 ** 53)
    return ((2.0 * u - 1.0) * math.sqrt(3.0) * scale).astype(np.float32).reshape(shape)


def gate_logits(x, wg) -> np.ndarray:
    """fp32 router logits of bf16-valued x[T,d] and fp32 Wg[d,E]."""
    return (np.asarray(x, np.float64) @ np.asarray(wg, np.float64)).astype(np.float32)


def topk_route(logits, top_k: int, norm_topk: bool, slot_map=None):
    """Returns (expert_idx [T,k], group_idx [T,k], prob [T,k] fp64)."""
    logits = np.asarray(logits, np.float32)
    T, E = logits.shape
    # stable sort of -logit: equal logits keep ascending index order
    order = np.argsort(-logits.astype(np.float64), axis=1, kind="stable")
    idx = order[:, :top_k].astype(np.int64)
    l64 = logits.astype(np.float64)
    picked = np.take_along_axis(l64, idx, axis=1)
    if top_k == 1:
        if norm_topk:
            prob = np.ones((T, 1))
        else:
            m = l64.max(axis=1, keepdims=True)
            prob = 1.0 / np.exp(l64 - m).sum(axis=1, keepdims=True)
    elif norm_topk:
        z = np.exp(picked[:, 1] - picked[:, 0])
        prob = np.stack([1.0 / (1.0 + z), z / (1.0 + z)], axis=1)
    else:
        m = l64.max(axis=1, keepdims=True)
        s = np.exp(l64 - m).sum(axis=1, keepdims=True)
        prob = np.exp(picked - m) / s
    smap = np.arange(E) if slot_map is None else np.asarray(slot_map, np.int64)
    group = smap[idx]
    prob = prob.copy()
    if top_k == 2:
        same = group[:, 1] == group[:, 0]
        prob[same, 0] += prob[same, 1]
        prob[same, 1] = 0.0
        group = group.copy()
        group[same, 1] = -1
    return idx, group, prob


def capacity(T: int, n_groups: int, top_k: int, capacity_factor) -> int:
    if capacity_factor is None:
        return T * top_k
    return int(math.ceil(float(capacity_factor) * T * top_k / n_groups))


def dispatch(group, n_groups: int, cap: int):
    """Stream-order ranks, capacity and the compact permutation.

    Returns dict with rank [T,k] (-1 for no assignment), count [G] (before
    capacity), kept [G], base [G], pos [T,k] (row or -1), row_token [rows],
    row_slot [rows] (which choice j), local_rank [T,k] (rank inside the
    128-token tile) and tile_hist [k, ntiles, G].
    """
    group = np.asarray(group, np.int64)
    T, k = group.shape
    rank = np.full((T, k), -1, np.int64)
    count = np.zeros(n_groups, np.int64)
    for j in range(k):
        for t in range(T):
            g = group[t, j]
            if g >= 0:
                rank[t, j] = count[g]
                count[g] += 1
    kept = np.minimum(count, cap)
    base = np.concatenate([[0], np.cumsum(kept)[:-1]]).astype(np.int64)
    pos = np.full((T, k), -1, np.int64)
    rows = int(kept.sum())
    row_token = np.full(rows, -1, np.int64)
    row_choice = np.full(rows, -1, np.int64)
    for j in range(k):
        for t in range(T):
            g = group[t, j]
            if g >= 0 and rank[t, j] < cap:
                p = base[g] + rank[t, j]
                pos[t, j] = p
                row_token[p] = t
                row_choice[p] = j
    ntiles = (T + GATE_TILE - 1) // GATE_TILE
    local = np.full((T, k), -1, np.int64)
    hist = np.zeros((k, ntiles, n_groups), np.int64)
    for j in range(k):
        for tile in range(ntiles):
            seen = {}
            for t in range(tile * GATE_TILE, min(T, (tile + 1) * GATE_TILE)):
                g = group[t, j]
                if g >= 0:
                    local[t, j] = seen.get(g, 0)
                    seen[g] = local[t, j] + 1
            for g, c in seen.items():
                hist[j, tile, g] = c
    return dict(rank=rank, count=count, kept=kept, base=base, pos=pos, row_token=row_token,
                row_choice=row_choice, local_rank=local, tile_hist=hist)


def expert_ffn(xrows, w_in, w_out, act: str, round_h: bool = True) -> np.ndarray:
    """Y = act(X W_in^T) W_out^T for one expert, fp64 math.

    w_in: [N1, d] (N1 = d_ff, or 2*d_ff interleaved gate/up blocks for
    SwiGLU), w_out: [d, d_ff]."""
    x = np.asarray(xrows, np.float64)
    a = x @ np.asarray(w_in, np.float64).T
    if act == "relu":
        h = np.maximum(a, 0.0)
    elif act == "swiglu":
        n1 = a.shape[1]
        blocks = a.reshape(a.shape[0], n1 // (2 * SWIGLU_BLOCK), 2, SWIGLU_BLOCK)
        g, u = blocks[:, :, 0, :], blocks[:, :, 1, :]
        h = (g / (1.0 + np.exp(-g)) * u).reshape(a.shape[0], n1 // 2)
    else:
        raise ValueError(act)
    if round_h:
        h = bf16_round(h.astype(np.float32)).astype(np.float64)
    return h @ np.asarray(w_out, np.float64).T


def split_expert(flat, d: int, d_ff: int, act: str):
    """Flat slot vector [W_in | W_out] -> (w_in [N1,d], w_out [d,d_ff])."""
    n1 = 2 * d_ff if act == "swiglu" else d_ff
    flat = np.asarray(flat)
    w_in = flat[: n1 * d].reshape(n1, d)
    w_out = flat[n1 * d: n1 * d + d * d_ff].reshape(d, d_ff)
    return w_in, w_out


def layer_forward(x, wg, experts, top_k=1, norm_topk=False, capacity_factor=1.25,
                  slot_map=None, group_experts=None, act="relu", d_ff=None, logits=None,
                  round_h=True):
    """Full oracle forward.

    x [T,d] bf16-valued, wg [d,E] fp32, experts: list of flat expert vectors
    indexed by GROUP (len G) — with no merging groups are the experts.
    `logits` lets a test feed the device's fp32 logits (parity "given
    identical fp32 logits"). Returns (y fp64 [T,d], info dict).
    """
    x = np.asarray(x, np.float32)
    T, d = x.shape
    if logits is None:
        logits = gate_logits(x, wg)
    E = logits.shape[1]
    G = len(experts) if group_experts is None else group_experts
    idx, group, prob = topk_route(logits, top_k, norm_topk, slot_map)
    cap = capacity(T, G, top_k, capacity_factor)
    disp = dispatch(group, G, cap)
    y = np.zeros((T, d), np.float64)
    Yrows = np.zeros((len(disp["row_token"]), d), np.float64)
    for g in range(G):
        lo, n = disp["base"][g], disp["kept"][g]
        if n == 0:
            continue
        toks = disp["row_token"][lo:lo + n]
        w_in, w_out = split_expert(experts[g], d, d_ff, act)
        Yrows[lo:lo + n] = expert_ffn(x[toks], w_in, w_out, act, round_h)
    for j in range(top_k):
        p = disp["pos"][:, j]
        m = p >= 0
        y[m] += prob[m, j][:, None] * Yrows[p[m]]
    info = dict(logits=logits, expert_idx=idx, group_idx=group, prob=prob, capacity=cap,
                y_rows=Yrows, **disp)
    return y, info


def normwise_error(got, ref) -> float:
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(got - ref) / (den if den > 0 else 1.0))


# ---------------------------------------------------------------------------
# vectorised CPU path (the timed CPU baseline; same semantics as above)


def dispatch_fast(group, n_groups: int, cap: int):
    """Vectorised `dispatch` (ranks by a stable sort in stream order)."""
    group = np.asarray(group, np.int64)
    T, k = group.shape
    flat = group.T.reshape(-1)            # stream order: choice-major, then token
    valid = flat >= 0
    order = np.argsort(np.where(valid, flat, n_groups), kind="stable")
    sorted_g = np.where(valid, flat, n_groups)[order]
    count_all = np.bincount(sorted_g, minlength=n_groups + 1)
    count = count_all[:n_groups]
    starts = np.concatenate([[0], np.cumsum(count_all)[:-1]])
    rank_sorted = np.arange(flat.size) - starts[sorted_g]
    rank_flat = np.empty(flat.size, np.int64)
    rank_flat[order] = rank_sorted
    rank_flat[~valid] = -1
    kept = np.minimum(count, cap)
    base = np.concatenate([[0], np.cumsum(kept)[:-1]]).astype(np.int64)
    keep = valid & (rank_flat < cap)
    pos_flat = np.full(flat.size, -1, np.int64)
    pos_flat[keep] = base[flat[keep]] + rank_flat[keep]
    pos = pos_flat.reshape(k, T).T.copy()
    rank = rank_flat.reshape(k, T).T.copy()
    row_token = np.full(int(kept.sum()), -1, np.int64)
    tok = np.tile(np.arange(T), k)
    row_token[pos_flat[keep]] = tok[keep]
    return dict(rank=rank, count=count, kept=kept, base=base, pos=pos, row_token=row_token)


def layer_forward_fast(x, wg, w_in, w_out, top_k=1, norm_topk=False, capacity_factor=1.25,
                       slot_map=None, act="relu", dtype=np.float32, logits=None, round_h=False):
    """CPU forward with NumPy BLAS: x [T,d], wg [d,E], w_in [G,N1,d],
    w_out [G,d,d_ff] (arrays or per-group lists, already `dtype`). Returns
    y [T,d] (dtype). `logits` feeds given fp32 logits (parity "given
    identical logits"); `round_h` rounds H to bf16 like the device."""
    x = np.asarray(x, dtype)
    if logits is None:
        logits = (x @ np.asarray(wg, dtype)).astype(np.float32)
    idx, group, prob = topk_route(logits, top_k, norm_topk, slot_map)
    G = len(w_in)
    cap = capacity(x.shape[0], G, top_k, capacity_factor)
    disp = dispatch_fast(group, G, cap)
    y = np.zeros_like(x)
    rows = np.zeros((len(disp["row_token"]), x.shape[1]), dtype)
    for g in range(G):
        lo, n = int(disp["base"][g]), int(disp["kept"][g])
        if n == 0:
            continue
        xs = x[disp["row_token"][lo:lo + n]]
        a = xs @ w_in[g].T
        if act == "relu":
            h = np.maximum(a, 0)
        else:
            n1 = a.shape[1]
            b = a.reshape(n, n1 // (2 * SWIGLU_BLOCK), 2, SWIGLU_BLOCK)
            h = (b[:, :, 0] / (1 + np.exp(-b[:, :, 0])) * b[:, :, 1]).reshape(n, n1 // 2)
        if round_h:
            h = bf16_round(h.astype(np.float32)).astype(dtype)
        rows[lo:lo + n] = h @ w_out[g].T
    for j in range(top_k):
        p = disp["pos"][:, j]
        m = p >= 0
        y[m] += prob[m, j][:, None].astype(dtype) * rows[p[m]]
    return y, dict(expert_idx=idx, group_idx=group, prob=prob, capacity=cap, **disp)
