"""Multi-layer MoE stack on HBM-budgeted expert caches with predictive
prefetch — the per-token policy loop of the reference simulator
(simulator.py:684-724: serve demand, predict the next MoE layer, prefetch,
evict) turned into a batched device pipeline.

For each MoE layer l of the stack:
  1. route layer l (gate + scan) and serve its demand from cache_l (hits,
     substitutions, demand fetches — CachedMoELayer);
  2. if l is an encoder layer with a successor (simulator.py:709-712), run
     the K8 predictor on layer l's routing for every token and reduce (in
     K8) to the probability that layer l+1 demands each expert from this
     batch, 1 - prod_t (1 - p_t) — the batched form of the per-token
     probability the reference compares with the threshold in
     decide_prefetch (a batch mean would wash out the peaked per-token
     predictions: no expert ever crossed the threshold at 16-1024 tokens,
     scripts/bench_stack.py) — and prefetch into cache_{l+1} with the
     resource-aware threshold. The copies run on cache_{l+1}'s copy stream
     and overlap layer l's grouped GEMMs;
  3. decoder layers can be pinned (pin_decoder, simulator.py:407-413).
Dense (non-MoE) sublayers are outside this hot path; hidden states pass
between MoE layers unchanged (x_{l+1} = y_l + x_l residual).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .offload import OffloadPolicy, prefetch_threshold


def fold_demand(demand, slot_map, n_groups: int, mode: str = "complement") -> np.ndarray:
    """Per-original-expert demand probabilities of the next layer -> its
    cache's group space (a fused variant's experts are (layer, group)).
    mode "sum": the reference's fold of one token's predictor output,
    np.add.at(merged, map_arrays[nxt], raw) (simulator.py:587-588);
    mode "complement": P(group g demanded by the batch) =
    1 - prod_{e in g} (1 - p_e), the consistent fold of batch demand
    probabilities (stays a probability)."""
    lut = np.asarray(slot_map, np.int64)
    demand = np.asarray(demand, np.float64)[:len(lut)]
    if mode == "sum":
        merged = np.zeros(n_groups)
        np.add.at(merged, lut, demand)
        return merged
    demand = np.clip(demand, 0.0, 1.0)
    miss = np.ones(n_groups)
    np.multiply.at(miss, lut, 1.0 - demand)
    return 1.0 - miss


class PrefetchGovernor:
    """Turns predictive prefetch off when it does not pay (an extension of
    the reference's threshold rule, which only gates individual experts).
    Prefetches compete with demand fetches for the host link and evict
    experts the batch would have hit, so whether they help depends on the
    batch size and routing skew (scripts/bench_stack.py). The governor
    measures it: per batch size it times `window` stack forwards with
    prefetch on and `window` with it off (CUDA events on the compute
    stream, read back without a sync one step later), keeps the faster
    setting for `hold` steps, then probes again."""

    def __init__(self, window: int = 3, hold: int = 24, margin: float = 0.0):
        self.window, self.hold, self.margin = int(window), int(hold), float(margin)
        self._st = {}
        self._pending = None

    def _state(self, T):
        return self._st.setdefault(T, {"phase": "on", "left": self.window, "on": [], "off": [],
                                       "choice": True})

    def enabled(self, T: int) -> bool:
        st = self._state(T)
        return st["choice"] if st["phase"] == "hold" else st["phase"] == "on"

    def begin(self, T: int):
        self._collect()
        start = torch.cuda.Event(enable_timing=True)
        start.record()
        return (T, self.enabled(T), start)

    def end(self, token) -> None:
        stop = torch.cuda.Event(enable_timing=True)
        stop.record()
        self._pending = (*token, stop)

    def _collect(self) -> None:
        if self._pending is None:
            return
        T, on, start, stop = self._pending
        stop.synchronize()
        self._pending = None
        self.record(T, on, start.elapsed_time(stop))

    def record(self, T: int, on: bool, ms: float) -> None:
        """One measured stack forward of T tokens, prefetch `on` or off."""
        st = self._state(T)
        if st["phase"] == "hold":
            st["left"] -= 1
            if st["left"] <= 0:
                st.update(phase="on", left=self.window, on=[], off=[])
            return
        st["on" if on else "off"].append(ms)
        st["left"] -= 1
        if st["left"] > 0:
            return
        if st["phase"] == "on":
            st.update(phase="off", left=self.window)
        else:
            m_on, m_off = float(np.median(st["on"])), float(np.median(st["off"]))
            st.update(phase="hold", left=self.hold, choice=m_on < m_off * (1.0 - self.margin),
                      last=(m_on, m_off))


@dataclass
class StackLayer:
    index: int
    layer: object            # CachedMoELayer
    encoder: bool = True


class CachedMoEStack:
    """One token step = one forward of every layer over the batch.

    The layers' caches may be one shared ExpertCache (the reference's single
    CacheState over all MoE layers) or one per layer. At a batch of one
    token the stack is the reference's per-token loop (simulator.py:684-724)
    with the same order of decisions — serve layer l, then predict layer
    l+1 (raw predictor output folded with the reference's sum) and prefetch
    — and its JSONL event log matches the simulator's decision stream
    (tests/test_cache_parity.py)."""

    def __init__(self, layers: list, predictor=None, policy: OffloadPolicy = None,
                 s_b: float = 1.0, mem_avail: float = 1.0, mem_total: float = 1.0,
                 theta: float = None, governor: PrefetchGovernor = None):
        self.layers = layers
        self.predictor = predictor
        self.governor = governor
        self.policy = policy or OffloadPolicy()
        self.theta = prefetch_threshold(self.policy, s_b, mem_avail, mem_total) \
            if theta is None else float(theta)
        self.prefetch_log = []
        self.steps = 0

    def caches(self) -> list:
        seen, out = set(), []
        for sl in self.layers:
            c = sl.layer.cache
            if id(c) not in seen:
                seen.add(id(c))
                out.append(c)
        return out

    def forward(self, x, emb=None, ctx=None, routings=None, tick: int = None):
        """x [T, d] bf16; emb/ctx [T, *] float64 device tensors for the
        predictor (token embedding / context, as TokenRecord carries);
        `routings` (optional, one (expert_idx, probs) per layer) replays a
        routing trace instead of running each layer's router; `tick` is the
        step's clock (default: one more than the last)."""
        T = x.shape[0]
        t = self.steps if tick is None else int(tick)
        self.steps = t + 1
        for c in self.caches():
            c.begin_step(t)
        token = self.governor.begin(T) if self.governor is not None else None
        predictive = self.predictor is not None and (token is None or token[1])
        h = x
        for i, sl in enumerate(self.layers):
            nxt = self.layers[i + 1] if i + 1 < len(self.layers) else None
            pre = post = None
            if nxt is not None and sl.encoder and predictive:
                mode = "sum" if T == 1 else "any"

                def pre(r, mode=mode):
                    # predictor right after routing (before this layer's
                    # GEMMs); its demand comes back by an async copy
                    _, demand = self.predictor.predict_slots(r.gate.expert_idx, emb, ctx,
                                                             want_demand=True, demand_mode=mode)
                    host = torch.empty(demand.shape, dtype=demand.dtype, pin_memory=True)
                    host.copy_(demand, non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record()
                    return host, ev

                def post(handle, sl=sl, nxt=nxt, T=T):
                    host, ev = handle
                    ev.synchronize()       # gate + predictor only, not the GEMMs
                    L = nxt.layer.layer
                    probs = fold_demand(host.numpy(), L.slot_map_host, L.G,
                                        mode="sum" if T == 1 else "complement")
                    chosen = nxt.layer.cache.prefetch(probs, self.theta, layer=nxt.layer.layer_id)
                    self.prefetch_log.append((sl.index, nxt.index, chosen))
            y = sl.layer.forward(h, after_route=pre, after_serve=post, step=False,
                                 routing=routings[i] if routings is not None else None)
            h = (y.float() + h.float()).to(torch.bfloat16)
        if token is not None:
            self.governor.end(token)
        return h
