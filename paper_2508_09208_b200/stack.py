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


def fold_demand(demand, slot_map, n_groups: int) -> np.ndarray:
    """Per-original-expert demand probabilities of the next layer -> its
    cache's group space (a fused variant's experts are (layer, group)):
    P(group g demanded) = 1 - prod_{e in g} (1 - p_e). The reference folds
    its per-token predictor output the same way before decide_prefetch,
    with a sum (np.add.at(merged, map_arrays[nxt], raw), simulator.py:587-588);
    for the batch demand probabilities here the complement product is the
    consistent fold (it stays a probability)."""
    demand = np.clip(np.asarray(demand, np.float64), 0.0, 1.0)
    lut = np.asarray(slot_map, np.int64)
    miss = np.ones(n_groups)
    np.multiply.at(miss, lut, 1.0 - demand[:len(lut)])
    return 1.0 - miss


@dataclass
class StackLayer:
    index: int
    layer: object            # CachedMoELayer
    encoder: bool = True


class CachedMoEStack:
    def __init__(self, layers: list, predictor=None, policy: OffloadPolicy = None,
                 s_b: float = 1.0, mem_avail: float = 1.0, mem_total: float = 1.0):
        self.layers = layers
        self.predictor = predictor
        self.policy = policy or OffloadPolicy()
        self.theta = prefetch_threshold(self.policy, s_b, mem_avail, mem_total)
        self.prefetch_log = []

    def forward(self, x, emb=None, ctx=None, routings=None):
        """x [T, d] bf16; emb/ctx [T, *] float64 device tensors for the
        predictor (token embedding / context, as TokenRecord carries);
        `routings` (optional, one (expert_idx, probs) per layer) replays a
        routing trace instead of running each layer's router."""
        h = x
        for i, sl in enumerate(self.layers):
            nxt = self.layers[i + 1] if i + 1 < len(self.layers) else None
            hook = None
            if nxt is not None and sl.encoder and self.predictor is not None:
                def hook(r, sl=sl, nxt=nxt):
                    _, demand = self.predictor.predict_slots(r.gate.expert_idx, emb, ctx,
                                                             want_demand=True, demand_mode="any")
                    L = nxt.layer.layer
                    demand = fold_demand(demand.cpu().numpy(), L.slot_map.cpu().numpy(), L.G)
                    chosen = nxt.layer.cache.prefetch(demand, self.theta)
                    self.prefetch_log.append((sl.index, nxt.index, chosen))
            y = sl.layer.forward(h, after_route=hook,
                                 routing=routings[i] if routings is not None else None)
            h = (y.float() + h.float()).to(torch.bfloat16)
        return h
