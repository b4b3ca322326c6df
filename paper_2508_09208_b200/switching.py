"""Live variant switching: the coarse-grained half of CoMoE's two-level
adaptation (the reference's `_Run._process_resource_tick` and
`_switch_variant`, pkg/src/comoe/simulator.py:624-680) driving real device
layers.

Every `reeval_interval` ticks the controller re-selects a variant for the
current (smoothed) GPU memory availability with the reference's rules —
`select_variant` under the resident-bytes requirement, the significant-
change bookkeeping, `should_switch` hysteresis, forced switches when the
current variant no longer fits — and, on a switch, rebuilds each MoE
layer's HBM expert cache for the new variant (`cache.activate_variant`,
i.e. `_activate_variant`, simulator.py:370-441): the experts that become
resident are copied host -> HBM on the cache's copy stream and the layer's
routing LUT is pointed at the new groups. Smoothing the resource signal
(the reference's EWMA, resource.py) is outside this path: callers pass the
smoothed value.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import torch

from .aggregation import SwitchPolicy, select_variant, should_switch
from .cache import CachedMoELayer, activate_variant
from .errors import InfeasibleError


@dataclass
class SwitchEvent:
    tick: int
    kind: str                 # "variant-switch" | "adjustment" | "no-feasible-variant"
    variant_from: str = ""
    variant_to: str = ""
    forced: bool = False
    migrated_bytes: float = 0.0
    seconds: float = 0.0      # wall time of the rebuild, copies completed


@dataclass
class VariantController:
    """`library`: VariantLibrary whose variants hold per-layer pinned host
    stores (`host_stores[variant_id][layer]`, rows in ascending principal
    order, as `activate_variant` expects); `layers`: {layer: (router wg,
    d_ff)}; budget/usable/required mirror simulator.py:646-647."""

    library: object
    stats: object
    host_stores: dict
    layers: dict
    d_ff: int
    policy: SwitchPolicy = field(default_factory=SwitchPolicy)
    reeval_interval: int = 8
    significant_change: float = 0.1
    usable: float = 1.0
    required_bytes: object = None
    workspace_slots: int = 2
    capacity_factor: object = 1.25
    variant: object = None
    events: list = field(default_factory=list)

    def __post_init__(self):
        self.policy.validate()
        self.last_eval_value = None
        self.last_change_tick = 0
        self.caches = {}
        self.model_layers = {}

    # ------------------------------------------------------------ activation
    def activate(self, variant, budget_bytes: float) -> float:
        """Build the cached layers of `variant` within `budget_bytes` per
        layer; returns the bytes copied host -> HBM for its resident experts
        (principals are re-indexed per variant, so every resident expert of
        a new variant is a fresh copy)."""
        caches, layers = {}, {}
        for l, (wg, _) in self.layers.items():
            cache = activate_variant(variant, l, self.stats, self.host_stores[variant.variant_id][l],
                                     budget_bytes, workspace_slots=self.workspace_slots)
            lut, _ = variant.group_table(l, wg.shape[1])
            cl = CachedMoELayer(wg, cache, self.d_ff, capacity_factor=self.capacity_factor)
            cl.set_groups(lut)
            caches[l], layers[l] = cache, cl
        self.caches, self.model_layers, self.variant = caches, layers, variant
        return float(sum(c.stats.h2d_bytes for c in caches.values()))

    def start(self, mem_available: float) -> SwitchEvent:
        """Initial variant for the starting memory level (tick 0)."""
        req = self.required_bytes or (lambda v: v.mem_required)
        cand = select_variant(self.library, self.usable * mem_available, required_bytes=req)
        self.last_eval_value = mem_available
        return self.switch(cand, 0, False, self.usable * mem_available)

    def forward(self, x, layer: int):
        return self.model_layers[layer].forward(x)

    # ------------------------------------------------------------ resource tick
    def tick(self, t: int, mem_available: float):
        """_process_resource_tick (simulator.py:624-661) on a smoothed
        memory signal; returns the SwitchEvent of a switch, else None."""
        if self.variant is None:
            raise RuntimeError("call start() before tick()")
        if t == 0 or t % self.reeval_interval != 0 or len(self.library.variants) < 2:
            return None
        ref, cur = self.last_eval_value, mem_available
        if ref > 0 and abs(cur - ref) / ref > self.significant_change:
            self.events.append(SwitchEvent(t, "adjustment"))
            self.last_change_tick = t
            self.last_eval_value = cur
        budget = self.usable * cur
        req = self.required_bytes or (lambda v: v.mem_required)
        try:
            cand = select_variant(self.library, budget, required_bytes=req)
        except InfeasibleError:
            self.events.append(SwitchEvent(t, "no-feasible-variant"))
            return None
        if cand.variant_id == self.variant.variant_id:
            return None
        t_stable = float(t - self.last_change_tick)
        forced = req(self.variant) > budget
        delta_p = cand.perf_estimate - self.variant.perf_estimate
        if forced or should_switch(self.variant, cand, delta_p, self.policy, t_stable):
            return self.switch(cand, t, forced, budget)
        return None

    def switch(self, cand, t: int, forced: bool, budget: float) -> SwitchEvent:
        """_switch_variant (simulator.py:663-680): rebuild the caches for the
        candidate; the event carries the migrated bytes and the measured
        rebuild time (host policy + H2D copies, synchronised)."""
        old = self.variant.variant_id if self.variant is not None else ""
        per_layer = budget / max(1, len(self.layers))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        migrated = self.activate(cand, per_layer)
        for c in self.caches.values():
            c.copy_stream.synchronize()
        dt = time.perf_counter() - t0
        self.last_change_tick = t
        ev = SwitchEvent(t, "variant-switch", old, cand.variant_id, forced, migrated, dt)
        self.events.append(ev)
        return ev
