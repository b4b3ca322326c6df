"""HBM-budgeted expert cache (K7) and the MoE layer that runs on it.

Every expert keeps a master copy in pinned host memory (weights are
read-only, so the reference's CACHE->HOST eviction, simulator.py:480, is a
free slot release). HBM holds `n_slots` expert slots (an ExpertPool). The
residency decisions are the reference policy, unchanged
(paper_2508_09208_b200.offload mirrors offload.py): tiers in a CacheState,
popularity placement, hybrid eviction scores, threshold-gated prefetch and
similarity substitution. Data movement is real: cudaMemcpyAsync (torch
copy_) host->slot on a dedicated copy stream, one CUDA event per slot
standing in for the simulator's `inflight[eid]` (simulator.py:617).

CachedMoELayer.forward(x):
  1. gate + capacity scan on the compute stream (as MoELayer);
  2. one D2H of the per-group kept counts — the demand set (the only host
     sync of the layer; the reference decides on the host too);
  3. hits are served in place; misses are either substituted (slot of the
     most similar resident expert, correct_misprediction) or fetched;
  4. experts are processed in waves that fit the slot pool: wave k's grouped
     GEMMs run while wave k+1's H2D copies stream into the other slots
     (the compute stream waits per-slot events; the copy stream waits for
     the GEMM event of the wave that last used a slot before overwriting it).
Outputs are bit-identical to MoELayer.forward with every expert resident:
the cache only changes where weights live, never the arithmetic.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels
from .errors import InfeasibleError
from .layer import MoELayer
from .offload import (CACHE, HOST, WORKSPACE, OffloadPolicy, build_cache_state,
                      correct_misprediction, decide_prefetch, eviction_score, evict,
                      plan_initial_placement)
from .pool import ExpertPool


@dataclass
class CacheStats:
    demand: int = 0
    hits: int = 0
    fetches: int = 0
    prefetch_issued: int = 0
    prefetch_hits: int = 0
    substitutions: int = 0
    evictions: int = 0
    h2d_bytes: int = 0
    waves: int = 0
    events: list = field(default_factory=list)  # (kind, expert[, used]) in decision order

    def hit_rate(self) -> float:
        return self.hits / self.demand if self.demand else 0.0


class EventLog:
    """Cache decision records in the reference simulator's event format
    (simulator.py:86-99: {"tick", "event", "seq", payload keys sorted}) with
    its event kinds (hit / fetch / substitute / prefetch / demote / evict,
    simulator.py:47-63) and payload keys (expert, tier_from, tier_to, bytes,
    used, penalty, theta, p). Timing fields of the analytic simulator
    (comm_s, completes_s) are absent: copies here are real and asynchronous.
    write_jsonl / the reference's read_events_jsonl round-trip."""

    def __init__(self):
        self.records = []
        self._seq = 0

    def emit(self, tick: int, kind: str, **payload):
        rec = {"tick": int(tick), "event": kind, "seq": self._seq}
        for key in sorted(payload):
            rec[key] = payload[key]
        self.records.append(rec)
        self._seq += 1
        return rec

    def write_jsonl(self, path: str) -> None:
        import json
        with open(path, "w", encoding="utf-8") as fh:
            for rec in self.records:
                fh.write(json.dumps(rec) + "\n")


class ExpertCache:
    """Slot manager + policy for the experts of one or more MoE layers (ids
    (layer, slot)) in ONE HBM budget, like the simulator's single CacheState
    over all layers (simulator.py:415-420). `host_experts` is a pinned
    [E, numel] tensor for the single layer `layer`, or {layer: tensor}."""

    def __init__(self, host_experts, layer: int = None, n_slots: int = 0,
                 workspace_slots: int = 2, policy: OffloadPolicy = None, freqs=None,
                 pinned=(), device=None, substitution=False, similarity=None,
                 priorities: dict = None, priority_threshold: float = 1.0,
                 half_life: float = 256.0):
        hosts = dict(host_experts) if isinstance(host_experts, dict) else {layer: host_experts}
        if any(not h.is_pinned() for h in hosts.values()):
            raise ValueError("host expert store must be pinned memory")
        shapes = {tuple(h.shape[1:]) for h in hosts.values()}
        if len(shapes) != 1:
            raise ValueError("every layer's experts must have one flat size")
        if not 1 <= workspace_slots < n_slots:
            raise ValueError("need 1 <= workspace_slots < n_slots")
        numel = next(iter(hosts.values())).shape[1]
        self.host = hosts
        self.layers = sorted(hosts)
        self.layer = self.layers[0]            # single-layer caches: the layer
        self.E = max(h.shape[0] for h in hosts.values())
        self.dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.pool = ExpertPool(n_slots, numel, device=self.dev)
        self.bytes = numel * next(iter(hosts.values())).element_size()
        self.policy = policy or OffloadPolicy()
        self.substitution = substitution
        self.similarity = similarity  # callable (eid_a, eid_b) -> float
        self.priorities = priorities or {}
        self.prio_threshold = priority_threshold
        self.copy_stream = torch.cuda.Stream(self.dev)
        self.ready = [torch.cuda.Event() for _ in range(n_slots)]   # slot filled
        self.free_ev = [torch.cuda.Event() for _ in range(n_slots)]  # slot's last reader done
        self._free_pending = [False] * n_slots
        self.slot_of = {}
        self._free_slots = list(range(n_slots - 1, -1, -1))
        self.stats = CacheStats()
        self.log = EventLog()
        self.tick = 0
        self.last_probs = {}       # layer -> predicted probabilities (eviction scores)
        self.prefetched = set()
        self.inflight = set()      # prefetched, pinned until demanded or the next step
        all_ids = [(l, s) for l in self.layers for s in range(hosts[l].shape[0])]
        freqs = freqs if freqs is not None else {e: 1.0 / self.E for e in all_ids}
        max_f = max(max(freqs.values()), 1e-12)
        self.importance = {e: f / max_f for e, f in freqs.items()}
        sizes = {e: float(self.bytes) for e in all_ids}
        ws_cap = workspace_slots * float(self.bytes)
        ca_cap = (n_slots - workspace_slots) * float(self.bytes)
        plan = plan_initial_placement(sizes, freqs, ws_cap, ca_cap, pinned=frozenset(pinned),
                                      working_set_bytes=float(self.bytes))
        self.state = build_cache_state(plan, sizes, ws_cap, ca_cap, pinned=set(pinned),
                                       importance=self.importance, half_life=half_life)
        for eid in self.state.gpu_resident_ids():
            self._load(eid)
        self.hard_pinned = set(pinned)

    # ------------------------------------------------------------ slots
    def _load(self, eid):
        slot = self._free_slots.pop()
        self.slot_of[eid] = slot
        with torch.cuda.stream(self.copy_stream):
            if self._free_pending[slot]:
                self.copy_stream.wait_event(self.free_ev[slot])
            self.pool.view(slot).copy_(self.host[eid[0]][eid[1]], non_blocking=True)
            self.ready[slot].record(self.copy_stream)
        self.stats.h2d_bytes += self.bytes
        return slot

    def _release(self, eid):
        slot = self.slot_of.pop(eid)
        self._free_slots.append(slot)

    def mark_used(self, slots, stream):
        """Record that `stream` reads these slots (copies into them must wait)."""
        for s in slots:
            self.free_ev[s].record(stream)
            self._free_pending[s] = True

    def wait_ready(self, slots, stream):
        for s in slots:
            stream.wait_event(self.ready[s])

    # ------------------------------------------------------------ steps
    def begin_step(self, tick: int = None) -> None:
        """Start of a token step (the simulator's token-start + arrival sweep,
        simulator.py:503-513, 684-687): prefetches issued in earlier steps
        have landed (their copies are stream-ordered before any reader), so
        their in-flight pins are dropped."""
        self.tick = self.tick + 1 if tick is None else int(tick)
        for e in sorted(self.inflight):
            if e not in self.hard_pinned:
                self.state.pinned.discard(e)
        self.inflight.clear()

    # ------------------------------------------------------------ policy
    def _scores(self):
        out = {}
        for eid in self.state.cache:
            if eid in self.state.pinned:
                continue
            probs = self.last_probs.get(eid[0])
            p = float(probs[eid[1]]) if probs is not None else 0.0
            out[eid] = eviction_score(p, self.state.recent_value(eid, self.tick),
                                      self.importance.get(eid, 0.0), self.policy.delta_evict,
                                      self.policy.lambda_evict)
        return out

    def _make_room_cache(self, nbytes) -> bool:
        try:
            victims = evict(self.state, nbytes, self._scores())
        except InfeasibleError:
            return False
        for v in victims:
            self.state.move(v, CACHE, HOST)
            self._release(v)
            self.prefetched.discard(v)
            self.stats.evictions += 1
            self.stats.events.append(("evict", v))
            self.log.emit(self.tick, "evict", expert=list(v), tier_from=CACHE, tier_to=HOST,
                          bytes=float(self.bytes))
        return True

    def _room_in_workspace(self) -> bool:
        """simulator._room_in_workspace (simulator.py:486-501) over a batch:
        demote unpinned workspace entries FIFO to the cache (evicting cache
        entries if needed, else to host). False when every workspace entry
        belongs to the active (pinned) wave."""
        b = float(self.bytes)
        while self.state.free_bytes(WORKSPACE) < b:
            victim = next((e for e in self.state.workspace if e not in self.state.pinned), None)
            if victim is None:
                return False
            if self.state.free_bytes(CACHE) >= b or self._make_room_cache(b):
                self.state.move(victim, WORKSPACE, CACHE)
                self.stats.events.append(("demote", victim))
                self.log.emit(self.tick, "demote", expert=list(victim), tier_from=WORKSPACE,
                              tier_to=CACHE, bytes=b)
            else:
                self.state.move(victim, WORKSPACE, HOST)
                self._release(victim)
                self.stats.events.append(("evict", victim))
                self.log.emit(self.tick, "evict", expert=list(victim), tier_from=WORKSPACE,
                              tier_to=HOST, bytes=b)
        return True

    def serve(self, demanded: list):
        """Serve one wave of demanded expert ids (layer, slot), pinning each
        so later misses of the same wave cannot evict it. Batched
        generalisation of _serve_demand (simulator.py:517-574): a miss goes
        to the workspace tier, or — when the workspace is full of this
        wave's experts — to the cache tier. Returns {eid: pool slot} (the
        substitute's slot for substituted experts)."""
        out = {}
        b = float(self.bytes)
        for eid in demanded:
            self.stats.demand += 1
            if self.state.resident(eid):
                tier = self.state.tier_of(eid)
                self.stats.hits += 1
                if eid in self.inflight:   # the prefetch has landed: in-flight pin off
                    self.inflight.discard(eid)
                    if eid not in self.hard_pinned:
                        self.state.pinned.discard(eid)
                if eid in self.prefetched:
                    self.stats.prefetch_hits += 1
                    self.prefetched.discard(eid)
                self.state.record_access(eid, self.tick)
                self.state.pinned.add(eid)
                out[eid] = self.slot_of[eid]
                self.stats.events.append(("hit", eid))
                self.log.emit(self.tick, "hit", expert=list(eid), tier_from=tier, tier_to=tier,
                              bytes=0.0)
                continue
            if self.substitution and self.similarity is not None:
                dec = correct_misprediction(eid, self.state, self.similarity, self.policy,
                                            priority=self.priorities.get(eid, 0.0),
                                            priority_threshold=self.prio_threshold)
                if dec.action == "substitute":
                    self.stats.substitutions += 1
                    self.state.record_access(dec.expert, self.tick)
                    self.state.pinned.add(dec.expert)
                    out[eid] = self.slot_of[dec.expert]
                    self.stats.events.append(("substitute", eid, dec.expert))
                    self.log.emit(self.tick, "substitute", expert=list(eid),
                                  used=list(dec.expert), penalty=dec.penalty, tier_from=HOST,
                                  tier_to=HOST, bytes=0.0)
                    continue
            if self._room_in_workspace():
                tier = WORKSPACE
            elif self.state.free_bytes(CACHE) >= b or self._make_room_cache(b):
                tier = CACHE
            else:
                raise InfeasibleError("wave does not fit the HBM expert slots")
            self.state.move(eid, HOST, tier)
            self.state.pinned.add(eid)
            self.state.record_access(eid, self.tick)
            out[eid] = self._load(eid)
            self.stats.fetches += 1
            self.stats.events.append(("fetch", eid))
            self.log.emit(self.tick, "fetch", expert=list(eid), tier_from=HOST, tier_to=tier,
                          bytes=b)
        return out

    def room(self) -> int:
        """Pool slots a wave of misses can use now: every slot not holding a
        pinned resident expert (pinned = this wave's, hard-pinned, or an
        in-flight prefetch)."""
        held = sum(1 for e in self.slot_of if e in self.state.pinned)
        return self.pool.n_slots - held

    def drop_inflight_pins(self) -> None:
        """Treat this step's in-flight prefetches as landed (the batched
        stand-in for the simulator's arrival sweep): their pins only guard
        the policy state, since a copy into a slot and any later reuse of
        that slot are ordered on the copy stream. Used when a wave of
        demand misses would otherwise find no slot."""
        for e in sorted(self.inflight):
            if e not in self.hard_pinned:
                self.state.pinned.discard(e)
        self.inflight.clear()

    def unpin(self, eids):
        for e in eids:
            if e not in self.hard_pinned and e not in self.inflight:
                self.state.pinned.discard(e)

    def prefetch(self, probs, theta: float, layer: int = None):
        """Threshold-gated prefetch of next-use experts of `layer` into the
        cache tier (simulator._predict_and_prefetch, simulator.py:578-620):
        `probs` (over the layer's cache experts) also become the layer's
        eviction-score probabilities; each prefetched expert is pinned while
        in flight (until it is demanded or the next step begins). Copies are
        asynchronous on the copy stream."""
        layer = self.layer if layer is None else layer
        probs = np.asarray(probs, dtype=float)
        self.last_probs[layer] = probs
        chosen = decide_prefetch(probs, theta, self.state, layer, lambda e: float(self.bytes))
        for eid in chosen:
            if self.state.free_bytes(CACHE) < self.bytes and not self._make_room_cache(self.bytes):
                break
            self.state.move(eid, HOST, CACHE)
            self.state.pinned.add(eid)   # guard the in-flight copy (simulator.py:612)
            self.inflight.add(eid)
            self._load(eid)
            self.prefetched.add(eid)
            self.stats.prefetch_issued += 1
            self.stats.events.append(("prefetch", eid))
            self.log.emit(self.tick, "prefetch", expert=list(eid), tier_from=HOST, tier_to=CACHE,
                          bytes=float(self.bytes), theta=float(theta), p=float(probs[eid[1]]))
        return chosen

    def check(self):
        self.state.check_invariants()
        assert len(self.slot_of) == len(self.state.workspace) + len(self.state.cache)
        assert len(set(self.slot_of.values())) == len(self.slot_of)


def resident_budget(variant_expert_bytes: float, cache_mode: str, cache_fraction: float,
                    total_expert_bytes: float, cache_bytes: float = None,
                    offload: bool = True) -> float:
    """GPU bytes kept resident for a variant's experts (simulator.py:275-286):
    fraction of the variant, fraction of the whole model, or absolute bytes,
    never more than the variant itself."""
    if not offload:
        return variant_expert_bytes
    if cache_mode == "fraction_of_variant":
        budget = cache_fraction * variant_expert_bytes
    elif cache_mode == "fraction_of_model":
        budget = cache_fraction * total_expert_bytes
    elif cache_mode == "absolute":
        budget = float(cache_bytes)
    else:
        raise ValueError(f"unknown cache_mode {cache_mode!r}")
    return min(budget, variant_expert_bytes)


def required_bytes_fn(cache_mode: str, cache_fraction: float, total_expert_bytes: float,
                      m_other: float, workspace_bytes: float, cache_bytes: float = None):
    """select_variant's resident-bytes requirement (simulator.py:289-293)."""
    def req(variant):
        return resident_budget(variant.expert_bytes, cache_mode, cache_fraction,
                               total_expert_bytes, cache_bytes) + m_other + workspace_bytes
    return req


def activate_variant(variant, layer: int, stats, host_experts: torch.Tensor, budget_bytes: float,
                     workspace_slots: int = 2, top_k: int = 1, policy: OffloadPolicy = None,
                     pin_decoder_layers=(), bandwidth: float = 55e9, substitution=False,
                     similarity=None, device=None) -> "ExpertCache":
    """Cache runtime for one layer of a variant, sized and seeded like
    _Run._activate_variant (simulator.py:370-441): importance = merged
    frequency / max, workspace = workspace_slots*K experts (capped by the
    budget), cache = the rest of the budget, decoder layers pinned, offload
    priorities with the priority-quantile threshold for substitution.
    `host_experts` holds the variant's retained experts of this layer in
    ascending principal order (row i <-> principal i of group_table)."""
    from .aggregation import variant_freqs
    from .offload import offload_priority
    policy = policy or OffloadPolicy()
    principals = sorted(variant.retained[layer])
    freqs_all = variant_freqs(variant, stats)
    freqs = {(layer, i): freqs_all[(layer, p)] for i, p in enumerate(principals)}
    numel = host_experts.shape[1]
    ebytes = float(numel * host_experts.element_size())
    # _resident_budget (simulator.py:275-286) never keeps more than the
    # variant itself resident; the batched runtime adds its workspace slots
    # (one wave of demanded experts) on top, and no more
    ws_cap = min(workspace_slots * top_k * ebytes, budget_bytes)
    ws_slots = max(1, int(ws_cap // ebytes))
    n_slots = min(int(budget_bytes // ebytes), len(principals) + ws_slots)
    if n_slots <= ws_slots:
        raise InfeasibleError(f"budget {budget_bytes:.3e} B holds {n_slots} experts; need more than "
                              f"the {ws_slots}-expert workspace")
    pinned = {(layer, i) for i in range(len(principals))} if layer in set(pin_decoder_layers) else set()
    est = ebytes / max(bandwidth, 1.0)
    prios = {e: offload_priority(f, ebytes, est, policy.gamma_prio, ebytes / est)
             for e, f in freqs.items()}
    thr = float(np.quantile(np.array(sorted(prios.values())), policy.priority_quantile)) if prios else 1.0
    return ExpertCache(host_experts, layer=layer, n_slots=n_slots, workspace_slots=ws_slots,
                       policy=policy, freqs=freqs, pinned=pinned, device=device,
                       substitution=substitution, similarity=similarity, priorities=prios,
                       priority_threshold=thr)


class CachedMoELayer:
    """MoELayer whose experts live in an ExpertCache (Switch / top-1 or top-2)."""

    def __init__(self, wg, cache: ExpertCache, d_ff: int, act="relu", top_k=1, norm_topk=None,
                 capacity_factor=1.25, wave_slots: int = None, layer: int = None):
        self.cache = cache
        self.layer_id = cache.layer if layer is None else layer  # cache ids (layer_id, group)
        if self.layer_id not in cache.host:
            raise ValueError(f"the cache holds no experts of layer {self.layer_id}")
        n_exp = wg.shape[1]
        # group g of the layer <-> cache expert (layer, g); set_variant(lut, ...) maps a
        # fused variant's original experts onto the cache's retained experts
        self.layer = MoELayer(wg, cache.pool, d_ff, act=act, top_k=top_k, norm_topk=norm_topk,
                              capacity_factor=capacity_factor, expert_slots=[0] * n_exp)
        self.E = max(n_exp, cache.E)
        free = cache.pool.n_slots - len(cache.hard_pinned)
        # half the free slots per wave: wave k+1 can stream in while wave k computes
        self.wave_slots = wave_slots or max(1, free // 2)
        self._tables = torch.zeros((self.E, 2, self.E), dtype=torch.int32).pin_memory()
        self._tables_dev = torch.zeros((self.E, 2, self.E), dtype=torch.int32, device=wg.device)

    def set_groups(self, slot_map) -> None:
        """Route through a fused variant: slot_map[E] -> group index, where
        group g is the cache's expert (layer, g) (ModelVariant.group_table)."""
        G = max(slot_map) + 1
        n = self.cache.host[self.layer_id].shape[0]
        if G > n:
            raise ValueError(f"{G} groups but the cache holds {n} experts of this layer")
        self.layer.set_variant(slot_map, [0] * G)  # slots come from the cache per wave

    def forward(self, x, out=None, after_route=None, after_serve=None, routing=None, step=True):
        """`after_route(routing)` runs right after routing (the stack launches
        the next-layer predictor there, so it runs before this layer's
        GEMMs); `after_serve(handle)` runs once this layer's demand is served
        and its GEMMs are enqueued — the reference order (serve, then
        predict and prefetch, simulator.py:700-712) — so the prefetch copies
        overlap this layer's GEMMs. `routing` = (expert_idx, probs) replays
        given choices (MoELayer.route). A standalone layer advances the
        cache clock itself (`step=True`); in a stack (`step=False` from
        CachedMoEStack) the stack does, once per token step."""
        L = self.layer
        T = x.shape[0]
        if out is None:
            out = torch.empty((T, L.d), dtype=torch.bfloat16, device=x.device)
        ws = L._workspace(T)
        comp = torch.cuda.current_stream()
        r = L.route(x, routing=routing)
        k1 = L.top_k == 1
        fused, gather = ws["fused"], ws["gather"]
        kernels.permute(x, r.gate, r.scan, r.capacity, r.rows, y_zero=out if k1 else None,
                        out=r.perm, copy_rows=not gather)
        handle = after_route(r) if after_route is not None else None
        kept = r.scan.group_kept.cpu().numpy()  # the demand set (the layer's one host sync)
        c = self.cache
        lid = self.layer_id
        if step:
            c.begin_step()
        n_here = c.host[lid].shape[0]
        if len(kept) > n_here:
            raise ValueError(f"layer has {len(kept)} groups but the cache holds {n_here} experts; "
                             "call layer.set_variant(lut, ...) for a fused variant")
        order = [int(g) for g in np.argsort(-kept, kind="stable") if kept[g] > 0]
        hits = [g for g in order if c.state.resident((lid, g))]
        misses = [g for g in order if not c.state.resident((lid, g))]
        n1 = 2 * L.d_ff if L.act == "swiglu" else L.d_ff
        dst = out if k1 else ws["y_perm"]
        epi1 = kernels.EPI_SWIGLU if L.act == "swiglu" else kernels.EPI_RELU
        epi2 = kernels.EPI_SCALE_SCATTER if k1 else kernels.EPI_STORE
        tab = self._tables.numpy()

        def waves():
            # every hit is already resident: one wave serves them all (no
            # copies, no slots needed); a wave of misses takes at most
            # wave_slots experts and never more than the slots free of pins
            # right now (in-flight prefetches of this step hold theirs)
            if hits:
                yield hits
            i = 0
            while i < len(misses):
                room = c.room()
                if room < 1:
                    c.drop_inflight_pins()
                    room = c.room()
                n = max(1, min(self.wave_slots, room))
                yield misses[i:i + n]
                i += n

        for w, wave in enumerate(waves()):
            if w >= self._tables.shape[0]:
                raise InfeasibleError("more expert waves than groups")
            ids = [(lid, g) for g in wave]
            slots = c.serve(ids)
            c.stats.waves += 1
            tab[w] = 0
            G = len(kept)
            for g in wave:
                tab[w, 0, g] = kept[g]
                tab[w, 1, g] = slots[(lid, g)]
            used = sorted({slots[e] for e in ids})
            self._tables_dev[w].copy_(self._tables[w], non_blocking=True)
            c.wait_ready(used, comp)
            g_rows, g_slot = self._tables_dev[w, 0, :G], self._tables_dev[w, 1, :G]
            if fused:  # K3F over this wave's groups (H on chip)
                kernels.fused_ffn(x if gather else r.perm.x_perm, c.pool.data, L.d_ff, g_rows,
                                  r.scan.group_base, g_slot, dst,
                                  gather_rows=r.perm.row_token if gather else None,
                                  row_token=r.perm.row_token if k1 else None,
                                  row_prob=r.perm.row_prob if k1 else None)
            else:
                kernels.grouped_gemm(r.perm.x_perm, c.pool.data, 0, n1, g_rows,
                                     r.scan.group_base, g_slot, epi1, ws["h"])
                kernels.grouped_gemm(ws["h"], c.pool.data, n1 * L.d, L.d, g_rows,
                                     r.scan.group_base, g_slot, epi2, dst,
                                     row_token=r.perm.row_token if k1 else None,
                                     row_prob=r.perm.row_prob if k1 else None)
            c.mark_used(used, comp)
            c.unpin(list(ids) + [e for e in c.slot_of if c.slot_of[e] in used])
        if not k1:
            kernels.combine(ws["y_perm"], r.perm.token_pos, r.gate.gate_prob, out=out)
        if after_serve is not None:
            after_serve(handle)
        c.check()
        L.last = r
        return out

    __call__ = forward
