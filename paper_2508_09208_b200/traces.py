"""Routing traces: the reference's synthetic routing source and JSONL trace
format (pkg/src/comoe/moe.py:114-230, 372-415), so reference traces can be
replayed through the device layer (MoELayer.forward(x, routing=...)).

generate_routing draws from the same seeded generators in the same order as
the reference (structure RNG: per-layer rank permutations then one shared
successor map; draw RNG: embeddings, contexts, then per token and layer one
follow/draw decision and inverse-CDF draws with rejection), so a spec yields
the identical trace (checked against reference fixtures in tests/golden).
This is host-side synthetic input generation, not a compute path.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np
import torch

from .errors import TraceError


@dataclass
class RoutingGeneratorSpec:
    """Zipf skew (scalar or {layer: skew}), follow probability rho, seeds
    (moe.py:114-143)."""

    skew: object = 1.0
    rho: float = 0.9
    seed: int = 0
    structure_seed: int = 0
    embed_dim: int = 16
    context_dim: int = 8

    def layer_skew(self, layer: int) -> float:
        if isinstance(self.skew, dict):
            return float(self.skew.get(layer, self.skew.get("default", 1.0)))
        return float(self.skew)

    def validate(self) -> None:
        if not 0.0 <= self.rho <= 1.0:
            raise ValueError(f"rho must be in [0, 1], got {self.rho}")
        values = self.skew.values() if isinstance(self.skew, dict) else (self.skew,)
        if any(float(v) < 0 for v in values):
            raise ValueError("skew must be nonnegative")


@dataclass
class TokenRecord:
    token_id: int
    layer_experts: dict  # layer -> tuple of slots
    embedding: np.ndarray
    context: np.ndarray


@dataclass
class RoutingTrace:
    tokens: list
    experts_per_layer: int
    moe_layer_indices: tuple
    top_k: int = 1

    def __len__(self) -> int:
        return len(self.tokens)

    def expert_indices(self, layer: int) -> np.ndarray:
        """[T, k] int32 expert choices of one layer (for the device path)."""
        return np.asarray([tok.layer_experts[layer] for tok in self.tokens], dtype=np.int32)

    def to_device(self, layer: int, device="cuda") -> torch.Tensor:
        return torch.as_tensor(self.expert_indices(layer), device=device)


def _slot_probs(E: int, skew: float, perm: np.ndarray) -> np.ndarray:
    w = np.arange(1, E + 1, dtype=float) ** (-skew)
    w /= w.sum()
    out = np.empty(E)
    out[perm] = w  # rank r is slot perm[r]
    return out


def _draw_distinct(rng, cdf: np.ndarray, k: int) -> tuple:
    picks = []
    last = cdf.size - 1
    while len(picks) < k:
        s = min(int(np.searchsorted(cdf, rng.random(), side="right")), last)
        if s not in picks:
            picks.append(s)
    return tuple(picks)


def generate_routing(gspec: RoutingGeneratorSpec, model_spec, n_tokens: int) -> RoutingTrace:
    """Zipf-over-permuted-ranks first layer, rho-follow of one shared
    successor map afterwards (moe.py:186-230)."""
    if n_tokens <= 0:
        raise ValueError("n_tokens must be positive")
    gspec.validate()
    model_spec.validate()
    E, K = model_spec.experts_per_layer, model_spec.top_k
    layers = model_spec.moe_layer_indices
    draw = np.random.default_rng(gspec.seed)
    struct = np.random.default_rng(gspec.structure_seed)
    perms = [struct.permutation(E) for _ in layers]
    successor = struct.permutation(E)
    cdfs = [np.cumsum(_slot_probs(E, gspec.layer_skew(l), perms[i])) for i, l in enumerate(layers)]
    emb = draw.normal(size=(n_tokens, gspec.embed_dim))
    ctx = draw.normal(size=(n_tokens, gspec.context_dim))
    tokens = []
    for t in range(n_tokens):
        chosen, prev = {}, None
        for i, l in enumerate(layers):
            follow = i > 0 and draw.random() < gspec.rho
            cur = tuple(int(successor[s]) for s in prev) if follow else _draw_distinct(draw, cdfs[i], K)
            chosen[l] = cur
            prev = cur
        tokens.append(TokenRecord(t, chosen, emb[t], ctx[t]))
    return RoutingTrace(tokens=tokens, experts_per_layer=E, moe_layer_indices=layers, top_k=K)


def trace_to_jsonl(trace: RoutingTrace, path: str) -> None:
    with open(path, "w") as fh:
        for tok in trace.tokens:
            fh.write(json.dumps({
                "token_id": tok.token_id,
                "layers": [{"layer": l, "experts": [int(s) for s in slots]}
                           for l, slots in sorted(tok.layer_experts.items())],
                "embedding": [float(v) for v in tok.embedding],
                "context": [float(v) for v in tok.context]}) + "\n")


def trace_from_jsonl(path: str, experts_per_layer: int = None) -> RoutingTrace:
    tokens, layers, top_k, max_slot = [], None, 1, -1
    with open(path) as fh:
        for line in fh:
            if not line.strip():
                continue
            rec = json.loads(line)
            le = {int(e["layer"]): tuple(int(s) for s in e["experts"]) for e in rec["layers"]}
            key = tuple(sorted(le))
            if layers is None:
                layers = key
            elif key != layers:
                raise ValueError("inconsistent MoE layer set across trace records")
            for slots in le.values():
                top_k = max(top_k, len(slots))
                max_slot = max(max_slot, max(slots))
            tokens.append(TokenRecord(int(rec["token_id"]), le,
                                      np.array(rec["embedding"], dtype=float),
                                      np.array(rec["context"], dtype=float)))
    if not tokens:
        raise ValueError(f"no records in trace file {path}")
    E = experts_per_layer if experts_per_layer is not None else max_slot + 1
    return RoutingTrace(tokens=tokens, experts_per_layer=E, moe_layer_indices=layers, top_k=top_k)


__all__ = ["RoutingGeneratorSpec", "TokenRecord", "RoutingTrace", "generate_routing",
           "trace_to_jsonl", "trace_from_jsonl", "TraceError"]
