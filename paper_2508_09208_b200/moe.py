"""Experts, activation statistics and expert similarity on the device.

Drop-in for the hot-path part of pkg/src/comoe/moe.py: the same names and
signatures, but `Expert.params` is a CUDA tensor (bf16 for the fast path,
float64 for the parity mode) — usually one slot of an ExpertPool — and the
similarity contraction runs in the K6 kernels. Plain NumPy parameter
vectors are accepted and uploaded as float64 (parity mode); there is no CPU
compute path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import kernels
from .traces import (RoutingGeneratorSpec, RoutingTrace, TokenRecord,  # noqa: F401
                     generate_routing, trace_from_jsonl, trace_to_jsonl)


@dataclass
class MoeModelSpec:
    """Layer geometry (pkg/src/comoe/moe.py:27-66)."""

    total_layers: int
    encoder_moe_layers: tuple
    decoder_moe_layers: tuple
    experts_per_layer: int
    expert_size_bytes: float
    top_k: int = 1
    expert_param_dim: int = 64

    @property
    def moe_layer_indices(self) -> tuple:
        return tuple(sorted((*self.encoder_moe_layers, *self.decoder_moe_layers)))

    @property
    def expert_count(self) -> int:
        return len(self.moe_layer_indices) * self.experts_per_layer

    @property
    def total_expert_bytes(self) -> float:
        return self.expert_count * self.expert_size_bytes

    def validate(self) -> None:
        if self.top_k < 1 or self.experts_per_layer < 1:
            raise ValueError("counts must be >= 1")
        if self.top_k > self.experts_per_layer:
            raise ValueError("top_k exceeds experts_per_layer")
        if self.expert_size_bytes <= 0:
            raise ValueError("expert_size_bytes must be positive")
        if self.expert_param_dim < 1:
            raise ValueError("expert_param_dim must be >= 1")
        idx = self.moe_layer_indices
        if len(set(idx)) != len(idx):
            raise ValueError("duplicate MoE layer indices")
        if any(not 1 <= l <= self.total_layers for l in idx):
            raise ValueError("MoE layer index outside the model")
        if set(self.encoder_moe_layers) & set(self.decoder_moe_layers):
            raise ValueError("encoder and decoder MoE layers overlap")


def as_device_params(params, device=None) -> torch.Tensor:
    """Expert parameters as a flat CUDA tensor (NumPy -> float64 upload)."""
    if isinstance(params, torch.Tensor):
        t = params
        if not t.is_cuda:
            t = t.to("cuda" if device is None else device)
    else:
        t = torch.as_tensor(np.asarray(params, dtype=np.float64),
                            device="cuda" if device is None else device)
    return t.reshape(-1)


@dataclass
class Expert:
    """One expert (pkg/src/comoe/moe.py:69-74). `params` is a flat device
    tensor; `size` is its byte footprint for memory accounting."""

    layer: int
    slot: int
    params: object
    size: float


@dataclass
class MoeModel:
    spec: MoeModelSpec
    experts: dict  # (layer, slot) -> Expert

    def layer_experts(self, layer: int) -> list:
        return [self.experts[(layer, s)] for s in range(self.spec.experts_per_layer)]


# ---------------------------------------------------------------------------
# activation statistics


@dataclass
class ActivationStats:
    """Per-layer activation counts (pkg/src/comoe/moe.py:233-247)."""

    counts: dict  # layer -> ndarray[E] float64
    totals: dict  # layer -> int
    experts_per_layer: int

    def freqs(self, layer: int) -> np.ndarray:
        total = self.totals[layer]
        if total <= 0:
            raise ValueError(f"no activations recorded for layer {layer}")
        return np.asarray(self.counts[layer], dtype=np.float64) / total

    @property
    def layers(self) -> tuple:
        return tuple(sorted(self.counts))


def collect_stats(trace) -> ActivationStats:
    """collect_stats (moe.py:250-262) over a host RoutingTrace."""
    if len(trace.tokens) == 0:
        raise ValueError("empty routing trace")
    E = trace.experts_per_layer
    counts = {l: np.zeros(E) for l in trace.moe_layer_indices}
    totals = {l: 0 for l in trace.moe_layer_indices}
    for tok in trace.tokens:
        for l, slots in tok.layer_experts.items():
            np.add.at(counts[l], list(slots), 1.0)
            totals[l] += len(slots)
    return ActivationStats(counts=counts, totals=totals, experts_per_layer=E)


def stats_from_routing(layer_expert_idx: dict, experts_per_layer: int) -> ActivationStats:
    """ActivationStats from device routing: {layer: expert_idx[T,k] int32
    CUDA tensor}. Counts every pick (pre-capacity), like collect_stats."""
    counts, totals = {}, {}
    for layer, idx in layer_expert_idx.items():
        h = kernels.expert_histogram(idx.contiguous(), experts_per_layer)
        counts[layer] = h.cpu().numpy().astype(np.float64)
        totals[layer] = int((idx >= 0).sum().item())
    return ActivationStats(counts=counts, totals=totals, experts_per_layer=experts_per_layer)


# ---------------------------------------------------------------------------
# similarity


@dataclass
class Calibration:
    """Probe inputs plus the fixed projection (moe.py:269-274)."""

    probes: np.ndarray      # (n_probes, dim)
    projection: np.ndarray  # (buckets, dim)

    def device(self, device="cuda"):
        if self.probes is None or len(self.probes) == 0:
            return None, None  # cosine-only calibration
        key = ("dev", str(device))
        cache = self.__dict__.setdefault("_dev_cache", {})
        if key not in cache:
            cache[key] = (torch.as_tensor(np.ascontiguousarray(self.probes, np.float64), device=device),
                          torch.as_tensor(np.ascontiguousarray(self.projection, np.float64), device=device))
        return cache[key]


def cosine_only_calibration() -> Calibration:
    """Calibration with no probes: similarity_matrix then returns
    alpha*cos + (1-alpha) (the functional term is the constant 1). For
    real-scale experts, where the reference's n x D fp64 probe/projection
    matrices would not fit in memory."""
    return Calibration(probes=None, projection=None)


def make_calibration(dim: int, n_probes: int = 8, seed: int = 7, buckets: int = 8) -> Calibration:
    """Same seeded draws as moe.py:277-283 so calibrations are interchangeable."""
    if n_probes < 1:
        raise ValueError("need at least one probe")
    rng = np.random.default_rng(seed)
    probes = rng.normal(size=(n_probes, dim))
    projection = rng.normal(size=(buckets, dim))
    return Calibration(probes=probes, projection=projection)


def _rows(experts) -> list:
    rows = [as_device_params(e.params) for e in experts]
    dt = rows[0].dtype
    if dt not in (torch.bfloat16, torch.float64):
        rows = [r.to(torch.float64) for r in rows]
    elif any(r.dtype != dt for r in rows):
        rows = [r.to(torch.float64) for r in rows]
    if any(r.numel() != rows[0].numel() for r in rows):
        raise ValueError("parameter dimension mismatch")
    return [r.contiguous() for r in rows]


def similarity_matrix(experts: list, alpha_sim: float, calib: Calibration) -> np.ndarray:
    """similarity_matrix (moe.py:339-365) computed by the K6 kernels.

    Returns a host float64 [E, E] array (the reference returns an ndarray
    that group_experts indexes). Surrogate distributions use log-softmax, so
    the result stays finite where the reference's log(softmax) underflows."""
    if not (0.0 <= alpha_sim <= 1.0):
        raise ValueError(f"alpha_sim must be in [0, 1], got {alpha_sim}")
    rows = _rows(experts)
    if not hasattr(calib, "device"):  # the reference's own Calibration (drop-in use)
        calib = Calibration(probes=calib.probes, projection=calib.projection)
    probes, proj = calib.device(rows[0].device)
    sim, gram, _ = kernels.similarity(rows, probes, proj, alpha_sim)
    if torch.any(torch.diagonal(gram) == 0):
        raise ValueError("zero parameter vector has no direction")
    return sim.cpu().numpy()


def param_similarity(a: Expert, b: Expert) -> float:
    """Cosine similarity (moe.py:286-294), via the K6 Gram."""
    s = similarity_matrix([a, b], 1.0, _unit_calib(as_device_params(a.params).numel()))
    return float(s[0, 1])


def func_similarity(a: Expert, b: Expert, calib: Calibration) -> float:
    """1 - mean symmetric KL of the surrogate outputs (moe.py:318-328)."""
    if calib.probes.shape[0] < 1:
        raise ValueError("empty calibration set")
    return float(similarity_matrix([a, b], 0.0, calib)[0, 1])


def combined_similarity(a: Expert, b: Expert, alpha_sim: float, calib: Calibration) -> float:
    """alpha*param + (1-alpha)*functional similarity (moe.py:331-336)."""
    if not (0.0 <= alpha_sim <= 1.0):
        raise ValueError(f"alpha_sim must be in [0, 1], got {alpha_sim}")
    return float(similarity_matrix([a, b], alpha_sim, calib)[0, 1])


def kl_divergence(p, q) -> float:
    """KL(p || q) over p > 0 (moe.py:311-315); tiny host helper."""
    p = np.asarray(p, dtype=float)
    q = np.asarray(q, dtype=float)
    m = p > 0
    return float(np.sum(p[m] * (np.log(p[m]) - np.log(q[m]))))


_UNIT = {}


def _unit_calib(dim: int) -> Calibration:
    if dim not in _UNIT:
        _UNIT[dim] = Calibration(probes=np.ones((1, dim)), projection=np.ones((1, dim)))
    return _UNIT[dim]
