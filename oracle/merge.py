"""NumPy restatement of the CoMoE fusion math (TEST INFRASTRUCTURE ONLY).

Each function cites the reference code it restates; tests pin these against
golden vectors the reference itself produced (oracle/gen_golden.py ->
tests/golden/fusion_*.json) before they are used to check the device path.
"""

from __future__ import annotations

import math

import numpy as np

EPS_FREQ = 1e-12  # pkg/src/comoe/aggregation.py:27


def merge_params(vectors, freqs) -> np.ndarray:
    """merge_group (aggregation.py:200-215): sum_j f_j v_j / sum f, or the
    plain mean when sum f <= EPS_FREQ. Sequential row order, as numpy."""
    V = [np.asarray(v, np.float64) for v in vectors]
    w = [float(f) for f in freqs]
    total = 0.0
    for f in w:
        total += f
    if total <= EPS_FREQ:
        acc = V[0].copy()
        for v in V[1:]:
            acc = acc + v
        return acc / len(V)
    acc = w[0] * V[0]
    for f, v in zip(w[1:], V[1:]):
        acc = acc + f * v
    return acc / total


def retention_fixed(E: int, r: float) -> int:
    """fixed_retention (aggregation.py:128-131)."""
    if not (0.0 < r <= 1.0):
        raise ValueError(r)
    return max(1, int(math.floor(r * E)))


def entropy(freqs):
    """layer_entropy (aggregation.py:134-141): (H, H / log E)."""
    f = np.asarray(freqs, np.float64)
    h = 0.0
    for x in f:
        if x > 0:
            h -= x * math.log(x)
    E = len(f)
    return h, (h / math.log(E) if E > 1 else 0.0)


def retention_adaptive(E, r_base, delta_r, hbar, e_min) -> int:
    """adaptive_retention (aggregation.py:144-149)."""
    return min(E, max(e_min, int(math.floor(E * (r_base + delta_r * hbar)))))


def principals(freqs, target: int, theta_act: float = 0.0) -> list:
    """identify_principals (aggregation.py:156-169), by repeated max scan."""
    f = list(np.asarray(freqs, np.float64))
    left = list(range(len(f)))
    out = []
    for _ in range(target):
        best = left[0]
        for s in left[1:]:
            if f[s] > f[best]:
                best = s
        out.append(best)
        left.remove(best)
    chosen = set(out)
    if theta_act > 0.0:
        chosen |= {s for s in range(len(f)) if f[s] >= theta_act}
    return sorted(chosen)


def assign(sim, principal_slots, E: int) -> dict:
    """group_experts (aggregation.py:172-197): secondary -> argmax principal,
    strict '>' so exact ties keep the lowest principal."""
    out = {}
    ps = sorted(principal_slots)
    for s in range(E):
        if s in ps:
            continue
        best, best_v = None, -np.inf
        for p in ps:
            if sim[s][p] > best_v:
                best, best_v = p, sim[s][p]
        out[s] = best
    return out


def cosine_matrix(P) -> np.ndarray:
    """Cosine part of similarity_matrix (moe.py:345-349)."""
    P = np.asarray(P, np.float64)
    n = np.linalg.norm(P, axis=1)
    Q = P / n[:, None]
    return Q @ Q.T


def surrogate_logits(P, probes, proj) -> np.ndarray:
    """einsum('nd,ed,bd->enb') of moe.py:351, as a matmul over D."""
    P = np.asarray(P, np.float64)
    probes = np.asarray(probes, np.float64)
    proj = np.asarray(proj, np.float64)
    n, B = probes.shape[0], proj.shape[0]
    Q = (probes[:, None, :] * proj[None, :, :]).reshape(n * B, -1)
    return (P @ Q.T).reshape(P.shape[0], n, B)


def similarity(P, probes, proj, alpha: float) -> np.ndarray:
    """similarity_matrix (moe.py:339-365) with log-softmax distributions."""
    cos = cosine_matrix(P)
    L = surrogate_logits(P, probes, proj)
    m = L.max(axis=2, keepdims=True)
    logd = L - m - np.log(np.exp(L - m).sum(axis=2, keepdims=True))
    D = np.exp(logd)
    E, n = L.shape[0], L.shape[1]
    kl = np.zeros((E, E))
    for i in range(n):
        Di, Li = D[:, i, :], logd[:, i, :]
        self_t = (Di * Li).sum(axis=1)
        k = self_t[:, None] - Di @ Li.T
        kl += 0.5 * (k + k.T)
    kl /= n
    return alpha * cos + (1.0 - alpha) * np.clip(1.0 - kl, 0.0, 1.0)


def fuse_layer(P, freqs, target, sim, theta_act=0.0):
    """Per-layer fusion (aggregation.py:282-300): principals, assignment,
    merged vectors per principal, slot_map."""
    E = len(freqs)
    ps = principals(freqs, target, theta_act)
    a = assign(sim, ps, E)
    members = {p: [] for p in ps}
    for s in range(E):
        if s in a:
            members[a[s]].append(s)
    merged = {}
    for p in ps:
        slots = [p] + members[p]
        merged[p] = merge_params([P[s] for s in slots], [freqs[s] for s in slots])
    slot_map = {s: (s if s in members else a[s]) for s in range(E)}
    return ps, members, merged, slot_map
