"""Naive restatement of the expert-cache policy (TEST INFRASTRUCTURE ONLY).

Mirrors pkg/src/comoe/offload.py decision functions with plain loops and
exhaustive search; tests pin these against reference-generated golden
decisions (tests/golden/policy_*.json) and then use them to check the
package's host policy (paper_2508_09208_b200/offload.py).
"""

from __future__ import annotations

SCORE_FLOOR = 1e-6  # offload.py:26


def threshold(mode, theta_base, delta_pref, gamma_cachethr, conservative, s_b, m_avail, m_total):
    """prefetch_threshold (offload.py:344-367)."""
    if m_total <= 0:
        raise ValueError("mem_total_gpu must be positive")
    frac = m_avail / m_total
    if mode == "constant":
        th = theta_base
    elif mode == "storage-fraction":
        th = gamma_cachethr * frac
    elif conservative:
        th = theta_base * (1.0 + delta_pref * frac) / max(s_b, 1e-3)
    else:
        th = theta_base * s_b * (1.0 + delta_pref * frac)
    return min(1.0, max(0.0, th))


def score(p_next, f_recent, importance, delta, lam):
    """eviction_score (offload.py:397-403)."""
    f = f_recent if f_recent > SCORE_FLOOR else SCORE_FLOOR
    imp = importance if importance > SCORE_FLOOR else SCORE_FLOOR
    return (1 - delta) * (1 - p_next) + delta * (lam / f + (1 - lam) / imp)


def victims(cache_sizes: dict, pinned: set, capacity: float, bytes_needed: float, scores: dict):
    """evict (offload.py:406-427) by exhaustive prefix search; None when no
    prefix frees enough (the reference raises InfeasibleError)."""
    if bytes_needed > capacity:
        return None
    free = capacity - sum(cache_sizes.values())
    if free >= bytes_needed:
        return []
    cands = sorted((e for e in cache_sizes if e not in pinned),
                   key=lambda e: (-scores.get(e, 0.0), e))
    for k in range(1, len(cands) + 1):
        if free + sum(cache_sizes[e] for e in cands[:k]) >= bytes_needed:
            return list(cands[:k])
    return None


def prefetch_choice(probs, theta, layer, resident: set, sizes, budget, exclude=()):
    """decide_prefetch (offload.py:370-394): p > theta strictly, by (-p, slot),
    skipping resident/excluded, greedy under the byte budget."""
    order = sorted(range(len(probs)), key=lambda s: (-probs[s], s))
    out, spent = [], 0.0
    for s in order:
        if not probs[s] > theta:
            break
        e = (layer, s)
        if e in resident or e in exclude:
            continue
        sz = sizes[e]
        if spent + sz > budget:
            continue
        spent += sz
        out.append(e)
    return out
