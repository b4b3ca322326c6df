"""Drop-in conformance: the UNMODIFIED reference package (installed offline
into baseline/_ref) runs its own fusion pipeline with this package's device
implementations patched in where INTEGRATION.md says a maintainer would
patch them — comoe.aggregation.merge_group (K5) and comoe.moe.
similarity_matrix (K6), the names fuse_model resolves at call time
(pkg/src/comoe/aggregation.py:263,290,297). The patched run must build the
same variants as the unpatched reference: principals, slot maps, groups,
byte accounting, perf estimate (rel 1e-9) and merged parameters (fp64,
bit-identical). The cases follow the reference's acceptance criterion 06
(pkg/tests/test_acceptance.py:169-221: E = 2..8, the r / theta_act grids),
built through the reference's public API. Skipped when baseline/_ref is
absent."""

import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
R_GRID = (0.25, 0.5, 0.75, 1.0)
THETA_GRID = (0.0, 0.1, 0.3)


@pytest.fixture(scope="module")
def ref():
    if not (REF / "comoe").is_dir():
        pytest.skip("baseline/_ref (the offline reference install) is absent")
    sys.path.insert(0, str(REF))
    try:
        import comoe.aggregation as agg
        import comoe.moe as moe
    finally:
        sys.path.remove(str(REF))
    return agg, moe


def _case(moe, seed, E, D=3072):
    rng = np.random.default_rng(1000 + seed)
    spec = moe.MoeModelSpec(total_layers=1, encoder_moe_layers=(1,), decoder_moe_layers=(),
                            experts_per_layer=E, expert_size_bytes=float(D * 8), top_k=1,
                            expert_param_dim=D)
    base = rng.normal(size=D)
    experts = {(1, s): moe.Expert(1, s, base * rng.uniform(0.2, 1.0) + rng.normal(size=D),
                                  float(D * 8)) for s in range(E)}
    counts = rng.integers(1, 400, size=E).astype(float)
    if seed % 5 == 0:
        counts[rng.integers(0, E)] = 0.0   # an idle expert (theta_act path)
    stats = moe.ActivationStats(counts={1: counts}, totals={1: int(counts.sum())},
                                experts_per_layer=E)
    return moe.MoeModel(spec, experts), stats, moe.make_calibration(D)


def _same_variant(a, b):
    assert a.variant_id == b.variant_id
    assert sorted(a.retained[1]) == sorted(b.retained[1])
    assert a.slot_map == b.slot_map
    assert [(g.principal_slot, g.member_slots) for g in a.groups[1]] == \
        [(g.principal_slot, g.member_slots) for g in b.groups[1]]
    assert a.expert_bytes == b.expert_bytes and a.mem_required == b.mem_required
    assert a.perf_estimate == pytest.approx(b.perf_estimate, rel=1e-9)
    for p, e in a.retained[1].items():
        got = b.retained[1][p].params
        got = got.cpu().numpy() if hasattr(got, "cpu") else np.asarray(got)
        assert np.array_equal(np.asarray(e.params), got), f"merged params of group {p}"


def test_reference_fuse_model_with_device_kernels_patched_in(ref, monkeypatch):
    agg, moe = ref
    from paper_2508_09208_b200 import aggregation as dev_agg, moe as dev_moe
    cases = []
    for seed in range(42):
        E = 2 + seed % 7
        model, stats, calib = _case(moe, seed, E)
        cfg = agg.FusionConfig(mode="fixed", r=R_GRID[seed % len(R_GRID)],
                               theta_act=THETA_GRID[seed % len(THETA_GRID)])
        cases.append((model, stats, calib, cfg))
    want = [agg.fuse_model(m, s, c, alpha_sim=0.5, calib=k) for m, s, k, c in cases]
    monkeypatch.setattr(agg, "merge_group", dev_agg.merge_group)
    monkeypatch.setattr(moe, "similarity_matrix", dev_moe.similarity_matrix)
    got = [agg.fuse_model(m, s, c, alpha_sim=0.5, calib=k) for m, s, k, c in cases]
    merged_groups = 0
    for a, b in zip(want, got):
        _same_variant(a, b)
        merged_groups += sum(1 for g in a.groups[1] if g.member_slots)
    assert merged_groups > 20   # real merges, not only singletons


def test_reference_build_library_with_device_kernels_patched_in(ref, monkeypatch):
    """build_library (aggregation.py:319-324) over a retention sweep, then the
    reference's own select_variant on the patched library."""
    agg, moe = ref
    from paper_2508_09208_b200 import aggregation as dev_agg, moe as dev_moe
    model, stats, calib = _case(moe, 7, 8)
    cfgs = [agg.FusionConfig(mode="fixed", r=r, theta_act=0.0) for r in (0.25, 0.5, 0.75)]
    want = agg.build_library(model, stats, cfgs, 0.5, calib)
    monkeypatch.setattr(agg, "merge_group", dev_agg.merge_group)
    monkeypatch.setattr(moe, "similarity_matrix", dev_moe.similarity_matrix)
    got = agg.build_library(model, stats, cfgs, 0.5, calib)
    assert [v.variant_id for v in want.variants] == [v.variant_id for v in got.variants]
    for a, b in zip(want.variants[1:], got.variants[1:]):
        _same_variant(a, b)
