"""Device merge (K5), similarity (K6) and predictor (K8) against the oracle
and against reference-generated golden vectors."""

import hashlib
import json

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import merge as M

pytestmark = pytest.mark.gpu


def _experts(P, dtype=torch.float64):
    from paper_2508_09208_b200.moe import Expert
    return [Expert(1, s, torch.as_tensor(np.asarray(p), dtype=dtype, device="cuda"), 1.0)
            for s, p in enumerate(P)]


def _stats(counts):
    from paper_2508_09208_b200.moe import ActivationStats
    c = np.asarray(counts, float)
    return ActivationStats(counts={1: c}, totals={1: max(int(c.sum()), 1)}, experts_per_layer=len(c))


def test_merge_hand_cases():
    from paper_2508_09208_b200.aggregation import ExpertGroup, merge_group
    for case in json.loads((GOLDEN / "merge_hand.json").read_text()):
        ex = _experts(case["vectors"])
        f = np.asarray(case["freqs"])
        counts = f * 4 if f.sum() > 0 else f
        st = _stats(counts)
        if f.sum() == 0:
            st.totals[1] = 10
        m = merge_group(ExpertGroup(0, (1,)), {0: ex[0], 1: ex[1]}, st, 1)
        np.testing.assert_array_equal(m.params.cpu().numpy(), np.asarray(case["expected"]))


def test_merge_f64_bit_exact_vs_reference_checksums():
    from paper_2508_09208_b200 import kernels
    for case in json.loads((GOLDEN / "merge_bigsum.json").read_text()):
        rng = np.random.default_rng(case["seed"])
        V = rng.normal(size=(case["n"], case["D"])) * 0.02
        f = np.asarray(case["counts"])
        Vd = torch.as_tensor(V, device="cuda")
        out = torch.empty(case["D"], dtype=torch.float64, device="cuda")
        freqs = f / max(int(f.sum()), 1)   # stats.freqs: counts / totals
        if freqs.sum() > 1e-12:
            w, div = list(freqs), float(freqs.sum())
        else:
            w, div = [1.0] * case["n"], float(case["n"])
        kernels.merge_groups([[Vd[i] for i in range(case["n"])]], [w], [div], [out], torch.float64)
        got = out.cpu().numpy()
        assert hashlib.sha256(got.tobytes()).hexdigest() == case["sha256"]


def test_merge_bf16_tolerance_sb8_shape():
    """Switch expert size (D = 4,718,592), groups of 2/4/8 members: every
    element within 1 bf16 ulp of bf16(fp64 merge) + 2^-24 max|input|."""
    from paper_2508_09208_b200 import kernels
    from oracle.switch_layer import bf16_round
    D = 4_718_592
    g = torch.Generator(device="cuda").manual_seed(2)
    V = (torch.randn(8, D, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    for n in (2, 4, 8):
        f = np.arange(1, n + 1, dtype=float)
        out = torch.empty(D, dtype=torch.bfloat16, device="cuda")
        kernels.merge_groups([[V[i] for i in range(n)]], [list(f)], [float(f.sum())], [out],
                             torch.bfloat16)
        Vh = V[:n].double().cpu().numpy()
        ref = M.merge_params(list(Vh), f)
        refb = bf16_round(ref.astype(np.float32)).astype(np.float64)
        got = out.double().cpu().numpy()
        ulp = np.abs(refb) * 2.0 ** -7
        bound = ulp + 2.0 ** -24 * np.abs(Vh).max()
        assert np.all(np.abs(got - refb) <= bound + 1e-30)


def test_fusion_pipeline_matches_reference_golden():
    """fuse_model on the device reproduces the reference's decisions
    (principals, groups, slot_map) and merged params to rel 1e-9, with the
    reference's own similarity matrix checked to 1e-9 as well."""
    from paper_2508_09208_b200 import aggregation as A
    from paper_2508_09208_b200.moe import Calibration, MoeModel, MoeModelSpec, similarity_matrix
    for case in json.loads((GOLDEN / "fusion_cases.json").read_text()):
        E = case["E"]
        P = np.asarray(case["params"])
        ex = _experts(P)
        calib = Calibration(np.asarray(case["probes"]), np.asarray(case["projection"]))
        S = similarity_matrix(ex, case["alpha"], calib)
        np.testing.assert_allclose(S, np.asarray(case["sim"]), rtol=1e-9, atol=1e-9)
        spec = MoeModelSpec(2, (1,), (), E, 1e6, 1, case["dim"])
        model = MoeModel(spec, {(1, e.slot): e for e in ex})
        st = _stats(case["counts"])
        cfg = A.FusionConfig(mode="fixed", r=case["r"], theta_act=case["theta_act"])
        var = A.fuse_model(model, st, cfg, case["alpha"], calib)
        assert {str(k): v for k, v in var.slot_map[1].items()} == case["slot_map"]
        assert sorted(var.retained[1]) == case["principals"]
        for p, ref in case["merged"].items():
            np.testing.assert_allclose(var.retained[1][int(p)].params.cpu().numpy(),
                                       np.asarray(ref), rtol=1e-9, atol=1e-12)
        assert var.perf_estimate == pytest.approx(case["perf_estimate"], rel=1e-9)


def test_similarity_bf16_switch_scale():
    """K6 on bf16 Switch-size experts (E=8, D=4.7M) vs fp64 oracle of the
    same bf16 values (sigma 0.02 keeps the reference surrogate finite)."""
    from paper_2508_09208_b200.moe import Expert, make_calibration, similarity_matrix
    D, E = 4_718_592, 8
    g = torch.Generator(device="cuda").manual_seed(5)
    V = (torch.randn(E, D, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    calib = make_calibration(D, n_probes=8, seed=7, buckets=8)
    S = similarity_matrix([Expert(1, s, V[s], 1.0) for s in range(E)], 0.5, calib)
    ref = M.similarity(V.double().cpu().numpy(), calib.probes, calib.projection, 0.5)
    np.testing.assert_allclose(S, ref, rtol=1e-7, atol=1e-7)


def test_predictor_matches_numpy():
    from paper_2508_09208_b200 import kernels
    rng = np.random.default_rng(0)
    E, emb, ctx, H, B, K = 128, 16, 8, 32, 1000, 1
    w1 = rng.normal(scale=0.1, size=(H, E + emb + ctx)); b1 = rng.normal(size=H) * 0.1
    w2 = rng.normal(scale=0.1, size=(E, H)); b2 = rng.normal(size=E) * 0.1
    slots = rng.integers(0, E, size=(B, K)).astype(np.int32)
    he = rng.normal(size=(B, emb)); ce = rng.normal(size=(B, ctx))
    X = np.zeros((B, E + emb + ctx))
    X[np.arange(B), slots[:, 0]] = 1.0
    X[:, E:E + emb] = he
    X[:, E + emb:] = ce
    z = np.maximum(X @ w1.T + b1, 0) @ w2.T + b2
    z -= z.max(1, keepdims=True)
    ref = np.exp(z) / np.exp(z).sum(1, keepdims=True)
    d = lambda a: torch.as_tensor(a, device="cuda")
    probs, demand = kernels.predictor_mlp(d(slots), d(he), d(ce), d(w1), d(b1), d(w2), d(b2),
                                          want_demand=True)
    np.testing.assert_allclose(probs.cpu().numpy(), ref, rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(demand.cpu().numpy(), ref.sum(0), rtol=1e-10)


@pytest.mark.parametrize("E", [3, 8, 13, 40, 128])
def test_similarity_cosine_tensor_core_paths(E):
    """bf16 cosine-only Gram (K6 tensor-core path: 8x8 tile for E <= 8,
    upper-triangle 32x32 tiles with mirroring above) vs fp64 of the same
    bf16 values, at a D that is not a multiple of the 32-d chunk."""
    from paper_2508_09208_b200 import kernels
    D = 100_000 + 8 * 3
    g = torch.Generator(device="cuda").manual_seed(E)
    base = torch.randn(4, D, device="cuda", generator=g) * 0.02
    V = (torch.randn(E, D, device="cuda", generator=g) * 0.02 + base[torch.arange(E) % 4])
    V = V.to(torch.bfloat16)
    sim, gram, _ = kernels.similarity([V[e] for e in range(E)], None, None, 1.0)
    ref = M.cosine_matrix(V.double().cpu().numpy())
    np.testing.assert_allclose(sim.cpu().numpy(), ref, rtol=1e-7, atol=1e-7)
    Vh = V.double().cpu().numpy()
    G = Vh @ Vh.T  # fp32 partial sums: absolute error ~1e-10 of the Gram scale
    np.testing.assert_allclose(gram.cpu().numpy(), G, rtol=1e-6, atol=1e-9 * np.abs(G).max())


@pytest.mark.parametrize("E", [2, 20])
def test_similarity_f64_and_probe_paths(E):
    """fp64 parameters (SIMT register path for E <= 8, tiled path above) and
    the calibration-probe surrogate (tiled fp64 path) vs the NumPy oracle."""
    from paper_2508_09208_b200 import kernels
    rng = np.random.default_rng(E)
    D, n, B = 5_000, 3, 4
    P = rng.normal(size=(E, D)) * 0.05
    probes = rng.normal(size=(n, D))
    proj = rng.normal(size=(B, D))
    Pd = torch.as_tensor(P, device="cuda")
    sim, _, _ = kernels.similarity([Pd[e] for e in range(E)], None, None, 1.0)
    np.testing.assert_allclose(sim.cpu().numpy(), M.cosine_matrix(P), rtol=1e-9, atol=1e-12)
    sim, _, _ = kernels.similarity([Pd[e] for e in range(E)], torch.as_tensor(probes, device="cuda"),
                                   torch.as_tensor(proj, device="cuda"), 0.5)
    np.testing.assert_allclose(sim.cpu().numpy(), M.similarity(P, probes, proj, 0.5), rtol=1e-9,
                               atol=1e-9)


def test_merge_many_groups_unstaged_path():
    """More groups than the shared-memory group table holds (1024): the
    kernel falls back to global group/weight lookups; results unchanged."""
    from paper_2508_09208_b200 import kernels
    G, D = 1100, 4096
    g = torch.Generator(device="cuda").manual_seed(3)
    V = (torch.randn(G + 1, D, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    outs = [torch.empty(D, dtype=torch.bfloat16, device="cuda") for _ in range(G)]
    members = [[V[i], V[i + 1]] for i in range(G)]
    w = [[1.0 + (i % 3), 2.0] for i in range(G)]
    kernels.merge_groups(members, w, [sum(x) for x in w], outs, torch.bfloat16)
    Vf = V.float()
    for i in (0, 517, G - 1):
        ref = (w[i][0] * Vf[i] + w[i][1] * Vf[i + 1]) / sum(w[i])
        torch.testing.assert_close(outs[i].float(), ref, rtol=1e-2, atol=1e-4)


@pytest.mark.parametrize("E,K,H,emb", [(20, 1, 32, 16), (64, 2, 32, 16), (200, 2, 32, 16),
                                        (64, 2, 40, 48)])
def test_predictor_expert_counts(E, K, H, emb):
    """Every experts-per-lane instantiation, duplicate K-hot slots, a ragged
    last token chunk, a hidden width that is not a multiple of 32 and more
    than 32 dense inputs."""
    from paper_2508_09208_b200 import kernels
    rng = np.random.default_rng(E + H)
    ctx, B = 8, 777
    w1 = rng.normal(scale=0.1, size=(H, E + emb + ctx)); b1 = rng.normal(size=H) * 0.1
    w2 = rng.normal(scale=0.1, size=(E, H)); b2 = rng.normal(size=E) * 0.1
    slots = rng.integers(0, E, size=(B, K)).astype(np.int32)
    slots[::7, -1] = slots[::7, 0]  # duplicates count once
    he = rng.normal(size=(B, emb)); ce = rng.normal(size=(B, ctx))
    X = np.zeros((B, E + emb + ctx))
    for k in range(K):
        X[np.arange(B), slots[:, k]] = 1.0
    X[:, E:E + emb] = he
    X[:, E + emb:] = ce
    z = np.maximum(X @ w1.T + b1, 0) @ w2.T + b2
    z -= z.max(1, keepdims=True)
    ref = np.exp(z) / np.exp(z).sum(1, keepdims=True)
    d = lambda a: torch.as_tensor(a, device="cuda")
    probs, demand = kernels.predictor_mlp(d(slots), d(he), d(ce), d(w1), d(b1), d(w2), d(b2),
                                          want_demand=True)
    np.testing.assert_allclose(probs.cpu().numpy(), ref, rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(demand.cpu().numpy(), ref.sum(0), rtol=1e-10)


def test_predictor_any_demand_mode():
    """demand_mode "any": 1 - prod_t (1 - p_t) per expert (the stack's
    batched prefetch probability), across several 256-token chunks."""
    from paper_2508_09208_b200 import kernels
    rng = np.random.default_rng(3)
    E, emb, ctx, H, B = 64, 16, 8, 32, 700
    w1 = rng.normal(scale=0.3, size=(H, E + emb + ctx)); b1 = rng.normal(size=H) * 0.1
    w2 = rng.normal(scale=0.8, size=(E, H)); b2 = rng.normal(size=E) * 0.1
    slots = rng.integers(0, E, size=(B, 1)).astype(np.int32)
    he = rng.normal(size=(B, emb)); ce = rng.normal(size=(B, ctx))
    d = lambda a: torch.as_tensor(a, device="cuda")
    probs, demand = kernels.predictor_mlp(d(slots), d(he), d(ce), d(w1), d(b1), d(w2), d(b2),
                                          want_demand=True, demand_mode="any")
    p = probs.cpu().numpy()
    ref = -np.expm1(np.log1p(-p).sum(0))
    np.testing.assert_allclose(demand.cpu().numpy(), ref, rtol=1e-10, atol=1e-14)


@pytest.mark.parametrize("E,D", [(9, 5 * 64 + 8), (128, 2048 + 8), (2, 2040), (1, 16), (8, 3 * 2048 + 24),
                                 (40, 64)])
def test_similarity_cosine_edge_shapes(E, D):
    """Gram paths at their edges: the tcgen05 path's smallest / largest E and
    a ragged last 64-d block, the streaming <= 8 path with a D shorter than
    one 2048-d chunk and with a ragged last chunk, a single expert, and the
    non-consecutive-row fallback (rows gathered out of order)."""
    from paper_2508_09208_b200 import kernels
    g = torch.Generator(device="cuda").manual_seed(100 + E)
    V = (torch.randn(E, D, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    Vh = V.double().cpu().numpy()
    G = Vh @ Vh.T
    for order in (list(range(E)), list(reversed(range(E)))):
        sim, gram, _ = kernels.similarity([V[e] for e in order], None, None, 1.0)
        Go = G[np.ix_(order, order)]
        # fp32 sums of <= 64 exact products per block: ~1 fp32 ulp of a block
        # partial per block, which at short D is ~1e-8 of the Gram scale
        np.testing.assert_allclose(gram.cpu().numpy(), Go, rtol=1e-6, atol=3e-8 * np.abs(G).max())
        np.testing.assert_allclose(sim.cpu().numpy(), M.cosine_matrix(Vh[order]), rtol=1e-7,
                                   atol=1e-7)


@pytest.mark.parametrize("E,n,B,D", [(8, 8, 8, 4096 + 8), (5, 3, 6, 1000), (2, 8, 1, 256 * 7)])
def test_surrogate_logits_bf16_paths(E, n, B, D):
    """Surrogate logits of bf16 experts (fp64 tensor-core path, and the
    vector path under COMOE_SIM_DMMA=0 in CI runs that set it) vs an fp64
    einsum of the same values: ragged chunks, fewer experts / probes /
    buckets than the 8x8x8 tile."""
    from paper_2508_09208_b200 import kernels
    g = torch.Generator(device="cuda").manual_seed(E * 100 + n * 10 + B)
    V = (torch.randn(E, D, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    probes = torch.randn(n, D, device="cuda", generator=g, dtype=torch.float64)
    proj = torch.randn(B, D, device="cuda", generator=g, dtype=torch.float64)
    _, _, logits = kernels.similarity([V[e] for e in range(E)], probes, proj, 0.5)
    P = V.double().cpu().numpy()
    ref = np.einsum("ed,nd,bd->enb", P, probes.cpu().numpy(), proj.cpu().numpy())
    np.testing.assert_allclose(logits.cpu().numpy(), ref, rtol=1e-10, atol=1e-12 * np.abs(ref).max())
