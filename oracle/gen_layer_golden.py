"""Golden MoE-layer fixtures from HuggingFace transformers (TEST INFRASTRUCTURE).

The reference (pkg/src/comoe) has no router, capacity, permutation, expert
FFN or combine, so oracle/switch_layer.py restates the
published Switch / Mixtral layer semantics. This script pins that
restatement to an independent implementation of the same layers, the
`transformers` package (5.5.0 in this image; third-party, absent from
/root/reference):

  * Switch-Transformer layer: `SwitchTransformersTop1Router` (fp32 router,
    softmax, top-1, gate value = the picked probability) and
    `SwitchTransformersExperts` / `SwitchTransformersDenseActDense` (ReLU
    FFN per expert, weighted by the gate value, dropped tokens -> 0), in
    eval mode with no jitter, one sequence of T tokens, expert_capacity =
    ceil(cf * T / E).
    Caveat, transformers 5.5.0: Top1Router takes `torch.max(..., keepdim=True)`
    before `one_hot`, so its `cumsum(dim=-2)` runs over a singleton axis and
    the capacity mask never fires. The published token-priority rule (Switch
    paper; transformers 4.x Top1Router: cumsum of the one-hot choices over
    the sequence axis, keep priority <= capacity) is therefore applied here
    to the router's own argmax before `SwitchTransformersExperts` runs.
    HF picks the argmax of the probabilities, the oracle of the logits; the
    inputs are drawn so no two logits of a token are within 1e-3 (no ties
    for either rule).
  * Mixtral layer: `MixtralSparseMoeBlock` (softmax over all E, top-2,
    renormalised, SiLU-gated experts with gate_up_proj = [W1; W3] and
    down_proj = W2), no capacity. The oracle's slot layout interleaves gate
    and up rows in 128-row blocks; the test maps one onto the other.

Run in the build container:  python oracle/gen_layer_golden.py
Writes tests/golden/layer_switch.npz and tests/golden/layer_mixtral.npz.
Inputs are not stored: they come from oracle.switch_layer.det_uniform (a
counter-based splitmix64 stream, bit-identical on any numpy), rounded to
bf16 (x, expert weights) or kept fp32 (router), so the fixtures hold only the
seeds, the shapes and the HF outputs (fp32 y).
"""

from __future__ import annotations

import math
from pathlib import Path

import numpy as np
import torch

import sys
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle.switch_layer import det_uniform  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
SWIGLU_BLOCK = 128


def _bf16(a: torch.Tensor) -> torch.Tensor:
    return a.to(torch.bfloat16)


def _u(shape, seed, scale):
    return torch.from_numpy(det_uniform(shape, seed, scale))


def _separated(logits: torch.Tensor, gap: float = 1e-3) -> bool:
    top = torch.topk(logits, 3, dim=-1).values
    return bool(((top[:, 0] - top[:, 1]) > gap).all() and ((top[:, 1] - top[:, 2]) > gap).all())


def switch_case(seed: int, T: int, d: int, d_ff: int, E: int, cf: float):
    from transformers import SwitchTransformersConfig
    from transformers.models.switch_transformers import modeling_switch_transformers as m
    cap = int(math.ceil(cf * T / E))
    cfg = SwitchTransformersConfig(d_model=d, d_ff=d_ff, num_experts=E, expert_capacity=cap,
                                   router_jitter_noise=0.0, router_dtype="float32",
                                   dense_act_fn="relu", dropout_rate=0.0, router_bias=False)
    for s in range(seed, seed + 200):
        x = _bf16(_u((T, d), s, 1.0)).double()
        wg = _u((d, E), s + 10_000, 1.0 / math.sqrt(d)).float()  # router weight, fp32
        if _separated(x.float() @ wg):
            break
    else:
        raise RuntimeError("no tie-free draw")
    router = m.SwitchTransformersTop1Router(cfg).eval()
    with torch.no_grad():
        router.classifier.weight.copy_(wg.t())
        probs_max, _, _ = router(x.float()[None])             # [1, T, 1] picked probability
        logits = router.classifier(x.float()[None])[0]        # fp32 router logits
        probs = torch.softmax(logits, dim=-1)
        idx = probs.argmax(dim=-1)                            # HF: argmax of the probabilities
        onehot = torch.nn.functional.one_hot(idx, E)
        kept = ((torch.cumsum(onehot, dim=0) * onehot).sum(-1) <= cap)  # token priority
        sel = (onehot * kept[:, None]).to(torch.int64)[:, None, :]      # [T, 1, E]
        experts = m.SwitchTransformersExperts(cfg).double().eval()
        w_in = _bf16(_u((E, d_ff, d), s + 20_000, 0.05)).double()
        w_out = _bf16(_u((E, d, d_ff), s + 30_000, 0.05)).double()
        for e in range(E):
            experts[f"expert_{e}"].wi.weight.copy_(w_in[e])
            experts[f"expert_{e}"].wo.weight.copy_(w_out[e])
        y = experts(x, sel, probs_max[0].double())
    return dict(kind="switch", seed=s, T=T, d=d, d_ff=d_ff, E=E, capacity_factor=cf,
                capacity=cap, hf_expert_idx=idx.numpy().astype(np.int16),
                hf_prob=probs_max[0, :, 0].numpy().astype(np.float32), hf_kept=kept.numpy(),
                hf_y=y.numpy().astype(np.float32))


def mixtral_case(seed: int, T: int, d: int, d_ff: int, E: int):
    from transformers import MixtralConfig
    from transformers.models.mixtral import modeling_mixtral as mx
    cfg = MixtralConfig(hidden_size=d, intermediate_size=d_ff, num_local_experts=E,
                        num_experts_per_tok=2, router_jitter_noise=0.0, hidden_act="silu")
    for s in range(seed, seed + 200):
        x = _bf16(_u((T, d), s, 1.0)).double()
        wg = _u((d, E), s + 10_000, 1.0 / math.sqrt(d)).float()
        if _separated(x.float() @ wg):
            break
    else:
        raise RuntimeError("no tie-free draw")
    block = mx.MixtralSparseMoeBlock(cfg).double().eval()
    gate_up = _bf16(_u((E, 2 * d_ff, d), s + 20_000, 0.05)).double()  # [W1; W3]
    down = _bf16(_u((E, d, d_ff), s + 30_000, 0.05)).double()          # W2
    with torch.no_grad():
        block.gate.weight.copy_(wg.t().double())
        block.experts.gate_up_proj.copy_(gate_up)
        block.experts.down_proj.copy_(down)
        _, weights, index = block.gate(x)
        y = block(x[None])[0]
    return dict(kind="mixtral", seed=s, T=T, d=d, d_ff=d_ff, E=E,
                hf_topk_index=index.numpy().astype(np.int16),
                hf_topk_weight=weights.numpy().astype(np.float32),
                hf_y=y.numpy().astype(np.float32))


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    sw = [switch_case(101, 512, 256, 256, 8, 1.0), switch_case(102, 256, 256, 512, 16, 1.25),
          switch_case(103, 384, 256, 256, 8, 2.0)]
    mixtral = [mixtral_case(201, 256, 256, 256, 4), mixtral_case(202, 128, 256, 512, 8)]
    for name, cases in (("layer_switch.npz", sw), ("layer_mixtral.npz", mixtral)):
        flat = {f"c{i}_{k}": np.asarray(v) for i, c in enumerate(cases) for k, v in c.items()}
        flat["n_cases"] = np.asarray(len(cases))
        np.savez_compressed(OUT / name, **flat)
        print(f"wrote {OUT / name}: {len(cases)} cases, "
              f"{(OUT / name).stat().st_size / 1e6:.2f} MB")
    for c in sw:
        print(f"switch T={c['T']} E={c['E']} cf={c['capacity_factor']}: C={c['capacity']}, "
              f"dropped {int((~c['hf_kept']).sum())} of {c['T']}")


if __name__ == "__main__":
    main()
