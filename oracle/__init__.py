"""CPU oracle for the CoMoE MoE-layer hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import anything here, and only as the checker or
the timed CPU baseline, never as the product path. The product package
(paper_2508_09208_b200) never imports this module; it has no CPU fallback.

Modules
  switch_layer  NumPy restatement of gate -> top-k -> slot remap -> capacity
                -> permutation -> expert FFN -> combine (the reference has no
                tensor forward; semantics are written down in DESIGN.md
                "Semantic ledger": PARITY UNPINNED by reference tests, pinned
                instead by hand-computed cases in tests/golden/).
  merge         NumPy restatement of the reference fusion math
                (pkg/src/comoe/aggregation.py:128-316, moe.py:286-365),
                pinned against golden vectors produced by the reference
                itself (oracle/gen_golden.py -> tests/golden/).
  policy        Naive restatements of the expert-cache policy
                (pkg/src/comoe/offload.py:34-546), pinned the same way.
"""
