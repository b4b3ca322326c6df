"""Grouped GEMM (K3, 2-SM kernel) on awkward group sizes against a torch
fp32 reference of the same op: rows that leave remainders of every kind
after 256-row tiles (1, 16, 31, 255, 257, 511, 513, 600, 639, 640), empty
groups, and long K, where the output GEMM splits each group into equal
token tiles (decode_tile2) — with the bulk-store epilogue (32-token
rounding) and the scale-and-scatter epilogue (16-token rounding), plus a
decode-sized batch that takes the 32/64-token tile configurations."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _case(rows, N, K, seed=0):
    from paper_2508_09208_b200 import ExpertPool
    g = torch.Generator(device="cuda").manual_seed(seed)
    G = len(rows)
    total = int(sum(rows))
    a = (torch.randn(max(total, 1), K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    pool = ExpertPool(G + 2, N * K, device="cuda")
    pool.data.normal_(0, 0.05, generator=g)
    slots = list(range(2, G + 2))[::-1]  # groups read non-trivial slots, reversed order
    base = np.concatenate([[0], np.cumsum(rows)[:-1]]).astype(np.int32)
    t = lambda v: torch.tensor(v, dtype=torch.int32, device="cuda")
    return a, pool, t(rows), t(base), t(slots)


def _ref(a, pool, rows, base, slots, N, K):
    out = torch.zeros(a.shape[0], N, dtype=torch.float32, device="cuda")
    for g in range(rows.numel()):
        n, b, s = int(rows[g]), int(base[g]), int(slots[g])
        if n:
            w = pool.data[s, : N * K].view(N, K).float()
            out[b:b + n] = a[b:b + n].float() @ w.t()
    return out


ROWS = [1, 16, 31, 255, 257, 0, 511, 513, 600, 639, 640, 256, 512]


@pytest.mark.parametrize("K", [768, 1536, 3072])
def test_store_epilogue_awkward_groups(K):
    from paper_2508_09208_b200 import kernels
    N = 512
    a, pool, rows, base, slots = _case(ROWS, N, K, seed=K)
    out = torch.full((a.shape[0], N), float("nan"), dtype=torch.bfloat16, device="cuda")
    kernels.grouped_gemm(a, pool.data, 0, N, rows, base, slots, kernels.EPI_STORE, out)
    torch.cuda.synchronize()
    ref = _ref(a, pool, rows, base, slots, N, K)
    torch.testing.assert_close(out.float(), ref, rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("K", [768, 3072])
def test_scatter_epilogue_awkward_groups(K):
    """EPI_SCALE_SCATTER: out[row_token[r]] = bf16(acc[r] * row_prob[r]); rows
    scattered to a permutation of the output rows."""
    from paper_2508_09208_b200 import kernels
    N = 256
    a, pool, rows, base, slots = _case(ROWS, N, K, seed=K + 1)
    R = a.shape[0]
    g = torch.Generator(device="cuda").manual_seed(7)
    row_token = torch.randperm(R, device="cuda", generator=g).to(torch.int32)
    row_prob = torch.rand(R, device="cuda", generator=g)
    out = torch.full((R, N), float("nan"), dtype=torch.bfloat16, device="cuda")
    kernels.grouped_gemm(a, pool.data, 0, N, rows, base, slots, kernels.EPI_SCALE_SCATTER, out,
                         row_token=row_token, row_prob=row_prob)
    torch.cuda.synchronize()
    ref = _ref(a, pool, rows, base, slots, N, K) * row_prob[:, None]
    want = torch.empty_like(ref)
    want[row_token.long()] = ref
    torch.testing.assert_close(out.float(), want, rtol=2e-2, atol=2e-2)


def test_decode_sized_groups_take_small_tiles():
    """<= 8 / <= 32 rows per group on average: 32- / 64-token tile configs."""
    from paper_2508_09208_b200 import kernels
    N, K = 256, 3072
    for rows_list in ([1, 3, 0, 7, 8, 2, 5, 4] * 4, [17, 30, 1, 32, 9, 25, 0, 31] * 4):
        a, pool, rows, base, slots = _case(rows_list, N, K, seed=len(rows_list))
        out = torch.full((a.shape[0], N), float("nan"), dtype=torch.bfloat16, device="cuda")
        kernels.grouped_gemm(a, pool.data, 0, N, rows, base, slots, kernels.EPI_STORE, out)
        torch.cuda.synchronize()
        ref = _ref(a, pool, rows, base, slots, N, K)
        torch.testing.assert_close(out.float(), ref, rtol=2e-2, atol=2e-2)
