// K2 permute (scatter-by-expert with capacity) and K4 combine (unpermute).
//
// Neither exists in the reference (its "forward" is the analytic charge at
// pkg/src/comoe/simulator.py:692-707); the semantics are the Switch/GShard
// ones written down in DESIGN.md: an assignment (token t, choice j) of group g
// has rank = tokens before it in stream order (all first choices in token
// order, then all second choices); it is kept iff rank < capacity and lands
// at row base[g] + rank of the compact, expert-sorted buffer.
#include <cstdlib>

#include "common.cuh"
#include "../../include/comoe_b200.h"

namespace comoe {

struct PermuteParams {
  const __nv_bfloat16* x;
  int T, d, top_k, G, capacity, ntiles;
  const int* group_idx;
  const float* gate_prob;
  const int* local_rank;
  const int* tile_offset;
  const int* group_base;
  __nv_bfloat16* x_perm;
  int* row_token;
  float* row_prob;
  int* token_pos;      // [T, k] destination row or -1
  __nv_bfloat16* y;    // optional: zero rows of fully-dropped tokens (top-1 fused combine)
  // expert parallelism over peer memory (kPeers): row r of the [dst][local
  // expert][C] send layout is written straight into rank r / block_rows's
  // receive buffer at row src_off + r % block_rows (src_off = my rank *
  // block_rows), i.e. the all-to-all is the store itself
  __nv_bfloat16* const* peer_rows;
  int block_rows, src_off;
  int rev;  // dev (COMOE_PERMUTE_REV=1): walk the tokens last-to-first
};

// Row address of destination row `dest` in the local buffer or, with peers,
// in the owning rank's receive buffer.
template <bool kPeers>
__device__ __forceinline__ int4* permute_row(const PermuteParams& p, int dest) {
  if constexpr (kPeers) {
    const int blk = dest / p.block_rows;
    return reinterpret_cast<int4*>(p.peer_rows[blk] +
                                   static_cast<long>(p.src_off + (dest - blk * p.block_rows)) * p.d);
  } else {
    return reinterpret_cast<int4*>(p.x_perm + static_cast<long>(dest) * p.d);
  }
}

constexpr int kRowUnroll = 3;  // d = 768: one slice covers the row

constexpr int kTokPerWarp = 4;

// One warp per kTokPerWarp consecutive tokens. The first slice of every row
// is loaded before the destinations are resolved (group -> tile offset ->
// base is a chain of dependent loads), so row traffic overlaps the index
// work; then each 32*kRowUnroll-vector slice is stored and the next loaded.
template <bool kPeers>
__global__ void __launch_bounds__(256, 3) permute_kernel(PermuteParams p) {
  pdl_wait();  // routing tables come from the gate / scan kernels
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int vec = p.d >> 3;  // uint4 per row
  const bool copy = kPeers || p.x_perm != nullptr;
  const int nb = (p.T + kTokPerWarp - 1) / kTokPerWarp;
  for (int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nb; b += warps) {
    const int t0 = (p.rev ? nb - 1 - b : b) * kTokPerWarp;
    int4 v[kTokPerWarp][kRowUnroll];
    auto load_slice = [&](int i0) {
#pragma unroll
      for (int u = 0; u < kTokPerWarp; ++u)
#pragma unroll
        for (int w = 0; w < kRowUnroll; ++w) {
          const int i = i0 + w * 32 + lane;
          if (copy && t0 + u < p.T && i < vec)
            v[u][w] = ld_nc_v4(reinterpret_cast<const int4*>(p.x + static_cast<long>(t0 + u) * p.d) + i);
        }
    };
    load_slice(0);
    // index chain in two independent phases over all tokens of the warp
    // (group/local rank, then tile offset/base), instead of serially per token
    int g[kTokPerWarp][2], lr[kTokPerWarp][2];
#pragma unroll
    for (int u = 0; u < kTokPerWarp; ++u)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const bool ok = t0 + u < p.T && j < p.top_k;
        const long o = static_cast<long>(t0 + u) * p.top_k + j;
        g[u][j] = ok ? __ldg(p.group_idx + o) : -1;
        lr[u][j] = ok ? __ldg(p.local_rank + o) : 0;
      }
    int dst[kTokPerWarp][2];
#pragma unroll
    for (int u = 0; u < kTokPerWarp; ++u)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int gg = g[u][j];
        int dest = -1;
        if (gg >= 0) {
          const int tile = (t0 + u) / 128;
          const int rank =
              __ldg(p.tile_offset + (static_cast<long>(j) * p.ntiles + tile) * p.G + gg) + lr[u][j];
          if (rank < p.capacity) dest = __ldg(p.group_base + gg) + rank;
        }
        dst[u][j] = dest;
      }
    if (lane < kTokPerWarp * 2) {  // one lane per (token, choice) writes the tables
      const int u = lane >> 1, j = lane & 1;
      int dest = -1, t = t0 + u;
#pragma unroll
      for (int uu = 0; uu < kTokPerWarp; ++uu)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
          if (uu == u && jj == j) dest = dst[uu][jj];
      if (t < p.T && j < p.top_k) {
        const long o = static_cast<long>(t) * p.top_k + j;
        p.token_pos[o] = dest;
        if (dest >= 0) {
          p.row_token[dest] = t;
          p.row_prob[dest] = __ldg(p.gate_prob + o);
        }
      }
    }
    // peers: destination rows resolved once per (token, choice); local rows
    // are addressed inline (holding 8 pointers costs the local kernel 20%)
    int4* rowp[kTokPerWarp][2];
    if constexpr (kPeers) {
#pragma unroll
      for (int u = 0; u < kTokPerWarp; ++u)
#pragma unroll
        for (int j = 0; j < 2; ++j)
          rowp[u][j] = dst[u][j] >= 0 ? permute_row<true>(p, dst[u][j]) : nullptr;
    }
    for (int i0 = 0; i0 < vec; i0 += 32 * kRowUnroll) {
#pragma unroll
      for (int u = 0; u < kTokPerWarp; ++u) {
        if (t0 + u >= p.T) continue;
        const bool any = dst[u][0] >= 0 || dst[u][1] >= 0;
#pragma unroll
        for (int w = 0; w < kRowUnroll; ++w) {
          const int i = i0 + w * 32 + lane;
          if (i >= vec) continue;
          if (any && copy) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              if constexpr (kPeers) {
                if (rowp[u][j]) rowp[u][j][i] = v[u][w];
              } else if (dst[u][j] >= 0) {
                permute_row<false>(p, dst[u][j])[i] = v[u][w];
              }
            }
          } else if (!any && p.y) {
            reinterpret_cast<int4*>(p.y + static_cast<long>(t0 + u) * p.d)[i] = make_int4(0, 0, 0, 0);
          }
        }
      }
      if (i0 + 32 * kRowUnroll < vec) load_slice(i0 + 32 * kRowUnroll);
    }
  }
}

// y[t] = sum_j prob_j * y_perm[pos_j]  (pos -1 contributes 0), fp32 accumulate.
// kPeers: row pos_j lives in rank pos_j / block_rows's output buffer at row
// src_off + pos_j % block_rows (peer_rows[rank]), read over peer memory.
template <bool kPeers>
__global__ void __launch_bounds__(256) combine_kernel(const __nv_bfloat16* __restrict__ y_perm,
                                                      const int* __restrict__ token_pos,
                                                      const float* __restrict__ gate_prob, int T,
                                                      int d, int top_k,
                                                      __nv_bfloat16* __restrict__ y,
                                                      const __nv_bfloat16* const* peer_rows,
                                                      int block_rows, int src_off) {
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int vec = d >> 3;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < T; t += warps) {
    int pos[2] = {-1, -1};
    float pr[2] = {0.f, 0.f};
    for (int j = 0; j < top_k; ++j) {
      pos[j] = __ldg(token_pos + static_cast<long>(t) * top_k + j);
      pr[j] = __ldg(gate_prob + static_cast<long>(t) * top_k + j);
    }
    int4* dst = reinterpret_cast<int4*>(y + static_cast<long>(t) * d);
    if constexpr (kPeers) {  // owner rank and row, once per choice
      for (int j = 0; j < top_k; ++j) {
        if (pos[j] < 0) continue;
        const int blk = pos[j] / block_rows;
        pos[j] = blk * (1 << 24) + src_off + (pos[j] - blk * block_rows);  // (rank, row) packed
      }
    }
    for (int i = lane; i < vec; i += 32) {
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int j = 0; j < top_k; ++j) {
        if (pos[j] < 0) continue;
        const __nv_bfloat16* row;
        if constexpr (kPeers)
          row = peer_rows[pos[j] >> 24] + static_cast<long>(pos[j] & 0xffffff) * d;
        else
          row = y_perm + static_cast<long>(pos[j]) * d;
        const int4 raw = ld_nc_v4(reinterpret_cast<const int4*>(row) + i);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float2 f = __bfloat1622float2(h[u]);
          acc[2 * u] = fmaf(pr[j], f.x, acc[2 * u]);
          acc[2 * u + 1] = fmaf(pr[j], f.y, acc[2 * u + 1]);
        }
      }
      int4 out;
      out.x = static_cast<int>(pack_bf16x2(acc[0], acc[1]));
      out.y = static_cast<int>(pack_bf16x2(acc[2], acc[3]));
      out.z = static_cast<int>(pack_bf16x2(acc[4], acc[5]));
      out.w = static_cast<int>(pack_bf16x2(acc[6], acc[7]));
      dst[i] = out;
    }
  }
}

static int grid_for_warps(long warps_needed) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long blocks = (warps_needed + 7) / 8;
  const long cap = static_cast<long>(sms) * 8;  // 8 x 256-thread CTAs per SM
  return static_cast<int>(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

}  // namespace comoe

extern "C" {

int comoe_permute(const void* x, int T, int d, int top_k, const int* group_idx,
                  const float* gate_prob, const int* local_rank, const int* tile_offset,
                  const int* group_base, int n_groups, int capacity, void* x_perm,
                  int* row_token, float* row_prob, int* token_pos, void* y_zero, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(x && group_idx && gate_prob && local_rank && tile_offset && group_base &&
                    row_token && row_prob && token_pos,
                kBadArg, "permute: null pointer");  // x_perm may be NULL: index-only
  COMOE_REQUIRE(top_k == 1 || top_k == 2, kUnsupportedShape, "permute: top_k=%d", top_k);
  COMOE_REQUIRE(d % 8 == 0 && d > 0, kUnsupportedShape, "permute: d=%d must be a multiple of 8", d);
  COMOE_REQUIRE(T >= 0 && n_groups >= 1, kBadArg, "permute: bad sizes");
  if (T == 0) return kOk;
  PermuteParams p{reinterpret_cast<const __nv_bfloat16*>(x), T, d, top_k, n_groups, capacity,
                  (T + 127) / 128, group_idx, gate_prob, local_rank, tile_offset, group_base,
                  reinterpret_cast<__nv_bfloat16*>(x_perm), row_token, row_prob, token_pos,
                  reinterpret_cast<__nv_bfloat16*>(y_zero), nullptr, 0, 0};
  static const int rev = [] {
    const char* e = std::getenv("COMOE_PERMUTE_REV");
    return e && e[0] == '1' ? 1 : 0;
  }();
  p.rev = rev;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid_for_warps((T + kTokPerWarp - 1) / kTokPerWarp));
  cfg.blockDim = dim3(256);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attrs[1];
  cfg.attrs = attrs;
  cfg.numAttrs = pdl_attr(&attrs[0]);
  cudaLaunchKernelEx(&cfg, permute_kernel<false>, p);
  return check_launch("permute_kernel");
}

int comoe_permute_peers(const void* x, int T, int d, int top_k, const int* group_idx,
                        const float* gate_prob, const int* local_rank, const int* tile_offset,
                        const int* group_base, int n_groups, int capacity, void* const* peer_rows,
                        int n_peers, long block_rows, int src_rank, int* row_token,
                        float* row_prob, int* token_pos, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(x && group_idx && gate_prob && local_rank && tile_offset && group_base &&
                    peer_rows && row_token && row_prob && token_pos,
                kBadArg, "permute_peers: null pointer");
  COMOE_REQUIRE(top_k == 1 || top_k == 2, kUnsupportedShape, "permute_peers: top_k=%d", top_k);
  COMOE_REQUIRE(d % 8 == 0 && d > 0, kUnsupportedShape, "permute_peers: d=%d must be a multiple of 8", d);
  COMOE_REQUIRE(T >= 0 && n_groups >= 1 && n_peers >= 1 && block_rows >= 1 && src_rank >= 0 &&
                    src_rank < n_peers && block_rows * n_peers < (1L << 24) && n_peers <= 127,
                kBadArg, "permute_peers: bad sizes");
  if (T == 0) return kOk;
  PermuteParams p{reinterpret_cast<const __nv_bfloat16*>(x), T, d, top_k, n_groups, capacity,
                  (T + 127) / 128, group_idx, gate_prob, local_rank, tile_offset, group_base,
                  nullptr, row_token, row_prob, token_pos, nullptr,
                  reinterpret_cast<__nv_bfloat16* const*>(peer_rows), static_cast<int>(block_rows),
                  src_rank * static_cast<int>(block_rows)};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid_for_warps((T + kTokPerWarp - 1) / kTokPerWarp));
  cfg.blockDim = dim3(256);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attrs[1];
  cfg.attrs = attrs;
  cfg.numAttrs = pdl_attr(&attrs[0]);
  cudaLaunchKernelEx(&cfg, permute_kernel<true>, p);
  return check_launch("permute_kernel(peers)");
}

int comoe_combine(const void* y_perm, const int* token_pos, const float* gate_prob, int T, int d,
                  int top_k, void* y, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(y_perm && token_pos && gate_prob && y, kBadArg, "combine: null pointer");
  COMOE_REQUIRE(top_k == 1 || top_k == 2, kUnsupportedShape, "combine: top_k=%d", top_k);
  COMOE_REQUIRE(d % 8 == 0 && d > 0, kUnsupportedShape, "combine: d=%d", d);
  if (T == 0) return kOk;
  combine_kernel<false><<<grid_for_warps(T), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(y_perm), token_pos, gate_prob, T, d, top_k,
      reinterpret_cast<__nv_bfloat16*>(y), nullptr, 0, 0);
  return check_launch("combine_kernel");
}

int comoe_combine_peers(const void* const* peer_rows, int n_peers, long block_rows, int src_rank,
                        const int* token_pos, const float* gate_prob, int T, int d, int top_k,
                        void* y, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(peer_rows && token_pos && gate_prob && y, kBadArg, "combine_peers: null pointer");
  COMOE_REQUIRE(top_k == 1 || top_k == 2, kUnsupportedShape, "combine_peers: top_k=%d", top_k);
  COMOE_REQUIRE(d % 8 == 0 && d > 0, kUnsupportedShape, "combine_peers: d=%d", d);
  COMOE_REQUIRE(n_peers >= 1 && block_rows >= 1 && src_rank >= 0 && src_rank < n_peers &&
                    block_rows * n_peers < (1L << 24) && n_peers <= 127,
                kBadArg, "combine_peers: bad sizes");
  if (T == 0) return kOk;
  combine_kernel<true><<<grid_for_warps(T), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      nullptr, token_pos, gate_prob, T, d, top_k, reinterpret_cast<__nv_bfloat16*>(y),
      reinterpret_cast<const __nv_bfloat16* const*>(peer_rows), static_cast<int>(block_rows),
      src_rank * static_cast<int>(block_rows));
  return check_launch("combine_kernel(peers)");
}

}  // extern "C"
