// K3F: fused expert FFN on CTA pairs — GEMM1 -> ReLU -> GEMM2 with the
// intermediate H kept on chip (TMEM -> registers -> shared memory), never
// written to HBM. Replaces the analytic expert charge of the reference
// simulator (pkg/src/comoe/simulator.py:705, expert_flops at
// pkg/src/comoe/scenario.py:471) with relu(X_e Wi_e^T) Wo_e^T per expert.
//
// One tile = up to 128 routed tokens of one expert group on one CTA pair
// (tcgen05 cta_group::2, M = 256). Swap-AB throughout: weights are the A
// operand, tokens the B operand (N = tokens, any multiple of 16).
//   GEMM1, per d_ff chunk c of 256 rows: H^T[256, N] = Wi[c] . X^T
//          -> TMEM columns [384, 512) (each SM: 128 d_ff rows x N tokens)
//   GEMM2: Y^T[d, N] += Wo[:, c] . H[c]^T
//          -> TMEM columns [0, 128*d/256) (3 M-tiles of 256 features at d=768)
// TMEM per SM: Y 3 x 128 + H 128 = 512 columns, which caps N at 128 tokens.
//
// The H hand-off: each SM holds 128 d_ff rows of H for all N tokens, but the
// GEMM2 B operand of CTA r must hold tokens [r*N/2, (r+1)*N/2) for all 256
// rows of the chunk. The H warps therefore write bf16 H in the MN-major
// 128B-swizzled layout (8 k-rows x 64 tokens per 1 KB atom; thread = d_ff
// row, 16-byte vectors of 8 consecutive tokens: no transpose) — their own
// token half into their CTA's buffer and the other half into the peer CTA's
// buffer over DSMEM (st.shared::cluster). MN-major SW128 descriptor: SBO =
// K-atom stride (pinned by scripts/mn_major_probe.cu).
//
// MMA issue order per tile: G1(0), G1(1), G2(0), G1(2), G2(1), ... G2(nc-1):
// GEMM1 of chunk c+1 runs on the tensor pipe while the H warps turn chunk c
// into shared memory, and GEMM2 of chunk c runs while they drain chunk c+1.
// Warp roles (384 threads): w0 weight TMA producer, w1 MMA issuer (leader
// CTA, one thread), w2 TMEM allocator, w3 token TMA producer (tile or
// gather4), w4-7 H epilogue, w8-11 output epilogue (scale by the gate
// probability and scatter to the token's row: the fused top-1 combine).
#pragma once

#include "grouped_gemm_2sm.cuh"

namespace comoe {

constexpr int kFTok = 128;        // tokens per tile (CTA pair)
constexpr int kFChunk = 256;      // d_ff rows per chunk
constexpr int kFMaxGroups = 256;
constexpr int kFMaxD = 768;
constexpr int kFThreads = 384;
constexpr int kFStageBytes = 128 * 64 * 2;      // 128 weight rows x 64 K per SM
constexpr int kFXBlockBytes = (kFTok / 2) * 128;  // 64 token rows x 64 K per SM
constexpr int kFHBytes = (kFChunk / 8) * 1024;    // 32 K-atoms of (8 rows x 64 tokens)
constexpr uint32_t kFColH = 384;                  // TMEM column of the H accumulator

struct FusedFfnParams {
  const int* group_rows;      // [G] kept rows per group
  const int* group_row_base;  // [G] first row of the group in the permuted order
  const int* group_slot;      // [G] expert slot in the pool
  int G, d, d_ff;
  __nv_bfloat16* out;
  int ldo;
  const int* row_token;   // non-null: out row = row_token[row], scaled by row_prob[row]
  const float* row_prob;  // (top-1 fused combine); null: out row = permuted row
  const int* gather_rows; // non-null: token row r of the permuted order is x[gather_rows[r]]
  int debug;              // dev attribution switches (COMOE_FUSED_DEBUG), 0 in production:
                          // 1 = every tile reads slot 0 (L2-resident weights), 2 = no weight
                          // TMA (MMA on stale smem), 4 = H warps skip TMEM loads and stores,
                          // 8 = output warps skip stores, 32 / 64 = no GEMM2 / GEMM1 MMAs,
                          // 128 = the MMA issuer skips the H / output hand-off waits
};

// kStages ring stages of kBoxes weight boxes (16 KB each) per SM
template <int kStages, int kBoxes>
struct FusedCfg {
  static constexpr int kStageBytes = kBoxes * kFStageBytes;
  static constexpr int kBars = 2 * kStages + 8;
  static constexpr int kCtrlBytes = kBars * 8 + 16 + (kFMaxGroups + 1) * 4;
  static int smem_bytes(int d) {
    return 1024 + (d / 64) * kFXBlockBytes + kFHBytes + kStages * kStageBytes + kCtrlBytes;
  }
};

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_rel_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
// MN-major, 128B-swizzled operand: 1 KB atoms of 8 K-rows x 64 MN elements,
// consecutive K-atoms SBO = 1024 B apart (single MN atom: LBO unused)
__device__ __forceinline__ uint64_t umma_desc_mn_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(16384 >> 4) << 16;  // LBO (MN-atom stride; one atom here)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;   // SBO: K-atom stride
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// 4-D weight maps: {64 k (inner), rows, k-block, slot}; a box {64, 128,
// kBoxes, 1} lands as kBoxes consecutive 16 KB K-major SW128 tiles
__device__ __forceinline__ void tma_load_4d_2sm(void* dst, const CUtensorMap* map, uint32_t bar,
                                                int32_t row, int32_t kblk, int32_t slot,
                                                uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(0), "r"(row), "r"(kblk), "r"(slot),
      "l"(policy)
      : "memory");
}

// dev (COMOE_FUSED_DEBUG bit 256): clock64 cycles the MMA issuer of each
// pair spends in each wait, read back with comoe_debug_fused_prof:
// [0] total, [1] x_full, [2] h_empty, [3] GEMM1 full, [4] y_empty,
// [5] hs_full, [6] GEMM2 full, [7] tiles; weight producer of CTA rank r:
// [8 + r] empty waits, [10 + r] loop total; [12] leader's per-box issue
// cycles outside the waits
constexpr int kFProf = 16;
static __device__ unsigned long long g_fprof[128][kFProf];
#define FPROF(i, stmt)                                          \
  do {                                                         \
    if (p.debug & 256) {                                       \
      const unsigned long long t0_ = clock64();                \
      stmt;                                                    \
      prof[i] += clock64() - t0_;                              \
    } else {                                                   \
      stmt;                                                    \
    }                                                          \
  } while (0)

struct FTile {
  int g, tok0, ntok, nmma;
};

__device__ __forceinline__ FTile decode_ftile(const int* prefix, const FusedFfnParams& p, int tile) {
  FTile t;
  t.g = find_group(prefix, p.G, tile);
  t.tok0 = (tile - prefix[t.g]) * kFTok;
  t.ntok = min(kFTok, __ldg(p.group_rows + t.g) - t.tok0);
  t.nmma = (t.ntok + 15) & ~15;
  return t;
}

template <int kStages, int kBoxes, bool kGather>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kFThreads, 1)
    fused_ffn_kernel(const __grid_constant__ CUtensorMap tmap_win,
                     const __grid_constant__ CUtensorMap tmap_wout,
                     const __grid_constant__ CUtensorMap tmap_x, FusedFfnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int kb1 = p.d / 64;      // GEMM1 k-blocks (= token blocks resident in smem)
  const int mtiles = p.d / 256;  // GEMM2 output M-tiles
  const int nc = p.d_ff / kFChunk;
  uint8_t* sx = smem;
  uint8_t* sh = sx + kb1 * kFXBlockBytes;
  uint8_t* sring = sh + kFHBytes;
  constexpr int kStageBytes = FusedCfg<kStages, kBoxes>::kStageBytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sring + kStages * kStageBytes);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* x_full = empty_bar + kStages;
  uint64_t* x_empty = x_full + 1;
  uint64_t* h_full = x_full + 2;
  uint64_t* h_empty = x_full + 3;
  uint64_t* hs_full = x_full + 4;
  uint64_t* hs_free = x_full + 5;
  uint64_t* y_full = x_full + 6;
  uint64_t* y_empty = x_full + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(x_full + 8);
  int* prefix = reinterpret_cast<int*>(tmem_slot + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int n_clusters = gridDim.x >> 1;
  const int cluster = blockIdx.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_win);
    tma_prefetch_desc(&tmap_wout);
    tma_prefetch_desc(&tmap_x);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 2);  // one arrive per CTA (leader's copy is used)
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(x_full, 2);
    mbar_init(x_empty, 1);
    mbar_init(h_full, 1);
    mbar_init(h_empty, 8);  // 4 H warps x 2 CTAs (leader's copy)
    mbar_init(hs_full, 8);
    mbar_init(hs_free, 1);
    mbar_init(y_full, 1);
    mbar_init(y_empty, 8);
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  pdl_wait();
  pdl_trigger();
  build_tile_prefix_2sm<kFTok>(p.group_rows, p.G, 1, prefix);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = prefix[p.G];

  if (warp == 0) {
    // ---------------------------------------------- weight producer (both CTAs)
    // One 4-D TMA per stage brings kBoxes consecutive 64-wide k-blocks of a
    // 128-row weight slab (kBoxes x 16 KB, each block a K-major SW128 tile).
    // The producer is a single thread whose per-TMA instruction chain costs
    // ~200 clocks, so a stage must carry more MMA time than that: one 16 KB
    // block is only 4 MMAs = 256 clocks at N = 128 (measured: producer-bound).
    if (lane == 0) {
      unsigned long long prof[kFProf] = {};
      const unsigned long long t_prod = clock64();
      const uint64_t pol_w = l2_policy_evict_last();  // re-read by the group's other tiles
      int stage = 0;
      uint32_t phase = 0;
      const int r128 = static_cast<int>(rank) * 128;
      for (int tile = cluster; tile < total_tiles; tile += n_clusters) {
        const int slot = (p.debug & 1) ? 0 : __ldg(p.group_slot + find_group(prefix, p.G, tile));
        for (int c = 0; c <= nc; ++c) {
          // GEMM1 boxes of chunk c, then GEMM2 boxes of chunk c-1 (the MMA order)
          const int n_in = c < nc ? kb1 / kBoxes : 0;
          const int n_out = c > 0 ? mtiles * (4 / kBoxes) : 0;
          for (int b = 0; b < n_in + n_out; ++b) {
            const uint32_t fb = smem_u32(&full_bar[stage]) & kPeerMask;
            FPROF(8, mbar_wait(&empty_bar[stage], phase ^ 1));
            if ((p.debug & 2) && leader) mbar_arrive(&full_bar[stage]);
            else if (leader) mbar_expect_tx(&full_bar[stage], 2 * kStageBytes);
            else mbar_arrive_cluster(fb);
            if (!(p.debug & 2)) {
              if (b < n_in)
                tma_load_4d_2sm(sring + stage * kStageBytes, &tmap_win, fb, c * kFChunk + r128,
                                b * kBoxes, slot, pol_w);
              else
                tma_load_4d_2sm(sring + stage * kStageBytes, &tmap_wout, fb,
                                ((b - n_in) / (4 / kBoxes)) * 256 + r128,
                                (c - 1) * 4 + ((b - n_in) % (4 / kBoxes)) * kBoxes, slot, pol_w);
            }
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
        }
      }
      if ((p.debug & 256) && cluster < 128) {
        g_fprof[cluster][8 + rank] = prof[8];
        g_fprof[cluster][10 + rank] = clock64() - t_prod;
      }
    }
  } else if (warp == 3) {
    // ---------------------------------------------- token producer (both CTAs)
    const uint64_t pol_x = l2_policy_evict_first();  // read once per tile
    int it = 0;
    for (int tile = cluster; tile < total_tiles; tile += n_clusters, ++it) {
      const FTile t = decode_ftile(prefix, p, tile);
      const int gbase = __ldg(p.group_row_base + t.g);
      const int row0 = t.tok0 + static_cast<int>(rank) * (t.nmma >> 1);
      const uint32_t xb = smem_u32(x_full) & kPeerMask;
      if (lane == 0) {
        mbar_wait(x_empty, (it & 1) ^ 1);
        if (leader) {
          if (p.debug & 1024) mbar_arrive(x_full);  // dev: no token loads
          else mbar_expect_tx(x_full, 2 * kb1 * kFXBlockBytes);
        } else {
          mbar_arrive_cluster(xb);
        }
      }
      __syncwarp();
      if (p.debug & 1024) continue;
      if constexpr (kGather) {
        // lane l < 16 gathers rows 4l..4l+3 of this CTA's token half (rows past
        // the tile repeat its first token; their columns are never stored)
        if (lane < 16) {
          int rr[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = row0 + 4 * lane + i;
            rr[i] = __ldg(p.gather_rows + gbase + (r < t.tok0 + t.ntok ? r : t.tok0));
          }
          for (int kb = 0; kb < kb1; ++kb)
            tma_gather4_2sm(sx + kb * kFXBlockBytes + lane * 512, &tmap_x, xb, kb * 64, rr[0], rr[1],
                            rr[2], rr[3], pol_x);
        }
      } else {
        if (lane == 0)
          for (int kb = 0; kb < kb1; ++kb)
            tma_load_2d_2sm(sx + kb * kFXBlockBytes, &tmap_x, xb, kb * 64, gbase + row0, pol_x);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------- MMA issuer (leader CTA only)
    if (leader && elect_one()) {
      unsigned long long prof[kFProf] = {};
      const unsigned long long t_start = clock64();
      int stage = 0;
      uint32_t phase = 0;
      int n = 0;  // chunks issued so far (all tiles)
      int it = 0;
      for (int tile = cluster; tile < total_tiles; tile += n_clusters, ++it) {
        const FTile t = decode_ftile(prefix, p, tile);
        const uint32_t idesc1 = umma_idesc_bf16_f32(256, t.nmma);
        const uint32_t idesc2 = idesc1 | (1u << 16);  // B (H) MN-major
        auto gemm2 = [&](int cc, int nn) {
          if (cc == 0 && !(p.debug & 128)) {  // Y drained by the previous tile's epilogue
            FPROF(4, mbar_wait_acq_cluster(y_empty, (it & 1) ^ 1));
            tc_fence_after();
          }
          if (!(p.debug & 128)) FPROF(5, mbar_wait_acq_cluster(hs_full, nn & 1));  // H in both CTAs
          tc_fence_after();
          for (int m = 0; m < mtiles; ++m)
            for (int kb = 0; kb < kFChunk / 64; kb += kBoxes) {
              FPROF(6, mbar_wait(&full_bar[stage], phase));
              tc_fence_after();
#pragma unroll
              for (int bi = 0; bi < kBoxes; ++bi) {
                const uint64_t adesc =
                    umma_desc_k_sw128(smem_u32(sring + stage * kStageBytes + bi * kFStageBytes));
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const uint64_t bdesc =
                      umma_desc_mn_sw128(smem_u32(sh) + ((kb + bi) * 4 + k) * 2048);
                  if (!(p.debug & 32))
                    umma_bf16_2sm(tmem_base + m * 128, adesc + 2 * k, bdesc, idesc2,
                                  (cc | (kb + bi) | k) != 0);
                }
              }
              umma_commit_2sm_mc(&empty_bar[stage]);
              if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
          umma_commit_2sm_mc(hs_free);
        };
        FPROF(1, mbar_wait(x_full, it & 1));
        tc_fence_after();
        for (int c = 0; c < nc; ++c, ++n) {
          if (n > 0 && !(p.debug & 128)) {  // H accumulator drained by the H warps
            FPROF(2, mbar_wait_acq_cluster(h_empty, (n - 1) & 1));
            tc_fence_after();
          }
          for (int kb = 0; kb < kb1; kb += kBoxes) {
            FPROF(3, mbar_wait(&full_bar[stage], phase));
            tc_fence_after();
#pragma unroll
            for (int bi = 0; bi < kBoxes; ++bi) {
              const uint64_t adesc =
                  umma_desc_k_sw128(smem_u32(sring + stage * kStageBytes + bi * kFStageBytes));
              const uint64_t bdesc = umma_desc_k_sw128(smem_u32(sx + (kb + bi) * kFXBlockBytes));
#pragma unroll
              for (int k = 0; k < 4; ++k)
                if (!(p.debug & 64))
                  umma_bf16_2sm(tmem_base + kFColH, adesc + 2 * k, bdesc + 2 * k, idesc1,
                                ((kb + bi) | k) != 0);
            }
            umma_commit_2sm_mc(&empty_bar[stage]);
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
          umma_commit_2sm_mc(h_full);
          if (c == nc - 1) umma_commit_2sm_mc(x_empty);
          if (c > 0) gemm2(c - 1, n - 1);
        }
        gemm2(nc - 1, n - 1);
        umma_commit_2sm_mc(y_full);
      }
      if ((p.debug & 256) && cluster < 128) {
        prof[0] = clock64() - t_start;
        prof[7] = it;
        for (int i = 0; i < 8; ++i) g_fprof[cluster][i] = prof[i];
      }
    }
  } else if (warp >= 4 && (p.debug & 512)) {
    // dev: no epilogue warps at all (with bit 128 the issuer does not wait for them)
  } else if (warp >= 4 && warp < 8) {
    // ---------------------------------------------- H epilogue (both CTAs)
    // thread = d_ff row k (chunk-local 128*rank + 32*q + lane) of the H
    // accumulator: relu -> bf16 -> 16-byte vectors of 8 consecutive tokens
    const int q = warp & 3;
    const uint32_t t_h = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + kFColH;
    const uint32_t h_local = smem_u32(sh);
    const uint32_t h_peer = mapa_u32(h_local, rank ^ 1);
    const uint32_t h_empty_l = mapa_u32(smem_u32(h_empty), 0);
    const uint32_t hs_full_l = mapa_u32(smem_u32(hs_full), 0);
    const int k = static_cast<int>(rank) * 128 + q * 32 + lane;
    const uint32_t krow = k & 7;
    const uint32_t koff = static_cast<uint32_t>(k >> 3) * 1024 + krow * 128;
    int n = 0;
    for (int tile = cluster; tile < total_tiles; tile += n_clusters) {
      const FTile t = decode_ftile(prefix, p, tile);
      const int half = t.nmma >> 1;
      for (int c = 0; c < nc; ++c, ++n) {
        mbar_wait(h_full, n & 1);
        tc_fence_after();
        uint32_t pk[64];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if (b * 32 < t.nmma && !(p.debug & 4)) {
            uint32_t v[32];
            tmem_ld32(t_h + b * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j)
              pk[b * 16 + j] = pack_bf16x2(fmaxf(__uint_as_float(v[2 * j]), 0.f),
                                           fmaxf(__uint_as_float(v[2 * j + 1]), 0.f));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_rel_cluster(h_empty_l);  // GEMM1 of the next chunk may start
        if (n > 0) mbar_wait(hs_free, (n - 1) & 1);          // GEMM2 done reading the buffer
#pragma unroll
        for (int gi = 0; gi < 16; ++gi) {
          const int tok = gi * 8;
          if (tok < t.nmma && !(p.debug & 4)) {
            const bool hi = tok >= half;
            const uint32_t gl = static_cast<uint32_t>((tok - (hi ? half : 0)) >> 3);
            const uint32_t off = koff + ((gl ^ krow) << 4);
            const uint4 v = make_uint4(pk[4 * gi], pk[4 * gi + 1], pk[4 * gi + 2], pk[4 * gi + 3]);
            if (static_cast<uint32_t>(hi) == rank) st_shared_v4(h_local + off, v);
            else st_cluster_v4(h_peer + off, v);
          }
        }
        asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_rel_cluster(hs_full_l);
      }
    }
  } else if (warp >= 8) {
    // ---------------------------------------------- output epilogue (both CTAs)
    // thread = output feature (M-tile m, 128*rank + 32*q + lane); per 32-token
    // chunk: TMEM -> regs, feature-pair swap with the neighbour lane, bf16x2
    // stores (16 lanes = one 64-byte segment of a token row)
    const int q = warp & 3;
    const uint32_t y_empty_l = mapa_u32(smem_u32(y_empty), 0);
    const bool scatter = p.row_token != nullptr;
    const int odd = lane & 1;
    int it = 0;
    for (int tile = cluster; tile < total_tiles; tile += n_clusters, ++it) {
      const FTile t = decode_ftile(prefix, p, tile);
      const long row_base = static_cast<long>(__ldg(p.group_row_base + t.g)) + t.tok0;
      mbar_wait(y_full, it & 1);
      tc_fence_after();
      const int nch = (t.nmma + 31) >> 5;
      for (int m = 0; m < mtiles; ++m) {
        const long col = static_cast<long>(m) * 256 + rank * 128 + q * 32 + 2 * (lane >> 1);
        for (int ci = 0; ci < nch; ++ci) {
          const int c = ci * 32;
          uint32_t v[32];
          tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + m * 128 + c, v);
          tmem_ld_wait();
          if (m == mtiles - 1 && ci == nch - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_rel_cluster(y_empty_l);
          }
          const int my_tok = c + lane;
          long my_dst = 0;
          float my_p = 1.f;
          if (my_tok < t.ntok) {
            my_dst = scatter ? static_cast<long>(__ldg(p.row_token + row_base + my_tok))
                             : row_base + my_tok;
            if (scatter) my_p = __ldg(p.row_prob + row_base + my_tok);
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float send = __uint_as_float(odd ? v[2 * j] : v[2 * j + 1]);
            const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
            const float lo = odd ? recv : __uint_as_float(v[2 * j]);
            const float hi = odd ? __uint_as_float(v[2 * j + 1]) : recv;
            const int tl = 2 * j + odd;
            const float pr = __shfl_sync(0xffffffffu, my_p, tl);
            const long dst = __shfl_sync(0xffffffffu, my_dst, tl);
            if (c + tl < t.ntok && !(p.debug & 8))
              *reinterpret_cast<uint32_t*>(p.out + dst * p.ldo + col) = pack_bf16x2(lo * pr, hi * pr);
          }
        }
      }
    }
  }

  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base)
                 : "memory");
  }
}

}  // namespace comoe
