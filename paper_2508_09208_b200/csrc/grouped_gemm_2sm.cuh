// K3 (2-SM variant): grouped expert GEMM on CTA pairs (tcgen05 cta_group::2).
//
// Swap-AB formulation: the expert weights are the MMA "A" operand (M = 256
// output features per CTA pair, 128 per SM) and the routed token rows are
// the "B" operand (N = up to 256 tokens, any multiple of 16, chosen per
// tile at run time). Consequences:
//   * ragged expert groups waste < 16 token columns per group instead of up
//     to 127 rows of a 128-row M tile;
//   * each SM stages only half of each operand (A: its 128 features, B: its
//     N/2 tokens) — half the shared-memory operand traffic of the 1-SM
//     128x256 tile, the limiter measured in profiles/r1 (tensor pipe ~66%).
// D[feature, token] lands in TMEM (lanes = features, columns = tokens);
// the epilogue transposes 32x32 blocks through shared memory so every
// global store writes whole 256-byte token-row segments.
#pragma once

#include "grouped_gemm.cuh"

namespace comoe {

constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // clear the peer-CTA bit -> leader's smem
constexpr int k2BM = 256;                    // features per CTA pair
constexpr int k2BN = 256;                    // max tokens per tile
constexpr int kMaxGroups2 = 1024;
constexpr int k2MaxThreads = 128 + 32 * 8;

// kStages: smem pipeline depth (32 KB per stage per SM); kEpiWarps: 4 or 8
// epilogue warps (1 or 2 per TMEM lane quarter). Measured and not kept
// (K3): 512-token tiles sharing each weight stage between two
// MMAs, dynamic tile claiming through a cross-CTA tile-id ring, split
// weight/token rings, and L2 prefetch of weight boxes.
// kBN: tokens per tile (256; 32 for decode-sized batches: 16-row token boxes,
// so more of the shared memory holds weight stages)
template <int kStages, int kEpiWarps, int kBN = 256>
struct Gemm2Cfg {
  static constexpr int kThreads = 128 + 32 * kEpiWarps;  // w0 TMA, w1 MMA, w2 TMEM, w3 idle
  static constexpr int kABytes = 128 * kGemmBK * 2;     // 128 feature rows x 64 K
  static constexpr int kBBytes = (kBN / 2) * kGemmBK * 2;  // up to kBN/2 token rows x 64 K
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTileBytes = kStages * kStageBytes;
  static constexpr int kXposeBytes = 0;                          // (register transpose)
  static constexpr int kStgBytes = kEpiWarps * 2 * 32 * 64;    // per-warp 2 x (32 tok x 32 feat)
  static constexpr int kCtrlBytes = (2 * kStages + 4) * 8 + 16 + (kMaxGroups2 + 1) * 4;
  static constexpr int kTotal = 1024 + kTileBytes + kXposeBytes + kStgBytes + kCtrlBytes;
  static_assert(kTotal <= 227 * 1024, "shared memory");
};

__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w)
               : "memory");
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  return v;
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint32_t bar,
                                                int32_t x, int32_t y, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_2sm(void* dst, const CUtensorMap* map, uint32_t bar,
                                                int32_t x, int32_t y, int32_t z, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y), "r"(z), "l"(policy)
      : "memory");
}
// 4 token rows (box {64 cols, 1 row}) into 512 contiguous smem bytes; the
// transaction completes on the pair leader's mbarrier (peer-masked address)
__device__ __forceinline__ void tma_gather4_2sm(void* dst, const CUtensorMap* map, uint32_t bar,
                                                int32_t x, int r0, int r1, int r2, int r3,
                                                uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      ".cta_group::2.L2::cache_hint [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "l"(policy)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit_2sm_mc(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], m;\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

// tiles of a group: ceil(rows/256) token tiles x (N/256) feature tiles
template <int kBN>
__device__ __forceinline__ void build_tile_prefix_2sm(const int* __restrict__ rows, int G,
                                                      int f_tiles, int* prefix) {
  __shared__ int warp_tot2[k2MaxThreads / 32];
  const int tid = threadIdx.x;
  const int nthreads = blockDim.x;
  const int per = (G + nthreads - 1) / nthreads;
  const int g0 = tid * per;
  int local = 0;
  for (int i = 0; i < per; ++i)
    if (g0 + i < G) local += ((__ldg(rows + g0 + i) + kBN - 1) / kBN) * f_tiles;
  int v = local;
  const int lane = tid & 31, w = tid >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  if (lane == 31) warp_tot2[w] = v;
  __syncthreads();
  int run = v - local;
  for (int i = 0; i < w; ++i) run += warp_tot2[i];
  for (int i = 0; i < per; ++i) {
    const int g = g0 + i;
    if (g < G) {
      prefix[g] = run;
      run += ((__ldg(rows + g) + kBN - 1) / kBN) * f_tiles;
    }
  }
  if (tid == nthreads - 1) prefix[G] = run;
  __syncthreads();
}

static __device__ unsigned long long g_gemm_clock[4];  // dev clock probe (debug bit 256)

struct Tile2 {
  int g, ft, tok0, ntok, nmma;
};

template <int kBN, bool kChunk32 = false>
__device__ __forceinline__ Tile2 decode_tile2(const int* prefix, const GroupedGemmParams& p,
                                              int f_tiles, int tile) {
  Tile2 t;
  t.g = find_group(prefix, p.G, tile);
  const int local = tile - prefix[t.g];
  const int rows = __ldg(p.group_rows + t.g);
  int tt;
  if (p.ft_major) {  // big weight blocks: neighbouring pairs share a weight tile
    const int n_tt = (rows + kBN - 1) / kBN;
    tt = local % n_tt;
    t.ft = local / n_tt;
  } else {
    tt = local / f_tiles;
    t.ft = local % f_tiles;
  }
  // Equal token tiles (p.equal_tiles, long-K launches): a group's rows are
  // split into ceil(rows/kBN) tiles of one size (rounded up to 16), e.g. 600
  // rows -> 208 + 208 + 184 instead of 256 + 256 + 88. Same tile count (same
  // weight traffic), but the tiles a round-robin deal hands the pairs are
  // near-equal in MMA work: in the output GEMM at C2 (13 tiles per pair) the
  // busiest pair's excess over the average drops from 21-32% to ~11%
  // (DESIGN §K3). The activation GEMM (52 tiles per pair) keeps fixed tiles:
  // there smaller tiles cost more operand ingest per MAC than balance gains.
  int size = kBN;
  if (p.equal_tiles) {
    // bulk-store epilogues: sizes in whole 32-token chunks, so every tile but
    // a group's last keeps the TMA store path (a partial chunk falls back to
    // 16-byte stores); the scatter epilogue stores rows anyway: 16
    const int n_tt = max(1, (rows + kBN - 1) / kBN);  // (a decoded tile's group has rows > 0)
    const int q = kChunk32 ? 31 : 15;
    size = min(kBN, (((rows + n_tt - 1) / n_tt) + q) & ~q);
  }
  t.tok0 = tt * size;
  t.ntok = min(size, rows - t.tok0);
  t.nmma = (t.ntok + 15) & ~15;
  return t;
}

template <int kMode, int k2Stages, int k2EpiWarps, bool kGather = false, int kBN = 256>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Gemm2Cfg<k2Stages, k2EpiWarps, kBN>::kThreads, 1)
    grouped_gemm_2sm_kernel(const __grid_constant__ CUtensorMap tmap_w,
                            const __grid_constant__ CUtensorMap tmap_x,
                            const __grid_constant__ CUtensorMap tmap_out, GroupedGemmParams p) {
  static_assert(kMode != kEpiSwiGLU, "SwiGLU uses the 1-SM kernel");
  using S = Gemm2Cfg<k2Stages, k2EpiWarps, kBN>;
  static_assert(!kGather || kBN == 256, "the token gather fills 128-row boxes");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* smem_a = smem;                                   // weights
  uint8_t* smem_b = smem + k2Stages * S::kABytes;           // tokens
  uint8_t* xpose = smem + S::kTileBytes;
  uint8_t* stg = smem + S::kTileBytes + S::kXposeBytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(stg + S::kStgBytes);
  uint64_t* empty_bar = full_bar + k2Stages;
  uint64_t* tfull_bar = empty_bar + k2Stages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int* prefix = reinterpret_cast<int*>(tmem_slot + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int f_tiles = p.N / k2BM;
  const int k_blocks = p.K / kGemmBK;
  const int n_clusters = gridDim.x >> 1;
  const int cluster = blockIdx.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_w);
    tma_prefetch_desc(&tmap_x);
    for (int s = 0; s < k2Stages; ++s) {
      mbar_init(&full_bar[s], 2);   // one arrive per CTA of the pair (leader's copy is used)
      mbar_init(&empty_bar[s], 1);  // MMA commit multicast
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 2 * k2EpiWarps);  // epilogue warps of both CTAs (leader's copy)
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  pdl_wait();     // group tables / token rows come from the preceding kernels
  pdl_trigger();  // persistent grid: the next kernel may launch and wait
  build_tile_prefix_2sm<kBN>(p.group_rows, p.G, f_tiles, prefix);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = prefix[p.G];
  // dev: SM clock during the launch (COMOE_GEMM_DEBUG bit 256): CTA 0 stamps
  // clock64 and the global ns timer at start and end (comoe_debug_gemm_clock)
  if ((p.debug & 256) && blockIdx.x == 0 && threadIdx.x == 0) {
    g_gemm_clock[0] = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_gemm_clock[1]));
  }

  if (warp == 0) {
    // ---------------------------------------------- TMA producer (both CTAs)
    const uint64_t pol_w = l2_policy_evict_last();
    // token rows are re-read by every feature tile of the group: keep them
    // (evict_first here doubled DRAM reads of H, profiles/r1_2sm_evict_first)
    const uint64_t pol_x = l2_policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = cluster; tile < total_tiles; tile += n_clusters) {
      const Tile2 t = decode_tile2<kBN, kMode != kEpiScaleScatter>(prefix, p, f_tiles, tile);
      // (dev attribution: debug 16 = every tile loads slot 0 and token row 0,
      // 128 = slot 0 only — L2-resident operands; +27-42% / +17% at C2)
      const int slot = (p.debug & (16 | 128)) ? 0 : __ldg(p.group_slot + t.g);
      const int feat = t.ft * k2BM + static_cast<int>(rank) * 128;
      // (dev 32768: token rows only L2-resident — every tile reads rows 0..255;
      // the weights still stream from HBM)
      const int gbase = (p.debug & (16 | 32768)) ? -t.tok0 : __ldg(p.group_row_base + t.g);
      const int half0 = t.tok0 + static_cast<int>(rank) * (t.nmma >> 1);
      int idx0 = 0, idx1 = 0, idx2 = 0, idx3 = 0;
      if constexpr (kGather) {
        // this lane gathers rows 4*lane .. 4*lane+3 of the CTA's token half
        // (padding rows point at the group's first token; their columns are dropped)
        int rr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = half0 + 4 * lane + i;
          rr[i] = __ldg(p.gather_rows + gbase + (r < t.tok0 + t.ntok ? r : t.tok0));
        }
        idx0 = rr[0]; idx1 = rr[1]; idx2 = rr[2]; idx3 = rr[3];
      }
      for (int kb = 0; kb < k_blocks; ++kb) {
        const uint32_t fb = smem_u32(&full_bar[stage]) & kPeerMask;
        if (lane == 0) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (p.debug & 2) {  // dev: no data movement
            if (leader) mbar_arrive(&full_bar[stage]);
            else mbar_arrive_cluster(fb);
          } else {
            if (leader) mbar_expect_tx(&full_bar[stage], 2 * S::kStageBytes);
            else mbar_arrive_cluster(fb);
            tma_load_3d_2sm(smem_a + stage * S::kABytes, &tmap_w, fb, kb * kGemmBK, feat, slot, pol_w);
            if constexpr (!kGather)
              tma_load_2d_2sm(smem_b + stage * S::kBBytes, &tmap_x, fb, kb * kGemmBK,
                              gbase + half0, pol_x);
          }
        }
        if constexpr (kGather) {
          __syncwarp();  // lane 0 has seen the stage free
          if (!(p.debug & 2))
            tma_gather4_2sm(smem_b + stage * S::kBBytes + lane * 512, &tmap_x, fb, kb * kGemmBK,
                            idx0, idx1, idx2, idx3, pol_x);
        }
        if (++stage == k2Stages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------- MMA issuer (leader CTA only)
    if (leader && elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = cluster; tile < total_tiles; tile += n_clusters, ++it) {
        const Tile2 t = decode_tile2<kBN, kMode != kEpiScaleScatter>(prefix, p, f_tiles, tile);
        const uint32_t idesc = umma_idesc_bf16_f32(k2BM, t.nmma);
        const int acc = it & 1;
        mbar_wait(&tempty_bar[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kBN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t adesc = umma_desc_k_sw128(smem_u32(smem_a + stage * S::kABytes));
          const uint64_t bdesc = umma_desc_k_sw128(smem_u32(smem_b + stage * S::kBBytes));
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k)
            umma_bf16_2sm(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          umma_commit_2sm_mc(&empty_bar[stage]);
          if (++stage == k2Stages) { stage = 0; phase ^= 1; }
        }
        umma_commit_2sm_mc(&tfull_bar[acc]);
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------- epilogue (both CTAs)
    // Warp w: TMEM lane quarter q = w%4 (features 32q..32q+31 of this SM's
    // 128), token chunks c = 32*(2j + sub). Per chunk: TMEM -> regs (thread =
    // feature) -> fp32 transpose in smem (thread = token) -> bf16 row staging
    // -> 16-byte stores, 4 lanes per 64-byte token-row segment. All smem
    // layouts are XOR-swizzled on 16-byte chunks: conflict-free both ways.
    const int ew = warp - 4;
    const int q = warp & 3, sub = ew >> 2;
    constexpr int kSubs = k2EpiWarps / 4;
    const uint32_t sg0 = smem_u32(stg) + ew * (2 * 32 * 64);
    constexpr bool kTmaStore = kMode != kEpiScaleScatter;  // contiguous rows: TMA bulk store
    int nbuf = 0;
    int it = 0;
    // chunks of one tile handled by this warp (ci = sub, sub + kSubs, ...)
    constexpr int kMaxIt = (kBN / 32 + kSubs - 1) / kSubs;
    for (int tile = cluster; tile < total_tiles; tile += n_clusters, ++it) {
      const Tile2 t = decode_tile2<kBN, kMode != kEpiScaleScatter>(prefix, p, f_tiles, tile);
      const int acc = it & 1;
      const long row_base = static_cast<long>(__ldg(p.group_row_base + t.g)) + t.tok0;
      const long col0 = static_cast<long>(t.ft) * k2BM + rank * 128 + q * 32;
      // Scatter epilogue: the tile's gate probabilities and destination rows
      // (lane = token c + lane of each chunk) are loaded before the wait on
      // the accumulator, so their L2 latency hides behind the mainloop instead
      // of sitting twice on every chunk's critical path (debug 4096: old form).
      float pre_p[kMaxIt] = {};
      int pre_t[kMaxIt] = {};
      const bool preload = kMode == kEpiScaleScatter && !(p.debug & 4096);
      if constexpr (kMode == kEpiScaleScatter) {
        if (preload) {
#pragma unroll
          for (int i = 0; i < kMaxIt; ++i) {
            const int tk = (sub + i * kSubs) * 32 + lane;
            const bool ok = tk < t.ntok;
            pre_p[i] = ok ? __ldg(p.row_prob + row_base + tk) : 0.f;
            pre_t[i] = ok ? __ldg(p.row_token + row_base + tk) : 0;
          }
        }
      }
      mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * kBN;
      const int chunks = (t.nmma + 31) >> 5;
      bool released = false;
#pragma unroll
      for (int i = 0; i < kMaxIt; ++i) {
        const int ci = sub + i * kSubs;
        if (ci >= chunks) break;
        const int c = ci * 32;
        uint32_t v[32];
        tmem_ld32(t_row + c, v);
        tmem_ld_wait();
        if (ci + kSubs >= chunks) {  // this warp's last TMEM read of the tile
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(smem_u32(&tempty_bar[acc]) & kPeerMask);
          released = true;
        }
        if (p.debug & 1) continue;  // dev: TMEM read only
        // epilogue math in the feature-major registers: v[j] = D[feature lane][token c+j]
        if constexpr (kMode == kEpiRelu) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(fmaxf(__uint_as_float(v[j]), 0.f));
        } else if constexpr (kMode == kEpiScaleScatter) {
          const float my_p = preload ? pre_p[i]
                                     : ((c + lane < t.ntok) ? __ldg(p.row_prob + row_base + c + lane) : 0.f);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            v[j] = __float_as_uint(__uint_as_float(v[j]) * __shfl_sync(0xffffffffu, my_p, j));
        }
        if (p.debug & 1024) continue;  // dev: epilogue math only (no staging, no stores)
        // register transpose of feature pairs: lanes (2p, 2p+1) hold features
        // (2p, 2p+1); for each token pair (2j, 2j+1) the even lane keeps token
        // 2j and the odd lane token 2j+1, one shfl_xor swapping the partner
        // feature in. Staging = bf16 [32 tokens][32 features], 64-B rows in
        // the TMA 64-byte swizzle (16-B chunk c at c ^ ((row/2)%4)): the
        // even/odd lanes land in opposite bank halves -> conflict-free STS.
        const int odd = lane & 1;
        const uint32_t pw = static_cast<uint32_t>(lane >> 1);  // feature-pair word 0..15
        const uint32_t sg = sg0 + nbuf * (32 * 64);
        if constexpr (kTmaStore) {
          if (lane == 0) bulk_wait_read<1>();  // this buffer's previous store has read smem
          __syncwarp();
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float send = __uint_as_float(odd ? v[2 * j] : v[2 * j + 1]);
          const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
          const float lo = odd ? recv : __uint_as_float(v[2 * j]);          // feature 2p
          const float hi = odd ? __uint_as_float(v[2 * j + 1]) : recv;      // feature 2p+1
          const uint32_t row = 2 * j + odd;
          const uint32_t addr = sg + row * 64 + (((pw >> 2) ^ ((row >> 1) & 3)) << 4) + ((pw & 3) << 2);
          asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(pack_bf16x2(lo, hi)) : "memory");
        }
        __syncwarp();
        bool stored = false;
        if constexpr (kTmaStore) {
          // whole chunk valid: one bulk tensor store (debug 4: dev, force st.global)
          if (c + 32 <= t.ntok && !(p.debug & 4)) {
            fence_async_smem();
            __syncwarp();
            if (lane == 0 && !(p.debug & 512)) {  // (dev 512: staged, not stored)
              tma_store_2d(&tmap_out, stg + (sg - smem_u32(stg)), static_cast<int>(col0),
                           (p.debug & 2048) ? 0 : static_cast<int>(row_base + c));
              bulk_commit();
            }
            nbuf ^= 1;
            stored = true;
          }
        }
        if (!stored) {  // scatter rows or a partial chunk: 16-B stores, 4 lanes per row
#pragma unroll
          for (int ii = 0; ii < 4; ++ii) {
            const int r = 8 * ii + (lane >> 2), j = lane & 3;
            const uint4 x = lds128(sg + r * 64 + ((j ^ ((r >> 1) & 3)) << 4));
            const int tk = c + r;
            int pre_dst = 0;
            if constexpr (kMode == kEpiScaleScatter) pre_dst = __shfl_sync(0xffffffffu, pre_t[i], r);
            if (tk < t.ntok && !(p.debug & 512)) {
              long dst;
              if constexpr (kMode == kEpiScaleScatter)
                dst = preload ? pre_dst : __ldg(p.row_token + row_base + tk);
              else dst = row_base + tk;
              if (p.debug & 2048) dst = r;  // dev: every tile writes the same 32 rows (L2-resident)
              st_global_v4(p.out + dst * p.ldo + col0 + j * 8, x.x, x.y, x.z, x.w);
            }
          }
          __syncwarp();
        }
      }
      if (!released) {  // no chunk for this warp in a narrow tile
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(smem_u32(&tempty_bar[acc]) & kPeerMask);
      }
    }
  }

  if (warp >= 4 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base)
                 : "memory");
  }
  if ((p.debug & 256) && blockIdx.x == 0 && threadIdx.x == 0) {
    g_gemm_clock[2] = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_gemm_clock[3]));
  }
}

}  // namespace comoe
