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

// kStages: smem pipeline depth; kEpiWarps: 4 or 8 epilogue warps (1 or 2
// per TMEM lane quarter); kWide: token tiles of up to 512 rows computed as
// two N<=256 MMAs per k-step that share the weight (A) stage, each into
// its own 256-column TMEM half — one weight pass per 512 routed tokens
// instead of per 256 (a C2 expert holds ~512 tokens, so a 256-token tiling
// re-streams every expert's weights 2-3 times, the last time for a ragged
// tail of a few dozen tokens).
template <int kStages, int kEpiWarps, bool kWide = false>
struct Gemm2Cfg {
  static constexpr int kThreads = 128 + 32 * kEpiWarps;  // w0 TMA, w1 MMA, w2 TMEM, w3 idle
  static constexpr int kHalves = kWide ? 2 : 1;          // token MMAs (TMEM halves) per tile
  static constexpr int kTokTile = 256 * kHalves;         // max tokens per tile
  static constexpr int kABytes = 128 * kGemmBK * 2;     // 128 feature rows x 64 K
  static constexpr int kBHalfBytes = 128 * kGemmBK * 2; // up to 128 token rows x 64 K per MMA
  static constexpr int kBBytes = kHalves * kBHalfBytes;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTileBytes = kStages * kStageBytes;
  static constexpr int kXposeBytes = 0;                          // (register transpose)
  static constexpr int kStgBytes = kEpiWarps * 2 * 32 * 64;    // per-warp 2 x (32 tok x 32 feat)
  static constexpr int kSchedDepth = 8;                  // tile-id ring (dynamic scheduling)
  static constexpr int kCtrlBytes =
      (2 * kStages + 4 + 2 * kSchedDepth) * 8 + 16 + kSchedDepth * 4 + (kMaxGroups2 + 1) * 4;
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
// shared::cluster address of `local` in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_rank(const void* local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_release_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void st_cluster_u32(uint32_t cluster_addr, int v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}

// Dynamic tile claiming for a persistent CTA pair. The leader's producer
// thread claims tile ids from a global counter (atomicAdd, in order, so
// concurrently running pairs still work on neighbouring tiles and share
// weights/tokens in L2) and publishes the i-th claim into slot i % depth of
// a tile-id ring held by BOTH CTAs. Consumers — the peer's producer, the
// MMA thread and every epilogue warp of both CTAs — read claims in the same
// order and release the slot on the leader's empty barrier. A pair claims
// its next tile only when it is ready to load it, so the load imbalance of
// ragged expert groups (round-robin: max/mean 1.08-1.23 at C2) drops to
// at most one tile.
struct TileRing {
  int* tile;            // [depth] local ring
  uint64_t* full;       // [depth] local, count 1 (the leader's publish)
  uint64_t* empty;      // [depth] leader's copy counts every consumer of both CTAs
  int depth;
  // publish claim i (= t, drawn earlier so the atomic's L2 round trip
  // overlaps the previous tile's loads)
  __device__ __forceinline__ void publish(uint32_t i, int t, bool peer_too) const {
    const int s = static_cast<int>(i % depth);
    const uint32_t par = (i / depth) & 1;
    mbar_wait(&empty[s], par ^ 1);
    tile[s] = t;
    if (peer_too) {
      st_cluster_u32(mapa_rank(&tile[s], 1), t);
      mbar_arrive_release_cluster(mapa_rank(&full[s], 1));
    }
    mbar_arrive(&full[s]);
  }
  // consumers in the leader CTA: everything is CTA-local (cta-scope
  // acquire/release); the peer's consumers need cluster scope
  __device__ __forceinline__ int consume(uint32_t i, bool is_leader) const {
    const int s = static_cast<int>(i % depth);
    const uint32_t par = (i / depth) & 1;
    if (is_leader) {
      mbar_wait(&full[s], par);
      const int t = *reinterpret_cast<volatile int*>(&tile[s]);
      // relaxed: a release here would also order the MMA thread's in-flight
      // tcgen05 work and drain the tensor pipe at every tile boundary
      asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s]))
                   : "memory");
      return t;
    }
    mbar_wait(&full[s], par);
    asm volatile("fence.acq_rel.cluster;" ::: "memory");  // pairs with the leader's release
    const int t = *reinterpret_cast<volatile int*>(&tile[s]);
    mbar_arrive_release_cluster(mapa_rank(&empty[s], 0));
    return t;
  }
};
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

// tiles of a group: ceil(rows/kTokTile) token tiles x (N/256) feature tiles
template <int kTokTile>
__device__ __forceinline__ void build_tile_prefix_2sm(const int* __restrict__ rows, int G,
                                                      int f_tiles, int* prefix) {
  __shared__ int warp_tot2[k2MaxThreads / 32];
  const int tid = threadIdx.x;
  const int nthreads = blockDim.x;
  const int per = (G + nthreads - 1) / nthreads;
  const int g0 = tid * per;
  int local = 0;
  for (int i = 0; i < per; ++i)
    if (g0 + i < G) local += ((__ldg(rows + g0 + i) + kTokTile - 1) / kTokTile) * f_tiles;
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
      run += ((__ldg(rows + g) + kTokTile - 1) / kTokTile) * f_tiles;
    }
  }
  if (tid == nthreads - 1) prefix[G] = run;
  __syncthreads();
}

// A tile = (group, feature tile, token tile). Its tokens split into halves of
// <= 256 (one MMA and one TMEM half each): ntok[j] valid, nmma[j] padded to 16.
struct Tile2 {
  int g, ft, tok0, nh;
  int ntok[2], nmma[2];
};

template <int kTokTile>
__device__ __forceinline__ Tile2 decode_tile2(const int* prefix, const GroupedGemmParams& p,
                                              int f_tiles, int tile) {
  Tile2 t;
  t.g = find_group(prefix, p.G, tile);
  const int local = tile - prefix[t.g];
  const int rows = __ldg(p.group_rows + t.g);
  int tt;
  if (p.ft_major) {  // big weight blocks: neighbouring pairs share a weight tile
    const int n_tt = (rows + kTokTile - 1) / kTokTile;
    tt = local % n_tt;
    t.ft = local / n_tt;
  } else {
    tt = local / f_tiles;
    t.ft = local % f_tiles;
  }
  t.tok0 = tt * kTokTile;
  const int n = min(kTokTile, rows - t.tok0);
  t.ntok[0] = min(k2BN, n);
  t.ntok[1] = n - t.ntok[0];
  t.nh = t.ntok[1] > 0 ? 2 : 1;
  t.nmma[0] = (t.ntok[0] + 15) & ~15;
  t.nmma[1] = (t.ntok[1] + 15) & ~15;
  return t;
}

template <int kMode, int k2Stages, int k2EpiWarps, bool kGather = false, bool kWide = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Gemm2Cfg<k2Stages, k2EpiWarps, kWide>::kThreads, 1)
    grouped_gemm_2sm_kernel(const __grid_constant__ CUtensorMap tmap_w,
                            const __grid_constant__ CUtensorMap tmap_x,
                            const __grid_constant__ CUtensorMap tmap_out, GroupedGemmParams p) {
  static_assert(kMode != kEpiSwiGLU, "SwiGLU uses the 1-SM kernel");
  static_assert(!(kGather && kWide), "row gather uses 256-token tiles");
  using S = Gemm2Cfg<k2Stages, k2EpiWarps, kWide>;
  constexpr int kTT = S::kTokTile;
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
  uint64_t* sched_full = tempty_bar + 2;
  uint64_t* sched_empty = sched_full + S::kSchedDepth;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sched_empty + S::kSchedDepth);
  int* sched_tile = reinterpret_cast<int*>(tmem_slot + 4);
  int* prefix = sched_tile + S::kSchedDepth;
  const TileRing ring{sched_tile, sched_full, sched_empty, S::kSchedDepth};

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
    for (int s = 0; s < S::kSchedDepth; ++s) {
      mbar_init(&sched_full[s], 1);
      // leader's MMA thread + peer's producer + epilogue warps of both CTAs
      mbar_init(&sched_empty[s], 2 + 2 * k2EpiWarps);
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
  build_tile_prefix_2sm<kTT>(p.group_rows, p.G, f_tiles, prefix);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = prefix[p.G];
  const bool dyn = p.sched != nullptr;

  if (warp == 0) {
    // ---------------------------------------------- TMA producer (both CTAs)
    const uint64_t pol_w = l2_policy_evict_last();
    // token rows are re-read by every feature tile of the group: keep them
    // (evict_first here doubled DRAM reads of H, profiles/r1_2sm_evict_first)
    const uint64_t pol_x = l2_policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    // leader: claims run two ahead of the tile being loaded and are
    // published one ahead, so neither the atomic's L2 round trip nor the
    // cross-CTA hand-off to the peer sits on the load path
    int c_cur = 0, c_nxt = 0, c_nxt2 = 0;
    if (dyn && leader && lane == 0) {
      c_cur = atomicAdd(p.sched, 1);
      ring.publish(0, c_cur, true);
      if (c_cur < total_tiles) c_nxt = atomicAdd(p.sched, 1);
    }
    for (uint32_t i = 0;; ++i) {
      int tile = cluster + static_cast<int>(i) * n_clusters;
      if (dyn) {
        if (lane == 0) {
          if (leader) {
            tile = c_cur;
            if (tile < total_tiles) {
              ring.publish(i + 1, c_nxt, true);
              if (c_nxt < total_tiles) c_nxt2 = atomicAdd(p.sched, 1);
              c_cur = c_nxt;
              c_nxt = c_nxt2;
            }
          } else {
            tile = ring.consume(i, false);
          }
        }
        tile = __shfl_sync(0xffffffffu, tile, 0);
      }
      if (tile >= total_tiles) break;
      const Tile2 t = decode_tile2<kTT>(prefix, p, f_tiles, tile);
      // (dev attribution: debug 16 = every tile loads slot 0 and token row 0,
      // 128 = slot 0 only — L2-resident operands; +27-42% / +17% at C2)
      const int slot = (p.debug & (16 | 128)) ? 0 : __ldg(p.group_slot + t.g);
      const int feat = t.ft * k2BM + static_cast<int>(rank) * 128;
      const int gbase = (p.debug & 16) ? -t.tok0 : __ldg(p.group_row_base + t.g);
      // this CTA's token rows of MMA j: the rank-th half of its nmma[j] columns
      const int row0 = gbase + t.tok0 + static_cast<int>(rank) * (t.nmma[0] >> 1);
      const int row1 = gbase + t.tok0 + k2BN + static_cast<int>(rank) * (t.nmma[1] >> 1);
      const uint32_t tx = 2 * (S::kABytes + t.nh * S::kBHalfBytes);
      int idx0 = 0, idx1 = 0, idx2 = 0, idx3 = 0;
      if constexpr (kGather) {
        // this lane gathers rows 4*lane .. 4*lane+3 of the CTA's token half
        // (padding rows point at the group's first token; their columns are dropped)
        const int half0 = t.tok0 + static_cast<int>(rank) * (t.nmma[0] >> 1);
        int rr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = half0 + 4 * lane + i;
          rr[i] = __ldg(p.gather_rows + gbase + (r < t.tok0 + t.ntok[0] ? r : t.tok0));
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
            if (leader) mbar_expect_tx(&full_bar[stage], kGather ? 2 * S::kStageBytes : tx);
            else mbar_arrive_cluster(fb);
            tma_load_3d_2sm(smem_a + stage * S::kABytes, &tmap_w, fb, kb * kGemmBK, feat, slot, pol_w);
            if constexpr (!kGather) {
              uint8_t* b = smem_b + stage * S::kBBytes;
              tma_load_2d_2sm(b, &tmap_x, fb, kb * kGemmBK, row0, pol_x);
              if (kWide && t.nh == 2)
                tma_load_2d_2sm(b + S::kBHalfBytes, &tmap_x, fb, kb * kGemmBK, row1, pol_x);
            }
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
    // TMEM = two 256-column accumulator halves used as a ring: half sequence
    // number h -> columns (h&1)*256, use count h>>1. A tile takes nh halves.
    if (leader && elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t hseq = 0;
      for (uint32_t i = 0;; ++i) {
        const int tile = dyn ? ring.consume(i, true) : cluster + static_cast<int>(i) * n_clusters;
        if (tile >= total_tiles) break;
        const Tile2 t = decode_tile2<kTT>(prefix, p, f_tiles, tile);
        const uint32_t idesc0 = umma_idesc_bf16_f32(k2BM, t.nmma[0]);
        const uint32_t idesc1 = umma_idesc_bf16_f32(k2BM, kWide && t.nh == 2 ? t.nmma[1] : 16);
        const uint32_t h0 = hseq, h1 = hseq + 1;
        mbar_wait(&tempty_bar[h0 & 1], ((h0 >> 1) & 1) ^ 1);
        if (kWide && t.nh == 2) mbar_wait(&tempty_bar[h1 & 1], ((h1 >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem_base + (h0 & 1) * k2BN;
        const uint32_t d1 = tmem_base + (h1 & 1) * k2BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t adesc = umma_desc_k_sw128(smem_u32(smem_a + stage * S::kABytes));
          const uint64_t bdesc0 = umma_desc_k_sw128(smem_u32(smem_b + stage * S::kBBytes));
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k)
            umma_bf16_2sm(d0, adesc + 2 * k, bdesc0 + 2 * k, idesc0, (kb | k) != 0);
          if (kWide && t.nh == 2) {
            const uint64_t bdesc1 =
                umma_desc_k_sw128(smem_u32(smem_b + stage * S::kBBytes + S::kBHalfBytes));
#pragma unroll
            for (int k = 0; k < kGemmBK / 16; ++k)
              umma_bf16_2sm(d1, adesc + 2 * k, bdesc1 + 2 * k, idesc1, (kb | k) != 0);
          }
          umma_commit_2sm_mc(&empty_bar[stage]);
          if (++stage == k2Stages) { stage = 0; phase ^= 1; }
        }
        umma_commit_2sm_mc(&tfull_bar[h0 & 1]);
        if (kWide && t.nh == 2) umma_commit_2sm_mc(&tfull_bar[h1 & 1]);
        hseq += t.nh;
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
    uint32_t hseq = 0;
    for (uint32_t i = 0;; ++i) {
      int tile = cluster + static_cast<int>(i) * n_clusters;
      if (dyn) {
        if (lane == 0) tile = ring.consume(i, leader);
        tile = __shfl_sync(0xffffffffu, tile, 0);
      }
      if (tile >= total_tiles) break;
      const Tile2 t = decode_tile2<kTT>(prefix, p, f_tiles, tile);
      const long col0 = static_cast<long>(t.ft) * k2BM + rank * 128 + q * 32;
      for (int j = 0; j < t.nh; ++j, ++hseq) {
        const int acc = hseq & 1;
        const int ntok = t.ntok[j];
        const long row_base = static_cast<long>(__ldg(p.group_row_base + t.g)) + t.tok0 + j * k2BN;
        mbar_wait(&tfull_bar[acc], (hseq >> 1) & 1);
        tc_fence_after();
        const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * k2BN;
        const int chunks = (t.nmma[j] + 31) >> 5;
        bool released = false;
        for (int ci = sub; ci < chunks; ci += kSubs) {
          const int c = ci * 32;
          uint32_t v[32];
          tmem_ld32(t_row + c, v);
          tmem_ld_wait();
          if (ci + kSubs >= chunks) {  // this warp's last TMEM read of the half
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(smem_u32(&tempty_bar[acc]) & kPeerMask);
            released = true;
          }
          if (p.debug & 1) continue;  // dev: TMEM read only
          // epilogue math in the feature-major registers: v[i] = D[feature lane][token c+i]
          if constexpr (kMode == kEpiRelu) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(fmaxf(__uint_as_float(v[i]), 0.f));
          } else if constexpr (kMode == kEpiScaleScatter) {
            const float my_p = (c + lane < ntok) ? __ldg(p.row_prob + row_base + c + lane) : 0.f;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              v[i] = __float_as_uint(__uint_as_float(v[i]) * __shfl_sync(0xffffffffu, my_p, i));
          }
          // register transpose of feature pairs: lanes (2p, 2p+1) hold features
          // (2p, 2p+1); for each token pair (2i, 2i+1) the even lane keeps token
          // 2i and the odd lane token 2i+1, one shfl_xor swapping the partner
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
          for (int i = 0; i < 16; ++i) {
            const float send = __uint_as_float(odd ? v[2 * i] : v[2 * i + 1]);
            const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
            const float lo = odd ? recv : __uint_as_float(v[2 * i]);          // feature 2p
            const float hi = odd ? __uint_as_float(v[2 * i + 1]) : recv;      // feature 2p+1
            const uint32_t row = 2 * i + odd;
            const uint32_t addr = sg + row * 64 + (((pw >> 2) ^ ((row >> 1) & 3)) << 4) + ((pw & 3) << 2);
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(pack_bf16x2(lo, hi)) : "memory");
          }
          __syncwarp();
          bool stored = false;
          if constexpr (kTmaStore) {
            // whole chunk valid: one bulk tensor store (debug 4: dev, force st.global)
            if (c + 32 <= ntok && !(p.debug & 4)) {
              fence_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(&tmap_out, stg + (sg - smem_u32(stg)), static_cast<int>(col0),
                             static_cast<int>(row_base + c));
                bulk_commit();
              }
              nbuf ^= 1;
              stored = true;
            }
          }
          if (!stored) {  // scatter rows or a partial chunk: 16-B stores, 4 lanes per row
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int r = 8 * i + (lane >> 2), jj = lane & 3;
              const uint4 x = lds128(sg + r * 64 + ((jj ^ ((r >> 1) & 3)) << 4));
              const int tk = c + r;
              if (tk < ntok) {
                long dst;
                if constexpr (kMode == kEpiScaleScatter) dst = __ldg(p.row_token + row_base + tk);
                else dst = row_base + tk;
                st_global_v4(p.out + dst * p.ldo + col0 + jj * 8, x.x, x.y, x.z, x.w);
              }
            }
            __syncwarp();
          }
        }
        if (!released) {  // no chunk for this warp in a narrow half
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(smem_u32(&tempty_bar[acc]) & kPeerMask);
        }
      }
    }
  }
  if (warp >= 4 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  tc_fence_before();
  cluster_sync_all();
  if (dyn && leader && threadIdx.x == 0) {
    // every pair has drawn its end-of-work claim before counting itself
    // finished, so the last one can rearm the counters for the next launch
    __threadfence();
    if (atomicAdd(p.sched + 1, 1) == n_clusters - 1) {
      atomicExch(p.sched, 0);
      atomicExch(p.sched + 1, 0);
    }
  }
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base)
                 : "memory");
  }
}

}  // namespace comoe
