// K1 gate, router resident in tensor memory (EP = 128 padded router experts,
// d <= 768, CTA pair, two split router terms). Included from gate.cu.
//
// Why: the pair gate (gate_kernel) re-reads one router term per SM from L2
// with every token k-block, so each SM ingests twice the bytes of x; its
// timeline (scripts/gate_timeline.py) shows the TMA stream at ~4.8 µs per
// 256-token unit and 4 units on the busiest pairs (256 units over 74 pairs),
// i.e. ingest-bound and quantised. Here the router is loaded ONCE per CTA
// into TMEM and used as the MMA's A operand (tcgen05.mma ... [a_tmem]):
//   * A = router rows, M = 256 per pair: SM s holds the hi and mid terms of
//     experts [64s, 64s+64), lane 32q + l = expert 64s + 16q + l%16, term
//     l/16 (K = d packed two bf16 per 32-bit column: columns [0, d/2));
//   * B = the tile's 128 tokens (N = 128, each SM stages its 64 rows);
//   * D = x.term^T in TMEM columns [384, 512): SM s ends up with the hi and
//     mid partial logits of its 64 experts for all 128 tokens of the tile.
// The x stream is the only operand traffic (half the per-SM ingest of the
// pair kernel) and a unit is one 128-token tile (512 units / 74 pairs: a
// 1.4% tail instead of 13%).
//
// Warp roles: w0 TMA, w1 MMA (leader), w2 TMEM alloc, w4-11 epilogue. All
// eight epilogue warps load the router into TMEM at the start. Per tile, w4-7
// drain the single accumulator into a double-buffered fp32 stash in shared
// memory (hi + mid added with one shuffle: an expert's two rows sit in lanes
// l and l + 16 of the same warp), which frees TMEM for the next tile's MMAs
// at once; then all eight warps run the token pass (two threads per token,
// 32 experts each: top-2, max, softmax sum). SM1 hands its partials to SM0
// through distributed shared memory and SM0 merges them (its experts have
// the lower ids, so ties keep the reference's lowest-id rule) and runs the
// same finalisation as gate_kernel: probabilities, slot remap, in-tile
// ranks, outputs, tile histogram (+ the folded capacity scan).
#pragma once
// (included inside namespace comoe)

constexpr int kTmKbPerStage = 2;   // 64-d k-blocks per ring stage
constexpr uint32_t kTmAccCol = 384;  // D columns [384, 512); A (router) in [0, d/2)

template <int kStages>
struct GateTmSmem {
  static constexpr int kBoxBytes = 64 * kGemmBK * 2;             // 64 token rows x 64 d
  static constexpr int kStageBytes = kTmKbPerStage * kBoxBytes;  // 16 KB
  static constexpr int kRingBytes = kStages * kStageBytes;
  static constexpr int kStashFloats = 128 * 64;                  // [128 tokens][64 experts]
  static constexpr int kStashBytes = 2 * kStashFloats * 4;       // double-buffered (router staging at start)
  static constexpr int kPartBytes = 2 * 2 * 128 * 8 * 4;         // own + peer partials [2][128][8]
  static constexpr int kCntBytes = kGateMaxK * 4 * kGateMaxE * 4;
  static constexpr int kMapBytes = kGateMaxE * 4;
  static constexpr int kBars = 2 * kStages + 24;
  static constexpr int kTotal =
      1024 + kRingBytes + kStashBytes + kPartBytes + kCntBytes + kMapBytes + kBars * 8 + 16;
};
constexpr int kTmRouterRounds = 3;  // router -> TMEM in rounds of 4 64-d chunks (d <= 768)

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(cta));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote_release(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
// D[tmem] (+)= A[tmem] . B[smem]^T on the CTA pair (M = 256: 128 A rows per SM)
__device__ __forceinline__ void umma_ts_bf16_2sm(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                                 uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// Stash float index of (token t, local expert e): 16-byte chunks XOR-swizzled
// by g(t) (bits 0 and 2 of t swapped, bit 1 kept) so the drain (16 experts of
// two consecutive tokens per warp store) and the token pass (16 tokens x 2
// halves, one chunk each) are both bank-conflict-free.
__device__ __forceinline__ int tm_stash_idx(int t, int e) {
  const int g = ((t & 1) << 2) | (t & 2) | ((t >> 2) & 1);
  return t * 64 + ((((e >> 2) ^ g)) << 2) + (e & 3);
}

// One token's partial over a set of experts: top-2 (value, id) and the
// softmax max / sum.
struct TmPart {
  float v1, v2, m, s;
  int i1, i2;
};
__device__ __forceinline__ void tm_part_store(uint32_t* dst, const TmPart& a) {
  *reinterpret_cast<uint4*>(dst) = make_uint4(__float_as_uint(a.v1), static_cast<uint32_t>(a.i1),
                                              __float_as_uint(a.v2), static_cast<uint32_t>(a.i2));
  *reinterpret_cast<uint2*>(dst + 4) = make_uint2(__float_as_uint(a.m), __float_as_uint(a.s));
}
__device__ __forceinline__ TmPart tm_part_load(const uint32_t* src) {
  const uint4 a = *reinterpret_cast<const uint4*>(src);
  const uint2 b = *reinterpret_cast<const uint2*>(src + 4);
  TmPart r;
  r.v1 = __uint_as_float(a.x); r.i1 = static_cast<int>(a.y);
  r.v2 = __uint_as_float(a.z); r.i2 = static_cast<int>(a.w);
  r.m = __uint_as_float(b.x); r.s = __uint_as_float(b.y);
  return r;
}
// merge b (higher expert ids) into a
__device__ __forceinline__ void tm_part_merge(TmPart& a, const TmPart& b, bool need_sum) {
  constexpr float kLog2e = 1.4426950408889634f;
  GateTop2 x, y;
  x.v1 = a.v1; x.i1 = a.i1; x.v2 = a.v2; x.i2 = a.i2;
  y.v1 = b.v1; y.i1 = b.i1; y.v2 = b.v2; y.i2 = b.i2;
  gate_top2_merge(x, y, a.v1, a.i1, a.v2, a.i2);
  if (need_sum) {
    const float mt = fmaxf(a.m, b.m);
    a.s = (a.m == -INFINITY ? 0.f : a.s * ex2_approx((a.m - mt) * kLog2e)) +
          (b.m == -INFINITY ? 0.f : b.s * ex2_approx((b.m - mt) * kLog2e));
    a.m = mt;
  }
}

template <int kStages>
__global__ void __launch_bounds__(kGateThreads, 1)
    gate_tm_kernel(const __grid_constant__ CUtensorMap tmap_x,
                   const __grid_constant__ CUtensorMap tmap_r, GateParams p) {
  using S = GateTmSmem<kStages>;
  constexpr uint32_t kIdesc = umma_idesc_bf16_f32(256, 128);
  constexpr float kLog2e = 1.4426950408889634f;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* ring = smem;
  float* stash = reinterpret_cast<float*>(smem + S::kRingBytes);
  uint32_t* own = reinterpret_cast<uint32_t*>(smem + S::kRingBytes + S::kStashBytes);  // [2][128][8]
  uint32_t* xch = own + 2 * 128 * 8;  // [2][128][8], SM0: SM1's partials (written over DSMEM)
  int* cnt = reinterpret_cast<int*>(xch + 2 * 128 * 8);
  int* smap = cnt + kGateMaxK * 4 * kGateMaxE;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smap + kGateMaxE);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* b0 = empty_bar + kStages;
  uint64_t* router_bar = b0;          // [3] leader's copies: router round r in both CTAs' TMEM
  uint64_t* stage_bar = b0 + 3;       // [3] local: router round r staged in shared memory
  uint64_t* tfull_bar = b0 + 6;       // MMA commit (multicast to both CTAs)
  uint64_t* tempty_bar = b0 + 7;      // leader's copy: both CTAs drained TMEM
  uint64_t* stash_full = b0 + 8;      // [2]
  uint64_t* stash_empty = b0 + 10;    // [2]
  uint64_t* own_full = b0 + 12;       // [2] SM0: own partials written
  uint64_t* own_empty = b0 + 14;      // [2] SM0: finalise has read them
  uint64_t* xch_full = b0 + 16;       // [2] SM0: SM1's partials arrived
  uint64_t* xch_empty = b0 + 18;      // [2] SM1: SM0 has read them
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(b0 + 20);

  const long long tl0 = clock64();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int k_blocks = p.d / kGemmBK;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int n_units = p.ntiles;  // one unit = one 128-token tile
  const int unit0 = static_cast<int>(blockIdx.x >> 1);
  const int unit_step = static_cast<int>(gridDim.x >> 1);
  const bool need_sum = !p.norm_topk;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_x);
    tma_prefetch_desc(&tmap_r);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 2);
      mbar_init(&empty_bar[s], 1);
    }
    for (int r = 0; r < kTmRouterRounds; ++r) {
      mbar_init(&router_bar[r], 16);  // 8 epilogue warps x 2 CTAs
      mbar_init(&stage_bar[r], 1);
    }
    mbar_init(tfull_bar, 1);
    mbar_init(tempty_bar, 8);  // 4 drain warps x 2 CTAs
    for (int b = 0; b < 2; ++b) {
      mbar_init(&stash_full[b], 128);
      mbar_init(&stash_empty[b], 256);
      // every thread that writes or reads an exchange slot arrives itself
      // (a lane-0 arrive after __syncwarp is also ordered, but this form is
      // the one compute-sanitizer racecheck models)
      mbar_init(&own_full[b], 256);
      mbar_init(&own_empty[b], 128);
      mbar_init(&xch_full[b], 256);
      mbar_init(&xch_empty[b], 128);
    }
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
  __shared__ uint32_t s_ep;
  if (threadIdx.x == 0 && p.lb) s_ep = *reinterpret_cast<volatile unsigned int*>(p.lb_ctrl) + 1u;
  for (int e = threadIdx.x; e < kGateMaxE; e += blockDim.x)
    smap[e] = e < p.E ? (p.slot_map ? __ldg(p.slot_map + e) : e) : -1;
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t ep = p.lb ? s_ep : 0u;
  if (threadIdx.x == 0) gate_tl(p, tl0, 1, 0);

  if (warp == 0) {
    // ------------------------------------------------ TMA producer (both CTAs)
    if (elect_one()) {
      const uint64_t pol_x = l2_policy_evict_last();  // the permute re-reads x next
      int stage = 0;
      uint32_t phase = 0;
      for (int u = unit0; u < n_units; u += unit_step) {
        for (int kb = 0; kb < k_blocks; kb += kTmKbPerStage) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (kb == 0) gate_tl(p, tl0, 2, u);
          const uint32_t fb = smem_u32(&full_bar[stage]) & kPeerMask;
          if (leader) mbar_expect_tx(&full_bar[stage], 2 * S::kStageBytes);
          else mbar_arrive_cluster(fb);
#pragma unroll
          for (int j = 0; j < kTmKbPerStage; ++j)
            tma_load_2d_2sm(ring + stage * S::kStageBytes + j * S::kBoxBytes, &tmap_x, fb,
                            (kb + j) * kGemmBK, u * kGemmBM + static_cast<int>(rank) * 64, pol_x);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (leader only)
    if (leader && elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = unit0; u < n_units; u += unit_step, ++it) {
        mbar_wait(tempty_bar, (it & 1) ^ 1);
        tc_fence_after();
        gate_tl(p, tl0, 4, u);
        const uint32_t d_tmem = tmem_base + kTmAccCol;
        for (int kb = 0; kb < k_blocks; kb += kTmKbPerStage) {
          if (it == 0 && kb % 4 == 0) {  // first tile: router round kb/4 in TMEM
            mbar_wait(&router_bar[kb / 4], 0);
            tc_fence_after();
          }
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (kb == 0) gate_tl(p, tl0, 5, u);
#pragma unroll
          for (int j = 0; j < kTmKbPerStage; ++j) {
            const uint64_t bdesc =
                umma_desc_k_sw128(smem_u32(ring + stage * S::kStageBytes + j * S::kBoxBytes));
#pragma unroll
            for (int k = 0; k < kGemmBK / 16; ++k) {
              const int ks = (kb + j) * (kGemmBK / 16) + k;  // global 16-deep k-step
              umma_ts_bf16_2sm(d_tmem, tmem_base + static_cast<uint32_t>(ks) * 8, bdesc + 2 * k,
                               kIdesc, ks != 0);
            }
          }
          umma_commit_2sm_mc(&empty_bar[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        umma_commit_2sm_mc(tfull_bar);
        gate_tl(p, tl0, 6, u);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue warps 4-11
    // TMEM lane quarter q = warp % 4. Row layout of A (and D): lane 32q + l
    // holds expert 64*rank + 16q + (l % 16), term l / 16 (0 = hi, 1 = mid), so
    // a warp adds the two partial logits of an expert with one shuffle.
    const int q = warp & 3;
    const bool drain = warp < 8;
    const bool lo = lane < 16;
    const int el = 16 * q + (lane & 15);  // local expert of this lane's TMEM row
    {
      // router -> TMEM through the (still idle) stash: per round one TMA of
      // four 64-d chunks x the 8 (quarter, term) 16-row blocks of this SM,
      // 128B-swizzled; each thread copies its own row into its TMEM lane
      // (K packed two bf16 per 32-bit column). Warps 4-7 copy chunks 0-1 of
      // a round, warps 8-11 chunks 2-3.
      const int n_chunks = p.d / 64;
      const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
      uint8_t* rst = reinterpret_cast<uint8_t*>(stash);
      for (int r = 0; r * 4 < n_chunks; ++r) {
        const int nc = min(4, n_chunks - 4 * r);
        if (warp == 4 && lane == 0) {
          mbar_expect_tx(&stage_bar[r], nc * 8 * 2048);
          for (int c = 0; c < nc; ++c)
            for (int qq = 0; qq < 4; ++qq)
              for (int term = 0; term < 2; ++term)
                tma_load_2d(rst + ((c * 4 + qq) * 2 + term) * 2048, &tmap_r, &stage_bar[r],
                            (4 * r + c) * 64, term * 128 + 64 * static_cast<int>(rank) + 16 * qq);
        }
        mbar_wait(&stage_bar[r], 0);
        const int R = lane & 15, term = lane >> 4;
        for (int c = drain ? 0 : 2; c < (drain ? 2 : 4); ++c) {
          if (c >= nc) break;
          const uint8_t* box = rst + ((c * 4 + q) * 2 + term) * 2048 + R * 128;
          uint32_t v[32];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint4 w = *reinterpret_cast<const uint4*>(box + ((j ^ (R & 7)) << 4));
            v[4 * j] = w.x; v[4 * j + 1] = w.y; v[4 * j + 2] = w.z; v[4 * j + 3] = w.w;
          }
          tmem_st32(t_lane + (4 * r + c) * 32, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_u32(smem_u32(&router_bar[r]), 0));
        named_bar_sync(2, 256);  // the staging area is read: next round may overwrite it
      }
      for (int r = (n_chunks + 3) / 4; r < kTmRouterRounds; ++r) {  // unused rounds (d < 768)
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_u32(smem_u32(&router_bar[r]), 0));
      }
    }
    const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + kTmAccCol;
    // token pass: thread (token tt, expert half hh) of warp w8 = warp - 4
    const int w8 = warp - 4;
    const int tt = w8 * 16 + (lane & 15);
    const int hh = lane >> 4;
    const int gsw = ((tt & 1) << 2) | (tt & 2) | ((tt >> 2) & 1);
    const int e0 = 64 * static_cast<int>(rank) + 32 * hh;  // first expert of this thread
    // finalisation (SM0, warps 8-11): thread = token ft of the tile
    const int fq = warp - 8;
    const int ft = fq * 32 + lane;
    const uint32_t lt_mask = (1u << lane) - 1u;

    // SM0 finalisation of the tile finished one iteration earlier (its own
    // and SM1's partials have had a whole tile to arrive)
    auto finalize = [&](int fu, int fit) {
      const int b = fit & 1;
      const uint32_t par = (fit >> 1) & 1;
      mbar_wait(&own_full[b], par);
      mbar_wait_cluster(&xch_full[b], par);
      TmPart a = tm_part_load(own + (b * 128 + ft) * 8);
      const TmPart c = tm_part_load(xch + (b * 128 + ft) * 8);
      mbar_arrive(&own_empty[b]);
      mbar_arrive_remote_release(mapa_u32(smem_u32(&xch_empty[b]), 1));
      tm_part_merge(a, c, need_sum);  // SM0's experts have the lower ids
      const float s = need_sum ? a.s : 1.f;
      const int t = fu * kGemmBM + ft;
      const bool valid = t < p.T;
      float pr0, pr1 = 0.f;
      if (p.top_k == 1) {
        pr0 = p.norm_topk ? 1.f : 1.f / s;
      } else if (p.norm_topk) {
        const float z = expf(a.v2 - a.v1);
        pr0 = 1.f / (1.f + z);
        pr1 = z / (1.f + z);
      } else {
        pr0 = 1.f / s;
        pr1 = expf(a.v2 - a.v1) / s;
      }
      int gr0 = (valid && a.i1 >= 0) ? smap[a.i1] : -1;
      int gr1 = (valid && p.top_k == 2 && a.i2 >= 0) ? smap[a.i2] : -1;
      if (gr1 >= 0 && gr1 == gr0) {
        pr0 += pr1;
        pr1 = 0.f;
        gr1 = -1;
      }
      named_bar_sync(1, 128);
      for (int i = ft; i < p.top_k * 4 * kGateMaxE; i += 128) cnt[i] = 0;
      named_bar_sync(1, 128);
      int wr0, wr1 = 0;
      {
        const unsigned mm0 = __match_any_sync(0xffffffffu, gr0);
        wr0 = __popc(mm0 & lt_mask);
        if (gr0 >= 0 && wr0 == 0) cnt[fq * kGateMaxE + gr0] = __popc(mm0);
        if (p.top_k == 2) {
          const unsigned mm1 = __match_any_sync(0xffffffffu, gr1);
          wr1 = __popc(mm1 & lt_mask);
          if (gr1 >= 0 && wr1 == 0) cnt[(4 + fq) * kGateMaxE + gr1] = __popc(mm1);
        }
      }
      named_bar_sync(1, 128);
      if (valid) {
        int rank0 = -1, rank1 = -1;
        if (gr0 >= 0) {
          rank0 = wr0;
          for (int qq = 0; qq < fq; ++qq) rank0 += cnt[qq * kGateMaxE + gr0];
        }
        if (gr1 >= 0) {
          rank1 = wr1;
          for (int qq = 0; qq < fq; ++qq) rank1 += cnt[(4 + qq) * kGateMaxE + gr1];
        }
        const long o = static_cast<long>(t) * p.top_k;
        p.expert_idx[o] = a.i1;
        p.group_idx[o] = gr0;
        p.gate_prob[o] = gr0 >= 0 ? pr0 : 0.f;
        p.local_rank[o] = rank0;
        if (p.top_k == 2) {
          p.expert_idx[o + 1] = a.i2;
          p.group_idx[o + 1] = gr1;
          p.gate_prob[o + 1] = gr1 >= 0 ? pr1 : 0.f;
          p.local_rank[o + 1] = rank1;
        }
      }
      for (int j = 0; j < p.top_k; ++j)
        for (int g = ft; g < p.G; g += 128) {
          int h = 0;
          if (g < kGateMaxE)
            for (int qq = 0; qq < 4; ++qq) h += cnt[(j * 4 + qq) * kGateMaxE + g];
          gate_publish_hist(p, j, fu, g, h, ep);
        }
      if (lane == 0 && fq == 0) gate_tl(p, tl0, 9, fu);
    };

    int it = 0, prev_u = -1;
    for (int u = unit0; u < n_units; u += unit_step, ++it) {
      const int buf = it & 1;
      const uint32_t par = (it >> 1) & 1;
      float* sb = stash + buf * S::kStashFloats;
      if (drain) {
        // TMEM -> stash[buf]: logit = hi + mid, two tokens per shuffle
        mbar_wait(tfull_bar, it & 1);
        tc_fence_after();
        if (lane == 0 && q == 0) gate_tl(p, tl0, 7, u);
        mbar_wait(&stash_empty[buf], par ^ 1);
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2) {
          uint32_t v[2][32];
          tmem_ld32(t_row + c2 * 64, v[0]);
          tmem_ld32(t_row + c2 * 64 + 32, v[1]);
          tmem_ld_wait();
          if (c2 == 1) {  // accumulator drained: the next tile's MMAs may start
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_u32(smem_u32(tempty_bar), 0));
            if (lane == 0 && q == 0) gate_tl(p, tl0, 8, u);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int jj = 0; jj < 32; jj += 2) {
              const float a = __uint_as_float(v[h][jj]), b = __uint_as_float(v[h][jj + 1]);
              const float recv = __shfl_xor_sync(0xffffffffu, lo ? b : a, 16);
              const int tok = c2 * 64 + h * 32 + jj + (lo ? 0 : 1);
              sb[tm_stash_idx(tok, el)] = (lo ? a : b) + recv;  // hi + mid (commutative)
            }
        }
        mbar_arrive(&stash_full[buf]);
        if (lane == 0 && q == 0) gate_tl(p, tl0, 13, u);
      }
      // ---- token pass (8 warps, 16 tokens each): 32 experts of token tt per thread
      const int t = u * kGemmBM + tt;
      mbar_wait(&stash_full[buf], par);
      float v[32];
      const float* srow = sb + tt * 64;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 x4 = *reinterpret_cast<const float4*>(srow + (((8 * hh + i) ^ gsw) << 2));
        v[4 * i] = x4.x; v[4 * i + 1] = x4.y; v[4 * i + 2] = x4.z; v[4 * i + 3] = x4.w;
      }
      mbar_arrive(&stash_empty[buf]);
      if (lane == 0 && w8 == 0) gate_tl(p, tl0, 14, u);
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (e0 + j >= p.E) v[j] = -INFINITY;
      if (p.logits && t < p.T) {
        float* lrow = p.logits + static_cast<long>(t) * p.E;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (e0 + j < p.E) lrow[e0 + j] = v[j];
      }
      TmPart pa;
      {
        GateTop2 ta, tb;
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          ta.push(v[j], e0 + j);
          tb.push(v[j + 1], e0 + j + 1);
        }
        gate_top2_merge(ta, tb, pa.v1, pa.i1, pa.v2, pa.i2);
        pa.m = pa.v1;  // two-pass softmax denominator over the 32 experts
        pa.s = 0.f;
        if (need_sum && pa.m != -INFINITY) {
          const float mb = pa.m * kLog2e;
          float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int j = 0; j < 32; ++j) s4[j & 3] += ex2_approx(fmaf(v[j], kLog2e, -mb));
          pa.s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
        }
      }
      {  // merge the two expert halves of the token (lanes l and l ^ 16)
        TmPart pb;
        pb.v1 = __shfl_xor_sync(0xffffffffu, pa.v1, 16);
        pb.i1 = __shfl_xor_sync(0xffffffffu, pa.i1, 16);
        pb.v2 = __shfl_xor_sync(0xffffffffu, pa.v2, 16);
        pb.i2 = __shfl_xor_sync(0xffffffffu, pa.i2, 16);
        pb.m = __shfl_xor_sync(0xffffffffu, pa.m, 16);
        pb.s = __shfl_xor_sync(0xffffffffu, pa.s, 16);
        if (lo) tm_part_merge(pa, pb, need_sum);  // lo lanes hold the lower half
      }
      if (lane == 0 && w8 == 0) gate_tl(p, tl0, 15, u);
      if (!leader) {
        // SM1: partials over experts 64..127 into SM0's exchange buffer
        mbar_wait_cluster(&xch_empty[buf], par ^ 1);
        if (lo) {
          const uint32_t dst = mapa_u32(smem_u32(xch + (buf * 128 + tt) * 8), 0);
          asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst),
                       "r"(__float_as_uint(pa.v1)), "r"(static_cast<uint32_t>(pa.i1)),
                       "r"(__float_as_uint(pa.v2)), "r"(static_cast<uint32_t>(pa.i2))
                       : "memory");
          asm volatile("st.shared::cluster.v2.b32 [%0], {%1, %2};" ::"r"(dst + 16),
                       "r"(__float_as_uint(pa.m)), "r"(__float_as_uint(pa.s))
                       : "memory");
        }
        mbar_arrive_remote_release(mapa_u32(smem_u32(&xch_full[buf]), 0));
        if (lane == 0 && w8 == 0) gate_tl(p, tl0, 17, u);
        continue;
      }
      // SM0: own partials for the lagged finalisation
      mbar_wait(&own_empty[buf], par ^ 1);
      if (lo) tm_part_store(own + (buf * 128 + tt) * 8, pa);
      mbar_arrive(&own_full[buf]);
      if (!drain && prev_u >= 0) finalize(prev_u, it - 1);
      prev_u = u;
    }
    if (leader && !drain && prev_u >= 0) finalize(prev_u, it - 1);
  }

  if (threadIdx.x == 0 || threadIdx.x == 32 || threadIdx.x == 128 || threadIdx.x == 256)
    gate_tl(p, tl0, 10, warp);
  tc_fence_before();
  cluster_sync_all();
  if (threadIdx.x == 0) gate_tl(p, tl0, 11, 0);
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base)
                 : "memory");
  }
  if (p.lb) gate_fold_scan(p, ep);
  if (threadIdx.x == 0) gate_tl(p, tl0, 12, 0);
}

template <int kStages>
static int launch_gate_tm(const CUtensorMap& tx, const CUtensorMap& tr, const GateParams& p,
                          cudaStream_t stream) {
  using S = GateTmSmem<kStages>;
  static_assert(S::kTotal <= 227 * 1024, "gate_tm shared memory");
  auto kern = gate_tm_kernel<kStages>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kTotal);
    attr = true;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kGateThreads);
  cfg.dynamicSmemBytes = S::kTotal;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  static int max_pairs = -1;  // co-resident pairs (the folded scan's grid barrier)
  if (max_pairs < 0) {
    cfg.gridDim = dim3(sms);
    cfg.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess || clusters < 1) {
      cudaGetLastError();
      clusters = sms / 2;
    }
    max_pairs = clusters < sms / 2 ? clusters : sms / 2;
  }
  const int pairs = p.ntiles < max_pairs ? p.ntiles : max_pairs;
  cfg.gridDim = dim3(2 * pairs);
  cfg.numAttrs = 1 + pdl_attr(&attrs[1]);
  cudaLaunchKernelEx(&cfg, kern, tx, tr, p);
  return check_launch("gate_tm_kernel");
}

