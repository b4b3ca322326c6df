// K1 gate + routing scan.
//
// The reference has no router: routing decisions come from the synthetic
// Zipf/rho generator (pkg/src/comoe/moe.py:186-230) and are remapped to the
// merged expert set by ModelVariant.resolve (pkg/src/comoe/aggregation.py:101-103).
// Here the router is real: fp32 logits x.Wg on the tensor cores, softmax,
// top-k on the logits (ties -> lowest expert index, the reference's universal
// tie rule, aggregation.py:165,193), slot remap through the variant's
// slot_map, and per-tile token-order ranks that feed deterministic capacity.
//
// fp32-router logits on bf16 tensor cores: X is bf16 (exact); the fp32
// router weight is split Wg = hi + mid + lo with each term bf16 (exactly),
// so every product x*term is exact in the fp32 accumulator; the MMAs over
// the first gate_terms() terms sum to the fp32 logit up to accumulation
// rounding (2 terms: ~3e-7 at d = 768, see gate_terms()).
#include <cooperative_groups.h>
#include <cstdlib>

#include "grouped_gemm_2sm.cuh"
#include "../../include/comoe_b200.h"

namespace comoe {

constexpr int kGateMaxE = 128;
constexpr int kGateMaxK = 2;
// w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4-7 epilogue group 0 (accumulator 0,
// even tiles of this CTA), w8-11 epilogue group 1 (accumulator 1, odd tiles):
// two softmax/top-k/rank epilogues in flight per SM so the tensor core is not
// paced by one (profiles: the MMA warp waited on tmem_empty with one group).
constexpr int kGateThreads = 384;

// ------------------------------------------------------------ weight split
__global__ void gate_split_kernel(const float* __restrict__ wg, int d, int E, int EP,
                                  __nv_bfloat16* __restrict__ out) {
  const long n = static_cast<long>(EP) * d;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const int e = static_cast<int>(i / d), k = static_cast<int>(i % d);
    const float w = e < E ? wg[static_cast<long>(k) * E + e] : 0.f;  // Wg is [d, E]
    const __nv_bfloat16 hi = __float2bfloat16_rn(w);
    const float r1 = w - __bfloat162float(hi);
    const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
    const float r2 = r1 - __bfloat162float(mid);
    const __nv_bfloat16 lo = __float2bfloat16_rn(r2);
    out[i] = hi;
    out[n + i] = mid;
    out[2 * n + i] = lo;
  }
}

struct GateParams {
  int T, d, E, top_k, norm_topk, G, ntiles;
  const int* slot_map;  // [E] -> group, may be null (identity)
  float* logits;        // [T, E] optional
  int* expert_idx;      // [T, k]
  int* group_idx;       // [T, k]  (-1: no assignment)
  float* gate_prob;     // [T, k]
  int* local_rank;      // [T, k]
  int* tile_hist;       // [k][ntiles][G]
  int debug;            // dev attribution (COMOE_GATE_DEBUG): 1 no router loads, 2 x from tile 0, 4 no x loads
  // Folded capacity scan (comoe_gate_route; lb == null: histograms only).
  // The epilogue stores each tile's group histogram group-major and adds it
  // to the per-group totals; after the last tile every CTA meets at a grid
  // barrier (the persistent grid is co-resident), scans whole histogram
  // columns into stream-order tile offsets, and one CTA turns the totals
  // into count / kept / base. A device-side epoch advances once per launch
  // and selects the parity of the barrier counter and totals, which that
  // launch zeroes for the next one: the workspace is zero-filled once and
  // never reset again (CUDA-graph replays included).
  int* lb;                // [G][k * ntiles] histograms, group-major
  unsigned int* lb_ctrl;  // [0] epoch of the last completed launch, [2 + parity] barrier arrivals
  int* lb_total;          // [2 parities][kGateMaxE] assignments per group
  int* tile_offset;       // [k][ntiles][G] exclusive stream-order prefix
  int* group_count;       // [G]
  int* group_kept;        // [G]
  int* group_base;        // [G]
  int capacity;
  int xpol;  // dev: L2 policy of the x loads (0 evict_last, 1 normal, 2 first)
};

// ------------------------------------------------------------ folded scan
// Publish one tile's histogram entry: group-major plus the running total for
// the folded scan, the [k][ntiles][G] histogram for comoe_gate_topk +
// comoe_route_scan.
__device__ __forceinline__ void gate_publish_hist(const GateParams& p, int j, int tile, int g,
                                                  int h, uint32_t ep) {
  if (p.lb) {
    p.lb[static_cast<long>(g) * p.top_k * p.ntiles + static_cast<long>(j) * p.ntiles + tile] = h;
    if (h) atomicAdd(p.lb_total + (ep & 1u) * kGateMaxE + g, h);
  } else {
    p.tile_hist[(static_cast<long>(j) * p.ntiles + tile) * p.G + g] = h;
  }
}

__device__ __forceinline__ unsigned int ld_acquire_gpu_u32(const unsigned int* a) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu_add(unsigned int* a, unsigned int v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

// dev timeline (COMOE_GATE_DEBUG bit 256): CTAs 0 and 1 (one pair) stamp
// clock64 - entry at slot [code][unit iteration] (plain stores, no atomics,
// so the stamps do not delay the warps they time); comoe_debug_gate_timeline
// copies them out
constexpr int kGateTlMax = 1024;
constexpr int kGateTlIters = 32;
static __device__ unsigned long long g_gate_tl[2][kGateTlMax];
__device__ __forceinline__ void gate_tl(const GateParams& p, long long t0, int code, int u) {
  if (!(p.debug & 256) || blockIdx.x > 1) return;
  // codes 1, 10-12 carry a raw value (warp); the rest a unit -> its iteration
  const int iter = (code == 1 || (code >= 10 && code <= 12)) ? u : u / static_cast<int>(gridDim.x >> 1);
  if (iter >= kGateTlIters) return;
  g_gate_tl[blockIdx.x][code * kGateTlIters + iter] = static_cast<unsigned long long>(clock64() - t0) + 1ull;
}

constexpr int kFoldPer = 4;  // histogram entries per thread loaded before the scan

// After the main loop (all kGateThreads threads of every CTA): grid barrier,
// column scans in stream order (all first choices in token order, then all
// second choices), and count / kept / base from the per-group totals. Same
// results as route_scan_coop below.
__device__ __forceinline__ void gate_fold_scan(const GateParams& p, uint32_t ep) {
  __shared__ int warp_tot[kGateThreads / 32];
  unsigned int* arrivals = p.lb_ctrl + 2 + (ep & 1u);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();  // the CTA's histogram stores and totals, before the arrival
    red_release_gpu_add(arrivals, 1u);
    while (ld_acquire_gpu_u32(arrivals) < gridDim.x) {
    }
  }
  __syncthreads();
  const int S = p.top_k * p.ntiles;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int nw = kGateThreads / 32;
  // the CTA that finalises the totals: the last one when it has no column
  const int fin = static_cast<int>(gridDim.x) > p.G ? static_cast<int>(gridDim.x) - 1 : 0;
  if (static_cast<int>(blockIdx.x) == fin) {
    if (threadIdx.x < 128) {
      const int g = threadIdx.x;
      const int cnt = g < p.G ? __ldcg(p.lb_total + (ep & 1u) * kGateMaxE + g) : 0;
      const int kept = min(cnt, p.capacity);
      int v = kept;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
      }
      if (lane == 31) warp_tot[w] = v;
      named_bar_sync(1, 128);
      int base = v - kept;
      for (int i = 0; i < w; ++i) base += warp_tot[i];
      if (g < p.G) {
        p.group_count[g] = cnt;
        p.group_kept[g] = kept;
        p.group_base[g] = base;
      }
      // the next launch's totals and barrier start from zero
      p.lb_total[((ep + 1u) & 1u) * kGateMaxE + g] = 0;
      if (g == 0) {
        p.lb_ctrl[2 + ((ep + 1u) & 1u)] = 0u;
        p.lb_ctrl[0] = ep;
      }
    }
    __syncthreads();
  }
  for (int g = blockIdx.x; g < p.G; g += gridDim.x) {
    const int* col = p.lb + static_cast<long>(g) * S;
    int carry = 0;
    for (int b0 = 0; b0 < S; b0 += kFoldPer * kGateThreads) {
      int x[kFoldPer];
#pragma unroll
      for (int c = 0; c < kFoldPer; ++c) {  // every load in flight before the scan
        const int s = b0 + c * kGateThreads + threadIdx.x;
        x[c] = s < S ? __ldcg(col + s) : 0;
      }
#pragma unroll
      for (int c = 0; c < kFoldPer; ++c) {
        if (b0 + c * kGateThreads >= S) break;
        const int s = b0 + c * kGateThreads + threadIdx.x;
        int v = x[c];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int n = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += n;
        }
        if (lane == 31) warp_tot[w] = v;
        __syncthreads();
        int wb = 0, tot = 0;
#pragma unroll
        for (int i = 0; i < nw; ++i) {
          if (i < w) wb += warp_tot[i];
          tot += warp_tot[i];
        }
        if (s < S) p.tile_offset[static_cast<long>(s) * p.G + g] = carry + wb + v - x[c];
        carry += tot;
        __syncthreads();
      }
    }
  }
}

// kPair: CTA pair (cta_group::2, M = 256 tokens): each SM stages its own 128
// tokens and half of every router term (EP/2 experts), cutting per-SM shared-
// memory traffic ~30% (the 1-SM gate is smem-bound: the token tile is re-read
// once per term); each SM's TMEM still holds full logit rows of its tokens.
template <int EP, int kStages, bool kPair = false, int kTerms = 3>
struct GateSmem {
  static constexpr int kBRows = kPair ? EP / 2 : EP;
  static constexpr int kABytes = kGemmBM * kGemmBK * 2;
  static constexpr int kBBytes = kTerms * kBRows * kGemmBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTileBytes = kStages * kStageBytes;
  static constexpr int kCtrlBytes = (2 * kStages + 4) * 8 + 16 + 2 * kGateMaxK * 4 * kGateMaxE * 4 + kGateMaxE * 4;
  static constexpr int kTotal = 1024 + kTileBytes + kCtrlBytes;
};

// kCat (pair, two terms): the two router terms are one N = 2*EP operand —
// CTA rank r stages term r for every expert, so D[:, e] = x.hi_e and
// D[:, EP+e] = x.mid_e and logit_e = D[:, e] + D[:, EP+e] (one fp32 add in
// the epilogue). One MMA per k-step instead of one per term: the token tile
// is read from shared memory once, not once per term (the per-term form kept
// the tensor pipe ~50% busy with the TMA ring full: profiles/r1_ncu_gate_*).
// Running top-2 of (value, expert id) for ascending ids (strict '>': the
// lowest id wins ties).
struct GateTop2 {
  float v1 = -INFINITY, v2 = -INFINITY;
  int i1 = -1, i2 = -1;
  __device__ __forceinline__ void push(float v, int e) {
    const bool g1 = v > v1, g2 = v > v2;
    v2 = g1 ? v1 : (g2 ? v : v2);
    i2 = g1 ? i1 : (g2 ? e : i2);
    v1 = g1 ? v : v1;
    i1 = g1 ? e : i1;
  }
};
// (va, ia) ranks before (vb, ib): larger value, then lower id; an empty entry
// (id -1) ranks last.
__device__ __forceinline__ bool gate_before(float va, int ia, float vb, int ib) {
  return va > vb || (va == vb && static_cast<unsigned>(ia) < static_cast<unsigned>(ib));
}
__device__ __forceinline__ void gate_top2_merge(const GateTop2& a, const GateTop2& b, float& v1,
                                                int& i1, float& v2, int& i2) {
  if (gate_before(a.v1, a.i1, b.v1, b.i1)) {
    v1 = a.v1; i1 = a.i1;
    const bool x = gate_before(a.v2, a.i2, b.v1, b.i1);
    v2 = x ? a.v2 : b.v1; i2 = x ? a.i2 : b.i1;
  } else {
    v1 = b.v1; i1 = b.i1;
    const bool x = gate_before(a.v1, a.i1, b.v2, b.i2);
    v2 = x ? a.v1 : b.v2; i2 = x ? a.i1 : b.i2;
  }
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Chunk loads for the pipelined epilogue: 16 columns (plus the 16 mid-term
// columns EP further with kCat) issued without waiting; gate_ld_wait names
// the destination registers so the compiler cannot read them before the wait.
template <bool kCat, int EP>
__device__ __forceinline__ void gate_ld_chunk(uint32_t col, uint32_t (&r)[kCat ? 32 : 16]) {
  tmem_ld16(col, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
  if constexpr (kCat) tmem_ld16(col + EP, *reinterpret_cast<uint32_t(*)[16]>(&r[16]));
}
template <bool kCat>
__device__ __forceinline__ void gate_ld_wait(uint32_t (&r)[kCat ? 32 : 16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]),
                 "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]),
                 "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
  if constexpr (kCat)
    asm volatile(""
                 : "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                   "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]),
                   "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
                 :
                 : "memory");
}

// 16 logits of this thread's token starting at TMEM column `col`; with kCat
// the hi and mid partial logits sit EP columns apart and are summed here.
template <bool kCat, int EP>
__device__ __forceinline__ void gate_logits16(uint32_t col, uint32_t (&r)[16]) {
  tmem_ld16(col, r);
  if constexpr (kCat) {
    uint32_t m[16];
    tmem_ld16(col + EP, m);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) + __uint_as_float(m[j]));
  } else {
    tmem_ld_wait();
  }
}

template <int EP, int kStages, bool kPair, int kTerms>
__global__ void __launch_bounds__(kGateThreads, 1)
    gate_kernel(const __grid_constant__ CUtensorMap tmap_x,
                const __grid_constant__ CUtensorMap tmap_w, GateParams p) {
  using S = GateSmem<EP, kStages, kPair, kTerms>;
  constexpr bool kCat = kPair && kTerms == 2;
  constexpr int kAccCols = kCat ? 2 * EP : EP;  // TMEM columns of one accumulator
  constexpr uint32_t kTmemCols =
      2 * kAccCols <= 32 ? 32 : (2 * kAccCols <= 64 ? 64 : (2 * kAccCols <= 128 ? 128 : (2 * kAccCols <= 256 ? 256 : 512)));
  constexpr uint32_t kIdesc = umma_idesc_bf16_f32(kPair ? 256 : kGemmBM, kAccCols);
  constexpr int kBRows = S::kBRows;
  // kSplitEpi: both epilogue groups work on every unit, each on half of the
  // experts of the same tokens (warps 4+q and 8+q share TMEM lane quarter q);
  // group 1 hands its partial top-2 / softmax sum to group 0 through shared
  // memory and group 0 finishes. Halves each unit's epilogue latency, which
  // set the tail of the MMA -> epilogue chain (the alternating-groups form
  // left one full epilogue after the last MMA).
  constexpr bool kSplitEpi = kCat && EP >= 32;
  if (p.debug & 32) return;  // dev: empty launch
  const long long tl0 = clock64();

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + kStages * S::kABytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S::kTileBytes);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int* cnt_all = reinterpret_cast<int*>(tmem_slot + 4);   // [2 groups][kMaxK][4][kGateMaxE]
  int* smap = cnt_all + 2 * kGateMaxK * 4 * kGateMaxE;     // [kGateMaxE]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int k_blocks = p.d / kGemmBK;
  // work units: 128-token tiles (1-SM) or 256-token pair tiles (kPair); this
  // CTA's 128-token tile of unit u is 2u + rank
  const uint32_t rank = kPair ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int n_units = kPair ? (p.ntiles + 1) / 2 : p.ntiles;
  const int unit0 = kPair ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int unit_step = kPair ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_x);
    tma_prefetch_desc(&tmap_w);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], kPair ? 2 : 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], kPair ? (kSplitEpi ? 16 : 8) : 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc<kTmemCols>(tmem_slot);
    }
  }
  pdl_wait();     // x / slot_map may come from the preceding kernel
  pdl_trigger();  // persistent grid: the next kernel may launch and wait
  __shared__ uint32_t s_ep;
  if (threadIdx.x == 0 && p.lb) s_ep = *reinterpret_cast<volatile unsigned int*>(p.lb_ctrl) + 1u;
  for (int e = threadIdx.x; e < kGateMaxE; e += blockDim.x)
    smap[e] = e < p.E ? (p.slot_map ? __ldg(p.slot_map + e) : e) : -1;
  tc_fence_before();
  if constexpr (kPair) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t ep = p.lb ? s_ep : 0u;
  if (threadIdx.x == 0) gate_tl(p, tl0, 1, 0);  // prologue done

  if (p.debug & 64) {  // dev: prologue + epilogue of the kernel only
  } else if (warp == 0) {
    if (elect_one()) {
      // keep x in L2: the permute re-reads every row right after the gate
      // (dev: COMOE_GATE_XPOL=1 evict_normal, 2 evict_first)
      const uint64_t pol_x = p.xpol == 2 ? l2_policy_evict_first()
                             : p.xpol == 1 ? l2_policy_evict_normal() : l2_policy_evict_last();
      const uint64_t pol_w = l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = unit0; u < n_units; u += unit_step) {
        const int tile = kPair ? 2 * u + static_cast<int>(rank) : u;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (kb == 0 || kb == k_blocks - 1) gate_tl(p, tl0, kb == 0 ? 2 : 3, u);
          uint8_t* b = smem_b + stage * S::kBBytes;
          if constexpr (kPair) {
            const uint32_t fb = smem_u32(&full_bar[stage]) & kPeerMask;
            const int dbg = p.debug;
            if (leader)
              mbar_expect_tx(&full_bar[stage], 2 * ((dbg & 4 ? 0 : S::kABytes) + (dbg & 1 ? 0 : S::kBBytes)));
            else mbar_arrive_cluster(fb);
            if (!(dbg & 4))
              tma_load_2d_2sm(smem_a + stage * S::kABytes, &tmap_x, fb, kb * kGemmBK,
                              (dbg & 2 ? static_cast<int>(rank) : tile) * kGemmBM, pol_x);
            if constexpr (kCat) {
              if (!(dbg & 1))
                tma_load_2d_2sm(b, &tmap_w, fb, kb * kGemmBK, static_cast<int>(rank) * EP, pol_w);
            } else {
#pragma unroll
              for (int term = 0; term < kTerms; ++term)
                tma_load_2d_2sm(b + term * kBRows * 128, &tmap_w, fb, kb * kGemmBK,
                                term * EP + static_cast<int>(rank) * kBRows, pol_w);
            }
          } else {
            mbar_expect_tx(&full_bar[stage], S::kStageBytes);
            tma_load_2d_hint(smem_a + stage * S::kABytes, &tmap_x, &full_bar[stage], kb * kGemmBK,
                             tile * kGemmBM, pol_x);
#pragma unroll
            for (int term = 0; term < kTerms; ++term)
              tma_load_2d(b + term * EP * 128, &tmap_w, &full_bar[stage], kb * kGemmBK, term * EP);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = unit0; u < n_units; u += unit_step, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty_bar[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        gate_tl(p, tl0, 4, u);
        const uint32_t d_tmem = tmem_base + acc * kAccCols;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (kb == 0) gate_tl(p, tl0, 5, u);
          const uint64_t adesc = umma_desc_k_sw128(smem_u32(smem_a + stage * S::kABytes));
#pragma unroll
          for (int term = 0; term < (kCat ? 1 : kTerms); ++term) {
            const uint64_t bdesc =
                umma_desc_k_sw128(smem_u32(smem_b + stage * S::kBBytes + term * kBRows * 128));
#pragma unroll
            for (int k = 0; k < kGemmBK / 16; ++k) {
              if (p.debug & 16) continue;  // dev: no MMAs
              if constexpr (kPair)
                umma_bf16_2sm(d_tmem, adesc + 2 * k, bdesc + 2 * k, kIdesc, (kb | k | term) != 0);
              else
                umma_bf16(d_tmem, adesc + 2 * k, bdesc + 2 * k, kIdesc, (kb | k | term) != 0);
            }
          }
          if constexpr (kPair) umma_commit_2sm_mc(&empty_bar[stage]);
          else umma_commit(&empty_bar[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if constexpr (kPair) umma_commit_2sm_mc(&tfull_bar[acc]);
        else umma_commit(&tfull_bar[acc]);
        gate_tl(p, tl0, 6, u);
      }
    }
  } else if (kSplitEpi && warp >= 4) {
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;  // 0: experts [0, EP/2) and the finish; 1: [EP/2, EP)
    const int et = threadIdx.x - 128;  // 0..127 in group 0
    int* cnt = cnt_all;
    // group 1's counters are unused here: they hold the hand-off [128 tokens][6]
    uint32_t* xch = reinterpret_cast<uint32_t*>(cnt_all + kGateMaxK * 4 * kGateMaxE);
    const uint32_t lt_mask = (1u << lane) - 1u;
    constexpr int kHalf = EP / 2;
    constexpr int kChunks = kHalf / 16;
    constexpr float kLog2e = 1.4426950408889634f;
    const bool need_sum = !p.norm_topk;
    int it = 0;
    for (int u = unit0; u < n_units; u += unit_step, ++it) {
      const int acc = it & 1;
      const int tile = 2 * u + static_cast<int>(rank);
      const bool tile_ok = tile < p.ntiles;
      const int t = tile * kGemmBM + q * 32 + lane;
      const bool valid = tile_ok && t < p.T;
      mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
      tc_fence_after();
      if (lane == 0 && q == 0) gate_tl(p, tl0, 7 + half * 8, u);
      const int e0 = half * kHalf;
      const uint32_t t_row =
          tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * kAccCols + e0;
      GateTop2 ta, tb;
      float m = -INFINITY, s4[2] = {0.f, 0.f};
      float* lrow = (p.logits && valid) ? p.logits + static_cast<long>(t) * p.E : nullptr;
      uint32_t buf[2][32];
      gate_ld_chunk<true, EP>(t_row, buf[0]);
#pragma unroll
      for (int c = 0; c < kChunks; ++c) {
        uint32_t(&cur)[32] = buf[c & 1];
        gate_ld_wait<true>(cur);
        if (c + 1 < kChunks) {
          gate_ld_chunk<true, EP>(t_row + (c + 1) * 16, buf[(c + 1) & 1]);
        } else {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(smem_u32(&tempty_bar[acc]) & kPeerMask);
          if (lane == 0 && q == 0) gate_tl(p, tl0, 8 + half * 8, u);
        }
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int e = e0 + c * 16 + j;
          const float x = __uint_as_float(cur[j]) + __uint_as_float(cur[16 + j]);
          v[j] = e < p.E ? x : -INFINITY;
        }
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          ta.push(v[j], e0 + c * 16 + j);
          tb.push(v[j + 1], e0 + c * 16 + j + 1);
        }
        if (lrow) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (e0 + c * 16 + j < p.E) lrow[e0 + c * 16 + j] = v[j];
        }
        if (need_sum) {
          const float mn = fmaxf(m, fmaxf(ta.v1, tb.v1));
          const float mb = mn * kLog2e;
          const float sc = m == -INFINITY ? 0.f : ex2_approx((m - mn) * kLog2e);
          s4[0] *= sc;
          s4[1] *= sc;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            s4[j & 1] += (mn == -INFINITY) ? 0.f : ex2_approx(fmaf(v[j], kLog2e, -mb));
          m = mn;
        }
      }
      float v1, v2;
      int i1, i2;
      gate_top2_merge(ta, tb, v1, i1, v2, i2);
      float s = s4[0] + s4[1];
      uint32_t* slot = xch + (q * 32 + lane) * 6;
      if (half == 1) {
        slot[0] = __float_as_uint(v1);
        slot[1] = static_cast<uint32_t>(i1);
        slot[2] = __float_as_uint(v2);
        slot[3] = static_cast<uint32_t>(i2);
        slot[4] = __float_as_uint(m);
        slot[5] = __float_as_uint(s);
      }
      named_bar_sync(3 + q, 64);  // half 1's partials are in shared memory
      if (half == 1) {
        named_bar_sync(7 + q, 64);  // group 0 has read them
        if (lane == 0 && q == 0) gate_tl(p, tl0, 17, u);
        continue;
      }
      GateTop2 a0, a1;
      a0.v1 = v1; a0.i1 = i1; a0.v2 = v2; a0.i2 = i2;
      a1.v1 = __uint_as_float(slot[0]);
      a1.i1 = static_cast<int>(slot[1]);
      a1.v2 = __uint_as_float(slot[2]);
      a1.i2 = static_cast<int>(slot[3]);
      const float m1 = __uint_as_float(slot[4]), s1 = __uint_as_float(slot[5]);
      named_bar_sync(7 + q, 64);
      gate_top2_merge(a0, a1, v1, i1, v2, i2);  // expert ids of half 0 are all lower
      if (need_sum) {
        const float mt = fmaxf(m, m1);
        s = (m == -INFINITY ? 0.f : s * ex2_approx((m - mt) * kLog2e)) +
            (m1 == -INFINITY ? 0.f : s1 * ex2_approx((m1 - mt) * kLog2e));
      } else {
        s = 1.f;
      }

      float pr0, pr1 = 0.f;
      if (p.top_k == 1) {
        pr0 = p.norm_topk ? 1.f : 1.f / s;
      } else if (p.norm_topk) {
        const float z = expf(v2 - v1);
        pr0 = 1.f / (1.f + z);
        pr1 = z / (1.f + z);
      } else {
        pr0 = 1.f / s;
        pr1 = expf(v2 - v1) / s;
      }
      int gr0 = (valid && i1 >= 0) ? smap[i1] : -1;
      int gr1 = (valid && p.top_k == 2 && i2 >= 0) ? smap[i2] : -1;
      if (gr1 >= 0 && gr1 == gr0) {
        pr0 += pr1;
        pr1 = 0.f;
        gr1 = -1;
      }
      named_bar_sync(1, 128);
      for (int i = et; i < p.top_k * 4 * kGateMaxE; i += 128) cnt[i] = 0;
      named_bar_sync(1, 128);
      int wr0, wr1 = 0;
      {
        const unsigned mm0 = __match_any_sync(0xffffffffu, gr0);
        wr0 = __popc(mm0 & lt_mask);
        if (gr0 >= 0 && wr0 == 0) cnt[q * kGateMaxE + gr0] = __popc(mm0);
        if (p.top_k == 2) {
          const unsigned mm1 = __match_any_sync(0xffffffffu, gr1);
          wr1 = __popc(mm1 & lt_mask);
          if (gr1 >= 0 && wr1 == 0) cnt[(4 + q) * kGateMaxE + gr1] = __popc(mm1);
        }
      }
      named_bar_sync(1, 128);
      if (valid) {
        int rank0 = -1, rank1 = -1;
        if (gr0 >= 0) {
          rank0 = wr0;
          for (int qq = 0; qq < q; ++qq) rank0 += cnt[qq * kGateMaxE + gr0];
        }
        if (gr1 >= 0) {
          rank1 = wr1;
          for (int qq = 0; qq < q; ++qq) rank1 += cnt[(4 + qq) * kGateMaxE + gr1];
        }
        const long o = static_cast<long>(t) * p.top_k;
        p.expert_idx[o] = i1;
        p.group_idx[o] = gr0;
        p.gate_prob[o] = gr0 >= 0 ? pr0 : 0.f;
        p.local_rank[o] = rank0;
        if (p.top_k == 2) {
          p.expert_idx[o + 1] = i2;
          p.group_idx[o + 1] = gr1;
          p.gate_prob[o + 1] = gr1 >= 0 ? pr1 : 0.f;
          p.local_rank[o + 1] = rank1;
        }
      }
      if (tile_ok)
        for (int j = 0; j < p.top_k; ++j)
          for (int g = et; g < p.G; g += 128) {
            int h = 0;
            if (g < kGateMaxE)
              for (int qq = 0; qq < 4; ++qq) h += cnt[(j * 4 + qq) * kGateMaxE + g];
            gate_publish_hist(p, j, tile, g, h, ep);
          }
      if (lane == 0 && q == 0) gate_tl(p, tl0, 9, u);
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int eg = (warp - 4) >> 2;                 // epilogue group = accumulator
    const int et = threadIdx.x - 128 - 128 * eg;    // 0..127 inside the group
    int* cnt = cnt_all + eg * kGateMaxK * 4 * kGateMaxE;
    const uint32_t lt_mask = (1u << lane) - 1u;
    int it = eg;
    for (int u = unit0 + eg * unit_step; u < n_units; u += 2 * unit_step, it += 2) {
      const int acc = it & 1;
      const int tile = kPair ? 2 * u + static_cast<int>(rank) : u;
      const bool tile_ok = tile < p.ntiles;  // the odd pair's second tile may not exist
      const int t = tile * kGemmBM + q * 32 + lane;
      const bool valid = tile_ok && t < p.T;
      mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * kAccCols;

      // One pass over this token's logits, 16 columns per chunk, the TMEM
      // load of chunk c+1 in flight while chunk c is reduced; the accumulator
      // is released right after the last load. Two interleaved top-2 trackers
      // (even / odd columns; strict '>' in ascending expert order keeps the
      // lowest id on ties, and the final merge breaks ties by id) and an
      // online softmax denominator s = sum_e 2^((v_e - m) log2 e), rescaled
      // when the running max m moves (once per chunk).
      if (p.debug & 8) {  // dev: no epilogue work
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (kPair) mbar_arrive_cluster(smem_u32(&tempty_bar[acc]) & kPeerMask);
          else mbar_arrive(&tempty_bar[acc]);
        }
        continue;
      }
      GateTop2 ta, tb;
      const bool need_sum = !p.norm_topk;
      constexpr float kLog2e = 1.4426950408889634f;
      float m = -INFINITY, s4[2] = {0.f, 0.f};
      float* lrow = (p.logits && valid) ? p.logits + static_cast<long>(t) * p.E : nullptr;
      constexpr int kChunks = EP / 16;
      uint32_t buf[2][kCat ? 32 : 16];
      gate_ld_chunk<kCat, EP>(t_row, buf[0]);
#pragma unroll
      for (int c = 0; c < kChunks; ++c) {
        uint32_t(&cur)[kCat ? 32 : 16] = buf[c & 1];
        gate_ld_wait<kCat>(cur);
        if (c + 1 < kChunks) {
          gate_ld_chunk<kCat, EP>(t_row + (c + 1) * 16, buf[(c + 1) & 1]);
        } else {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (kPair) mbar_arrive_cluster(smem_u32(&tempty_bar[acc]) & kPeerMask);
            else mbar_arrive(&tempty_bar[acc]);
          }
        }
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int e = c * 16 + j;
          float x = __uint_as_float(cur[j]);
          if constexpr (kCat) x += __uint_as_float(cur[16 + j]);
          v[j] = e < p.E ? x : -INFINITY;
        }
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          ta.push(v[j], c * 16 + j);
          tb.push(v[j + 1], c * 16 + j + 1);
        }
        if (lrow) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c * 16 + j < p.E) lrow[c * 16 + j] = v[j];
        }
        if (need_sum) {
          const float mn = fmaxf(m, fmaxf(ta.v1, tb.v1));
          const float mb = mn * kLog2e;
          const float sc = m == -INFINITY ? 0.f : ex2_approx((m - mn) * kLog2e);
          s4[0] *= sc;
          s4[1] *= sc;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            s4[j & 1] += ex2_approx(fmaf(v[j], kLog2e, -mb));
          m = mn;
        }
      }
      float v1, v2;
      int i1, i2;
      gate_top2_merge(ta, tb, v1, i1, v2, i2);
      const float s = need_sum ? s4[0] + s4[1] : 1.f;

      // probabilities, slot remap, top-2 fold (all in registers)
      float pr0, pr1 = 0.f;
      if (p.top_k == 1) {
        pr0 = p.norm_topk ? 1.f : 1.f / s;
      } else if (p.norm_topk) {
        const float z = expf(v2 - v1);
        pr0 = 1.f / (1.f + z);
        pr1 = z / (1.f + z);
      } else {
        pr0 = 1.f / s;
        pr1 = expf(v2 - v1) / s;
      }
      int gr0 = (valid && i1 >= 0) ? smap[i1] : -1;
      int gr1 = (valid && p.top_k == 2 && i2 >= 0) ? smap[i2] : -1;
      if (gr1 >= 0 && gr1 == gr0) {  // both picks merged into one expert
        pr0 += pr1;
        pr1 = 0.f;
        gr1 = -1;
      }

      // token-order ranks inside the tile: warp match + per-warp counts
      named_bar_sync(1 + eg, 128);
      for (int i = et; i < p.top_k * 4 * kGateMaxE; i += 128) cnt[i] = 0;
      named_bar_sync(1 + eg, 128);
      int wr0, wr1 = 0;
      {
        const unsigned m0 = __match_any_sync(0xffffffffu, gr0);
        wr0 = __popc(m0 & lt_mask);
        if (gr0 >= 0 && wr0 == 0) cnt[q * kGateMaxE + gr0] = __popc(m0);
        if (p.top_k == 2) {
          const unsigned m1 = __match_any_sync(0xffffffffu, gr1);
          wr1 = __popc(m1 & lt_mask);
          if (gr1 >= 0 && wr1 == 0) cnt[(4 + q) * kGateMaxE + gr1] = __popc(m1);
        }
      }
      named_bar_sync(1 + eg, 128);
      if (valid) {
        int rank0 = -1, rank1 = -1;
        if (gr0 >= 0) {
          rank0 = wr0;
          for (int qq = 0; qq < q; ++qq) rank0 += cnt[qq * kGateMaxE + gr0];
        }
        if (gr1 >= 0) {
          rank1 = wr1;
          for (int qq = 0; qq < q; ++qq) rank1 += cnt[(4 + qq) * kGateMaxE + gr1];
        }
        const long o = static_cast<long>(t) * p.top_k;
        p.expert_idx[o] = i1;
        p.group_idx[o] = gr0;
        p.gate_prob[o] = gr0 >= 0 ? pr0 : 0.f;
        p.local_rank[o] = rank0;
        if (p.top_k == 2) {
          p.expert_idx[o + 1] = i2;
          p.group_idx[o + 1] = gr1;
          p.gate_prob[o + 1] = gr1 >= 0 ? pr1 : 0.f;
          p.local_rank[o + 1] = rank1;
        }
      }
      if (tile_ok)
        for (int j = 0; j < p.top_k; ++j)
          for (int g = et; g < p.G; g += 128) {
            int h = 0;
            if (g < kGateMaxE)
              for (int qq = 0; qq < 4; ++qq) h += cnt[(j * 4 + qq) * kGateMaxE + g];
            gate_publish_hist(p, j, tile, g, h, ep);
          }
    }
  }

  if (threadIdx.x == 0 || threadIdx.x == 32 || threadIdx.x == 128) gate_tl(p, tl0, 10, warp);
  tc_fence_before();
  if constexpr (kPair) cluster_sync_all();
  else __syncthreads();
  if (threadIdx.x == 0) gate_tl(p, tl0, 11, 0);
  if (warp == 2) {
    tc_fence_after();
    if constexpr (kPair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(kTmemCols)
                   : "memory");
    else
      tmem_dealloc<kTmemCols>(tmem_base);
  }
  if (p.lb) gate_fold_scan(p, ep);  // folded capacity scan (comoe_gate_route)
  if (threadIdx.x == 0) gate_tl(p, tl0, 12, 0);
}

#include "gate_tm.cuh"

template <int EP, bool kPair, int kTerms, int kStages>
static int launch_gate_stages(const CUtensorMap& tx, const CUtensorMap& tw, const GateParams& p,
                              cudaStream_t stream) {
  using S = GateSmem<EP, kStages, kPair, kTerms>;
  static_assert(S::kTotal <= 227 * 1024, "gate shared memory");
  auto kern = gate_kernel<EP, kStages, kPair, kTerms>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kTotal);
    attr = true;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if constexpr (kPair) {
    const int units = (p.ntiles + 1) / 2;
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
    // the persistent grid must be co-resident (the folded scan meets at a
    // grid barrier): at most as many pairs as can be resident at once
    static int max_pairs = -1;
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
    const int pairs = units < max_pairs ? units : max_pairs;
    cfg.gridDim = dim3(2 * pairs);
    cfg.numAttrs = 1 + pdl_attr(&attrs[1]);
    cudaLaunchKernelEx(&cfg, kern, tx, tw, p);
    return check_launch("gate_kernel(pair)");
  } else {
    const int grid = p.ntiles < sms ? p.ntiles : sms;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kGateThreads);
    cfg.dynamicSmemBytes = S::kTotal;
    cfg.stream = stream;
    cudaLaunchAttribute attrs[1];
    cfg.attrs = attrs;
    cfg.numAttrs = pdl_attr(&attrs[0]);
    cudaLaunchKernelEx(&cfg, kern, tx, tw, p);
    return check_launch("gate_kernel");
  }
}

template <int EP, bool kPair, int kTerms>
static int launch_gate_terms(const CUtensorMap& tx, const CUtensorMap& tw, const GateParams& p,
                             cudaStream_t stream) {
  if constexpr (kPair && kTerms == 2) {
    // 6 ring stages (192 KB of x + router tiles in flight per SM) by default:
    // the load stream is bound by bytes in flight, ~4.3 vs ~5.0 µs per unit
    // (profiles/r2_gate_stages_ab.jsonl); COMOE_GATE_STAGES=5 for A/B
    static const bool six = [] {
      const char* e = std::getenv("COMOE_GATE_STAGES");
      return !(e && e[0] == '5');
    }();
    return six ? launch_gate_stages<EP, kPair, kTerms, 6>(tx, tw, p, stream)
               : launch_gate_stages<EP, kPair, kTerms, 5>(tx, tw, p, stream);
  } else {
    constexpr int kStages = kTerms == 2 ? 4 : (kPair ? 4 : (EP >= 128 ? 3 : 4));
    return launch_gate_stages<EP, kPair, kTerms, kStages>(tx, tw, p, stream);
  }
}

// Router split terms used by the MMAs (COMOE_GATE_TERMS=2|3, default 2).
// Wg = hi + mid + lo is exact; hi + mid keeps 16 of fp32's 24 mantissa bits
// (|lo| <= 2^-17 |Wg|): logit error ~3e-7 at d = 768 (the fp32 accumulation
// itself contributes ~1e-7; the parity bar vs the fp64 oracle is 2e-5, and
// routing parity is defined on the device logits). Two terms cut the
// gate's tensor work and router traffic by a third.
static int gate_terms() {
  static const int t = [] {
    const char* e = std::getenv("COMOE_GATE_TERMS");
    return (e && e[0] == '3') ? 3 : 2;
  }();
  return t;
}

template <int EP, bool kPair>
static int launch_gate(const CUtensorMap& tx, const CUtensorMap& tw, const GateParams& p,
                       cudaStream_t stream) {
  return gate_terms() == 3 ? launch_gate_terms<EP, kPair, 3>(tx, tw, p, stream)
                           : launch_gate_terms<EP, kPair, 2>(tx, tw, p, stream);
}

// Router-in-TMEM gate (gate_tm.cuh) for EP = 128, d <= 768: opt-in
// (COMOE_GATE_TM=1, or comoe_debug_set_gate_tm at run time) — measured slower
// than the pair kernel (K1, "router in tensor memory").
static int g_gate_tm_override = -1;
static bool gate_tm_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("COMOE_GATE_TM");
    return e && e[0] == '1';
  }();
  return g_gate_tm_override >= 0 ? g_gate_tm_override != 0 : on;
}

static bool gate_pair_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("COMOE_GATE_1SM");
    return !(e && e[0] == '1');
  }();
  return on;
}

// ------------------------------------------------------------ routing scan
// Column g of tile_hist in stream order (k-major, then tile): exclusive scan
// -> tile_offset, total -> group_count.
__global__ void route_scan_columns(const int* __restrict__ hist, int n_rows, int G,
                                   int* __restrict__ offset, int* __restrict__ count) {
  __shared__ int warp_tot[32];
  const int g = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int carry = 0;
  for (int base = 0; base < n_rows; base += blockDim.x) {
    const int r = base + threadIdx.x;
    const int x = r < n_rows ? hist[static_cast<long>(r) * G + g] : 0;
    int v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += n;
    }
    if (lane == 31) warp_tot[w] = v;
    __syncthreads();
    int wb = 0, tot = 0;
    for (int i = 0; i < nw; ++i) {
      if (i < w) wb += warp_tot[i];
      tot += warp_tot[i];
    }
    if (r < n_rows) offset[static_cast<long>(r) * G + g] = carry + wb + v - x;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) count[g] = carry;
}

// One cooperative launch (block g = group g): column scan -> grid sync ->
// kept[g] = min(count[g], C), base[g] = sum_{h<g} kept[h] (each block sums
// the earlier groups' kept counts itself). Replaces columns + bases.
__global__ void __launch_bounds__(256) route_scan_coop(const int* __restrict__ hist, int n_rows,
                                                       int G, int capacity,
                                                       int* __restrict__ offset,
                                                       int* __restrict__ count,
                                                       int* __restrict__ kept,
                                                       int* __restrict__ base) {
  __shared__ int warp_tot[32];
  const int g = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int carry = 0;
  for (int b0 = 0; b0 < n_rows; b0 += blockDim.x) {
    const int r = b0 + threadIdx.x;
    const int x = r < n_rows ? hist[static_cast<long>(r) * G + g] : 0;
    int v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += n;
    }
    if (lane == 31) warp_tot[w] = v;
    __syncthreads();
    int wb = 0, tot = 0;
    for (int i = 0; i < nw; ++i) {
      if (i < w) wb += warp_tot[i];
      tot += warp_tot[i];
    }
    if (r < n_rows) offset[static_cast<long>(r) * G + g] = carry + wb + v - x;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) count[g] = carry;
  cooperative_groups::this_grid().sync();
  int part = 0;
  for (int h = threadIdx.x; h < g; h += blockDim.x) part += min(__ldcg(count + h), capacity);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) warp_tot[w] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    int sum = 0;
    for (int i = 0; i < nw; ++i) sum += warp_tot[i];
    kept[g] = min(carry, capacity);
    base[g] = sum;
  }
  pdl_trigger();
}

// kept = min(count, C); base = exclusive scan of kept.
__global__ void route_scan_bases(const int* __restrict__ count, int G, int capacity,
                                 int* __restrict__ kept, int* __restrict__ base) {
  __shared__ int warp_tot[32];
  const int per = (G + blockDim.x - 1) / blockDim.x;
  const int g0 = threadIdx.x * per;
  int local = 0;
  for (int i = 0; i < per; ++i) {
    const int g = g0 + i;
    if (g < G) local += min(count[g], capacity);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int v = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  if (lane == 31) warp_tot[w] = v;
  __syncthreads();
  int run = v - local;
  for (int i = 0; i < w; ++i) run += warp_tot[i];
  for (int i = 0; i < per; ++i) {
    const int g = g0 + i;
    if (g < G) {
      const int kk = min(count[g], capacity);
      kept[g] = kk;
      base[g] = run;
      run += kk;
    }
  }
}

__global__ void expert_hist_kernel(const int* __restrict__ idx, long n, int E,
                                   int* __restrict__ counts) {
  extern __shared__ int h[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) h[e] = 0;
  __syncthreads();
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const int e = idx[i];
    if (e >= 0 && e < E) atomicAdd(&h[e], 1);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    if (h[e]) atomicAdd(&counts[e], h[e]);
}

// Replayed routing (trace-driven runs): the same tile ranks / histograms as the
// gate epilogue, from given expert choices instead of logits. One 128-thread
// block per 128-token tile, thread = token.
__global__ void __launch_bounds__(128) route_from_indices_kernel(
    const int* __restrict__ expert_idx, const float* __restrict__ probs, int T, int E, int top_k,
    const int* __restrict__ slot_map, int G, int ntiles, int* __restrict__ group_idx,
    float* __restrict__ gate_prob, int* __restrict__ local_rank, int* __restrict__ tile_hist) {
  __shared__ int cnt[kGateMaxK * 4 * 1024];
  const int tile = blockIdx.x;
  const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = tile * 128 + threadIdx.x;
  const bool valid = t < T;
  for (int i = threadIdx.x; i < top_k * 4 * G; i += 128) cnt[i] = 0;
  __syncthreads();
  int e0 = -1, e1 = -1;
  float p0 = 0.f, p1 = 0.f;
  if (valid) {
    e0 = expert_idx[static_cast<long>(t) * top_k];
    p0 = probs ? probs[static_cast<long>(t) * top_k] : 1.f / top_k;
    if (top_k == 2) {
      e1 = expert_idx[static_cast<long>(t) * top_k + 1];
      p1 = probs ? probs[static_cast<long>(t) * top_k + 1] : 0.5f;
    }
  }
  int g0 = (e0 >= 0 && e0 < E) ? (slot_map ? slot_map[e0] : e0) : -1;
  int g1 = (e1 >= 0 && e1 < E) ? (slot_map ? slot_map[e1] : e1) : -1;
  if (g1 >= 0 && g1 == g0) {
    p0 += p1;
    p1 = 0.f;
    g1 = -1;
  }
  const uint32_t lt_mask = (1u << lane) - 1u;
  const unsigned m0 = __match_any_sync(0xffffffffu, g0);
  const int wr0 = __popc(m0 & lt_mask);
  if (g0 >= 0 && wr0 == 0) cnt[q * G + g0] = __popc(m0);
  int wr1 = 0;
  if (top_k == 2) {
    const unsigned m1 = __match_any_sync(0xffffffffu, g1);
    wr1 = __popc(m1 & lt_mask);
    if (g1 >= 0 && wr1 == 0) cnt[(4 + q) * G + g1] = __popc(m1);
  }
  __syncthreads();
  if (valid) {
    const long o = static_cast<long>(t) * top_k;
    int r0 = -1, r1 = -1;
    if (g0 >= 0) {
      r0 = wr0;
      for (int qq = 0; qq < q; ++qq) r0 += cnt[qq * G + g0];
    }
    group_idx[o] = g0;
    gate_prob[o] = g0 >= 0 ? p0 : 0.f;
    local_rank[o] = r0;
    if (top_k == 2) {
      if (g1 >= 0) {
        r1 = wr1;
        for (int qq = 0; qq < q; ++qq) r1 += cnt[(4 + qq) * G + g1];
      }
      group_idx[o + 1] = g1;
      gate_prob[o + 1] = g1 >= 0 ? p1 : 0.f;
      local_rank[o + 1] = r1;
    }
  }
  for (int j = 0; j < top_k; ++j)
    for (int g = threadIdx.x; g < G; g += 128) {
      int h = 0;
      for (int qq = 0; qq < 4; ++qq) h += cnt[(j * 4 + qq) * G + g];
      tile_hist[(static_cast<long>(j) * ntiles + tile) * G + g] = h;
    }
}

}  // namespace comoe

extern "C" {

int comoe_route_from_indices(const int* expert_idx, const float* probs, int T, int E, int top_k,
                             const int* slot_map, int n_groups, int* group_idx, float* gate_prob,
                             int* local_rank, int* tile_hist, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(expert_idx && group_idx && gate_prob && local_rank && tile_hist, kBadArg,
                "route_from_indices: null pointer");
  COMOE_REQUIRE(top_k == 1 || top_k == 2, kUnsupportedShape, "route_from_indices: top_k=%d", top_k);
  COMOE_REQUIRE(n_groups >= 1 && n_groups <= 1024 && E >= 1, kBadArg,
                "route_from_indices: n_groups=%d", n_groups);
  if (T <= 0) return kOk;
  const int nt = (T + 127) / 128;
  route_from_indices_kernel<<<nt, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      expert_idx, probs, T, E, top_k, slot_map, n_groups, nt, group_idx, gate_prob, local_rank,
      tile_hist);
  return check_launch("route_from_indices_kernel");
}

int comoe_gate_padded_experts(int E) {
  if (E < 1 || E > comoe::kGateMaxE) return -1;
  int ep = 16;
  while (ep < E) ep <<= 1;
  return ep;
}

int comoe_gate_prepare(const float* wg, int d, int E, void* wg_split, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(wg && wg_split, kBadArg, "gate_prepare: null pointer");
  const int EP = comoe_gate_padded_experts(E);
  COMOE_REQUIRE(EP > 0, kUnsupportedShape, "gate_prepare: E=%d must be in [1,%d]", E, kGateMaxE);
  COMOE_REQUIRE(d > 0 && d % 64 == 0, kUnsupportedShape, "gate_prepare: d=%d must be a multiple of 64", d);
  const long n = static_cast<long>(EP) * d;
  const int grid = static_cast<int>((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
  gate_split_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      wg, d, E, EP, reinterpret_cast<__nv_bfloat16*>(wg_split));
  return check_launch("gate_split_kernel");
}

}  // extern "C"

namespace comoe {
// Shared launch path of comoe_gate_topk (histograms) and comoe_gate_route
// (folded scan: p.lb set).
static int gate_launch(const void* x, int T, int d, const void* wg_split, int E, int top_k,
                       int norm_topk, const int* slot_map, int n_groups, float* logits_out,
                       int* expert_idx, int* group_idx, float* gate_prob, int* local_rank,
                       int* tile_hist, GateParams fold, cudaStream_t s) {
  COMOE_REQUIRE(x && wg_split && expert_idx && group_idx && gate_prob && local_rank &&
                    (tile_hist || fold.lb),
                kBadArg, "gate: null pointer");
  COMOE_REQUIRE(T > 0, kBadArg, "gate: T=%d", T);
  COMOE_REQUIRE(top_k == 1 || top_k == 2, kUnsupportedShape, "gate: top_k=%d not in {1,2}", top_k);
  COMOE_REQUIRE(top_k <= E, kBadArg, "gate: top_k > E");
  const int EP = comoe_gate_padded_experts(E);
  COMOE_REQUIRE(EP > 0, kUnsupportedShape, "gate: E=%d must be in [1,%d]", E, kGateMaxE);
  COMOE_REQUIRE(d % 64 == 0, kUnsupportedShape, "gate: d=%d must be a multiple of 64", d);
  COMOE_REQUIRE(n_groups >= 1 && n_groups <= E, kBadArg, "gate: n_groups=%d", n_groups);
  const bool pair = gate_pair_enabled();
  CUtensorMap tx, tw;
  int rc = make_tmap_bf16_2d(&tx, x, T, d, kGemmBM);
  if (rc) return rc;
  // box rows: a whole term per CTA for the concatenated-terms pair kernel
  rc = make_tmap_bf16_2d(&tw, wg_split, 3ull * EP, d, pair ? (gate_terms() == 2 ? EP : EP / 2) : EP);
  if (rc) return rc;
  GateParams p = fold;
  p.T = T; p.d = d; p.E = E; p.top_k = top_k; p.norm_topk = norm_topk; p.G = n_groups;
  p.ntiles = (T + kGemmBM - 1) / kGemmBM;
  p.slot_map = slot_map; p.logits = logits_out; p.expert_idx = expert_idx;
  p.group_idx = group_idx; p.gate_prob = gate_prob; p.local_rank = local_rank;
  p.tile_hist = tile_hist;
  static const int dbg = [] {
    const char* e = std::getenv("COMOE_GATE_DEBUG");
    return e ? std::atoi(e) : 0;
  }();
  p.debug = dbg;
  static const int xpol = [] {
    const char* e = std::getenv("COMOE_GATE_XPOL");
    return e ? std::atoi(e) : 0;
  }();
  p.xpol = xpol;
  COMOE_REQUIRE(!(p.lb && (dbg & ~256)), kBadArg,
                "gate_route: COMOE_GATE_DEBUG switches need comoe_gate_topk + comoe_route_scan");
  if (EP == 128 && pair && gate_terms() == 2 && gate_tm_enabled() && d <= 768 && d % 128 == 0) {
    CUtensorMap tx64, tr;
    rc = make_tmap_bf16_2d(&tx64, x, T, d, 64);
    if (rc) return rc;
    // router rows [3 terms x 128, d], 16-row boxes (one TMEM lane half-quarter)
    rc = make_tmap_bf16_2d_box(&tr, wg_split, 3ull * EP, d, d, 64, 16, 128);
    if (rc) return rc;
    return launch_gate_tm<8>(tx64, tr, p, s);
  }
  switch (EP) {
    case 16: return pair ? launch_gate<16, true>(tx, tw, p, s) : launch_gate<16, false>(tx, tw, p, s);
    case 32: return pair ? launch_gate<32, true>(tx, tw, p, s) : launch_gate<32, false>(tx, tw, p, s);
    case 64: return pair ? launch_gate<64, true>(tx, tw, p, s) : launch_gate<64, false>(tx, tw, p, s);
    case 128: return pair ? launch_gate<128, true>(tx, tw, p, s) : launch_gate<128, false>(tx, tw, p, s);
    default: break;
  }
  set_error("gate: no kernel for EP=%d", EP);
  return kUnsupportedShape;
}
}  // namespace comoe

extern "C" {

int comoe_gate_topk(const void* x, int T, int d, const void* wg_split, int E, int top_k,
                    int norm_topk, const int* slot_map, int n_groups, float* logits_out,
                    int* expert_idx, int* group_idx, float* gate_prob, int* local_rank,
                    int* tile_hist, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(tile_hist, kBadArg, "gate_topk: null pointer");
  return gate_launch(x, T, d, wg_split, E, top_k, norm_topk, slot_map, n_groups, logits_out,
                     expert_idx, group_idx, gate_prob, local_rank, tile_hist, GateParams{},
                     static_cast<cudaStream_t>(stream));
}

// dev: the gate timeline of CTAs 0 and 1 (COMOE_GATE_DEBUG bit 256), then
// reset; out: [2][kGateTlMax] records, counts: [2]
int comoe_debug_gate_timeline(unsigned long long* out, unsigned int* counts) {
  using namespace comoe;
  COMOE_REQUIRE(out && counts, kBadArg, "debug_gate_timeline: null pointer");
  cudaError_t e = cudaMemcpyFromSymbol(out, g_gate_tl, sizeof(g_gate_tl));
  counts[0] = counts[1] = kGateTlMax;
  static unsigned long long zero[2][kGateTlMax];
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_gate_tl, zero, sizeof(zero));
  COMOE_REQUIRE(e == cudaSuccess, kCudaError, "debug_gate_timeline: %s", cudaGetErrorString(e));
  return kOk;
}

// dev: select the router-in-TMEM gate for later launches (1 on, 0 off, -1 env)
int comoe_debug_set_gate_tm(int on) {
  comoe::g_gate_tm_override = on;
  return comoe::kOk;
}

long comoe_gate_route_workspace_bytes(int T, int top_k, int n_groups) {
  const long nt = (static_cast<long>(T) + comoe::kGemmBM - 1) / comoe::kGemmBM;
  return 16 + 8L * comoe::kGateMaxE + 4L * top_k * nt * n_groups;
}

int comoe_gate_route(const void* x, int T, int d, const void* wg_split, int E, int top_k,
                     int norm_topk, const int* slot_map, int n_groups, int capacity,
                     float* logits_out, int* expert_idx, int* group_idx, float* gate_prob,
                     int* local_rank, int* tile_offset, int* group_count, int* group_kept,
                     int* group_base, void* workspace, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(tile_offset && group_count && group_kept && group_base && workspace, kBadArg,
                "gate_route: null pointer");
  COMOE_REQUIRE(capacity >= 0, kBadArg, "gate_route: capacity=%d", capacity);
  COMOE_REQUIRE((reinterpret_cast<uintptr_t>(workspace) & 15) == 0, kBadArg,
                "gate_route: workspace must be 16-byte aligned");
  GateParams f{};
  f.lb_ctrl = static_cast<unsigned int*>(workspace);
  f.lb_total = reinterpret_cast<int*>(static_cast<char*>(workspace) + 16);
  f.lb = f.lb_total + 2 * kGateMaxE;
  f.tile_offset = tile_offset;
  f.group_count = group_count;
  f.group_kept = group_kept;
  f.group_base = group_base;
  f.capacity = capacity;
  return gate_launch(x, T, d, wg_split, E, top_k, norm_topk, slot_map, n_groups, logits_out,
                     expert_idx, group_idx, gate_prob, local_rank, nullptr, f,
                     static_cast<cudaStream_t>(stream));
}

int comoe_gate_num_tiles(int T) { return (T + comoe::kGemmBM - 1) / comoe::kGemmBM; }

int comoe_route_scan(const int* tile_hist, int top_k, int ntiles, int G, int capacity,
                     int* tile_offset, int* group_count, int* group_kept, int* group_base,
                     void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(tile_hist && tile_offset && group_count && group_kept && group_base, kBadArg,
                "route_scan: null pointer");
  COMOE_REQUIRE(G >= 1 && G <= 32 * 1024, kBadArg, "route_scan: G=%d", G);
  COMOE_REQUIRE(capacity >= 0, kBadArg, "route_scan: capacity=%d", capacity);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  static int coop_blocks = -1;  // co-resident capacity of the cooperative scan
  if (coop_blocks < 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, route_scan_coop, 256, 0);
    coop_blocks = sms * per_sm;
  }
  if (G <= coop_blocks) {
    int n_rows = top_k * ntiles;
    void* args[] = {const_cast<int**>(&tile_hist), &n_rows, &G, &capacity, &tile_offset,
                    &group_count, &group_kept, &group_base};
    cudaLaunchCooperativeKernel(reinterpret_cast<void*>(route_scan_coop), dim3(G), dim3(256),
                                args, 0, s);
    return check_launch("route_scan_coop");
  }
  route_scan_columns<<<G, 256, 0, s>>>(tile_hist, top_k * ntiles, G, tile_offset, group_count);
  int rc = check_launch("route_scan_columns");
  if (rc) return rc;
  route_scan_bases<<<1, 1024, 0, s>>>(group_count, G, capacity, group_kept, group_base);
  return check_launch("route_scan_bases");
}

int comoe_expert_histogram(const int* expert_idx, long n, int E, int* counts, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(expert_idx && counts && E > 0 && n >= 0, kBadArg, "expert_histogram: bad args");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaMemsetAsync(counts, 0, sizeof(int) * E, s);
  if (n == 0) return check_launch("expert_histogram");
  const long blocks = (n + 1023) / 1024;
  expert_hist_kernel<<<static_cast<int>(blocks < 296 ? blocks : 296), 1024, E * sizeof(int), s>>>(
      expert_idx, n, E, counts);
  return check_launch("expert_hist_kernel");
}

}  // extern "C"
