// K3: grouped expert GEMM on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// One persistent CTA per SM walks a device-side tile list built from the
// per-group row counts that the routing kernels left in HBM (no host sync).
// A tile is 128 rows of one expert group x BN output columns:
//   A  = permuted token rows      [total_rows, K] bf16, K-major (TMA, SW128)
//   B  = expert slot pool         [n_slots][N, K] bf16, K-major (3-D TMA, SW128)
//   D  = 128 x BN fp32 accumulator in TMEM, double-buffered (2*BN columns)
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer (one thread),
// w2 TMEM allocator, w3 idle, w4..w7 epilogue (thread = accumulator row).
//
// Replaces the analytic expert charge `len(ids)*expert_flops*comp_rate`
// of the reference simulator (pkg/src/comoe/simulator.py:705) with the real
// expert FFN: relu(X_e Wi_e^T) Wo_e^T (Switch) or (silu(X W1^T)*(X W3^T)) W2^T.
#pragma once

#include "common.cuh"

namespace comoe {

enum EpiMode : int {
  kEpiRelu = 0,          // out[arow, n] = bf16(relu(acc))
  kEpiSwiGLU = 1,        // BN cols = [gate 128 | up 128] -> out[arow, n/2] = silu(g)*u
  kEpiScaleScatter = 2,  // out[row_token[arow], n] = bf16(acc * row_prob[arow])
  kEpiStore = 3,         // out[arow, n] = bf16(acc)
};

struct GroupedGemmParams {
  const int* group_rows;      // [G] valid rows per group
  const int* group_row_base;  // [G] first A row of the group
  const int* group_slot;      // [G] expert slot in the pool (3rd TMA coordinate)
  int G;
  int N;  // MMA output columns per group (multiple of BN)
  int K;  // reduction length (multiple of 64)
  __nv_bfloat16* out;
  int ldo;  // elements
  const int* row_token;   // kEpiScaleScatter
  const float* row_prob;  // kEpiScaleScatter
  const int* gather_rows; // 2-SM kernel: B-operand row r of group g is row
                          // gather_rows[row_base[g] + r] of the token tensor (TMA gather4)
  int debug;              // dev-only attribution switches (COMOE_GEMM_DEBUG): 1 = no epilogue
                          // math/stores, 2 = no TMA (MMA on stale smem), 4 = no TMA store,
                          // 16/128 = L2-resident operands (see the producer); 0 in production
  int ft_major;           // tile order inside a group (0: token tile major,
                          // 1: feature tile major — consecutive CTAs share a weight tile)
  int equal_tiles;        // 2-SM kernel: split a group's rows into equal token tiles
                          // (long-K GEMMs, where few tiles per pair make the deal uneven)
};

constexpr int kGemmBM = 128;
constexpr int kGemmBK = 64;
constexpr int kGemmThreads = 256;
constexpr int kMaxGroups = 2048;

template <int BN, int kStages>
struct GemmSmem {
  static constexpr int kABytes = kGemmBM * kGemmBK * 2;
  static constexpr int kBBytes = BN * kGemmBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTileBytes = kStages * kStageBytes;
  // epilogue staging: 4 warps x (32 rows x 128 B), 128B-swizzled chunks
  static constexpr int kStageOutBytes = 4 * 32 * 128;
  // barriers + tmem slot + tile prefix table
  static constexpr int kCtrlBytes = (2 * kStages + 4) * 8 + 16 + (kMaxGroups + 1) * 4;
  static constexpr int kTotal = 1024 /*align slack*/ + kTileBytes + kStageOutBytes + kCtrlBytes;
};

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Tile-list prefix over groups: prefix[g] = sum_{h<g} ceil(rows_h/128)*n_tiles.
__device__ __forceinline__ void build_tile_prefix(const int* __restrict__ rows, int G,
                                                  int n_tiles, int* prefix) {
  __shared__ int warp_tot[kGemmThreads / 32];
  const int tid = threadIdx.x;
  const int per = (G + kGemmThreads - 1) / kGemmThreads;
  const int g0 = tid * per;
  int local = 0;
  for (int i = 0; i < per; ++i) {
    int g = g0 + i;
    if (g < G) local += ((__ldg(rows + g) + kGemmBM - 1) / kGemmBM) * n_tiles;
  }
  // block exclusive scan of `local`
  int v = local;
  const int lane = tid & 31, w = tid >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  if (lane == 31) warp_tot[w] = v;
  __syncthreads();
  int wbase = 0;
  for (int i = 0; i < w; ++i) wbase += warp_tot[i];
  int run = wbase + v - local;  // exclusive
  for (int i = 0; i < per; ++i) {
    int g = g0 + i;
    if (g < G) {
      prefix[g] = run;
      run += ((__ldg(rows + g) + kGemmBM - 1) / kGemmBM) * n_tiles;
    }
  }
  if (tid == kGemmThreads - 1) prefix[G] = run;
  __syncthreads();
}

__device__ __forceinline__ int find_group(const int* prefix, int G, int tile) {
  int lo = 0, hi = G - 1;  // largest g with prefix[g] <= tile
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// (token tile mt, feature tile nt) of tile `local` of group g
__device__ __forceinline__ void tile_coords(const GroupedGemmParams& p, int g, int local,
                                            int n_tiles, int& mt, int& nt) {
  if (p.ft_major) {
    const int n_mt = (__ldg(p.group_rows + g) + kGemmBM - 1) / kGemmBM;
    mt = local % n_mt;
    nt = local / n_mt;
  } else {
    mt = local / n_tiles;
    nt = local % n_tiles;
  }
}

template <int BN, int kStages, int kMode>
__global__ void __launch_bounds__(kGemmThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a,
                        const __grid_constant__ CUtensorMap tmap_b, GroupedGemmParams p) {
  using S = GemmSmem<BN, kStages>;
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN");
  constexpr uint32_t kTmemCols = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  constexpr uint32_t kIdesc = umma_idesc_bf16_f32(kGemmBM, BN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + kStages * S::kABytes;
  uint8_t* smem_out = smem + S::kTileBytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S::kTileBytes + S::kStageOutBytes);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;   // [2]
  uint64_t* tempty_bar = tfull_bar + 2;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int* prefix = reinterpret_cast<int*>(tmem_slot + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_tiles = p.N / BN;
  const int k_blocks = p.K / kGemmBK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  build_tile_prefix(p.group_rows, p.G, n_tiles, prefix);  // contains __syncthreads
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = prefix[p.G];

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (elect_one()) {
      const uint64_t pol_w = l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const int g = find_group(prefix, p.G, tile);
        const int local = tile - prefix[g];
        int mt, nt;
        tile_coords(p, g, local, n_tiles, mt, nt);
        const int a_row = __ldg(p.group_row_base + g) + mt * kGemmBM;
        const int b_slot = __ldg(p.group_slot + g);
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_expect_tx(&full_bar[stage], S::kStageBytes);
          tma_load_2d(smem_a + stage * S::kABytes, &tmap_a, &full_bar[stage], kb * kGemmBK, a_row);
          tma_load_3d_hint(smem_b + stage * S::kBBytes, &tmap_b, &full_bar[stage], kb * kGemmBK,
                           nt * BN, b_slot, pol_w);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t adesc = umma_desc_k_sw128(smem_u32(smem_a + stage * S::kABytes));
          const uint64_t bdesc = umma_desc_k_sw128(smem_u32(smem_b + stage * S::kBBytes));
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k) {
            // +32 bytes per UMMA_K=16 step inside the 128B swizzle atom (>>4 => +2)
            umma_bf16(d_tmem, adesc + 2 * k, bdesc + 2 * k, kIdesc, (kb | k) != 0);
          }
          umma_commit(&empty_bar[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull_bar[acc]);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue
    // TMEM -> registers (thread = row) -> bf16 -> swizzled smem staging ->
    // warp-cooperative stores of whole 128-byte row segments (8 lanes/row),
    // so every store instruction touches 4 full lines instead of 32 partial ones.
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    uint8_t* stg = smem_out + q * (32 * 128);
    const int sub_row = lane >> 3, sub_chunk = lane & 7;
    int it = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int g = find_group(prefix, p.G, tile);
      const int local = tile - prefix[g];
      int mt, nt;
      tile_coords(p, g, local, n_tiles, mt, nt);
      const int rows = __ldg(p.group_rows + g);
      const int r0 = mt * kGemmBM + q * 32;  // first row (within the group) of this warp
      const long arow0 = static_cast<long>(__ldg(p.group_row_base + g)) + r0;
      const bool valid = r0 + lane < rows;
      long my_row = -1;  // destination row of this thread's accumulator row
      float scale = 1.f;
      if (valid) {
        if constexpr (kMode == kEpiScaleScatter) {
          my_row = __ldg(p.row_token + arow0 + lane);
          scale = __ldg(p.row_prob + arow0 + lane);
        } else {
          my_row = arow0 + lane;
        }
      }
      constexpr int kOutCols = kMode == kEpiSwiGLU ? BN / 2 : BN;
      const long col0 = static_cast<long>(nt) * kOutCols;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < kOutCols; c += 64) {
        uint32_t packed[32];
        if constexpr (kMode == kEpiSwiGLU) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t gv[32], uv[32];
            tmem_ld32(t_row + c + 32 * h, gv);
            tmem_ld32(t_row + BN / 2 + c + 32 * h, uv);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float g0 = __uint_as_float(gv[2 * j]), g1 = __uint_as_float(gv[2 * j + 1]);
              const float u0 = __uint_as_float(uv[2 * j]), u1 = __uint_as_float(uv[2 * j + 1]);
              packed[16 * h + j] = pack_bf16x2(__fdividef(g0, 1.f + __expf(-g0)) * u0,
                                               __fdividef(g1, 1.f + __expf(-g1)) * u1);
            }
          }
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t v[32];
            tmem_ld32(t_row + c + 32 * h, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              float a0 = __uint_as_float(v[2 * j]), a1 = __uint_as_float(v[2 * j + 1]);
              if constexpr (kMode == kEpiRelu) {
                a0 = fmaxf(a0, 0.f);
                a1 = fmaxf(a1, 0.f);
              } else if constexpr (kMode == kEpiScaleScatter) {
                a0 *= scale;
                a1 *= scale;
              }
              packed[16 * h + j] = pack_bf16x2(a0, a1);
            }
          }
        }
        // stage my row: 8 chunks of 16 B, chunk j at (j ^ row%8) — conflict-free both ways
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t a = smem_u32(stg + lane * 128 + ((j ^ (lane & 7)) << 4));
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(packed[4 * j]),
                       "r"(packed[4 * j + 1]), "r"(packed[4 * j + 2]), "r"(packed[4 * j + 3])
                       : "memory");
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int row = 4 * k + sub_row;
          const long dst_row = __shfl_sync(0xffffffffu, my_row, row);
          const uint32_t a = smem_u32(stg + row * 128 + ((sub_chunk ^ (row & 7)) << 4));
          uint32_t x0, x1, x2, x3;
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
                       : "r"(a));
          if (dst_row >= 0)
            st_global_v4(p.out + dst_row * p.ldo + col0 + c + sub_chunk * 8, x0, x1, x2, x3);
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

}  // namespace comoe
