// K5: CoMoE frequency-weighted expert merge, one launch per layer.
//
// Restates merge_group (pkg/src/comoe/aggregation.py:200-215):
//     merged = (sum_j f_j * e_j) / sum_j f_j      (plain mean if sum f <= 1e-12)
// for every multi-member group of a layer at once. Inputs are flat expert
// parameter vectors (the reference's `Expert.params`, moe.py:69-74), here
// [W_in | W_out] bf16 slots of the HBM expert pool, or fp64 vectors in the
// parity mode. The host passes per-member weights and per-group divisors
// (weights = f_j, divisor = sum f; or weights = 1, divisor = n for the mean).
//
// fp64 mode reproduces numpy's evaluation order exactly: products rounded
// separately, rows summed in member order, one final division — no FMA
// contraction — so results are bit-identical to the reference.
// bf16 mode streams 16-byte vectors with fp32 accumulation (w_j/divisor
// divided in fp64, then rounded to fp32), reading each member once and
// writing the merge once.
#include <cstdlib>

#include "common.cuh"
#include "../../include/comoe_b200.h"

namespace comoe {

constexpr int kMergeMaxMembers = 64;

// Work item = (group, 512-vector chunk), items interleaved over groups
// (item w -> group w % G) and grid-strided by a persistent grid, so groups
// of 2..N members share the machine in proportion to their bytes (one
// block range per group left the 5-member groups as a long tail). Each
// thread keeps up to kMergeBatch members x 2 vectors of loads in flight.
constexpr int kMergeBatch = 2;
constexpr int kMergeSmemMembers = 2048;
constexpr int kMergeSmemGroups = 1024;
constexpr int kMergeThreads = 256;

__global__ void __launch_bounds__(kMergeThreads, 4) merge_bf16_kernel(
    const void* const* __restrict__ members, const int* __restrict__ offsets,
    const double* __restrict__ weights, const double* __restrict__ divisor,
    void* const* __restrict__ outs, long D, int G) {
  const long nvec = D >> 3;
  constexpr long kChunk = 2L * kMergeThreads;
  const long chunks = (nvec + kChunk - 1) / kChunk;
  const long items = chunks * G;
  // member pointers, group offsets and normalised fp32 weights w_j / divisor_g
  // staged in shared memory once per block: per work item only the data
  // loads remain on the critical path (chained global loads offsets ->
  // pointer -> data per item, plus an fp64 division per member, cost 1.5x)
  __shared__ float wn[kMergeSmemMembers];
  __shared__ const int4* mp[kMergeSmemMembers];
  __shared__ int offs[kMergeSmemGroups + 1];
  const int n_members = __ldg(offsets + G);
  const bool staged = n_members <= kMergeSmemMembers && G <= kMergeSmemGroups;
  if (staged) {
    for (int g = threadIdx.x; g <= G; g += blockDim.x) offs[g] = __ldg(offsets + g);
    __syncthreads();
    for (int m = threadIdx.x; m < n_members; m += blockDim.x) {
      int lo = 0, hi = G - 1;  // group of member m: largest g with offs[g] <= m
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (offs[mid] <= m) lo = mid; else hi = mid - 1;
      }
      wn[m] = static_cast<float>(__ldg(weights + m) / __ldg(divisor + lo));
      mp[m] = reinterpret_cast<const int4*>(members[m]);
    }
    __syncthreads();
  }
  for (long item = blockIdx.x; item < items; item += gridDim.x) {
    const int g = static_cast<int>(item % G);
    const long i = (item / G) * kChunk + threadIdx.x;
    const long i2 = i + kMergeThreads;
    const bool one = i < nvec, two = i2 < nvec;
    const int m0 = staged ? offs[g] : __ldg(offsets + g);
    const int n = (staged ? offs[g + 1] : __ldg(offsets + g + 1)) - m0;
    const double dv = staged ? 1.0 : __ldg(divisor + g);
    float acc[2][8];
#pragma unroll
    for (int v = 0; v < 2; ++v)
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[v][u] = 0.f;
    for (int j0 = 0; j0 < n; j0 += kMergeBatch) {
      int4 r[kMergeBatch][2];
      float wj[kMergeBatch];
#pragma unroll
      for (int b = 0; b < kMergeBatch; ++b) {
        const bool live = j0 + b < n;
        const int4* src = !live ? nullptr : staged ? mp[m0 + j0 + b]
                                                   : reinterpret_cast<const int4*>(members[m0 + j0 + b]);
        wj[b] = !live ? 0.f : staged ? wn[m0 + j0 + b]
                                     : static_cast<float>(__ldg(weights + m0 + j0 + b) / dv);
        r[b][0] = live && one ? ld_nc_v4(src + i) : make_int4(0, 0, 0, 0);
        r[b][1] = live && two ? ld_nc_v4(src + i2) : make_int4(0, 0, 0, 0);
      }
#pragma unroll
      for (int b = 0; b < kMergeBatch; ++b) {
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r[b][v]);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float2 f = __bfloat1622float2(h[u]);
            acc[v][2 * u] = fmaf(wj[b], f.x, acc[v][2 * u]);
            acc[v][2 * u + 1] = fmaf(wj[b], f.y, acc[v][2 * u + 1]);
          }
        }
      }
    }
    int4* dst = reinterpret_cast<int4*>(outs[g]);
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      if (!(v ? two : one)) continue;
      int4 o;
      o.x = static_cast<int>(pack_bf16x2(acc[v][0], acc[v][1]));
      o.y = static_cast<int>(pack_bf16x2(acc[v][2], acc[v][3]));
      o.z = static_cast<int>(pack_bf16x2(acc[v][4], acc[v][5]));
      o.w = static_cast<int>(pack_bf16x2(acc[v][6], acc[v][7]));
      dst[v ? i2 : i] = o;
    }
  }
}

// Bulk-copy variant (default; COMOE_MERGE_BULK=0 for the register one): one
// thread streams each (group, 8192-element chunk) item's member rows, one
// 16 KB row per stage of an 8-stage shared-memory ring (cp.async.bulk), and
// 8 consumer warps fold them with the same fp32 weights and member order as
// merge_bf16_kernel (bit-identical output), 4 x 16 bytes per thread per
// row. ~128 KB per SM in flight where the register version held ~64 KB
// (DRAM-latency-bound at 83% of HBM). Measured: 4 KB rows or 8-row stages
// were slower (per-row barrier cost; stages of 2-3-member groups half empty).
constexpr int kMbChunk = 8192, kMbRows = 1, kMbStages = 8, kMbThreads = 288;
constexpr int kMbVec = kMbChunk / 8 / 256;  // 16-byte vectors per consumer thread per row
constexpr int kMbStage = kMbRows * kMbChunk * 2;
constexpr int kMbSmem = 1024 + kMbStages * kMbStage + 2 * kMbStages * 8;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(kMbThreads, 1) merge_bulk_kernel(
    const void* const* __restrict__ members, const int* __restrict__ offsets,
    const double* __restrict__ weights, const double* __restrict__ divisor,
    void* const* __restrict__ outs, long D, int G) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(ring + kMbStages * kMbStage);
  uint64_t* empty_bar = full_bar + kMbStages;
  __shared__ float wn[kMergeSmemMembers];
  __shared__ int offs[kMergeSmemGroups + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int g = threadIdx.x; g <= G; g += blockDim.x) offs[g] = __ldg(offsets + g);
  __syncthreads();
  const int n_members = offs[G];
  for (int m = threadIdx.x; m < n_members; m += blockDim.x) {
    int lo = 0, hi = G - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (offs[mid] <= m) lo = mid; else hi = mid - 1;
    }
    wn[m] = static_cast<float>(__ldg(weights + m) / __ldg(divisor + lo));
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMbStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 8);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const long chunks = (D + kMbChunk - 1) / kMbChunk;
  const long items = chunks * G;
  if (warp == 0) {
    if (lane != 0) return;
    int it = 0;  // stage fills issued
    for (long item = blockIdx.x; item < items; item += gridDim.x) {
      const int g = static_cast<int>(item % G);
      const long c0 = (item / G) * kMbChunk;
      const uint32_t bytes = static_cast<uint32_t>((D - c0 < kMbChunk ? D - c0 : kMbChunk) * 2);
      const int m0 = offs[g], n = offs[g + 1] - m0;
      for (int j0 = 0; j0 < n; j0 += kMbRows, ++it) {
        const int s = it % kMbStages;
        if (it >= kMbStages) mbar_wait(&empty_bar[s], ((it / kMbStages) - 1) & 1);
        const int rows = n - j0 < kMbRows ? n - j0 : kMbRows;
        mbar_expect_tx(&full_bar[s], bytes * static_cast<uint32_t>(rows));
        for (int j = 0; j < rows; ++j)
          bulk_g2s(ring + s * kMbStage + j * kMbChunk * 2,
                   static_cast<const __nv_bfloat16*>(members[m0 + j0 + j]) + c0, bytes, &full_bar[s]);
      }
    }
    return;
  }
  const int t = threadIdx.x - 32;  // vectors t, t + 256, ... of the chunk
  int it = 0;
  for (long item = blockIdx.x; item < items; item += gridDim.x) {
    const int g = static_cast<int>(item % G);
    const long c0 = (item / G) * kMbChunk;
    const long len = D - c0 < kMbChunk ? D - c0 : kMbChunk;
    const int m0 = offs[g], n = offs[g + 1] - m0;
    float acc[kMbVec][8];
#pragma unroll
    for (int v = 0; v < kMbVec; ++v)
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[v][u] = 0.f;
    for (int j0 = 0; j0 < n; j0 += kMbRows, ++it) {
      const int s = it % kMbStages;
      mbar_wait(&full_bar[s], (it / kMbStages) & 1);
      const int rows = n - j0 < kMbRows ? n - j0 : kMbRows;
      for (int j = 0; j < rows; ++j) {
        const float wj = wn[m0 + j0 + j];
#pragma unroll
        for (int v = 0; v < kMbVec; ++v) {
          const int vi = t + 256 * v;
          if (8L * vi >= len) continue;
          const int4 raw = *reinterpret_cast<const int4*>(ring + s * kMbStage + j * kMbChunk * 2 + vi * 16);
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float2 f = __bfloat1622float2(h[u]);
            acc[v][2 * u] = fmaf(wj, f.x, acc[v][2 * u]);
            acc[v][2 * u + 1] = fmaf(wj, f.y, acc[v][2 * u + 1]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
    }
#pragma unroll
    for (int v = 0; v < kMbVec; ++v) {
      const int vi = t + 256 * v;
      if (8L * vi >= len) continue;
      int4 o;
      o.x = static_cast<int>(pack_bf16x2(acc[v][0], acc[v][1]));
      o.y = static_cast<int>(pack_bf16x2(acc[v][2], acc[v][3]));
      o.z = static_cast<int>(pack_bf16x2(acc[v][4], acc[v][5]));
      o.w = static_cast<int>(pack_bf16x2(acc[v][6], acc[v][7]));
      reinterpret_cast<int4*>(static_cast<__nv_bfloat16*>(outs[g]) + c0)[vi] = o;
    }
  }
}

__global__ void __launch_bounds__(256) merge_f64_kernel(const void* const* __restrict__ members,
                                                        const int* __restrict__ offsets,
                                                        const double* __restrict__ weights,
                                                        const double* __restrict__ divisor,
                                                        void* const* __restrict__ outs, long D) {
  const int g = blockIdx.y;
  const int m0 = offsets[g], m1 = offsets[g + 1];
  const int n = m1 - m0;
  __shared__ double w[kMergeMaxMembers];
  __shared__ const double* src[kMergeMaxMembers];
  if (threadIdx.x < n) {
    w[threadIdx.x] = weights[m0 + threadIdx.x];
    src[threadIdx.x] = reinterpret_cast<const double*>(members[m0 + threadIdx.x]);
  }
  __syncthreads();
  const double div = divisor[g];
  double* dst = reinterpret_cast<double*>(outs[g]);
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  // scalar, 8-byte aligned rows (parity mode: odd D and row views allowed)
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < D; i += stride) {
    double a = __dmul_rn(w[0], src[0][i]);
    for (int j = 1; j < n; ++j) a = __dadd_rn(a, __dmul_rn(w[j], src[j][i]));
    dst[i] = __ddiv_rn(a, div);
  }
}

}  // namespace comoe

extern "C" {

int comoe_merge(int dtype, const void* const* member_ptrs, const int* group_offsets,
                const double* weights, const double* divisor, void* const* out_ptrs, int n_groups,
                int max_members, long D, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(member_ptrs && group_offsets && weights && divisor && out_ptrs, kBadArg,
                "merge: null pointer");
  COMOE_REQUIRE(n_groups >= 0 && n_groups <= 65535, kBadArg, "merge: n_groups=%d", n_groups);
  COMOE_REQUIRE(max_members >= 1 && max_members <= kMergeMaxMembers, kUnsupportedShape,
                "merge: groups of %d members exceed %d", max_members, kMergeMaxMembers);
  COMOE_REQUIRE(D > 0, kBadArg, "merge: D=%ld", D);
  if (n_groups == 0) return kOk;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // ~8 resident 256-thread CTAs per SM spread over the groups of this layer
  const long per_vec = dtype == COMOE_DTYPE_BF16 ? 8 : 1;
  const long nvec = D / per_vec;
  long bx = (static_cast<long>(sms) * 8 + n_groups - 1) / n_groups;
  const long need = (nvec + 255) / 256;
  if (bx > need) bx = need;
  if (bx < 1) bx = 1;
  dim3 grid(static_cast<unsigned>(bx), static_cast<unsigned>(n_groups));
  if (dtype == COMOE_DTYPE_BF16) {
    COMOE_REQUIRE(D % 8 == 0, kUnsupportedShape, "merge(bf16): D=%ld must be a multiple of 8", D);
    static const bool bulk = [] {
      const char* e = std::getenv("COMOE_MERGE_BULK");
      return !(e && e[0] == '0');
    }();
    if (bulk && n_groups <= kMergeSmemGroups && max_members * n_groups <= kMergeSmemMembers) {
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(merge_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMbSmem);
        attr = true;
      }
      const long items = ((D + kMbChunk - 1) / kMbChunk) * n_groups;
      const long blocks = items < sms ? items : sms;
      merge_bulk_kernel<<<static_cast<unsigned>(blocks), kMbThreads, kMbSmem, s>>>(
          member_ptrs, group_offsets, weights, divisor, out_ptrs, D, n_groups);
      return check_launch("merge_bulk_kernel");
    }
    const long items = ((D / 8 + 2 * kMergeThreads - 1) / (2 * kMergeThreads)) * n_groups;
    const long blocks = items < static_cast<long>(sms) * 4 ? items : static_cast<long>(sms) * 4;
    merge_bf16_kernel<<<static_cast<unsigned>(blocks), kMergeThreads, 0, s>>>(
        member_ptrs, group_offsets, weights, divisor, out_ptrs, D, n_groups);
    return check_launch("merge_bf16_kernel");
  }
  if (dtype == COMOE_DTYPE_F64) {
    merge_f64_kernel<<<grid, 256, 0, s>>>(member_ptrs, group_offsets, weights, divisor, out_ptrs, D);
    return check_launch("merge_f64_kernel");
  }
  set_error("merge: unsupported dtype %d", dtype);
  return kBadArg;
}

}  // extern "C"
