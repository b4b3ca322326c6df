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
// pre-divided in fp64), reading each member once and writing the merge once.
#include "common.cuh"
#include "../../include/comoe_b200.h"

namespace comoe {

constexpr int kMergeMaxMembers = 64;

__global__ void __launch_bounds__(256) merge_bf16_kernel(const void* const* __restrict__ members,
                                                         const int* __restrict__ offsets,
                                                         const double* __restrict__ weights,
                                                         const double* __restrict__ divisor,
                                                         void* const* __restrict__ outs, long D) {
  const int g = blockIdx.y;
  const int m0 = offsets[g], m1 = offsets[g + 1];
  const int n = m1 - m0;
  __shared__ float w[kMergeMaxMembers];
  __shared__ const int4* src[kMergeMaxMembers];
  if (threadIdx.x < n) {
    w[threadIdx.x] = static_cast<float>(weights[m0 + threadIdx.x] / divisor[g]);
    src[threadIdx.x] = reinterpret_cast<const int4*>(members[m0 + threadIdx.x]);
  }
  __syncthreads();
  int4* dst = reinterpret_cast<int4*>(outs[g]);
  const long nvec = D >> 3;
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  // two 16-byte vectors per thread per member in flight (i and i + stride)
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < nvec;
       i += 2 * stride) {
    const long i2 = i + stride;
    const bool two = i2 < nvec;
    float acc[2][8];
#pragma unroll
    for (int v = 0; v < 2; ++v)
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[v][u] = 0.f;
    for (int j = 0; j < n; ++j) {
      const int4 r0 = ld_nc_v4(src[j] + i);
      const int4 r1 = two ? ld_nc_v4(src[j] + i2) : make_int4(0, 0, 0, 0);
      const float wj = w[j];
      const __nv_bfloat162* h0 = reinterpret_cast<const __nv_bfloat162*>(&r0);
      const __nv_bfloat162* h1 = reinterpret_cast<const __nv_bfloat162*>(&r1);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2 f0 = __bfloat1622float2(h0[u]);
        const float2 f1 = __bfloat1622float2(h1[u]);
        acc[0][2 * u] = fmaf(wj, f0.x, acc[0][2 * u]);
        acc[0][2 * u + 1] = fmaf(wj, f0.y, acc[0][2 * u + 1]);
        acc[1][2 * u] = fmaf(wj, f1.x, acc[1][2 * u]);
        acc[1][2 * u + 1] = fmaf(wj, f1.y, acc[1][2 * u + 1]);
      }
    }
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      if (v == 1 && !two) break;
      int4 o;
      o.x = static_cast<int>(pack_bf16x2(acc[v][0], acc[v][1]));
      o.y = static_cast<int>(pack_bf16x2(acc[v][2], acc[v][3]));
      o.z = static_cast<int>(pack_bf16x2(acc[v][4], acc[v][5]));
      o.w = static_cast<int>(pack_bf16x2(acc[v][6], acc[v][7]));
      dst[v ? i2 : i] = o;
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
    merge_bf16_kernel<<<grid, 256, 0, s>>>(member_ptrs, group_offsets, weights, divisor, out_ptrs, D);
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
