// Dev probe: which descriptor field (LBO or SBO) carries the K-direction
// stride of an MN-major, 128B-swizzled bf16 B operand for tcgen05.mma, and
// does the A-from-smem K-major / B MN-major combination give D = A.B^T?
// The fused FFN (csrc/fused_ffn.cuh) feeds GEMM2 its H operand in this layout.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/mn_major_probe.cu -o scripts/mn_major_probe.bin
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../paper_2508_09208_b200/csrc/grouped_gemm_2sm.cuh"

using namespace comoe;

constexpr int M = 128, N = 64, K = 64;

__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

__global__ void __launch_bounds__(128, 1) probe(const float* a, const float* b, float* d, int variant) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;            // 128 x 64 K-major SW128: 16 KB
  uint8_t* sb = smem + 16384;    // MN-major: 8 K-atoms of (8 k x 64 n), 1024 B each
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += 128) {
    const int m = i / K, k = i % K;
    const uint32_t off = (m / 8) * 1024 + (m % 8) * 128 + ((((k / 8) ^ (m % 8)) & 7) << 4) + (k % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sa + off) = __float2bfloat16(a[i]);
  }
  for (int i = tid; i < N * K; i += 128) {
    const int n = i / K, k = i % K;
    const uint32_t off = (k / 8) * 1024 + (k % 8) * 128 + ((((n / 8) ^ (k % 8)) & 7) << 4) + (n % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sb + off) = __float2bfloat16(b[i]);
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<64>(&slot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1 && elect_one()) {
    const uint32_t idesc = umma_idesc_bf16_f32(M, N) | (1u << 16);  // B MN-major
    const uint32_t lbo = variant == 0 ? 16384 : 1024;
    const uint32_t sbo = variant == 0 ? 1024 : 16384;
    for (int k = 0; k < K / 16; ++k) {
      const uint64_t ad = umma_desc_k_sw128(smem_u32(sa)) + 2 * k;
      const uint64_t bd = desc_mn_sw128(smem_u32(sb) + k * 2048, lbo, sbo);
      umma_bf16(tmem, ad, bd, idesc, k > 0);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t v[32];
  for (int c = 0; c < N; c += 32) {
    tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) d[(warp * 32 + lane) * N + c + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<64>(tmem);
}

int main() {
  float *a, *b, *d;
  cudaMallocManaged(&a, M * K * 4);
  cudaMallocManaged(&b, N * K * 4);
  cudaMallocManaged(&d, M * N * 4);
  srand(1);
  for (int i = 0; i < M * K; ++i) a[i] = (rand() % 17) - 8;
  for (int i = 0; i < N * K; ++i) b[i] = (rand() % 13) - 6;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  for (int variant = 0; variant < 2; ++variant) {
    cudaMemset(d, 0, M * N * 4);
    probe<<<1, 128, 40 * 1024>>>(a, b, d, variant);
    cudaError_t e = cudaDeviceSynchronize();
    double maxerr = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += (double)a[m * K + k] * b[n * K + k];
        maxerr = fmax(maxerr, fabs(s - d[m * N + n]));
      }
    printf("variant %d (%s): err=%d max|D-ref|=%g\n", variant,
           variant == 0 ? "SBO = K-atom stride" : "LBO = K-atom stride", (int)e, maxerr);
  }
  return 0;
}
