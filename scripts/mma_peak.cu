// Micro-benchmark: tcgen05.mma issue rate on resident shared memory (dev tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2508_09208_b200/csrc \
//      scripts/mma_peak.cu -o build/mma_peak
#include <cstdio>
#include "../paper_2508_09208_b200/csrc/grouped_gemm_2sm.cuh"

using namespace comoe;

template <int N, bool kTwo>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma_loop(int iters, unsigned long long* cycles) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<int4*>(smem)[i] = make_int4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) {
    if (kTwo) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc<512>(&slot);
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1 && (!kTwo || rank == 0) && elect_one()) {
    const uint64_t a = umma_desc_k_sw128(smem_u32(smem));
    const uint64_t b = umma_desc_k_sw128(smem_u32(smem + 32768));
    const uint32_t idesc = umma_idesc_bf16_f32(kTwo ? 256 : 128, N);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (kTwo) umma_bf16_2sm(tmem + (it & 1) * 256, a + 2 * k, b + 2 * k, idesc, 1);
        else umma_bf16(tmem + (it & 1) * 256, a + 2 * k, b + 2 * k, idesc, 1);
      }
    }
    if (kTwo) umma_commit_2sm_mc(&bar); else umma_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  } else if (kTwo && rank == 1 && warp == 1 && elect_one()) {
    mbar_wait(&bar, 0);  // multicast commit arrives here too
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    if (kTwo) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    else tmem_dealloc<512>(tmem);
  }
}

template <int N, bool kTwo>
void run(const char* name, int sms) {
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * sms);
  cudaMemset(d, 0, sizeof(unsigned long long) * sms);
  auto k = mma_loop<N, kTwo>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  const int iters = 20000;
  k<<<sms & ~1, 128, 70 * 1024>>>(iters, d);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<sms & ~1, 128, 70 * 1024>>>(iters, d);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float ms = 0; cudaEventElapsedTime(&ms, a, b);
  unsigned long long h[256] = {0};
  cudaMemcpy(h, d, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
  unsigned long long cyc = 0; int n = 0;
  for (int i = 0; i < sms; ++i) if (h[i]) { cyc += h[i]; ++n; }
  cyc /= (n ? n : 1);
  const double M = kTwo ? 256 : 128;
  const double macs_per_mma = M * N * 16;
  const double per_sm_cyc = macs_per_mma * 4.0 * iters / cyc / (kTwo ? 2 : 1);
  const double flops = 2.0 * macs_per_mma * 4.0 * iters * ((sms & ~1) / (kTwo ? 2 : 1));
  printf("%-22s err=%d cycles/MMA=%.1f MAC/cyc/SM=%.0f  TFLOP/s=%.1f  (%.3f ms)\n", name, (int)e,
         (double)cyc / (4.0 * iters), per_sm_cyc, flops / (ms * 1e-3) / 1e12, ms);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<256, false>("1SM M128 N256", sms);
  run<128, false>("1SM M128 N128", sms);
  run<256, true>("2SM M256 N256", sms);
  run<128, true>("2SM M256 N128", sms);
  return 0;
}
