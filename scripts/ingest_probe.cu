// Per-SM operand ingest (dev probe): L2-resident data into shared memory by
// (a) TMA bulk copies only, (b) cp.async 16-byte LSU copies only, (c) both at
// once from separate warps. If (c) exceeds (a), the ~53 B/clk per SM TMA
// figure is a TMA-path limit that a second load path can add to.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ingest_probe.bin scripts/ingest_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

constexpr int kStages = 8, kChunk = 16384;   // TMA ring: 128 KB
constexpr int kLsuBytes = 64 * 1024;         // LSU ring: 64 KB, 4 warps

__global__ void __launch_bounds__(160, 1) ingest(const char* a, const char* b, long foot, int tma_iters,
                                                 int lsu_iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) uint64_t bar[kStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane != 0) return;
    for (int s = 0; s < kStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const long n = foot / kChunk;
    long c = blockIdx.x;
    for (int i = 0; i < tma_iters; ++i) {
      const int s = i % kStages;
      if (i >= kStages) {
        const uint32_t ph = ((i / kStages) - 1) & 1;
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(
                         su32(&bar[s])), "r"(ph) : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(kChunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(smem + s * kChunk)), "l"(a + (c % n) * kChunk), "r"(kChunk), "r"(su32(&bar[s]))
                   : "memory");
      c += gridDim.x;
    }
    for (int i = tma_iters > kStages ? tma_iters - kStages : 0; i < tma_iters; ++i) {
      const int s = i % kStages;
      const uint32_t ph = (i / kStages) & 1;
      asm volatile("{\n.reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}" ::"r"(
                       su32(&bar[s])), "r"(ph) : "memory");
    }
  } else {
    // 128 threads, each copies 16 B x 8 per iteration into its slice of the LSU ring
    const int t = threadIdx.x - 32;
    char* ring = smem + kStages * kChunk;
    const long n = foot / 16;
    long v = static_cast<long>(blockIdx.x) * 1024 + t;
    for (int i = 0; i < lsu_iters; ++i) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t dst = su32(ring + ((i * 4 + u) % 32) * 2048 + t * 16);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(b + (v % n) * 16) : "memory");
        v += 128;
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 6;" ::: "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
}

int main() {
  char *a, *b;
  const long foot = 32L << 20;
  cudaMalloc(&a, foot);
  cudaMalloc(&b, foot);
  cudaMemset(a, 1, foot);
  cudaMemset(b, 2, foot);
  const int smem = kStages * kChunk + kLsuBytes;
  cudaFuncSetAttribute(ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long tma_bytes_per_cta = 64L << 20;  // 64 MB per CTA
  struct Mode { const char* name; int tma, lsu; } modes[] = {
      {"tma_only", 1, 0}, {"lsu_only", 0, 1}, {"tma+lsu", 1, 1}};
  for (auto m : modes) {
    const int tma_iters = m.tma ? static_cast<int>(tma_bytes_per_cta / kChunk) : 0;
    const int lsu_iters = m.lsu ? static_cast<int>(tma_bytes_per_cta / 4 / (128 * 16 * 4)) : 0;
    ingest<<<sms, 160, smem>>>(a, b, foot, tma_iters / 16, lsu_iters / 16, nullptr);  // warm
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    ingest<<<sms, 160, smem>>>(a, b, foot, tma_iters, lsu_iters, nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = static_cast<double>(sms) *
                         (static_cast<double>(tma_iters) * kChunk + static_cast<double>(lsu_iters) * 128 * 16 * 4);
    printf("{\"mode\": \"%s\", \"TBps\": %.2f, \"per_sm_GBps\": %.1f, \"ms\": %.3f, \"err\": \"%s\"}\n", m.name,
           bytes / (ms * 1e-3) / 1e12, bytes / sms / (ms * 1e-3) / 1e9, ms, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
