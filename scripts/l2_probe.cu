// L2 -> SM bandwidth ceiling on this GPU (dev probe): every CTA streams
// 16 KB cp.async.bulk copies from an L2-resident buffer (footprint << 126 MB)
// into a shared-memory ring, no compute. Prints TB/s for footprints and CTA
// counts; a DRAM-sized footprint gives the HBM figure for comparison.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2_probe scripts/l2_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int kStages, int kChunk>
__global__ void __launch_bounds__(32, 1) stream_kernel(const char* buf, long footprint, int iters) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar[kStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const long n_chunks = footprint / kChunk;
  long c = blockIdx.x;
  for (int i = 0; i < iters; ++i) {
    const int s = i % kStages;
    if (i >= kStages) {
      const uint32_t ph = ((i / kStages) - 1) & 1;
      asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(
                       su32(&bar[s])), "r"(ph) : "memory");
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(kChunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(smem + s * kChunk)), "l"(buf + (c % n_chunks) * kChunk), "r"(kChunk), "r"(su32(&bar[s]))
                 : "memory");
    c += gridDim.x;
  }
  for (int s = 0; s < kStages; ++s) {
    const int i = iters - kStages + s;
    if (i < 0) continue;
    const int st = i % kStages;
    const uint32_t ph = (i / kStages) & 1;
    asm volatile("{\n.reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}" ::"r"(
                     su32(&bar[st])), "r"(ph) : "memory");
  }
}

int main() {
  constexpr int kStages = 12, kChunk = 16384;
  char* buf;
  const long big = 4L << 30;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  auto k = stream_kernel<kStages, kChunk>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kChunk);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long foots[] = {32L << 20, 2L << 30};
  for (long f : foots)
    for (int grid : {sms / 8, sms / 4, sms / 2, (3 * sms) / 4, sms}) {
      const int iters = static_cast<int>((8L << 30) / kChunk / grid);
      k<<<grid, 32, kStages * kChunk>>>(buf, f, 20);  // warm the footprint into L2
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      k<<<grid, 32, kStages * kChunk>>>(buf, f, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = static_cast<double>(iters) * grid * kChunk;
      printf("{\"footprint_MB\": %ld, \"ctas\": %d, \"TBps\": %.2f, \"err\": \"%s\"}\n", f >> 20, grid,
             bytes / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
