// Dev probe: throughput of the producer -> MMA -> commit ring on CTA pairs
// with no data movement. A stage = wait(empty) -> arrive(full) by the
// producer thread of each CTA, wait(full) -> K tcgen05.mma (M256, N) ->
// commit(empty, multicast) by the leader's issuer. Reports clocks per stage
// for S stages; with enough stages the cost is the MMA time (64 clk per
// N=128 MMA), otherwise the sync round trip divided by S.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/ring_probe.cu -o scripts/ring_probe.bin \
//      -Lpaper_2508_09208_b200 -lcomoe_b200 -lcuda -Xlinker -rpath=\$ORIGIN/../paper_2508_09208_b200
#include <cstdio>
#include "../paper_2508_09208_b200/csrc/grouped_gemm_2sm.cuh"

using namespace comoe;

template <int S, int K, int N, bool kPeerArrive, int kTma = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) ring(int iters, unsigned long long* out,
                                                                     const __grid_constant__ CUtensorMap tm) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[S], empty[S];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<int4*>(smem)[i] = make_int4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], kPeerArrive ? 2 : 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0 && lane == 0) {
    int st = 0; uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&empty[st], ph ^ 1);
      const uint32_t fb = smem_u32(&full[st]) & kPeerMask;
      if (kTma) {
        if (leader) mbar_expect_tx(&full[st], 2 * kTma * 16384);
        else mbar_arrive_cluster(fb);
        for (int b = 0; b < kTma; ++b)
          tma_load_3d_2sm(smem + (st % 2) * 16384, &tm, fb, (i % 12) * 64, (b & 1) * 128 + rank * 64, 0, 0);
      } else {
        if (leader) mbar_arrive(&full[st]);
        else if (kPeerArrive) mbar_arrive_cluster(fb);
      }
      if (++st == S) { st = 0; ph ^= 1; }
    }
  } else if (warp == 1 && leader && elect_one()) {
    const uint64_t a = umma_desc_k_sw128(smem_u32(smem));
    const uint64_t b = umma_desc_k_sw128(smem_u32(smem + 32768));
    const uint32_t idesc = umma_idesc_bf16_f32(256, N);
    int st = 0; uint32_t ph = 0;
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&full[st], ph);
      tc_fence_after();
#pragma unroll
      for (int k = 0; k < K; ++k) umma_bf16_2sm(tmem, a + 2 * (k & 3), b + 2 * (k & 3), idesc, 1);
      umma_commit_2sm_mc(&empty[st]);
      if (++st == S) { st = 0; ph ^= 1; }
    }
    // drain: wait for the last commit of each stage
    mbar_wait(&empty[(st + S - 1) % S], ((iters - 1) / S) & 1);
    out[blockIdx.x >> 1] = clock64() - t0;
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

static CUtensorMap g_tm;
template <int S, int K, int N, bool kPeer, int kTma = 0>
void run(int sms) {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 256);
  cudaMemset(d, 0, 8 * 256);
  auto k = ring<S, K, N, kPeer, kTma>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  const int iters = 6000;
  k<<<sms & ~1, 128, 70 * 1024>>>(iters, d, g_tm);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, 8 * 256, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms / 2; ++i) avg += h[i];
  avg /= (sms / 2);
  printf("tma=%d S=%2d K=%d N=%d peer_arrive=%d err=%d  clk/stage=%.0f  (MMA-bound %d)\n", kTma, S, K, N,
         (int)kPeer, (int)e, avg / iters, K * N / 2);
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* buf;
  cudaMalloc(&buf, 1 << 22);  // 2 slots of [256 rows x 768] bf16 (L2-resident)
  cudaMemset(buf, 0, 1 << 22);
  if (make_tmap_bf16_3d(&g_tm, buf, 2, 256, 768, 256 * 768, 128)) { printf("tmap failed\n"); return 1; }
  run<6, 4, 128, true, 1>(sms);
  run<6, 0, 128, true, 1>(sms);
  run<3, 8, 128, true, 2>(sms);
  run<8, 4, 128, true, 1>(sms);
  run<2, 0, 128, true>(sms);
  run<6, 0, 128, true>(sms);
  run<2, 4, 128, true>(sms);
  run<4, 4, 128, true>(sms);
  run<6, 4, 128, true>(sms);
  run<8, 4, 128, true>(sms);
  run<12, 4, 128, true>(sms);
  run<6, 4, 128, false>(sms);
  run<6, 4, 256, true>(sms);
  run<3, 8, 128, true>(sms);
  return 0;
}
