// HBM -> SM streaming by load mechanism (dev probe): one thread per CTA
// keeps a ring of 16 KB stages full with either (a) 1-D cp.async.bulk copies
// of 16 KB contiguous, or (b) 2-D tensor-map boxes of 128 rows x 128 B,
// SWIZZLE_128B (the operand loads of the gate, grouped GEMM and Gram), over
// a 2 GiB buffer viewed as [rows, cols] bf16 with a row pitch of cols * 2 B:
// pitch 128 B makes every box one contiguous 16 KB, 1536 B is the token-row
// pitch of x at d = 768. No compute. Prints TB/s per (mode, pitch, stages).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe scripts/tma_dram_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(
                   su32(b)), "r"(ph) : "memory");
}

template <int kMode>  // 0 bulk, 1 tensor 2-D box
__global__ void __launch_bounds__(32, 1) stream_kernel(const __grid_constant__ CUtensorMap map,
                                                       const char* buf, long n_boxes,
                                                       int col_blocks, int stages, int iters) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar[16];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  long b = blockIdx.x;
  for (int i = 0; i < iters; ++i) {
    const int s = i % stages;
    if (i >= stages) wait_bar(&bar[s], ((i / stages) - 1) & 1);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(16384)
                 : "memory");
    const long bb = b % n_boxes;
    if constexpr (kMode == 0) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(smem + s * 16384)), "l"(buf + bb * 16384), "r"(16384), "r"(su32(&bar[s]))
                   : "memory");
    } else {
      const int x = static_cast<int>(bb % col_blocks) * 64, y = static_cast<int>(bb / col_blocks) * 128;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              su32(smem + s * 16384)), "l"(reinterpret_cast<uint64_t>(&map)), "r"(su32(&bar[s])), "r"(x), "r"(y)
          : "memory");
    }
    b += gridDim.x;
  }
  for (int i = iters - stages; i < iters; ++i)
    if (i >= 0) wait_bar(&bar[i % stages], (i / stages) & 1);
}

int main(int argc, char** argv) {
  const long bytes = 2L << 30;
  char* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  // Gram-like: 128 rows (whole experts) of `pitch` bytes, boxes walk the columns
  // argv: pitches (bytes) of the gram-like sweep; default: the round-2 set
  std::vector<long> pitches = {9437184L, 4L << 20, 2L << 20, 1572864L, 1L << 20, 512L << 10, 256L << 10, 64L << 10};
  if (argc > 1) {
    pitches.clear();
    for (int i = 1; i < argc; ++i) pitches.push_back(std::atol(argv[i]));
  }
  for (long pitch : pitches) {
    const long rows = 128, cols = (bytes / rows / 1024) * 512;  // row length in elements
    CUtensorMap map{};
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)pitch};
    if (pitch * rows > bytes) continue;
    const long cols_fit = pitch / 2;
    dims[0] = (cuuint64_t)cols_fit;
    cuuint32_t box[2] = {64, 128}, estr[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box,
                                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    const int col_blocks = static_cast<int>(cols_fit / 64);
    const long n_boxes = col_blocks;
    const int stages = 8, smem = stages * 16384 + 1024;
    auto k = stream_kernel<1>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = static_cast<int>(n_boxes / sms);
    k<<<sms, 32, smem>>>(map, buf, n_boxes, col_blocks, stages, iters);
    cudaEventRecord(a);
    for (int rep = 0; rep < 3; ++rep) k<<<sms, 32, smem>>>(map, buf, n_boxes, col_blocks, stages, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"mode\": \"gram-like 128 rows\", \"pitch\": %ld, \"TBps\": %.3f}\n", pitch,
           3.0 * iters * (double)sms * 16384 / (ms * 1e-3) / 1e12);
    (void)cols;
  }
  for (int mode = 0; mode < (argc > 1 ? 0 : 2); ++mode)
    for (long pitch : {128L, 1536L, 6144L}) {
      if (mode == 0 && pitch != 128) continue;
      const long cols = pitch / 2, rows = bytes / pitch;
      CUtensorMap map{};
      cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
      cuuint64_t strides[1] = {(cuuint64_t)pitch};
      cuuint32_t box[2] = {64, 128}, estr[2] = {1, 1};
      CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box,
                                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
      const int col_blocks = static_cast<int>(cols / 64);
      const long n_boxes = (rows / 128) * col_blocks;
      for (int stages : {4, 8, 12}) {
        const int smem = stages * 16384 + 1024;
        auto k = mode == 0 ? stream_kernel<0> : stream_kernel<1>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int iters = static_cast<int>(n_boxes / sms);
        k<<<sms, 32, smem>>>(map, buf, n_boxes, col_blocks, stages, iters);  // warm
        cudaEventRecord(a);
        for (int rep = 0; rep < 3; ++rep) k<<<sms, 32, smem>>>(map, buf, n_boxes, col_blocks, stages, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double tb = 3.0 * iters * (double)sms * 16384 / (ms * 1e-3) / 1e12;
        printf("{\"mode\": \"%s\", \"pitch\": %ld, \"stages\": %d, \"TBps\": %.3f}\n",
               mode == 0 ? "bulk16K" : "tensor128x128B", pitch, stages, tb);
      }
    }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
