// Expert parallelism over NVLink peer memory.
//
// The NCCL path (ep.py: ep_forward) permutes into a local send buffer laid
// out [dst rank][local expert][C][d] and moves it with two all-to-alls. Here
// every rank maps its peers' receive / output buffers (CUDA IPC) and
//   - the permute stores each kept token row straight into the owning
//     rank's receive buffer (comoe_permute_peers, permute.cu),
//   - the per-(source, expert) row counts are scattered the same way
//     (comoe_peer_scatter_counts),
//   - a flag barrier over peer memory orders the phases
//     (comoe_peer_barrier),
//   - the combine reads the expert outputs from the owners' buffers
//     (comoe_combine_peers, permute.cu),
// so the dispatch and combine exchanges are the permute's stores and the
// combine's loads themselves, with no staging copy and no collective launch.
#include <cuda.h>

#include "common.cuh"
#include "../../include/comoe_b200.h"

namespace comoe {

__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Thread q < world: publish `epoch` into rank q's pad slot [rank], then wait
// until rank q has published `epoch` (or later) into my pad slot [q]. Epochs
// only grow, so a pad never needs resetting. Writes of earlier kernels in
// this stream are complete at kernel start; the system fence orders them
// (and the scattered counts) before the flag. A wait that exceeds
// `timeout_ns` sets *err = 1 + q and gives up instead of hanging the GPU.
__global__ void peer_barrier_kernel(int* const* pads, int world, int rank, int epoch,
                                    long long timeout_ns, int* err) {
  const int q = threadIdx.x;
  if (q >= world) return;
  __threadfence_system();
  st_release_sys(pads[q] + rank, epoch);
  const int* mine = pads[rank] + q;
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (ld_acquire_sys(mine) < epoch) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      atomicCAS(err, 0, 1 + q);
      return;
    }
    __nanosleep(64);
  }
}

// counts[e] (rows of global expert e from this rank) -> rank e / El's
// receive counts at [src * El + e % El].
__global__ void peer_scatter_counts_kernel(const int* __restrict__ counts, int E, int El,
                                           int src_rank, int* const* peer_counts) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x)
    peer_counts[e / El][src_rank * El + e % El] = counts[e];
}

}  // namespace comoe

extern "C" {

int comoe_ipc_handle_size(void) { return static_cast<int>(sizeof(cudaIpcMemHandle_t)); }

int comoe_ipc_get_handle(const void* ptr, void* handle_out, long* offset_out) {
  using namespace comoe;
  COMOE_REQUIRE(ptr && handle_out && offset_out, kBadArg, "ipc_get_handle: null pointer");
  // the allocation base (IPC handles name whole allocations; a caching
  // allocator hands out pointers inside them), via the driver entry point
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<GetRange>(fn);
  }();
  COMOE_REQUIRE(get_range, kNoDriver, "ipc_get_handle: cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  const CUresult r = get_range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr));
  COMOE_REQUIRE(r == CUDA_SUCCESS, kCudaError, "ipc_get_handle: cuMemGetAddressRange failed (%d)",
                static_cast<int>(r));
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  COMOE_REQUIRE(e == cudaSuccess, kCudaError, "ipc_get_handle: %s", cudaGetErrorString(e));
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = static_cast<long>(reinterpret_cast<CUdeviceptr>(ptr) - base);
  return kOk;
}

int comoe_ipc_open(const void* handle, long offset, void** ptr_out) {
  using namespace comoe;
  COMOE_REQUIRE(handle && ptr_out, kBadArg, "ipc_open: null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  const cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  COMOE_REQUIRE(e == cudaSuccess, kCudaError, "ipc_open: %s", cudaGetErrorString(e));
  *ptr_out = static_cast<char*>(base) + offset;
  return kOk;
}

int comoe_ipc_close(void* ptr, long offset) {
  using namespace comoe;
  COMOE_REQUIRE(ptr, kBadArg, "ipc_close: null pointer");
  const cudaError_t e = cudaIpcCloseMemHandle(static_cast<char*>(ptr) - offset);
  COMOE_REQUIRE(e == cudaSuccess, kCudaError, "ipc_close: %s", cudaGetErrorString(e));
  return kOk;
}

int comoe_peer_barrier(int* const* pads, int world, int rank, int epoch, long long timeout_ns,
                       int* err, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(pads && err, kBadArg, "peer_barrier: null pointer");
  COMOE_REQUIRE(world >= 1 && world <= 1024 && rank >= 0 && rank < world && epoch > 0, kBadArg,
                "peer_barrier: world=%d rank=%d epoch=%d", world, rank, epoch);
  peer_barrier_kernel<<<1, ((world + 31) / 32) * 32, 0, static_cast<cudaStream_t>(stream)>>>(
      pads, world, rank, epoch, timeout_ns, err);
  return check_launch("peer_barrier_kernel");
}

int comoe_peer_scatter_counts(const int* counts, int E, int world, int src_rank,
                              int* const* peer_counts, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(counts && peer_counts, kBadArg, "peer_scatter_counts: null pointer");
  COMOE_REQUIRE(world >= 1 && E % world == 0 && src_rank >= 0 && src_rank < world, kBadArg,
                "peer_scatter_counts: E=%d world=%d rank=%d", E, world, src_rank);
  peer_scatter_counts_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      counts, E, E / world, src_rank, peer_counts);
  return check_launch("peer_scatter_counts_kernel");
}

}  // extern "C"
