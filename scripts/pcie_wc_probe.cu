// H2D from write-combined vs ordinary pinned host memory, alone and with a
// concurrent D2H (dev probe for the host pipeline): 100 MB per direction in
// 4 chunks over 2 streams per direction, GB/s per direction.
//   nvcc -O2 -o /tmp/pcie_wc scripts/pcie_wc_probe.cu
#include <cuda_runtime.h>
#include <cstdio>

static float run(char* h_in, char* h_out, char* d_in, char* d_out, size_t n, bool both) {
  cudaStream_t s[4];
  for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaDeviceSynchronize();
  cudaEventRecord(a, s[0]);
  for (int i = 1; i < 4; ++i) cudaStreamWaitEvent(s[i], a, 0);
  const int reps = 5, chunks = 4;
  const size_t step = n / chunks;
  for (int r = 0; r < reps; ++r)
    for (int c = 0; c < chunks; ++c) {
      cudaMemcpyAsync(d_in + c * step, h_in + c * step, step, cudaMemcpyHostToDevice, s[c % 2]);
      if (both)
        cudaMemcpyAsync(h_out + c * step, d_out + c * step, step, cudaMemcpyDeviceToHost,
                        s[2 + c % 2]);
    }
  for (int i = 1; i < 4; ++i) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s[i]);
    cudaStreamWaitEvent(s[0], e, 0);
  }
  cudaEventRecord(b, s[0]);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return static_cast<float>(n) * reps / (ms * 1e-3f) / 1e9f;
}

int main() {
  const size_t n = 100663296;
  char *h_pin, *h_wc, *h_out, *d_in, *d_out;
  cudaHostAlloc(&h_pin, n, cudaHostAllocDefault);
  cudaHostAlloc(&h_wc, n, cudaHostAllocWriteCombined);
  cudaHostAlloc(&h_out, n, cudaHostAllocDefault);
  cudaMalloc(&d_in, n);
  cudaMalloc(&d_out, n);
  for (size_t i = 0; i < n; i += 4096) { h_pin[i] = 1; h_wc[i] = 1; h_out[i] = 1; }
  for (int rep = 0; rep < 2; ++rep) {
    printf("{\"h2d_pinned\": %.1f, \"h2d_wc\": %.1f, \"duplex_h2d_pinned\": %.1f, \"duplex_h2d_wc\": %.1f}\n",
           run(h_pin, h_out, d_in, d_out, n, false), run(h_wc, h_out, d_in, d_out, n, false),
           run(h_pin, h_out, d_in, d_out, n, true), run(h_wc, h_out, d_in, d_out, n, true));
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
