// K8: batched next-layer expert predictor.
//
// PredictorMLP.forward_batch (pkg/src/comoe/offload.py:147-154) over inputs
// built like predict_next_layer (offload.py:157-172): x = [K-hot(slots) over
// E | token embedding | context]. The K-hot part is never materialised: its
// contribution to W1 x is the sum of the K selected W1 columns. fp64 end to
// end (the reference is fp64).
//
// Layout: each block stages W1^T [in_dim][hidden] and W2^T [hidden][E] in
// shared memory once, so in both layers the 32 lanes of a warp read 32
// consecutive doubles (lane = hidden unit, then lane = expert) instead of 32
// different weight rows — the first version (one lane per row, weights read
// through L1) issued ~5000 L1 wavefronts per token and ran at 72 GB/s.
// A block owns 256-token chunks (one warp per token, 8 warps); the optional
// per-expert demand is reduced per chunk in token order into `work`, then
// across chunks in chunk order — deterministic, independent of the grid.
#include "common.cuh"
#include "../../include/comoe_b200.h"

namespace comoe {

constexpr int kPredMaxHidden = 256;
constexpr int kPredWarps = 16;
constexpr int kPredChunk = 256;  // tokens per demand partial
constexpr int kPredEPL = 8;      // experts per lane in registers (E <= 256)
constexpr int kPredTok = 4;      // tokens per warp pass

static long pred_smem_bytes(int in_dim, int hidden, int E) {
  return 8L * (static_cast<long>(in_dim) * hidden + hidden + static_cast<long>(hidden) * E + E +
               kPredWarps * kPredTok * hidden);
}

// A warp evaluates kPredTok tokens at once so every weight read from shared
// memory feeds kPredTok FMAs; EPL = experts per lane (E <= 32 * EPL) is a
// template parameter so no predicated-off FMA chains are issued.
template <int EPL>
__global__ void __launch_bounds__(kPredWarps * 32, 2) predictor_kernel(
    const int* __restrict__ slots, int B, int K, const double* __restrict__ emb, int emb_dim,
    const double* __restrict__ ctx, int ctx_dim, const double* __restrict__ w1,
    const double* __restrict__ b1, int hidden, const double* __restrict__ w2,
    const double* __restrict__ b2, int E, double* __restrict__ probs,
    double* __restrict__ partial, int demand_mode) {
  extern __shared__ double psm[];
  const int in_dim = E + emb_dim + ctx_dim;
  double* w1t = psm;                                        // [in_dim][hidden]
  double* b1s = w1t + static_cast<long>(in_dim) * hidden;   // [hidden]
  double* w2t = b1s + hidden;                               // [hidden][E]
  double* b2s = w2t + static_cast<long>(hidden) * E;        // [E]
  double* hs = b2s + E;                                     // [warps][kPredTok][hidden]
  for (long i = threadIdx.x; i < static_cast<long>(in_dim) * hidden; i += blockDim.x) {
    const int h = static_cast<int>(i / in_dim), j = static_cast<int>(i % in_dim);
    w1t[static_cast<long>(j) * hidden + h] = w1[i];  // coalesced read of W1 [hidden][in_dim]
  }
  for (long i = threadIdx.x; i < static_cast<long>(E) * hidden; i += blockDim.x) {
    const int e = static_cast<int>(i / hidden), h = static_cast<int>(i % hidden);
    w2t[static_cast<long>(h) * E + e] = w2[i];       // W2 [E][hidden]
  }
  for (int i = threadIdx.x; i < hidden; i += blockDim.x) b1s[i] = b1[i];
  for (int i = threadIdx.x; i < E; i += blockDim.x) b2s[i] = b2[i];
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* hw = hs + warp * kPredTok * hidden;
  const int n_chunks = (B + kPredChunk - 1) / kPredChunk;
  for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const int t_end = min(B, (c + 1) * kPredChunk);
    for (int t0 = c * kPredChunk + warp * kPredTok; t0 < t_end; t0 += kPredWarps * kPredTok) {
      // hidden = relu(W1 x + b1): the reference's dense x.w sum, with the
      // K-hot block contributing its selected columns (x[s] = 1, duplicates once)
      for (int h0 = 0; h0 < hidden; h0 += 32) {  // warp-uniform (the shuffles below)
        const int h = h0 + lane < hidden ? h0 + lane : hidden - 1;  // lanes past hidden: discarded
        double z[kPredTok];
#pragma unroll
        for (int q = 0; q < kPredTok; ++q) {
          z[q] = b1s[h];
          const int t = min(t0 + q, t_end - 1);
          const int* st = slots + static_cast<long>(t) * K;
          for (int k = 0; k < K; ++k) {
            const int s = __ldg(st + k);
            bool dup = false;
            for (int kk = 0; kk < k; ++kk) dup |= __ldg(st + kk) == s;
            if (!dup && s >= 0 && s < E) z[q] += w1t[static_cast<long>(s) * hidden + h];
          }
        }
        // dense inputs [emb | ctx] of the kPredTok tokens: 32 at a time, one
        // coalesced load per lane, then broadcast by shuffle (each lane read
        // every element through L1 before: a dependent load per FMA)
        const int dense = emb_dim + ctx_dim;
        for (int j0 = 0; j0 < dense; j0 += 32) {
          double xv[kPredTok];
#pragma unroll
          for (int q = 0; q < kPredTok; ++q) {
            const int t = min(t0 + q, t_end - 1);
            const int j = j0 + lane;
            xv[q] = j < emb_dim ? __ldg(emb + static_cast<long>(t) * emb_dim + j)
                    : j < dense ? __ldg(ctx + static_cast<long>(t) * ctx_dim + (j - emb_dim))
                                : 0.0;
          }
          const int jn = dense - j0 < 32 ? dense - j0 : 32;
          for (int jj = 0; jj < jn; ++jj) {
            const double w = w1t[static_cast<long>(E + j0 + jj) * hidden + h];
#pragma unroll
            for (int q = 0; q < kPredTok; ++q) z[q] = fma(w, __shfl_sync(0xffffffffu, xv[q], jj), z[q]);
          }
        }
        if (h0 + lane < hidden)
#pragma unroll
          for (int q = 0; q < kPredTok; ++q) hw[q * hidden + h] = z[q] > 0.0 ? z[q] : 0.0;
      }
      __syncwarp();
      // logits = W2 h + b2 ; softmax over E. Lane owns experts lane + 32u.
      double z[kPredTok][EPL];
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        const double bv = (lane + 32 * u < E) ? b2s[lane + 32 * u] : 0.0;
#pragma unroll
        for (int q = 0; q < kPredTok; ++q) z[q][u] = bv;
      }
      for (int h = 0; h < hidden; ++h) {
        double w[EPL];
#pragma unroll
        for (int u = 0; u < EPL; ++u)
          w[u] = (lane + 32 * u < E) ? w2t[static_cast<long>(h) * E + lane + 32 * u] : 0.0;
#pragma unroll
        for (int q = 0; q < kPredTok; ++q) {
          const double hv = hw[q * hidden + h];
#pragma unroll
          for (int u = 0; u < EPL; ++u) z[q][u] = fma(w[u], hv, z[q][u]);
        }
      }
#pragma unroll
      for (int q = 0; q < kPredTok; ++q) {
        const int t = t0 + q;
        if (t >= t_end) break;  // warp-uniform
        double mx = -INFINITY;
#pragma unroll
        for (int u = 0; u < EPL; ++u)
          if (lane + 32 * u < E) mx = fmax(mx, z[q][u]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        double sum = 0.0;
#pragma unroll
        for (int u = 0; u < EPL; ++u)
          if (lane + 32 * u < E) {
            z[q][u] = exp(z[q][u] - mx);
            sum += z[q][u];
          }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        double* pt = probs + static_cast<long>(t) * E;
#pragma unroll
        for (int u = 0; u < EPL; ++u)
          if (lane + 32 * u < E) pt[lane + 32 * u] = z[q][u] / sum;
      }
      __syncwarp();
    }
    if (partial) {
      __syncthreads();  // every token of the chunk written (block-visible)
      for (int e = threadIdx.x; e < E; e += blockDim.x) {
        double s = 0.0;  // mode 0: sum_t p; mode 1: sum_t log(1 - p)
        for (int t = c * kPredChunk; t < t_end; ++t) {
          const double pt = probs[static_cast<long>(t) * E + e];
          s += demand_mode ? log1p(-pt) : pt;
        }
        partial[static_cast<long>(c) * E + e] = s;
      }
    }
  }
}

// demand[e] = sum over chunks (in order) of the chunk partials; mode 1
// turns the summed log(1 - p) into P(some token of the batch picks e)
__global__ void demand_kernel(const double* __restrict__ partial, int n_chunks, int E,
                              int demand_mode, double* __restrict__ demand) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < n_chunks; ++c) s += partial[static_cast<long>(c) * E + e];
    demand[e] = demand_mode ? -expm1(s) : s;
  }
}

}  // namespace comoe

extern "C" {

long comoe_predictor_workspace_bytes(int B, int E) {
  if (B <= 0 || E <= 0) return 0;
  return 8L * ((B + comoe::kPredChunk - 1) / comoe::kPredChunk) * E;
}

int comoe_predictor_mlp(const int* slots, int B, int K, const double* emb, int emb_dim,
                        const double* ctx, int ctx_dim, const double* w1, const double* b1,
                        int hidden, const double* w2, const double* b2, int E, double* probs,
                        double* demand, int demand_mode, void* work, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(slots && w1 && b1 && w2 && b2 && probs, kBadArg, "predictor: null pointer");
  COMOE_REQUIRE((emb_dim == 0 || emb) && (ctx_dim == 0 || ctx), kBadArg, "predictor: null emb/ctx");
  COMOE_REQUIRE(hidden >= 1 && hidden <= kPredMaxHidden, kUnsupportedShape,
                "predictor: hidden=%d > %d", hidden, kPredMaxHidden);
  COMOE_REQUIRE(B >= 0 && K >= 1 && E >= 1 && emb_dim >= 0 && ctx_dim >= 0, kBadArg,
                "predictor: bad sizes");
  COMOE_REQUIRE(!demand || work, kBadArg, "predictor: demand needs the workspace");
  COMOE_REQUIRE(demand_mode == 0 || demand_mode == 1, kBadArg, "predictor: demand_mode=%d",
                demand_mode);
  COMOE_REQUIRE(E <= 32 * kPredEPL, kUnsupportedShape, "predictor: E=%d > %d", E, 32 * kPredEPL);
  const long smem = pred_smem_bytes(E + emb_dim + ctx_dim, hidden, E);
  COMOE_REQUIRE(smem <= 227 * 1024, kUnsupportedShape,
                "predictor: weights need %ld B of shared memory (> 227 KB)", smem);
  if (B == 0) {
    if (demand) cudaMemsetAsync(demand, 0, sizeof(double) * E, static_cast<cudaStream_t>(stream));  // both modes: 0
    return check_launch("predictor(empty)");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int n_chunks = (B + kPredChunk - 1) / kPredChunk;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int per_sm = smem <= 72 * 1024 ? 3 : smem <= 110 * 1024 ? 2 : 1;
  const int blocks = n_chunks < sms * per_sm ? n_chunks : sms * per_sm;
  double* partial = demand ? static_cast<double*>(work) : nullptr;
  auto launch = [&](auto kern) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<blocks, kPredWarps * 32, smem, s>>>(slots, B, K, emb, emb_dim, ctx, ctx_dim, w1, b1,
                                                hidden, w2, b2, E, probs, partial, demand_mode);
  };
  if (E <= 32) launch(predictor_kernel<1>);
  else if (E <= 64) launch(predictor_kernel<2>);
  else if (E <= 128) launch(predictor_kernel<4>);
  else launch(predictor_kernel<8>);
  int rc = check_launch("predictor_kernel");
  if (rc || !demand) return rc;
  demand_kernel<<<(E + 127) / 128, 128, 0, s>>>(partial, n_chunks, E, demand_mode, demand);
  return check_launch("demand_kernel");
}

}  // extern "C"
