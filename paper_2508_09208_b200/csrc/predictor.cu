// K8: batched next-layer expert predictor.
//
// PredictorMLP.forward_batch (pkg/src/comoe/offload.py:147-154) over inputs
// built like predict_next_layer (offload.py:157-172): x = [K-hot(slots) over
// E | token embedding | context]. The K-hot part is never materialised: its
// contribution to W1 x is the sum of the K selected W1 columns. One warp per
// token, fp64 end to end (the reference is fp64).
#include "common.cuh"
#include "../../include/comoe_b200.h"

namespace comoe {

constexpr int kPredMaxHidden = 256;
constexpr int kPredWarps = 4;

__global__ void __launch_bounds__(kPredWarps * 32) predictor_kernel(
    const int* __restrict__ slots, int B, int K, const double* __restrict__ emb, int emb_dim,
    const double* __restrict__ ctx, int ctx_dim, const double* __restrict__ w1,
    const double* __restrict__ b1, int hidden, const double* __restrict__ w2,
    const double* __restrict__ b2, int E, double* __restrict__ probs) {
  __shared__ double hs[kPredWarps][kPredMaxHidden];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int in_dim = E + emb_dim + ctx_dim;
  const int warps_total = gridDim.x * kPredWarps;
  for (int t = blockIdx.x * kPredWarps + warp; t < B; t += warps_total) {
    // hidden = relu(W1 x + b1)
    for (int h = lane; h < hidden; h += 32) {
      const double* row = w1 + static_cast<long>(h) * in_dim;
      double z = b1[h];
      // the reference builds a dense x and sums x[j]*w[j] over all j via BLAS;
      // here the K-hot block contributes its selected columns (x[s] = 1)
      for (int k = 0; k < K; ++k) {
        const int s = slots[static_cast<long>(t) * K + k];
        bool dup = false;
        for (int kk = 0; kk < k; ++kk) dup |= slots[static_cast<long>(t) * K + kk] == s;
        if (!dup && s >= 0 && s < E) z += row[s];
      }
      for (int j = 0; j < emb_dim; ++j) z = fma(row[E + j], emb[static_cast<long>(t) * emb_dim + j], z);
      for (int j = 0; j < ctx_dim; ++j)
        z = fma(row[E + emb_dim + j], ctx[static_cast<long>(t) * ctx_dim + j], z);
      hs[warp][h] = z > 0.0 ? z : 0.0;
    }
    __syncwarp();
    // logits = W2 h + b2 ; softmax over E
    double mx = -INFINITY;
    for (int e = lane; e < E; e += 32) {
      const double* row = w2 + static_cast<long>(e) * hidden;
      double z = b2[e];
      for (int h = 0; h < hidden; ++h) z = fma(row[h], hs[warp][h], z);
      probs[static_cast<long>(t) * E + e] = z;
      mx = fmax(mx, z);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    double sum = 0.0;
    for (int e = lane; e < E; e += 32) {
      const double v = exp(probs[static_cast<long>(t) * E + e] - mx);
      probs[static_cast<long>(t) * E + e] = v;
      sum += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    for (int e = lane; e < E; e += 32) probs[static_cast<long>(t) * E + e] /= sum;
    __syncwarp();
  }
}

// demand[e] = sum_t probs[t, e], tokens summed in order (deterministic).
__global__ void demand_kernel(const double* __restrict__ probs, int B, int E,
                              double* __restrict__ demand) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int t = 0; t < B; ++t) s += probs[static_cast<long>(t) * E + e];
    demand[e] = s;
  }
}

}  // namespace comoe

extern "C" {

int comoe_predictor_mlp(const int* slots, int B, int K, const double* emb, int emb_dim,
                        const double* ctx, int ctx_dim, const double* w1, const double* b1,
                        int hidden, const double* w2, const double* b2, int E, double* probs,
                        double* demand, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(slots && w1 && b1 && w2 && b2 && probs, kBadArg, "predictor: null pointer");
  COMOE_REQUIRE((emb_dim == 0 || emb) && (ctx_dim == 0 || ctx), kBadArg, "predictor: null emb/ctx");
  COMOE_REQUIRE(hidden >= 1 && hidden <= kPredMaxHidden, kUnsupportedShape,
                "predictor: hidden=%d > %d", hidden, kPredMaxHidden);
  COMOE_REQUIRE(B >= 0 && K >= 1 && E >= 1, kBadArg, "predictor: bad sizes");
  if (B == 0) return kOk;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int blocks = (B + kPredWarps - 1) / kPredWarps;
  if (blocks > 148 * 16) blocks = 148 * 16;
  predictor_kernel<<<blocks, kPredWarps * 32, 0, s>>>(slots, B, K, emb, emb_dim, ctx, ctx_dim, w1,
                                                       b1, hidden, w2, b2, E, probs);
  int rc = check_launch("predictor_kernel");
  if (rc || !demand) return rc;
  demand_kernel<<<(E + 127) / 128, 128, 0, s>>>(probs, B, E, demand);
  return check_launch("demand_kernel");
}

}  // extern "C"
