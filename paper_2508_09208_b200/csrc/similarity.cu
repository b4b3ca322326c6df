// K6: expert similarity (cosine Gram + functional surrogate) on the device.
//
// Restates similarity_matrix (pkg/src/comoe/moe.py:339-365). The surrogate
// einsum "nd,ed,bd->enb" (moe.py:351) is the same contraction as the Gram
// once the probe/projection product Q[(n,b),d] = probes[n,d]*proj[b,d] is
// formed on the fly, so both are one split-K "rows x columns" contraction:
//     C[e, j] = sum_d P[e,d] * Col_j[d],  Col = [P rows ; Q rows]
// computed in 32x32 output tiles over D-slices, then reduced over slices in a
// fixed order (deterministic). Always accumulated in fp64 (the reference is
// fp64 and its surrogate softmax is sensitive to logit error).
#include "common.cuh"
#include "../../include/comoe_b200.h"

namespace comoe {

constexpr int kSimTile = 32;
constexpr int kSimKc = 32;

template <typename T>
__device__ __forceinline__ double to_f64(T v);
template <>
__device__ __forceinline__ double to_f64<double>(double v) { return v; }
template <>
__device__ __forceinline__ double to_f64<__nv_bfloat16>(__nv_bfloat16 v) {
  return static_cast<double>(__bfloat162float(v));
}

// grid: x = output tile (tiles over [E] x [E + n*B]), y = D-slice.
template <typename T>
__global__ void __launch_bounds__(256) sim_contract_kernel(const void* const* __restrict__ rows, int E,
                                                           long D, const double* __restrict__ probes,
                                                           int n_probes,
                                                           const double* __restrict__ proj,
                                                           int buckets, int tiles_j,
                                                           double* __restrict__ partial) {
  const int ncols = E + n_probes * buckets;
  const int ti = blockIdx.x / tiles_j, tj = blockIdx.x % tiles_j;
  const int i0 = ti * kSimTile, j0 = tj * kSimTile;
  const long slice = (D + gridDim.y - 1) / gridDim.y;
  const long d0 = blockIdx.y * slice;
  const long d1 = d0 + slice < D ? d0 + slice : D;

  __shared__ double sa[kSimKc][kSimTile + 1];
  __shared__ double sb[kSimKc][kSimTile + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 2x2 outputs each
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};

  for (long k0 = d0; k0 < d1; k0 += kSimKc) {
    // stage 32 rows x 32 d of A (expert rows) and of the column operand
    for (int idx = threadIdx.x; idx < kSimTile * kSimKc; idx += blockDim.x) {
      const int r = idx / kSimKc, c = idx % kSimKc;
      const long d = k0 + c;
      double av = 0.0, bv = 0.0;
      if (d < d1) {
        const int i = i0 + r;
        if (i < E) av = to_f64(static_cast<const T*>(rows[i])[d]);
        const int j = j0 + r;
        if (j < E) {
          bv = to_f64(static_cast<const T*>(rows[j])[d]);
        } else if (j < ncols) {
          const int q = j - E;
          bv = probes[static_cast<long>(q / buckets) * D + d] * proj[static_cast<long>(q % buckets) * D + d];
        }
      }
      sa[c][r] = av;
      sb[c][r] = bv;
    }
    __syncthreads();
#pragma unroll 8
    for (int c = 0; c < kSimKc; ++c) {
      const double a0 = sa[c][ty * 2], a1 = sa[c][ty * 2 + 1];
      const double b0 = sb[c][tx * 2], b1 = sb[c][tx * 2 + 1];
      acc[0][0] = fma(a0, b0, acc[0][0]);
      acc[0][1] = fma(a0, b1, acc[0][1]);
      acc[1][0] = fma(a1, b0, acc[1][0]);
      acc[1][1] = fma(a1, b1, acc[1][1]);
    }
    __syncthreads();
  }
  double* out = partial + static_cast<long>(blockIdx.y) * E * ncols;
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int i = i0 + ty * 2 + u, j = j0 + tx * 2 + v;
      if (i < E && j < ncols) out[static_cast<long>(i) * ncols + j] = acc[u][v];
    }
}

__global__ void sim_reduce_kernel(const double* __restrict__ partial, int splits, int E, int ncols,
                                  double* __restrict__ gram, double* __restrict__ logits) {
  const long n = static_cast<long>(E) * ncols;
  for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < n;
       idx += static_cast<long>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < splits; ++k) s += partial[k * n + idx];
    const int i = static_cast<int>(idx / ncols), j = static_cast<int>(idx % ncols);
    if (j < E) gram[static_cast<long>(i) * E + j] = s;
    else logits[static_cast<long>(i) * (ncols - E) + (j - E)] = s;
  }
}

// One thread per (e1, e2): cosine from the Gram, symmetric KL of the
// log-softmax surrogate distributions averaged over probes.
__global__ void sim_finalize_kernel(const double* __restrict__ gram,
                                    const double* __restrict__ logits, int E, int n_probes,
                                    int buckets, double alpha, double* __restrict__ sim) {
  const long pairs = static_cast<long>(E) * E;
  for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < pairs;
       idx += static_cast<long>(gridDim.x) * blockDim.x) {
    const int a = static_cast<int>(idx / E), b = static_cast<int>(idx % E);
    const double cosv = gram[static_cast<long>(a) * E + b] /
                        (sqrt(gram[static_cast<long>(a) * E + a]) * sqrt(gram[static_cast<long>(b) * E + b]));
    double mean_kl = 0.0;
    for (int n = 0; n < n_probes; ++n) {
      const double* la = logits + (static_cast<long>(a) * n_probes + n) * buckets;
      const double* lb = logits + (static_cast<long>(b) * n_probes + n) * buckets;
      double ma = -INFINITY, mb = -INFINITY;
      for (int k = 0; k < buckets; ++k) {
        ma = fmax(ma, la[k]);
        mb = fmax(mb, lb[k]);
      }
      double sa = 0.0, sb = 0.0;
      for (int k = 0; k < buckets; ++k) {
        sa += exp(la[k] - ma);
        sb += exp(lb[k] - mb);
      }
      const double lsa = ma + log(sa), lsb = mb + log(sb);
      double kab = 0.0, kba = 0.0;
      for (int k = 0; k < buckets; ++k) {
        const double lpa = la[k] - lsa, lpb = lb[k] - lsb;
        const double pa = exp(lpa), pb = exp(lpb);
        if (pa > 0.0) kab += pa * (lpa - lpb);
        if (pb > 0.0) kba += pb * (lpb - lpa);
      }
      mean_kl += 0.5 * (kab + kba);
    }
    if (n_probes > 0) mean_kl /= n_probes;
    double sf = 1.0 - mean_kl;
    sf = sf < 0.0 ? 0.0 : (sf > 1.0 ? 1.0 : sf);
    sim[idx] = alpha * cosv + (1.0 - alpha) * sf;
  }
}

static int sim_splits(int E, int ncols, long D) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long tiles = static_cast<long>((E + kSimTile - 1) / kSimTile) * ((ncols + kSimTile - 1) / kSimTile);
  long splits = (static_cast<long>(sms) * 4 + tiles - 1) / tiles;
  const long max_by_d = (D + 4095) / 4096;  // at least 4096 d per slice
  if (splits > max_by_d) splits = max_by_d;
  if (splits > 1024) splits = 1024;
  if (splits < 1) splits = 1;
  return static_cast<int>(splits);
}

}  // namespace comoe

extern "C" {

long comoe_sim_workspace_bytes(int E, int n_probes, int buckets, long D) {
  const int ncols = E + (n_probes > 0 ? n_probes * buckets : 0);
  return static_cast<long>(comoe::sim_splits(E, ncols, D)) * E * ncols * sizeof(double);
}

int comoe_sim_contract(int dtype, const void* const* rows, int E, long D, const double* probes,
                       int n_probes, const double* proj, int buckets, double* gram,
                       double* logits, void* work, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(rows && gram && work, kBadArg, "sim_contract: null pointer");
  COMOE_REQUIRE(n_probes == 0 || (probes && proj && logits && buckets >= 1), kBadArg,
                "sim_contract: null calibration");
  COMOE_REQUIRE(E >= 1 && D >= 1 && n_probes >= 0, kBadArg, "sim_contract: bad sizes");
  if (n_probes == 0) buckets = 0;  // cosine only
  const int ncols = E + n_probes * buckets;
  const int splits = sim_splits(E, ncols, D);
  const int tiles_i = (E + kSimTile - 1) / kSimTile, tiles_j = (ncols + kSimTile - 1) / kSimTile;
  dim3 grid(tiles_i * tiles_j, splits);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* partial = static_cast<double*>(work);
  if (dtype == COMOE_DTYPE_BF16)
    sim_contract_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(rows, E, D, probes, n_probes, proj,
                                                            buckets, tiles_j, partial);
  else if (dtype == COMOE_DTYPE_F64)
    sim_contract_kernel<double><<<grid, 256, 0, s>>>(rows, E, D, probes, n_probes, proj, buckets,
                                                     tiles_j, partial);
  else {
    set_error("sim_contract: dtype %d", dtype);
    return kBadArg;
  }
  int rc = check_launch("sim_contract_kernel");
  if (rc) return rc;
  const long n = static_cast<long>(E) * ncols;
  const int blocks = static_cast<int>((n + 255) / 256 < 2048 ? (n + 255) / 256 : 2048);
  sim_reduce_kernel<<<blocks, 256, 0, s>>>(partial, splits, E, ncols, gram, logits);
  return check_launch("sim_reduce_kernel");
}

int comoe_sim_finalize(const double* gram, const double* logits, int E, int n_probes, int buckets,
                       double alpha, double* sim, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(gram && sim && (logits || n_probes == 0), kBadArg, "sim_finalize: null pointer");
  COMOE_REQUIRE(alpha >= 0.0 && alpha <= 1.0, kBadArg, "sim_finalize: alpha=%g", alpha);
  const long pairs = static_cast<long>(E) * E;
  const int blocks = static_cast<int>((pairs + 127) / 128 < 1024 ? (pairs + 127) / 128 : 1024);
  sim_finalize_kernel<<<blocks, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      gram, logits, E, n_probes, buckets, alpha, sim);
  return check_launch("sim_finalize_kernel");
}

}  // extern "C"
