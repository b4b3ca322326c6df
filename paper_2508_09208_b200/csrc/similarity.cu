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
#include <cstdlib>
#include <utility>

#include "grouped_gemm.cuh"
#include "../../include/comoe_b200.h"

namespace comoe {

constexpr int kSimKc = 16;      // d per smem stage (a 32-byte sector of a bf16 row)
constexpr int kSimTJ = 64;      // output columns per tile
constexpr int kSimSmallE = 8;   // register-resident cosine path for E <= 8

template <typename T>
__device__ __forceinline__ double to_f64(T v);
template <>
__device__ __forceinline__ double to_f64<double>(double v) { return v; }
template <>
__device__ __forceinline__ double to_f64<__nv_bfloat16>(__nv_bfloat16 v) {
  return static_cast<double>(__bfloat162float(v));
}

// Row tile height: 64 (4x4 outputs per thread, 0.5 smem loads per FMA —
// the first version's 32x32 tile with 2x2 outputs did one load per FMA and
// ran L1-bound at 7 TF/s) or 16 for E <= 16 (small row counts would leave
// most of a 64-row tile empty).
static int sim_ti(int E) { return E <= 16 ? 16 : 64; }

// grid: x = output tile (tiles over [E] x [E + n*B]), y = D-slice.
// With 64x64 tiles the Gram block is symmetric: tiles strictly below the
// diagonal are skipped and mirrored by the reduction.
template <typename T, int TI>
__global__ void __launch_bounds__(256) sim_contract_kernel(const void* const* __restrict__ rows, int E,
                                                           long D, const double* __restrict__ probes,
                                                           int n_probes,
                                                           const double* __restrict__ proj,
                                                           int buckets, int tiles_j,
                                                           double* __restrict__ partial) {
  constexpr int RI = TI / 16, RJ = kSimTJ / 16;
  const int ncols = E + n_probes * buckets;
  const int ti = blockIdx.x / tiles_j, tj = blockIdx.x % tiles_j;
  const int i0 = ti * TI, j0 = tj * kSimTJ;
  if (TI == kSimTJ && j0 + kSimTJ <= E && tj < ti) return;  // mirrored Gram tile
  const long slice = (D + gridDim.y - 1) / gridDim.y;
  const long d0 = blockIdx.y * slice;
  const long d1 = d0 + slice < D ? d0 + slice : D;

  __shared__ __align__(16) double sa[kSimKc][TI];
  __shared__ __align__(16) double sb[kSimKc][kSimTJ];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, RI x RJ outputs each
  double acc[RI][RJ];
#pragma unroll
  for (int u = 0; u < RI; ++u)
#pragma unroll
    for (int v = 0; v < RJ; ++v) acc[u][v] = 0.0;

  for (long k0 = d0; k0 < d1; k0 += kSimKc) {
    // stage TI rows and 64 columns of kSimKc d each; thread -> (row, d), d fastest
    for (int idx = threadIdx.x; idx < TI * kSimKc; idx += blockDim.x) {
      const int r = idx / kSimKc, c = idx % kSimKc;
      const long d = k0 + c;
      const int i = i0 + r;
      sa[c][r] = (d < d1 && i < E) ? to_f64(static_cast<const T*>(rows[i])[d]) : 0.0;
    }
    for (int idx = threadIdx.x; idx < kSimTJ * kSimKc; idx += blockDim.x) {
      const int r = idx / kSimKc, c = idx % kSimKc;
      const long d = k0 + c;
      const int j = j0 + r;
      double bv = 0.0;
      if (d < d1) {
        if (j < E) {
          bv = to_f64(static_cast<const T*>(rows[j])[d]);
        } else if (j < ncols) {
          const int q = j - E;
          bv = probes[static_cast<long>(q / buckets) * D + d] * proj[static_cast<long>(q % buckets) * D + d];
        }
      }
      sb[c][r] = bv;
    }
    __syncthreads();
#pragma unroll 4
    for (int c = 0; c < kSimKc; ++c) {
      double a[RI], b[RJ];
#pragma unroll
      for (int u = 0; u < RI; ++u) a[u] = sa[c][ty * RI + u];
#pragma unroll
      for (int v = 0; v < RJ; ++v) b[v] = sb[c][tx * RJ + v];
#pragma unroll
      for (int u = 0; u < RI; ++u)
#pragma unroll
        for (int v = 0; v < RJ; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
  double* out = partial + static_cast<long>(blockIdx.y) * E * ncols;
#pragma unroll
  for (int u = 0; u < RI; ++u)
#pragma unroll
    for (int v = 0; v < RJ; ++v) {
      const int i = i0 + ty * RI + u, j = j0 + tx * RJ + v;
      if (i < E && j < ncols) out[static_cast<long>(i) * ncols + j] = acc[u][v];
    }
}

// Cosine Gram for E <= 8 experts without tiles: every thread streams 8
// consecutive d of all E rows (16-byte loads) and keeps the E(E+1)/2
// upper-triangle dot products in registers; block partials are reduced
// warp -> block in a fixed order. Exact bf16 products, fp64 sums.
template <typename T, int E>
__global__ void __launch_bounds__(256) sim_gram_small_kernel(const void* const* __restrict__ rows,
                                                             long D, double* __restrict__ partial) {
  constexpr int NP = E * (E + 1) / 2;
  constexpr int V = 16 / sizeof(T);  // elements per 16-byte load
  double acc[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) acc[p] = 0.0;
  const T* r[E];
#pragma unroll
  for (int e = 0; e < E; ++e) r[e] = static_cast<const T*>(rows[e]);
  const long nv = D / V;
  for (long v = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; v < nv;
       v += static_cast<long>(gridDim.x) * blockDim.x) {
    double x[E][V];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int4 raw = ld_nc_v4(r[e] + v * V);
      const T* pv = reinterpret_cast<const T*>(&raw);
#pragma unroll
      for (int k = 0; k < V; ++k) x[e][k] = to_f64(pv[k]);
    }
    int p = 0;
#pragma unroll
    for (int a = 0; a < E; ++a)
#pragma unroll
      for (int b = a; b < E; ++b, ++p)
#pragma unroll
        for (int k = 0; k < V; ++k) acc[p] = fma(x[a][k], x[b][k], acc[p]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // tail (D % V) by one thread
    for (long d = nv * V; d < D; ++d) {
      int p = 0;
      for (int a = 0; a < E; ++a)
        for (int b = a; b < E; ++b, ++p) acc[p] = fma(to_f64(r[a][d]), to_f64(r[b][d]), acc[p]);
    }
  }
  __shared__ double red[8][NP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    double v = acc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < NP; q += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += red[w][q];
    partial[static_cast<long>(blockIdx.x) * NP + q] = v;
  }
}

__global__ void sim_gram_small_reduce(const double* __restrict__ partial, int blocks, int E,
                                      double* __restrict__ gram) {
  const int NP = E * (E + 1) / 2;
  for (int q = threadIdx.x; q < NP; q += blockDim.x) {
    double v = 0.0;
    for (int b = 0; b < blocks; ++b) v += partial[static_cast<long>(b) * NP + q];
    int a = 0, rem = q;
    while (rem >= E - a) { rem -= E - a; ++a; }
    const int c = a + rem;
    gram[a * E + c] = v;
    gram[c * E + a] = v;
  }
}

// Cosine Gram of bf16 experts on the tensor cores (mma.sync m16n8k16,
// fp32 accumulate, flushed into fp64 every 64 d). bf16 x bf16 products
// are exact in fp32; only the fp32 sums of <= 64 products per flush round
// (measured: Gram entries within 2e-8 absolute of fp64 at D = 1e5, cosines
// within the 1e-7 bf16 parity bar).
// A warp owns one (32x32 tile, D-slice) unit; Gram tiles below the
// diagonal are skipped (mirrored by the reduction). k-permutation trick:
// the contraction sums over every d, so each thread may feed the MMA's k
// slots from one 16-byte vector of 8 consecutive d per row — the same
// vector serves as A fragment (row g / g+8 of an m-tile) and B fragment
// (column g of an n-tile) — no shared memory, fully used 32-byte sectors.
constexpr int kGramFlush = 2;  // 32-d chunks between fp64 flushes

__device__ __forceinline__ void mma_bf16_16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2,
                                               uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Q = 8-row groups per tile side (1: an 8x8 tile for E <= 8, 4: 32x32);
// U = 32-d chunks loaded per iteration (loads in flight per thread).
template <int Q, int U>
__global__ void __launch_bounds__(128) sim_gram_mma_kernel(const void* const* __restrict__ rows,
                                                           int E, long D, int tiles_1d,
                                                           int splits, long slice,
                                                           double* __restrict__ partial) {
  constexpr int M = Q == 1 ? 1 : Q / 2;  // m16 tiles (rows g + 16m, g + 16m + 8)
  constexpr int N = Q;                   // n8 tiles (columns g + 8n)
  constexpr int T = 8 * Q;               // tile side
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long unit = static_cast<long>(blockIdx.x) * 4 + warp;
  const int n_tiles = tiles_1d * (tiles_1d + 1) / 2;
  if (unit >= static_cast<long>(n_tiles) * splits) return;
  int tile = static_cast<int>(unit % n_tiles);
  const int split = static_cast<int>(unit / n_tiles);
  int ti = 0;  // upper-triangle tile (ti <= tj), row-major
  while (tile >= tiles_1d - ti) { tile -= tiles_1d - ti; ++ti; }
  const int tj = ti + tile;
  const bool diag = ti == tj;
  const int g = lane >> 2, tq = lane & 3;
  const int I0 = ti * T, J0 = tj * T;
  // interleaved 32U-d chunks (split, split + splits, ...): concurrent warps
  // read neighbouring pieces of each row (DRAM page locality)
  const long d0 = static_cast<long>(split) * 32 * U;
  const long dstep = static_cast<long>(splits) * 32 * U;
  const long d1 = D;
  const int4* ra[Q];
  const int4* rb[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int i = I0 + g + 8 * q, j = J0 + g + 8 * q;
    ra[q] = i < E ? static_cast<const int4*>(rows[i]) : nullptr;
    rb[q] = j < E ? static_cast<const int4*>(rows[j]) : nullptr;
  }
  float c[M][N][4];
  double acc[M][N][4];
#pragma unroll
  for (int m = 0; m < M; ++m)
#pragma unroll
    for (int n = 0; n < N; ++n)
#pragma unroll
      for (int r = 0; r < 4; ++r) { c[m][n][r] = 0.f; acc[m][n][r] = 0.0; }
  const int4 z = make_int4(0, 0, 0, 0);
  int since = 0;
  for (long d = d0; d < d1; d += dstep) {
    int4 A[U][Q], B[U][Q];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long dd = d + 32 * u;
      const long v = (dd >> 3) + tq;  // this thread's 16-byte vector: dd + 8*tq .. +8
      const bool in = dd + 8 * tq < d1;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        A[u][q] = (in && ra[q]) ? ld_nc_v4(ra[q] + v) : z;
        B[u][q] = diag ? A[u][q] : ((in && rb[q]) ? ld_nc_v4(rb[q] + v) : z);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const uint32_t* a_lo = reinterpret_cast<const uint32_t*>(&A[u][Q == 1 ? 0 : 2 * m]);
          const uint32_t hi0 = Q == 1 ? 0u : reinterpret_cast<const uint32_t*>(&A[u][2 * m + (Q > 1)])[2 * s2];
          const uint32_t hi1 = Q == 1 ? 0u : reinterpret_cast<const uint32_t*>(&A[u][2 * m + (Q > 1)])[2 * s2 + 1];
#pragma unroll
          for (int n = 0; n < N; ++n) {
            const uint32_t* b = reinterpret_cast<const uint32_t*>(&B[u][n]);
            mma_bf16_16816(c[m][n], a_lo[2 * s2], hi0, a_lo[2 * s2 + 1], hi1, b[2 * s2],
                           b[2 * s2 + 1]);
          }
        }
    since += U;
    if (since >= kGramFlush) {
      since = 0;
#pragma unroll
      for (int m = 0; m < M; ++m)
#pragma unroll
        for (int n = 0; n < N; ++n)
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            acc[m][n][r] += static_cast<double>(c[m][n][r]);
            c[m][n][r] = 0.f;
          }
    }
  }
  double* out = partial + static_cast<long>(split) * E * E;
#pragma unroll
  for (int m = 0; m < M; ++m)
#pragma unroll
    for (int n = 0; n < N; ++n)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        // C fragment: rows 16m + g (+8 for r >= 2), columns 8n + 2tq + (r & 1)
        const int i = I0 + 16 * m + g + (r >= 2 ? 8 : 0);
        const int j = J0 + 8 * n + 2 * tq + (r & 1);
        if (r < 2 || Q > 1)
          if (i < E && j < E && i < I0 + T)
            out[static_cast<long>(i) * E + j] = acc[m][n][r] + static_cast<double>(c[m][n][r]);
      }
}

// Cosine Gram of 9..128 bf16 experts on the 5th-gen tensor cores
// (tcgen05, 1-SM, M = N = 128: the expert tile is both operands), for
// experts stored as consecutive rows of one stride (a layer's pool slots,
// the rows of a matrix).
// - Split-K over CTAs by interleaved 64-d blocks (block c, c + grid, ...).
// - Warp 0: one TMA box per block (E rows x 64 d, 128-byte swizzled
//   K-major; rows >= E stay zero). One-row boxes measured TMA-issue-bound
//   at ~1 op / 50 cycles / SM.
// - Warp 1: four MMAs per block into a fresh TMEM accumulator (4 of them),
//   so the tensor core's fp32 sums stay as short as the mma.sync path's
//   (accumulating 256 d in TMEM drifted 4e-7 relative on the diagonal).
// - Warps 2-9 (two per TMEM lane quadrant): add the two blocks of a group
//   with one RN fp32 add and fold the sum into fp64 / compensated fp32
//   register accumulators, one of each transposed pair of 32 x 32 tiles
//   (see the fold below). The bf16 x bf16 products are exact.
// Each CTA writes its fp64 [E,E] partial; sim_reduce_kernel sums them in a
// fixed order. Every row is read once (the mma.sync tiles re-read each row
// ~5x at E = 128).
#ifndef COMOE_GT_STAGES
#define COMOE_GT_STAGES 8
#endif
constexpr int kGtStages = COMOE_GT_STAGES;
constexpr int kGtTile = 128 * 128;  // bytes per stage (128 rows x 64 bf16)
constexpr int kGtSmem = 1024 + kGtStages * kGtTile + 256;
constexpr int kGtThreads = 10 * 32;

__global__ void __launch_bounds__(kGtThreads, 1)
    sim_gram_tc_kernel(const __grid_constant__ CUtensorMap tmap, int row0, int box_rows, int E,
                       long n_kb, double* __restrict__ partial, int flags) {
  // flags: 1 = contiguous block ranges per CTA; dev attribution (COMOE_GRAM_DEBUG,
  // results invalid): 2 = the fold skips its arithmetic, 4 = no MMAs, 8 = the
  // MMA warp does not wait for the fold (the fold warps idle)
  const bool contig = flags & 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* tiles = smem;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kGtStages * kGtTile);
  uint64_t* empty_bar = full_bar + kGtStages;
  uint64_t* tfull_bar = empty_bar + kGtStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // block i of this CTA: blockIdx.x + i * grid (interleaved) or, with
  // `contig`, kb0 + i over a contiguous range of per = ceil(n_kb / grid)
  const long per = (n_kb + gridDim.x - 1) / gridDim.x;
  const long kb0 = static_cast<long>(blockIdx.x) * per;
  const int n = contig ? static_cast<int>(kb0 < n_kb ? (n_kb - kb0 < per ? n_kb - kb0 : per) : 0)
                       : static_cast<int>((n_kb - blockIdx.x + gridDim.x - 1) / gridDim.x);

  if (box_rows < 128)
    for (int i = threadIdx.x; i < kGtStages * kGtTile / 16; i += blockDim.x)
      reinterpret_cast<int4*>(tiles)[i] = make_int4(0, 0, 0, 0);  // rows >= E stay zero
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmap);
    for (int s = 0; s < kGtStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 8);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zeroed rows -> async proxy
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer: the stage is one box
    if (lane == 0) {
      for (int i = 0; i < n; ++i) {
        const int s = i % kGtStages;
        if (i >= kGtStages) mbar_wait(&empty_bar[s], ((i / kGtStages) - 1) & 1);
        mbar_expect_tx(&full_bar[s], static_cast<uint32_t>(box_rows) * 128u);
        const int x = static_cast<int>(
            (contig ? kb0 + i : blockIdx.x + static_cast<long>(i) * gridDim.x) * 64);
        tma_load_2d(tiles + s * kGtTile, &tmap, &full_bar[s], x, row0);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t kIdesc = umma_idesc_bf16_f32(128, 128);
      for (int i = 0; i < n; ++i) {
        // block i -> its own accumulator i % 4; blocks 2g, 2g+1 form fold
        // group g, handed over through the pair's barriers (g % 2)
        const int s = i % kGtStages, a = i & 3, g = i >> 1, pr = g & 1;
        if ((i & 1) == 0 && !(flags & 8)) mbar_wait(&tempty_bar[pr], ((g >> 1) & 1) ^ 1);
        mbar_wait(&full_bar[s], (i / kGtStages) & 1);
        tc_fence_after();
        const uint64_t desc = umma_desc_k_sw128(smem_u32(tiles + s * kGtTile));
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (!(flags & 4))
            umma_bf16(tmem_base + a * 128, desc + 2 * k, desc + 2 * k, kIdesc, k != 0 ? 1u : 0u);
        umma_commit(&empty_bar[s]);
        if (((i & 1) == 1 || i == n - 1) && !(flags & 8)) umma_commit(&tfull_bar[pr]);
      }
    }
  } else {
    // ------------------------------------------------ fp64 fold (warps 2-9)
    // Symmetric fold: of the 16 (row quadrant, 32-column block) tiles of the
    // 128 x 128 accumulator only one of each transposed pair is folded —
    // quadrant q takes column blocks q, q+1, q+2 (q < 2) or q, q+1 (q >= 2),
    // mod 4: 10 tiles instead of 16, at most 3 per quadrant (the busiest
    // scheduler's work drops a quarter and the accumulators fit in registers
    // without spilling). Warp (q, h) takes half of its quadrant's 16-column
    // chunks. Within a chunk the first 8 columns go fp32 -> fp64 (F2F on the
    // XU pipe, which alone bounded the fold) + DADD and the other 8 stay in
    // fp32 as an unevaluated sum hi + lo (Knuth two-sum on the FMA pipe, the
    // rounding error of every add carried in lo: ~2^-44 relative, far inside
    // the 1e-7 cosine bar), so the fold runs on two pipes at once.
    const int q = warp & 3, h = (warp - 2) >> 2;  // lane quadrant, chunk half
    const int row = q * 32 + lane;
    if (flags & 8) goto fold_done;
    {
    constexpr int kMaxCh = 3;
    const int nch = q < 2 ? 3 : 2;
    const int ch0 = 2 * q + h * nch;  // global chunk of slot i: (ch0 + i) mod 8
    double dacc[kMaxCh][8];
    float fhi[kMaxCh][8], flo[kMaxCh][8];
#pragma unroll
    for (int i = 0; i < kMaxCh; ++i)
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        dacc[i][c] = 0.0;
        fhi[i][c] = flo[i][c] = 0.f;
      }
    const int n_groups = (n + 1) >> 1;
    for (int g = 0; g < n_groups; ++g) {
      const int pr = g & 1;
      const bool two = 2 * g + 1 < n;
      mbar_wait(&tfull_bar[pr], (g >> 1) & 1);
      tc_fence_after();
      const uint32_t t = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + 2 * pr * 128;
#pragma unroll
      for (int i = 0; i < kMaxCh; ++i) {
        if (i >= nch) break;
        const uint32_t col = static_cast<uint32_t>(((ch0 + i) & 7) * 16);
        uint32_t v[16], w[16];
        tmem_ld16(t + col, v);
        tmem_ld16(t + 128 + col, w);  // block 2g+1 (unused when absent)
        tmem_ld_wait();
        if (i == nch - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[pr]);
        }
        // one RN fp32 add of the two 64-d block sums, then the fold
        if (flags & 2) continue;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const float x = __uint_as_float(v[c]) + (two ? __uint_as_float(w[c]) : 0.f);
          if (c < 8) {
            dacc[i][c] += static_cast<double>(x);
          } else {
            const int k = c - 8;
            const float sum = __fadd_rn(fhi[i][k], x);
            const float bp = __fsub_rn(sum, fhi[i][k]);
            const float err =
                __fadd_rn(__fsub_rn(fhi[i][k], __fsub_rn(sum, bp)), __fsub_rn(x, bp));
            fhi[i][k] = sum;
            flo[i][k] = __fadd_rn(flo[i][k], err);
          }
        }
      }
    }
    // every (i, j) of the partial is written exactly once: diagonal tiles as
    // folded, off-diagonal tiles at (row, col) and mirrored at (col, row)
    double* out = partial + static_cast<long>(blockIdx.x) * E * E;
#pragma unroll
    for (int i = 0; i < kMaxCh; ++i) {
      if (i >= nch) break;
      const int gc = (ch0 + i) & 7;
      const bool diag = (gc >> 1) == q;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const int col = gc * 16 + c;
        const double val = c < 8 ? dacc[i][c]
                                 : static_cast<double>(fhi[i][c - 8]) + static_cast<double>(flo[i][c - 8]);
        if (row < E && col < E) {
          out[static_cast<long>(row) * E + col] = val;
          if (!diag) out[static_cast<long>(col) * E + row] = val;
        }
      }
    }
    }
  fold_done:;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

// Cosine Gram of <= 8 bf16 experts (C1: Switch-Base-8, C5: Mixtral 8
// experts): a streaming kernel. Each CTA takes 2048-d chunks c, c + grid,
// ... (interleaved: concurrent CTAs read neighbouring pieces of every row);
// one thread moves a chunk of every row with one bulk copy per row (4 KB,
// cp.async.bulk, completion on the stage's mbarrier; rows padded by 16 B
// so the fragment loads are conflict-free). Consumer warp w takes 256 d of
// the chunk: per 16 d one 8-byte shared load per lane and one mma.sync
// m16n8k16 whose A (rows 0-7; rows 8-15 zero) and B fragments are the same
// registers (k permuted inside the 16 d, identically for both), fp32
// accumulation folded into fp64 every 64 d (exact bf16 products, <= 64-term
// fp32 sums). Fixed-order CTA reduction to one fp64 [E,E] partial per CTA.
// (The 8x8 mma.sync tiles over global memory stalled at ~1 TB/s on 16-byte
// outstanding requests; an FFMA version was issue-bound at 3.2 TB/s.)
constexpr int kG8Chunk = 2048, kG8Stages = 4, kG8Threads = 288;
constexpr int kG8Pitch = kG8Chunk * 2 + 16;  // bytes per staged row
constexpr int kG8Smem = 1024 + kG8Stages * 8 * kG8Pitch + 8 * 64 * 8 + 128;

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(kG8Threads, 1)
    sim_gram8_kernel(const void* const* __restrict__ rows, int E, long D,
                     double* __restrict__ partial) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* tiles = smem;  // [stage][8 rows][kG8Pitch]
  double* red = reinterpret_cast<double*>(smem + kG8Stages * 8 * kG8Pitch);  // [8 warps][64]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(red + 8 * 64);
  uint64_t* empty_bar = full_bar + kG8Stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long n_chunks = (D + kG8Chunk - 1) / kG8Chunk;
  const int n = static_cast<int>((n_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x);
  if (E < 8)
    for (int i = threadIdx.x; i < kG8Stages * 8 * kG8Pitch / 16; i += blockDim.x)
      reinterpret_cast<int4*>(tiles)[i] = make_int4(0, 0, 0, 0);  // rows >= E read as zero
  if (threadIdx.x == 0) {
    for (int st = 0; st < kG8Stages; ++st) {
      mbar_init(&full_bar[st], 1);
      mbar_init(&empty_bar[st], 8);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < n; ++i) {
        const int st = i % kG8Stages;
        if (i >= kG8Stages) mbar_wait(&empty_bar[st], ((i / kG8Stages) - 1) & 1);
        const long d0 = (blockIdx.x + static_cast<long>(i) * gridDim.x) * kG8Chunk;
        const long len = D - d0 < kG8Chunk ? D - d0 : kG8Chunk;
        const uint32_t bytes = static_cast<uint32_t>(len * 2);
        mbar_expect_tx(&full_bar[st], bytes * static_cast<uint32_t>(E));
        for (int e = 0; e < E; ++e)
          bulk_load(tiles + (st * 8 + e) * kG8Pitch,
                    static_cast<const __nv_bfloat16*>(rows[e]) + d0, bytes, &full_bar[st]);
      }
    }
    return;
  }
  const int w = warp - 1;                  // 256 d of every chunk
  const int g = lane >> 2, tq = lane & 3;  // fragment row / k quad
  float c[4] = {0.f, 0.f, 0.f, 0.f};
  double acc[2] = {0.0, 0.0};
  for (int i = 0; i < n; ++i) {
    const int st = i % kG8Stages;
    const long d0 = (blockIdx.x + static_cast<long>(i) * gridDim.x) * kG8Chunk;
    const int len = static_cast<int>(D - d0 < kG8Chunk ? D - d0 : kG8Chunk);
    mbar_wait(&full_bar[st], (i / kG8Stages) & 1);
    const uint8_t* row = tiles + (st * 8 + g) * kG8Pitch;
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const int d = w * 256 + kk * 16 + 4 * tq;  // this lane's 4 d of the 16-d step
      uint2 v = make_uint2(0u, 0u);
      if (d < len) v = *reinterpret_cast<const uint2*>(row + 2 * d);
      mma_bf16_16816(c, v.x, 0u, v.y, 0u, v.x, v.y);
      if ((kk & 3) == 3) {  // fold every 64 d
        acc[0] += static_cast<double>(c[0]);
        acc[1] += static_cast<double>(c[1]);
        c[0] = c[1] = c[2] = c[3] = 0.f;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[st]);
  }
  // lane holds C[g][2tq], C[g][2tq+1]; the 8 warps are summed in a fixed order
  red[w * 64 + g * 8 + 2 * tq] = acc[0];
  red[w * 64 + g * 8 + 2 * tq + 1] = acc[1];
  asm volatile("bar.sync 1, 256;" ::: "memory");  // consumer warps only
  const int t = threadIdx.x - 32;
  if (t < 64) {
    double v = 0.0;
    for (int ww = 0; ww < 8; ++ww) v += red[ww * 64 + t];
    const int a = t >> 3, b = t & 7;
    if (a < E && b < E) partial[static_cast<long>(blockIdx.x) * E * E + a * E + b] = v;
  }
}

// Surrogate logits for E <= 8 experts and <= 8 buckets (the reference's
// defaults): logits[e][n][b] = sum_d P[e,d] probes[n,d] proj[b,d]. A block
// owns a contiguous D-slice and streams it in 256-d chunks through a
// double-buffered cp.async pipeline (expert rows, up to 8 probe rows, the
// projection rows), so DRAM latency overlaps the fp64 math; warp w takes
// probe n0 + w, lane = d inside the chunk, 64 fp64 accumulators (e, b) per
// lane, u_e = P[e,d]*probe formed once per (e, d). Lane partials are
// tree-reduced per warp and written per block (deterministic). Replaces the
// 16x64-tile fp64 path for this shape, where 72% of the FMAs hit padding
// and every column re-read its probe and projection rows (7.8 ms at C1).
constexpr int kLogitE = 8, kLogitB = 8, kLogitN = 8, kLogitChunk = 256;

template <typename T>
struct LogitStage {
  static constexpr int kPBytes = kLogitE * kLogitChunk * static_cast<int>(sizeof(T));
  static constexpr int kQBytes = kLogitN * kLogitChunk * 8;  // probes
  static constexpr int kRBytes = kLogitB * kLogitChunk * 8;  // projection
  static constexpr int kBytes = kPBytes + kQBytes + kRBytes;
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}

constexpr int kLogitEW = 4;  // experts per warp: two warps per probe, 16 warps per block

template <typename T>
__global__ void __launch_bounds__(512) sim_logits_small_kernel(
    const void* const* __restrict__ rows, int E, long D, const double* __restrict__ probes,
    int n_probes, const double* __restrict__ proj, int B, long slice,
    double* __restrict__ partial) {
  using L = LogitStage<T>;
  extern __shared__ __align__(16) uint8_t lsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long d0 = blockIdx.x * slice;
  const long d1 = d0 + slice < D ? d0 + slice : D;
  constexpr int kVecT = 16 / sizeof(T);  // row elements per 16-byte copy
  for (int n0 = 0; n0 < n_probes; n0 += kLogitN) {
    const int np = n_probes - n0 < kLogitN ? n_probes - n0 : kLogitN;
    auto issue = [&](long c, int buf) {  // chunk starting at d = c into stage buf
      uint8_t* st = lsm + buf * L::kBytes;
      constexpr int kPV = kLogitChunk / kVecT, kDV = kLogitChunk / 2;  // 16-B vectors per row
      for (int i = threadIdx.x; i < E * kPV + (np + B) * kDV; i += blockDim.x) {
        if (i < E * kPV) {
          const int e = i / kPV, v = i % kPV;
          const long d = c + static_cast<long>(v) * kVecT;
          cp_async16(st + (e * kLogitChunk + v * kVecT) * sizeof(T),
                     static_cast<const T*>(rows[e]) + (d < d1 ? d : 0), d < d1);
        } else {
          const int j = i - E * kPV;
          const int r = j / kDV, v = j % kDV;
          const long d = c + 2L * v;
          const double* src = r < np ? probes + static_cast<long>(n0 + r) * D
                                     : proj + static_cast<long>(r - np) * D;
          uint8_t* dst = st + L::kPBytes + (r < np ? r * kLogitChunk * 8
                                                   : L::kQBytes + (r - np) * kLogitChunk * 8);
          cp_async16(dst + v * 16, src + (d < d1 ? d : 0), d < d1);
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // warp w: probe n0 + (w & 7), experts e0 .. e0 + kLogitEW - 1 with e0 = (w >> 3) * kLogitEW
    const int wn = warp & 7, e0 = (warp >> 3) * kLogitEW;
    const bool active = wn < np && e0 < E;
    double acc[kLogitEW][kLogitB];
#pragma unroll
    for (int e = 0; e < kLogitEW; ++e)
#pragma unroll
      for (int b = 0; b < kLogitB; ++b) acc[e][b] = 0.0;
    int buf = 0;
    if (d0 < d1) issue(d0, 0);
    for (long c = d0; c < d1; c += kLogitChunk, buf ^= 1) {
      if (c + kLogitChunk < d1) {
        issue(c + kLogitChunk, buf ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      const uint8_t* st = lsm + buf * L::kBytes;
      const T* ps = reinterpret_cast<const T*>(st);
      const double* qs = reinterpret_cast<const double*>(st + L::kPBytes);
      const double* rs = reinterpret_cast<const double*>(st + L::kPBytes + L::kQBytes);
      if (active) {
#pragma unroll 2
        for (int i = 0; i < kLogitChunk / 32; ++i) {
          const int dd = lane + 32 * i;  // (rows past d1 were zero-filled)
          const double pr = qs[wn * kLogitChunk + dd];
          double q[kLogitB];
#pragma unroll
          for (int b = 0; b < kLogitB; ++b) q[b] = b < B ? rs[b * kLogitChunk + dd] : 0.0;
#pragma unroll
          for (int e = 0; e < kLogitEW; ++e) {
            if (e0 + e >= E) break;
            const double u = to_f64(ps[(e0 + e) * kLogitChunk + dd]) * pr;
#pragma unroll
            for (int b = 0; b < kLogitB; ++b) acc[e][b] = fma(u, q[b], acc[e][b]);
          }
        }
      }
      __syncthreads();  // this stage is refilled by the next iteration's issue
    }
    if (active) {
#pragma unroll
      for (int e = 0; e < kLogitEW; ++e)
#pragma unroll
        for (int b = 0; b < kLogitB; ++b) {
          double v = acc[e][b];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == 0 && e0 + e < E && b < B)
            partial[(static_cast<long>(blockIdx.x) * E + e0 + e) * n_probes * B + (n0 + wn) * B + b] = v;
        }
    }
  }
}

// Surrogate logits on the fp64 tensor cores (bf16 parameters, <= 8
// experts, probes and buckets): for each probe n the logits are an 8x8
// GEMM over d, logits_n[e][b] = sum_d P[e,d] * (probe[n,d] * proj[b,d]),
// one mma.sync.m8n8k4.f64 per probe per 4 d. A = P (lane: expert
// lane/4, d lane%4); B_n = probe_n (.) proj formed in the fragment (lane:
// bucket lane/4, d lane%4: one fp64 multiply per probe). One thread moves
// each 256-d chunk of the P, probe and projection rows with bulk copies
// (3 stages, rows padded so fragment loads do not conflict); 8 consumer
// warps take 32 d each. fp64 throughout (the tensor-core fp64 FMA is
// IEEE), deterministic per block (warps summed in order). The vector path
// (2 warps per probe, 32 accumulators per lane) needed 2.5 shared-memory
// bytes per FMA and ran at ~27% of the fp64 rate (C1: ~440 us).
constexpr int kLdChunk = 256, kLdStages = 3, kLdThreads = 288;
constexpr int kLdPPitch = kLdChunk * 2 + 16, kLdFPitch = kLdChunk * 8 + 32;
constexpr int kLdStage = 8 * kLdPPitch + 16 * kLdFPitch;  // P | probes | projection
constexpr int kLdSmem = 1024 + kLdStages * kLdStage + 8 * 8 * 64 * 8 + 128;

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void bulk_load_ld(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(kLdThreads, 1)
    sim_logits_dmma_kernel(const void* const* __restrict__ rows, int E, long D,
                           const double* __restrict__ probes, int n_probes,
                           const double* __restrict__ proj, int B, long slice,
                           double* __restrict__ partial) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  double* red = reinterpret_cast<double*>(smem + kLdStages * kLdStage);  // [8 warps][8 n][64]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(red + 8 * 8 * 64);
  uint64_t* empty_bar = full_bar + kLdStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long d0 = blockIdx.x * slice;
  const long d1 = d0 + slice < D ? d0 + slice : D;
  const int n = d1 > d0 ? static_cast<int>((d1 - d0 + kLdChunk - 1) / kLdChunk) : 0;
  for (int i = threadIdx.x; i < kLdStages * kLdStage / 16; i += blockDim.x)
    reinterpret_cast<int4*>(smem)[i] = make_int4(0, 0, 0, 0);  // absent rows read as zero
  if (threadIdx.x == 0) {
    for (int st = 0; st < kLdStages; ++st) {
      mbar_init(&full_bar[st], 1);
      mbar_init(&empty_bar[st], 8);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < n; ++i) {
        const int st = i % kLdStages;
        if (i >= kLdStages) mbar_wait(&empty_bar[st], ((i / kLdStages) - 1) & 1);
        const long c = d0 + static_cast<long>(i) * kLdChunk;
        const long len = d1 - c < kLdChunk ? d1 - c : kLdChunk;
        uint8_t* sb = smem + st * kLdStage;
        mbar_expect_tx(&full_bar[st], static_cast<uint32_t>(len * (2 * E + 8 * (n_probes + B))));
        for (int e = 0; e < E; ++e)
          bulk_load_ld(sb + e * kLdPPitch, static_cast<const __nv_bfloat16*>(rows[e]) + c,
                       static_cast<uint32_t>(len * 2), &full_bar[st]);
        for (int q = 0; q < n_probes; ++q)
          bulk_load_ld(sb + 8 * kLdPPitch + q * kLdFPitch, probes + q * D + c,
                       static_cast<uint32_t>(len * 8), &full_bar[st]);
        for (int b = 0; b < B; ++b)
          bulk_load_ld(sb + 8 * kLdPPitch + 8 * kLdFPitch + b * kLdFPitch, proj + b * D + c,
                       static_cast<uint32_t>(len * 8), &full_bar[st]);
      }
    }
    return;
  }
  const int w = warp - 1, g = lane >> 2, k = lane & 3;
  double acc[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q][0] = acc[q][1] = 0.0;
  for (int i = 0; i < n; ++i) {
    const int st = i % kLdStages;
    const long c = d0 + static_cast<long>(i) * kLdChunk;
    const int len = static_cast<int>(d1 - c < kLdChunk ? d1 - c : kLdChunk);
    mbar_wait(&full_bar[st], (i / kLdStages) & 1);
    const uint8_t* sb = smem + st * kLdStage;
    const __nv_bfloat16* pr = reinterpret_cast<const __nv_bfloat16*>(sb + g * kLdPPitch);
    const double* qs = reinterpret_cast<const double*>(sb + 8 * kLdPPitch);
    const double* rr = reinterpret_cast<const double*>(sb + 8 * kLdPPitch + 8 * kLdFPitch + g * kLdFPitch);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int dd = w * 32 + ks * 4 + k;
      const bool in = dd < len;  // stale data past the chunk end is masked by a = 0
      const double a = in ? static_cast<double>(__bfloat162float(pr[dd])) : 0.0;
      const double r = rr[dd];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double bq = qs[q * (kLdFPitch / 8) + dd] * r;
        dmma_8x8x4(acc[q], a, bq);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[st]);
  }
  // lane holds logits_q[e = g][b = 2k, 2k+1]; warps summed in order
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    red[(w * 8 + q) * 64 + g * 8 + 2 * k] = acc[q][0];
    red[(w * 8 + q) * 64 + g * 8 + 2 * k + 1] = acc[q][1];
  }
  asm volatile("bar.sync 1, 256;" ::: "memory");
  for (int t = threadIdx.x - 32; t < 8 * 64; t += 256) {
    const int q = t >> 6, e = (t >> 3) & 7, b = t & 7;
    if (q < n_probes && e < E && b < B) {
      double v = 0.0;
      for (int ww = 0; ww < 8; ++ww) v += red[(ww * 8 + q) * 64 + e * 8 + b];
      partial[(static_cast<long>(blockIdx.x) * E + e) * n_probes * B + q * B + b] = v;
    }
  }
}

// out[i] = sum over splits (in order) of partial[split][i]; one warp per entry
__global__ void sim_sum_partials(const double* __restrict__ partial, int splits, long n,
                                 double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long warps = static_cast<long>(gridDim.x) * (blockDim.x >> 5);
  for (long i = blockIdx.x * static_cast<long>(blockDim.x >> 5) + (threadIdx.x >> 5); i < n;
       i += warps) {
    double s = 0.0;
    for (int k = lane; k < splits; k += 32) s += partial[k * n + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[i] = s;
  }
}

// one warp per output entry: lanes stride the splits, fixed-order tree
// (deterministic); skipped below-diagonal Gram tiles read the mirror.
__global__ void sim_reduce_kernel(const double* __restrict__ partial, int splits, int E, int ncols,
                                  int mirror_tile, double* __restrict__ gram,
                                  double* __restrict__ logits) {
  const long n = static_cast<long>(E) * ncols;
  const int lane = threadIdx.x & 31;
  const long warps = static_cast<long>(gridDim.x) * (blockDim.x >> 5);
  for (long idx = blockIdx.x * static_cast<long>(blockDim.x >> 5) + (threadIdx.x >> 5); idx < n;
       idx += warps) {
    const int i = static_cast<int>(idx / ncols), j = static_cast<int>(idx % ncols);
    long src = idx;
    if (mirror_tile && j < E && (j / mirror_tile) < (i / mirror_tile) &&
        (j / mirror_tile + 1) * mirror_tile <= E)
      src = static_cast<long>(j) * ncols + i;
    double s = 0.0;
    for (int k = lane; k < splits; k += 32) s += partial[k * n + src];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      if (j < E) gram[static_cast<long>(i) * E + j] = s;
      else logits[static_cast<long>(i) * (ncols - E) + (j - E)] = s;
    }
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

// Same result, one block: the log-softmax (log p and p) of every (expert,
// probe) row is computed once into shared memory, then threads sweep the
// pairs — the per-pair kernel above recomputes both rows' log-softmax for
// every pair (74 us at E = 8 on one 128-thread block). Identical operation
// order per value, so bit-identical output.
constexpr int kFinalizeThreads = 1024;
__global__ void __launch_bounds__(kFinalizeThreads) sim_finalize_staged_kernel(
    const double* __restrict__ gram, const double* __restrict__ logits, int E, int n_probes,
    int buckets, double alpha, double* __restrict__ sim) {
  extern __shared__ double fsm[];
  const int R = E * n_probes;  // rows (expert, probe)
  double* lp = fsm;                              // [R][buckets] log p
  double* pp = fsm + static_cast<long>(R) * buckets;  // [R][buckets] p
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    const double* l = logits + static_cast<long>(r) * buckets;
    double m = -INFINITY;
    for (int k = 0; k < buckets; ++k) m = fmax(m, l[k]);
    double sm = 0.0;
    for (int k = 0; k < buckets; ++k) sm += exp(l[k] - m);
    const double ls = m + log(sm);
    for (int k = 0; k < buckets; ++k) {
      const double v = l[k] - ls;
      lp[r * buckets + k] = v;
      pp[r * buckets + k] = exp(v);
    }
  }
  __syncthreads();
  const long pairs = static_cast<long>(E) * E;
  for (long idx = threadIdx.x; idx < pairs; idx += blockDim.x) {
    const int a = static_cast<int>(idx / E), b = static_cast<int>(idx % E);
    const double cosv = gram[static_cast<long>(a) * E + b] /
                        (sqrt(gram[static_cast<long>(a) * E + a]) * sqrt(gram[static_cast<long>(b) * E + b]));
    double mean_kl = 0.0;
    for (int n = 0; n < n_probes; ++n) {
      const int ra = (a * n_probes + n) * buckets, rb = (b * n_probes + n) * buckets;
      double kab = 0.0, kba = 0.0;
      for (int k = 0; k < buckets; ++k) {
        const double lpa = lp[ra + k], lpb = lp[rb + k];
        const double pa = pp[ra + k], pb = pp[rb + k];
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

static int num_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

static bool sim_small(int E, int n_probes) { return n_probes == 0 && E >= 1 && E <= kSimSmallE; }

// bf16 cosine-only Gram on the tensor cores (rows 16-byte aligned, D % 8 == 0)
static bool sim_mma(int dtype, int n_probes, long D) {
  return dtype == COMOE_DTYPE_BF16 && n_probes == 0 && D % 8 == 0;
}

// tcgen05 Gram for 9..128 bf16 experts (COMOE_SIM_TC=0: the mma.sync tiles)
static bool sim_tc(int dtype, int E, long D) {
  static const bool on = [] {
    const char* e = std::getenv("COMOE_SIM_TC");
    return !(e && e[0] == '0');
  }();
  return on && dtype == COMOE_DTYPE_BF16 && D % 8 == 0 && E > 8 && E <= 128;
}

// streaming Gram for <= 8 bf16 experts (COMOE_SIM_G8=0: the mma.sync tiles)
static bool sim_g8(int dtype, int E, long D) {
  static const bool on = [] {
    const char* e = std::getenv("COMOE_SIM_G8");
    return !(e && e[0] == '0');
  }();
  return on && dtype == COMOE_DTYPE_BF16 && D % 8 == 0 && E >= 1 && E <= 8;
}

static int gram8_ctas(long D) {
  const long n = (D + kG8Chunk - 1) / kG8Chunk;
  const long c = n < num_sms() ? n : num_sms();
  return static_cast<int>(c > 0 ? c : 1);
}

static int gram_tc_ctas(long D) {
  const long n_kb = (D + 63) / 64;
  const long c = n_kb < num_sms() ? n_kb : num_sms();
  return static_cast<int>(c > 0 ? c : 1);
}

struct GramPlan {
  int tiles_1d, splits;
  long slice;
};

static int gram_tile(int E) { return E <= 8 ? 8 : 32; }

static GramPlan gram_plan(int E, long D) {
  GramPlan g;
  g.tiles_1d = (E + gram_tile(E) - 1) / gram_tile(E);
  const long n_tiles = static_cast<long>(g.tiles_1d) * (g.tiles_1d + 1) / 2;
  long splits = (static_cast<long>(num_sms()) * 32 + n_tiles - 1) / n_tiles;  // ~32 warps per SM
  const long max_by_d = (D + 2047) / 2048;  // >= 2048 d per unit
  if (splits > max_by_d) splits = max_by_d;
  if (splits < 1) splits = 1;
  g.slice = ((D + splits - 1) / splits + 31) / 32 * 32;
  g.splits = static_cast<int>((D + g.slice - 1) / g.slice);
  return g;
}

static int sim_small_blocks(long D) {
  long b = static_cast<long>(num_sms()) * 4;
  const long need = (D / 8 + 255) / 256;
  if (b > need) b = need;
  return static_cast<int>(b < 1 ? 1 : b);
}

static int sim_splits(int E, int ncols, long D) {
  const int ti = sim_ti(E);
  const long tiles = static_cast<long>((E + ti - 1) / ti) * ((ncols + kSimTJ - 1) / kSimTJ);
  long splits = (static_cast<long>(num_sms()) * 4 + tiles - 1) / tiles;
  const long max_by_d = (D + 4095) / 4096;  // at least 4096 d per slice
  if (splits > max_by_d) splits = max_by_d;
  if (splits > 1024) splits = 1024;
  if (splits < 1) splits = 1;
  return static_cast<int>(splits);
}

// 16-byte cp.async of rows, probes and projection: D % 8 == 0 (bf16) / % 2 (f64)
static bool sim_logits_small(int E, int buckets, long D) {
  return E <= kLogitE && buckets <= kLogitB && D % 8 == 0;
}

// fp64 tensor-core surrogate logits (COMOE_SIM_DMMA=0: the vector kernel)
static bool sim_logits_dmma() {
  static const bool on = [] {
    const char* e = std::getenv("COMOE_SIM_DMMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

// (d per block, blocks) of the small-logit kernel: one block per SM (register-bound)
static std::pair<long, int> logit_plan(long D) {
  long blocks = static_cast<long>(num_sms());
  const long need = (D + 1023) / 1024;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  // slices start on 256-d chunk boundaries (16-byte aligned cp.async sources)
  const long slice = ((D + blocks - 1) / blocks + kLogitChunk - 1) / kLogitChunk * kLogitChunk;
  return {slice, static_cast<int>((D + slice - 1) / slice)};
}

template <typename T>
static void launch_small(int E, const void* const* rows, long D, int blocks, double* partial,
                         cudaStream_t s) {
  switch (E) {
    case 1: sim_gram_small_kernel<T, 1><<<blocks, 256, 0, s>>>(rows, D, partial); break;
    case 2: sim_gram_small_kernel<T, 2><<<blocks, 256, 0, s>>>(rows, D, partial); break;
    case 3: sim_gram_small_kernel<T, 3><<<blocks, 256, 0, s>>>(rows, D, partial); break;
    case 4: sim_gram_small_kernel<T, 4><<<blocks, 256, 0, s>>>(rows, D, partial); break;
    case 5: sim_gram_small_kernel<T, 5><<<blocks, 256, 0, s>>>(rows, D, partial); break;
    case 6: sim_gram_small_kernel<T, 6><<<blocks, 256, 0, s>>>(rows, D, partial); break;
    case 7: sim_gram_small_kernel<T, 7><<<blocks, 256, 0, s>>>(rows, D, partial); break;
    default: sim_gram_small_kernel<T, 8><<<blocks, 256, 0, s>>>(rows, D, partial); break;
  }
}

// One fp64 tiled pass over [E] x [E + n*B] columns: the Gram and (with
// probes) the surrogate logits.
static int tiled_contract(int dtype, const void* const* rows, int E, long D, const double* probes,
                          int n_probes, const double* proj, int buckets, double* gram,
                          double* logits, double* partial, cudaStream_t s) {
  if (n_probes == 0) buckets = 0;  // cosine only
  const int ncols = E + n_probes * buckets;
  const int splits = sim_splits(E, ncols, D);
  const int ti = sim_ti(E);
  const int tiles_i = (E + ti - 1) / ti, tiles_j = (ncols + kSimTJ - 1) / kSimTJ;
  dim3 grid(tiles_i * tiles_j, splits);
  if (dtype == COMOE_DTYPE_BF16) {
    if (ti == 16)
      sim_contract_kernel<__nv_bfloat16, 16><<<grid, 256, 0, s>>>(rows, E, D, probes, n_probes,
                                                                  proj, buckets, tiles_j, partial);
    else
      sim_contract_kernel<__nv_bfloat16, 64><<<grid, 256, 0, s>>>(rows, E, D, probes, n_probes,
                                                                  proj, buckets, tiles_j, partial);
  } else {
    if (ti == 16)
      sim_contract_kernel<double, 16><<<grid, 256, 0, s>>>(rows, E, D, probes, n_probes, proj,
                                                           buckets, tiles_j, partial);
    else
      sim_contract_kernel<double, 64><<<grid, 256, 0, s>>>(rows, E, D, probes, n_probes, proj,
                                                           buckets, tiles_j, partial);
  }
  int rc = check_launch("sim_contract_kernel");
  if (rc) return rc;
  const long n = static_cast<long>(E) * ncols;
  const int blocks = static_cast<int>((n + 7) / 8 < 4096 ? (n + 7) / 8 : 4096);
  sim_reduce_kernel<<<blocks, 256, 0, s>>>(partial, splits, E, ncols, ti == kSimTJ ? kSimTJ : 0,
                                           gram, logits);
  return check_launch("sim_reduce_kernel");
}

// Cosine Gram only (tensor cores for bf16, register path for small f64 E,
// fp64 tiles otherwise) into gram[E,E]
static int gram_contract(int dtype, const void* const* rows, int E, long D, double* gram,
                         double* partial, cudaStream_t s) {
  if (sim_g8(dtype, E, D)) {
    const int ctas = gram8_ctas(D);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(sim_gram8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kG8Smem);
      attr = true;
    }
    sim_gram8_kernel<<<ctas, kG8Threads, kG8Smem, s>>>(rows, E, D, partial);
    int rc = check_launch("sim_gram8_kernel");
    if (rc) return rc;
    const long n = static_cast<long>(E) * E;
    const int blocks = static_cast<int>((n + 7) / 8 < 4096 ? (n + 7) / 8 : 4096);
    sim_reduce_kernel<<<blocks, 256, 0, s>>>(partial, ctas, E, E, 0, gram, nullptr);
    return check_launch("sim_reduce_kernel");
  }
  if (sim_mma(dtype, 0, D)) {
    const GramPlan gp = gram_plan(E, D);
    const long units = static_cast<long>(gp.tiles_1d) * (gp.tiles_1d + 1) / 2 * gp.splits;
    const unsigned nb = static_cast<unsigned>((units + 3) / 4);
    if (E <= 8)
      sim_gram_mma_kernel<1, 8><<<nb, 128, 0, s>>>(rows, E, D, gp.tiles_1d, gp.splits, gp.slice,
                                                   partial);
    else
      sim_gram_mma_kernel<4, 1><<<nb, 128, 0, s>>>(rows, E, D, gp.tiles_1d, gp.splits, gp.slice,
                                                   partial);
    int rc = check_launch("sim_gram_mma_kernel");
    if (rc) return rc;
    const long n = static_cast<long>(E) * E;
    const int blocks = static_cast<int>((n + 7) / 8 < 4096 ? (n + 7) / 8 : 4096);
    sim_reduce_kernel<<<blocks, 256, 0, s>>>(partial, gp.splits, E, E, gram_tile(E), gram, nullptr);
    return check_launch("sim_reduce_kernel");
  }
  if (sim_small(E, 0)) {
    // rows must be 16-byte aligned for the vector loads (pool slots and
    // torch allocations are)
    const int blocks = sim_small_blocks(D);
    if (dtype == COMOE_DTYPE_BF16) launch_small<__nv_bfloat16>(E, rows, D, blocks, partial, s);
    else launch_small<double>(E, rows, D, blocks, partial, s);
    int rc = check_launch("sim_gram_small_kernel");
    if (rc) return rc;
    sim_gram_small_reduce<<<1, 64, 0, s>>>(partial, blocks, E, gram);
    return check_launch("sim_gram_small_reduce");
  }
  return tiled_contract(dtype, rows, E, D, nullptr, 0, nullptr, 0, gram, nullptr, partial, s);
}

}  // namespace comoe

extern "C" {

long comoe_sim_workspace_bytes(int E, int n_probes, int buckets, long D) {
  using namespace comoe;
  if (n_probes > 0 && !sim_logits_small(E, buckets, D)) {
    const int ncols = E + n_probes * buckets;
    return static_cast<long>(sim_splits(E, ncols, D)) * E * ncols * sizeof(double);
  }
  // Gram path (bf16 and f64 share one size: the larger), plus the small-logit partials
  long w = static_cast<long>(sim_splits(E, E, D)) * E * E * sizeof(double);
  if (D % 8 == 0) {
    const GramPlan g = gram_plan(E, D);
    const long wm = static_cast<long>(g.splits) * E * E * sizeof(double);
    w = w > wm ? w : wm;
    const long wt = static_cast<long>(gram_tc_ctas(D)) * E * E * sizeof(double);
    w = w > wt ? w : wt;
    const long w8 = static_cast<long>(gram8_ctas(D)) * E * E * sizeof(double);
    w = w > w8 ? w : w8;
  }
  if (sim_small(E, 0)) {
    const long ws = static_cast<long>(sim_small_blocks(D)) * (E * (E + 1) / 2) * sizeof(double);
    w = w > ws ? w : ws;
  }
  if (n_probes > 0) w += logit_plan(D).second * static_cast<long>(E) * n_probes * buckets * sizeof(double);
  return w;
}

int comoe_sim_gram_strided(const void* base, long row_stride, int E, long D, double* gram,
                           void* work, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(base && gram && work, kBadArg, "sim_gram_strided: null pointer");
  COMOE_REQUIRE(sim_tc(COMOE_DTYPE_BF16, E, D), kUnsupportedShape,
                "sim_gram_strided: needs bf16, 8 < E <= 128, D %% 8 == 0 (E=%d D=%ld)", E, D);
  COMOE_REQUIRE(row_stride >= D && row_stride % 8 == 0, kBadArg,
                "sim_gram_strided: row stride %ld", row_stride);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int box_rows = (E + 7) / 8 * 8;
  CUtensorMap tmap;
  int rc = make_tmap_bf16_2d_box(&tmap, base, static_cast<uint64_t>(E), static_cast<uint64_t>(D),
                                 static_cast<uint64_t>(row_stride), 64,
                                 static_cast<uint32_t>(box_rows), 128);
  if (rc) return rc;
  const int ctas = gram_tc_ctas(D);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sim_gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kGtSmem);
    attr = true;
  }
  double* partial = static_cast<double*>(work);
  static const int contig = [] {
    const char* e = std::getenv("COMOE_GRAM_CONTIG");
    const char* d = std::getenv("COMOE_GRAM_DEBUG");
    return (e && e[0] == '1' ? 1 : 0) | (d ? std::atoi(d) : 0);
  }();
  sim_gram_tc_kernel<<<ctas, kGtThreads, kGtSmem, s>>>(tmap, 0, box_rows, E, (D + 63) / 64,
                                                        partial, contig);
  rc = check_launch("sim_gram_tc_kernel");
  if (rc) return rc;
  const long nn = static_cast<long>(E) * E;
  const int blocks = static_cast<int>((nn + 7) / 8 < 4096 ? (nn + 7) / 8 : 4096);
  sim_reduce_kernel<<<blocks, 256, 0, s>>>(partial, ctas, E, E, 0, gram, nullptr);
  return check_launch("sim_reduce_kernel");
}

int comoe_sim_tc_supported(int E, long D) { return comoe::sim_tc(COMOE_DTYPE_BF16, E, D) ? 1 : 0; }

int comoe_sim_contract(int dtype, const void* const* rows, int E, long D, const double* probes,
                       int n_probes, const double* proj, int buckets, double* gram,
                       double* logits, void* work, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(rows && gram && work, kBadArg, "sim_contract: null pointer");
  COMOE_REQUIRE(n_probes == 0 || (probes && proj && logits && buckets >= 1), kBadArg,
                "sim_contract: null calibration");
  COMOE_REQUIRE(E >= 1 && D >= 1 && n_probes >= 0, kBadArg, "sim_contract: bad sizes");
  COMOE_REQUIRE(dtype == COMOE_DTYPE_BF16 || dtype == COMOE_DTYPE_F64, kBadArg,
                "sim_contract: dtype %d", dtype);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* partial = static_cast<double*>(work);
  if (n_probes > 0 && !sim_logits_small(E, buckets, D))  // one tiled pass: Gram and logits
    return tiled_contract(dtype, rows, E, D, probes, n_probes, proj, buckets, gram, logits,
                          partial, s);
  int rc = gram_contract(dtype, rows, E, D, gram, partial, s);
  if (rc || n_probes == 0) return rc;
  // small surrogate logits, partials after the Gram's (stream order keeps them apart)
  const std::pair<long, int> lp = logit_plan(D);
  double* lpart = partial + (comoe_sim_workspace_bytes(E, n_probes, buckets, D) / sizeof(double) -
                             static_cast<long>(lp.second) * E * n_probes * buckets);
  if (dtype == COMOE_DTYPE_BF16 && n_probes <= 8 && sim_logits_dmma()) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(sim_logits_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kLdSmem);
      attr = true;
    }
    sim_logits_dmma_kernel<<<lp.second, kLdThreads, kLdSmem, s>>>(rows, E, D, probes, n_probes,
                                                                  proj, buckets, lp.first, lpart);
  } else if (dtype == COMOE_DTYPE_BF16) {
    constexpr int smem = 2 * LogitStage<__nv_bfloat16>::kBytes;
    cudaFuncSetAttribute(sim_logits_small_kernel<__nv_bfloat16>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    sim_logits_small_kernel<__nv_bfloat16><<<lp.second, 512, smem, s>>>(
        rows, E, D, probes, n_probes, proj, buckets, lp.first, lpart);
  } else {
    constexpr int smem = 2 * LogitStage<double>::kBytes;
    cudaFuncSetAttribute(sim_logits_small_kernel<double>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    sim_logits_small_kernel<double><<<lp.second, 512, smem, s>>>(rows, E, D, probes, n_probes,
                                                                 proj, buckets, lp.first, lpart);
  }
  rc = check_launch("sim_logits_small_kernel");
  if (rc) return rc;
  const long n = static_cast<long>(E) * n_probes * buckets;
  sim_sum_partials<<<static_cast<int>((n + 7) / 8), 256, 0, s>>>(lpart, lp.second, n, logits);
  return check_launch("sim_sum_partials");
}

int comoe_sim_finalize(const double* gram, const double* logits, int E, int n_probes, int buckets,
                       double alpha, double* sim, void* stream) {
  using namespace comoe;
  COMOE_REQUIRE(gram && sim && (logits || n_probes == 0), kBadArg, "sim_finalize: null pointer");
  COMOE_REQUIRE(alpha >= 0.0 && alpha <= 1.0, kBadArg, "sim_finalize: alpha=%g", alpha);
  const long pairs = static_cast<long>(E) * E;
  const long smem = 2L * E * n_probes * buckets * static_cast<long>(sizeof(double));
  if (n_probes > 0 && smem <= 200 * 1024) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(sim_finalize_staged_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
    sim_finalize_staged_kernel<<<1, kFinalizeThreads, smem, static_cast<cudaStream_t>(stream)>>>(
        gram, logits, E, n_probes, buckets, alpha, sim);
    return check_launch("sim_finalize_staged_kernel");
  }
  const int blocks = static_cast<int>((pairs + 127) / 128 < 1024 ? (pairs + 127) / 128 : 1024);
  sim_finalize_kernel<<<blocks, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      gram, logits, E, n_probes, buckets, alpha, sim);
  return check_launch("sim_finalize_kernel");
}

}  // extern "C"
