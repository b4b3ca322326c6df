// K3 entry points: grouped expert GEMM and the two-pass expert FFN over the
// HBM expert slot pool. One slot holds one expert as a flat bf16 vector
// [W_in (N1 x d) | W_out (d x d_ff)], N1 = d_ff (ReLU) or 2*d_ff (SwiGLU with
// gate/up interleaved in 128-row blocks) — the device image of the
// reference's flat `Expert.params` (pkg/src/comoe/moe.py:69-74).
#include <cstdlib>

#include "fused_ffn.cuh"
#include "../../include/comoe_b200.h"

namespace comoe {

// ---------------------------------------------------------------- fused FFN
// Opt-in (COMOE_FUSED_FFN=1): comoe_grouped_ffn then runs the fused kernel
// for qualifying shapes. Measured slower than the two-launch FFN at every
// batch size of the C2 layer (K3F: 725 vs 574 us at 65,536 tokens,
// 317 vs 247 us at 16,384, 189 vs 171 us at 256), so it is not the default.
static bool fused_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("COMOE_FUSED_FFN");
    return e && e[0] == '1';
  }();
  return on;
}

static bool fused_supported(int d, int d_ff, int act, int G) {
  return act == COMOE_ACT_RELU && d > 0 && d % 256 == 0 && d <= kFMaxD && d_ff > 0 &&
         d_ff % kFChunk == 0 && G >= 1 && G <= kFMaxGroups;
}

// k-blocks per weight TMA / ring stage (COMOE_FUSED_BOXES: 1 = 6 x 16 KB,
// 2 = 3 x 32 KB, the default: the single producer thread needs >= 8 MMAs of
// work per TMA it issues)
static int fused_boxes() {
  static const int v = [] {
    const char* e = std::getenv("COMOE_FUSED_BOXES");
    return e && std::atoi(e) == 1 ? 1 : 2;
  }();
  return v;
}
static int fused_debug() {
  static const int v = [] {
    const char* e = std::getenv("COMOE_FUSED_DEBUG");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

template <int kStages, int kBoxes, bool kGather>
static int launch_fused(const CUtensorMap& twi, const CUtensorMap& two, const CUtensorMap& tx,
                        const FusedFfnParams& p, cudaStream_t stream) {
  auto kern = fused_ffn_kernel<kStages, kBoxes, kGather>;
  const int smem = FusedCfg<kStages, kBoxes>::smem_bytes(p.d);
  static int attr_set = 0;  // per instantiation: the largest size set so far
  if (attr_set < smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_set = smem;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  kern<<<sms & ~1, kFThreads, smem, stream>>>(twi, two, tx, p);
  return check_launch("fused_ffn_kernel");
}

static int fused_ffn_impl(const void* x, long x_rows, const int* gather_rows, int d, int d_ff,
                          const void* pool, int n_slots, long slot_stride, const int* group_rows,
                          const int* group_row_base, const int* group_slot, int G, void* out,
                          int ldo, const int* row_token, const float* row_prob,
                          cudaStream_t stream) {
  COMOE_REQUIRE(x && pool && out && group_rows && group_row_base && group_slot, kBadArg,
                "fused_ffn: null pointer");
  COMOE_REQUIRE(fused_supported(d, d_ff, COMOE_ACT_RELU, G), kUnsupportedShape,
                "fused_ffn: d=%d d_ff=%d G=%d unsupported (ReLU, d %% 256 == 0, d <= %d, "
                "d_ff %% 256 == 0, G <= %d)", d, d_ff, G, kFMaxD, kFMaxGroups);
  COMOE_REQUIRE(x_rows > 0 && n_slots > 0, kBadArg, "fused_ffn: empty operand");
  COMOE_REQUIRE(ldo % 2 == 0 && ldo >= d && (reinterpret_cast<uintptr_t>(out) & 3) == 0,
                kUnsupportedShape, "fused_ffn: out rows must be 4-byte aligned (ldo even)");
  COMOE_REQUIRE(slot_stride >= 2L * d * d_ff, kBadArg, "fused_ffn: slot smaller than the expert");
  COMOE_REQUIRE((row_token == nullptr) == (row_prob == nullptr), kBadArg,
                "fused_ffn: row_token and row_prob go together");
  CUtensorMap twi, two, tx;
  const int kbox = fused_boxes();
  int rc = make_tmap_bf16_kblk(&twi, pool, n_slots, d_ff, d, slot_stride, 128, kbox);
  if (rc) return rc;
  const void* wo = static_cast<const __nv_bfloat16*>(pool) + static_cast<long>(d_ff) * d;
  rc = make_tmap_bf16_kblk(&two, wo, n_slots, d, d_ff, slot_stride, 128, kbox);
  if (rc) return rc;
  rc = make_tmap_bf16_2d(&tx, x, static_cast<uint64_t>(x_rows), d, gather_rows ? 1 : kFTok / 2);
  if (rc) return rc;
  FusedFfnParams p{group_rows, group_row_base, group_slot, G, d, d_ff,
                   reinterpret_cast<__nv_bfloat16*>(out), ldo, row_token, row_prob, gather_rows,
                   fused_debug()};
  if (kbox == 1)
    return gather_rows ? launch_fused<6, 1, true>(twi, two, tx, p, stream)
                       : launch_fused<6, 1, false>(twi, two, tx, p, stream);
  return gather_rows ? launch_fused<3, 2, true>(twi, two, tx, p, stream)
                     : launch_fused<3, 2, false>(twi, two, tx, p, stream);
}

template <int BN, int kStages, int kMode>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GroupedGemmParams& p,
                       cudaStream_t stream) {
  using S = GemmSmem<BN, kStages>;
  auto kern = grouped_gemm_kernel<BN, kStages, kMode>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kTotal);
    attr_set = true;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  kern<<<sms, kGemmThreads, S::kTotal, stream>>>(ta, tb, p);
  return check_launch("grouped_gemm_kernel");
}

template <int kMode, int kStages, int kEpiWarps, int kBN = 256>
static int launch_gemm_2sm_cfg(const CUtensorMap& tw, const CUtensorMap& tx,
                               const CUtensorMap& to, const GroupedGemmParams& p,
                               cudaStream_t stream) {
  using C = Gemm2Cfg<kStages, kEpiWarps, kBN>;
  if (p.gather_rows) {
    if constexpr (kMode == kEpiRelu && kBN == 256) {
      auto kg = grouped_gemm_2sm_kernel<kMode, kStages, kEpiWarps, true>;
      static bool attr_g = false;
      if (!attr_g) {
        cudaFuncSetAttribute(kg, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kTotal);
        attr_g = true;
      }
      int dev = 0, sms = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      kg<<<sms & ~1, C::kThreads, C::kTotal, stream>>>(tw, tx, to, p);
      return check_launch("grouped_gemm_2sm_kernel(gather)");
    }
    set_error("grouped_gemm: row gather is only supported with the ReLU epilogue");
    return kUnsupportedShape;
  }
  auto kern = grouped_gemm_2sm_kernel<kMode, kStages, kEpiWarps, false, kBN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kTotal);
    attr_set = true;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(sms & ~1);
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = C::kTotal;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[1];  // (cluster shape comes from __cluster_dims__)
  cfg.attrs = attrs;
  cfg.numAttrs = pdl_attr(&attrs[0]);
  cudaLaunchKernelEx(&cfg, kern, tw, tx, to, p);
  return check_launch("grouped_gemm_2sm_kernel");
}

// pipeline config (COMOE_GEMM2_CFG for A/B runs): 0 = 5 stages x 8 epilogue
// warps, 1 = 4 x 8, 2 = 6 x 4 (default: deepest pipeline; ragged C2 +3-5%
// over 0 — the loads are latency-bound, 4 stages lose 7%)
static int gemm2_cfg() {
  static const int c = [] {
    const char* e = std::getenv("COMOE_GEMM2_CFG");
    return e ? std::atoi(e) : 2;
  }();
  return c;
}

template <int kMode>
static int launch_gemm_2sm(const CUtensorMap& tw, const CUtensorMap& tx, const CUtensorMap& to,
                           const GroupedGemmParams& p, cudaStream_t stream) {
  if (p.gather_rows) return launch_gemm_2sm_cfg<kMode, 5, 8>(tw, tx, to, p, stream);
  switch (gemm2_cfg()) {
    case 0: return launch_gemm_2sm_cfg<kMode, 5, 8>(tw, tx, to, p, stream);
    case 1: return launch_gemm_2sm_cfg<kMode, 4, 8>(tw, tx, to, p, stream);
    default: return launch_gemm_2sm_cfg<kMode, 6, 4>(tw, tx, to, p, stream);
  }
}

// Decode-sized batches (a few tokens per expert): 32-token tiles with
// 16-row token boxes leave room for 10 weight stages (the weight stream,
// first-touch from HBM, is the whole cost there). COMOE_GEMM_SMALLN=0 off.
// COMOE_GEMM_SMALLN: 0 = 256-token tiles only, 1 = + 32-token tiles, 2
// (default) = + 64-token tiles with 9 stages up to 32 rows per group
// (4096 tokens over 128 experts: 239 -> 233 us per layer)
static int small_mode() {
  static const int m = [] {
    const char* e = std::getenv("COMOE_GEMM_SMALLN");
    return e ? std::atoi(e) : 2;
  }();
  return m;
}
// token rows per tile: 32 (<= 8 rows per group on average), 64 (mode 2, <= 32), else 256
static int tile_tokens(long a_rows, int G) {
  const int m = small_mode();
  if (m >= 1 && a_rows <= 8L * G) return 32;
  if (m >= 2 && a_rows <= 32L * G) return 64;
  return 256;
}

template <int kMode>
static int launch_gemm_2sm_small(const CUtensorMap& tw, const CUtensorMap& tx,
                                 const CUtensorMap& to, const GroupedGemmParams& p, int bn,
                                 cudaStream_t stream) {
  if (bn == 64) return launch_gemm_2sm_cfg<kMode, 9, 4, 64>(tw, tx, to, p, stream);
  return launch_gemm_2sm_cfg<kMode, 10, 4, 32>(tw, tx, to, p, stream);
}

// dev switches (COMOE_GEMM_DEBUG, or comoe_debug_set_gemm at run time so
// A/B probes can alternate modes inside one process)
static int g_gemm_debug_override = -1;
static int gemm_debug() {
  static const int d = [] {
    const char* e = std::getenv("COMOE_GEMM_DEBUG");
    return e ? std::atoi(e) : 0;
  }();
  return g_gemm_debug_override >= 0 ? g_gemm_debug_override : d;
}

// Tile order (both kernels): feature-tile major when one group's weight block
// exceeds 32 MB (Mixtral: 235 MB per expert — token-tile major re-streamed
// every expert's weights from HBM once per 128-token tile); COMOE_GEMM_ORDER
// = 0 / 1 forces token- / feature-tile major.
static int ft_major(long weight_bytes) {
  static const int forced = [] {
    const char* e = std::getenv("COMOE_GEMM_ORDER");
    return e ? std::atoi(e) : -1;
  }();
  if (forced >= 0) return forced;
  return weight_bytes > (32L << 20) ? 1 : 0;
}

// Equal token tiles for the 2-SM kernel when K >= 1536 (COMOE_GEMM_EQUAL=0/1
// forces off/on): see decode_tile2.
static int equal_tiles(int K) {
  static const int forced = [] {
    const char* e = std::getenv("COMOE_GEMM_EQUAL");
    return e ? std::atoi(e) : -1;
  }();
  if (forced >= 0) return forced;
  return K >= 1536 ? 1 : 0;
}

static bool force_1sm() {
  static const bool f = [] {
    const char* e = std::getenv("COMOE_GEMM_1SM");
    return e && e[0] == '1';
  }();
  return f;
}

// B operand: `N x K` matrix at element offset `b_offset` inside every slot.
static int grouped_gemm_impl(const void* a, long a_rows, const void* pool, int n_slots,
                             long slot_stride, long b_offset, int N, int K,
                             const int* group_rows, const int* group_row_base,
                             const int* group_slot, int G, int epi_mode, void* out, int ldo,
                             const int* row_token, const float* row_prob, cudaStream_t stream,
                             const int* a_gather = nullptr) {
  COMOE_REQUIRE(a && pool && out && group_rows && group_row_base && group_slot, kBadArg,
                "grouped_gemm: null pointer");
  COMOE_REQUIRE(G >= 1 && G <= kMaxGroups, kBadArg, "grouped_gemm: G=%d out of [1,%d]", G,
                kMaxGroups);
  COMOE_REQUIRE(K % 64 == 0 && K > 0, kUnsupportedShape,
                "grouped_gemm: K=%d must be a multiple of 64", K);
  COMOE_REQUIRE(N % 256 == 0 && N > 0, kUnsupportedShape,
                "grouped_gemm: N=%d must be a multiple of 256", N);
  COMOE_REQUIRE(ldo % 8 == 0, kUnsupportedShape, "grouped_gemm: ldo must be a multiple of 8");
  COMOE_REQUIRE(a_rows > 0 && n_slots > 0, kBadArg, "grouped_gemm: empty operand");
  COMOE_REQUIRE(b_offset % 8 == 0 && b_offset + static_cast<long>(N) * K <= slot_stride, kBadArg,
                "grouped_gemm: B block exceeds the slot");
  if (epi_mode == kEpiScaleScatter)
    COMOE_REQUIRE(row_token && row_prob, kBadArg, "scatter epilogue needs row_token/row_prob");
  CUtensorMap ta, tb;
  const void* b = static_cast<const __nv_bfloat16*>(pool) + b_offset;
  GroupedGemmParams p{group_rows, group_row_base, group_slot, G, N, K,
                      reinterpret_cast<__nv_bfloat16*>(out), ldo, row_token, row_prob,
                      a_gather, gemm_debug(), ft_major(static_cast<long>(N) * K * 2),
                      equal_tiles(K)};
  int rc;
  // SwiGLU stays on the 1-SM kernel: a 2-SM variant (gate/up rows split into
  // 64-row boxes per SM, up values handed to the gate warps through shared
  // memory) measured 16% slower at the C2 shape and equal at C5
  if (epi_mode != kEpiSwiGLU && !force_1sm()) {
    COMOE_REQUIRE(G <= kMaxGroups2, kBadArg, "grouped_gemm: G=%d > %d", G, kMaxGroups2);
    // 2-SM swap-AB kernel: weights = A (128-feature boxes), tokens = B (128-row boxes)
    rc = make_tmap_bf16_3d(&tb, b, n_slots, N, K, slot_stride, 128);
    if (rc) return rc;
    const int bn = a_gather ? 256 : tile_tokens(a_rows, G);
    const bool small = bn < 256;
    rc = make_tmap_bf16_2d(&ta, a, static_cast<uint64_t>(a_rows), K, a_gather ? 1 : bn / 2);
    if (rc) return rc;
    // output map for the bulk-store epilogue: [a_rows, N] bf16 at ld ldo, box
    // 32 features x 32 tokens, 64-byte swizzle (unused by the scatter mode)
    CUtensorMap to;
    rc = make_tmap_bf16_2d_box(&to, out, static_cast<uint64_t>(a_rows), static_cast<uint64_t>(N),
                               static_cast<uint64_t>(ldo), 32, 32, 64);
    if (rc) return rc;
    if (small) {
      switch (epi_mode) {
        case kEpiRelu: return launch_gemm_2sm_small<kEpiRelu>(tb, ta, to, p, bn, stream);
        case kEpiScaleScatter: return launch_gemm_2sm_small<kEpiScaleScatter>(tb, ta, to, p, bn, stream);
        case kEpiStore: return launch_gemm_2sm_small<kEpiStore>(tb, ta, to, p, bn, stream);
        default: break;
      }
    }
    switch (epi_mode) {
      case kEpiRelu: return launch_gemm_2sm<kEpiRelu>(tb, ta, to, p, stream);
      case kEpiScaleScatter: return launch_gemm_2sm<kEpiScaleScatter>(tb, ta, to, p, stream);
      case kEpiStore: return launch_gemm_2sm<kEpiStore>(tb, ta, to, p, stream);
      default: break;
    }
    set_error("grouped_gemm: unknown epilogue mode %d", epi_mode);
    return kBadArg;
  }
  COMOE_REQUIRE(a_gather == nullptr, kUnsupportedShape,
                "grouped_gemm: row gather needs the 2-SM kernel (not SwiGLU / COMOE_GEMM_1SM)");
  rc = make_tmap_bf16_2d(&ta, a, static_cast<uint64_t>(a_rows), K, kGemmBM);
  if (rc) return rc;
  rc = make_tmap_bf16_3d(&tb, b, n_slots, N, K, slot_stride, 256);
  if (rc) return rc;
  switch (epi_mode) {
    case kEpiRelu: return launch_gemm<256, 4, kEpiRelu>(ta, tb, p, stream);
    case kEpiSwiGLU: return launch_gemm<256, 4, kEpiSwiGLU>(ta, tb, p, stream);
    case kEpiScaleScatter: return launch_gemm<256, 4, kEpiScaleScatter>(ta, tb, p, stream);
    case kEpiStore: return launch_gemm<256, 4, kEpiStore>(ta, tb, p, stream);
    default: break;
  }
  set_error("grouped_gemm: unknown epilogue mode %d", epi_mode);
  return kBadArg;
}

}  // namespace comoe

extern "C" {

int comoe_grouped_gemm(const void* a, long a_rows, const void* pool, int n_slots, long slot_stride,
                       long b_offset, int N, int K, const int* group_rows,
                       const int* group_row_base, const int* group_slot, int G, int epi_mode,
                       void* out, int ldo, const int* row_token, const float* row_prob,
                       const int* a_gather, void* stream) {
  return comoe::grouped_gemm_impl(a, a_rows, pool, n_slots, slot_stride, b_offset, N, K,
                                  group_rows, group_row_base, group_slot, G, epi_mode, out, ldo,
                                  row_token, row_prob, static_cast<cudaStream_t>(stream),
                                  a_gather);
}

int comoe_grouped_ffn(const void* x_perm, long total_rows, int d, int d_ff, int act,
                      const void* pool, int n_slots, long slot_stride, const int* group_rows,
                      const int* group_row_base, const int* group_slot, int G, void* h_work,
                      void* out, int ldo, const int* row_token, const float* row_prob,
                      void* stream) {
  using namespace comoe;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  COMOE_REQUIRE(act == COMOE_ACT_RELU || act == COMOE_ACT_SWIGLU, kBadArg, "grouped_ffn: act=%d",
                act);
  if (fused_enabled() && fused_supported(d, d_ff, act, G))  // H stays on chip
    return fused_ffn_impl(x_perm, total_rows, nullptr, d, d_ff, pool, n_slots, slot_stride,
                          group_rows, group_row_base, group_slot, G, out, ldo, row_token, row_prob,
                          s);
  COMOE_REQUIRE(h_work != nullptr, kBadArg, "grouped_ffn: null workspace");
  const int n1 = act == COMOE_ACT_SWIGLU ? 2 * d_ff : d_ff;
  int rc = grouped_gemm_impl(x_perm, total_rows, pool, n_slots, slot_stride, 0, n1, d, group_rows,
                             group_row_base, group_slot, G,
                             act == COMOE_ACT_SWIGLU ? kEpiSwiGLU : kEpiRelu, h_work, d_ff,
                             nullptr, nullptr, s);
  if (rc) return rc;
  const int mode2 = row_token ? kEpiScaleScatter : kEpiStore;
  return grouped_gemm_impl(h_work, total_rows, pool, n_slots, slot_stride,
                           static_cast<long>(n1) * d, d, d_ff, group_rows, group_row_base,
                           group_slot, G, mode2, out, ldo, row_token, row_prob, s);
}

int comoe_fused_ffn_supported(int d, int d_ff, int act, int G) {
  return comoe::fused_supported(d, d_ff, act, G) ? 1 : 0;
}

int comoe_fused_ffn_enabled(void) { return comoe::fused_enabled() ? 1 : 0; }

int comoe_fused_ffn(const void* x, long x_rows, const int* gather_rows, int d, int d_ff,
                    const void* pool, int n_slots, long slot_stride, const int* group_rows,
                    const int* group_row_base, const int* group_slot, int G, void* out, int ldo,
                    const int* row_token, const float* row_prob, void* stream) {
  return comoe::fused_ffn_impl(x, x_rows, gather_rows, d, d_ff, pool, n_slots, slot_stride,
                               group_rows, group_row_base, group_slot, G, out, ldo, row_token,
                               row_prob, static_cast<cudaStream_t>(stream));
}

// dev: per-pair wait cycles of the last fused FFN launched with
// COMOE_FUSED_DEBUG bit 256 (128 pairs x 16 counters, synchronises)
int comoe_debug_fused_prof(unsigned long long* out) {
  using namespace comoe;
  COMOE_REQUIRE(out, kBadArg, "debug_fused_prof: null pointer");
  const cudaError_t e = cudaMemcpyFromSymbol(out, g_fprof, sizeof(g_fprof));
  COMOE_REQUIRE(e == cudaSuccess, kCudaError, "debug_fused_prof: %s", cudaGetErrorString(e));
  return kOk;
}

// dev: {clock64, ns} at start and end of CTA 0 of the last 2-SM grouped GEMM
// launched with COMOE_GEMM_DEBUG bit 256 (synchronises)
int comoe_debug_gemm_clock(unsigned long long* out4) {
  using namespace comoe;
  COMOE_REQUIRE(out4, kBadArg, "debug_gemm_clock: null pointer");
  const cudaError_t e = cudaMemcpyFromSymbol(out4, g_gemm_clock, sizeof(unsigned long long) * 4);
  COMOE_REQUIRE(e == cudaSuccess, kCudaError, "debug_gemm_clock: %s", cudaGetErrorString(e));
  return kOk;
}

// dev: override COMOE_GEMM_DEBUG for later launches (-1 restores the env value)
int comoe_debug_set_gemm(int debug) {
  comoe::g_gemm_debug_override = debug;
  return comoe::kOk;
}

}  // extern "C"
