// C-ABI plumbing: error reporting, tensor-map encoding, version.
#include <cudaTypedefs.h>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "../../include/comoe_b200.h"

namespace comoe {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int pdl_attr(cudaLaunchAttribute* attr) {
  static const bool on = [] {
    const char* e = std::getenv("COMOE_PDL");
    return e && e[0] == '1';
  }();
  if (!on) return 0;
  attr->id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr->val.programmaticStreamSerializationAllowed = 1;
  return 1;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return kCudaError;
  }
  return kOk;
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

static void load_encode() {
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
          cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

int make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                      uint32_t box_rows) {
  std::call_once(g_encode_once, load_encode);
  COMOE_REQUIRE(g_encode != nullptr, kNoDriver, "cuTensorMapEncodeTiled unavailable (no driver)");
  COMOE_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0, kBadArg,
                "tensor base must be 16-byte aligned");
  COMOE_REQUIRE(cols % 64 == 0 && rows > 0, kUnsupportedShape, "tensor map %llux%llu unsupported",
                (unsigned long long)rows, (unsigned long long)cols);
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  COMOE_REQUIRE(r == CUDA_SUCCESS, kCudaError, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return kOk;
}

int make_tmap_bf16_2d_box(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                          uint64_t row_stride_elems, uint32_t box_cols, uint32_t box_rows,
                          int swizzle_bytes) {
  std::call_once(g_encode_once, load_encode);
  COMOE_REQUIRE(g_encode != nullptr, kNoDriver, "cuTensorMapEncodeTiled unavailable (no driver)");
  COMOE_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0 && row_stride_elems % 8 == 0,
                kBadArg, "tensor base/stride must be 16-byte aligned");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_elems * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                      : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  COMOE_REQUIRE(r == CUDA_SUCCESS, kCudaError, "cuTensorMapEncodeTiled(box) failed (%d)", (int)r);
  return kOk;
}

int make_tmap_bf16_3d(CUtensorMap* map, const void* base, uint64_t slots, uint64_t rows,
                      uint64_t cols, uint64_t slot_stride, uint32_t box_rows) {
  std::call_once(g_encode_once, load_encode);
  COMOE_REQUIRE(g_encode != nullptr, kNoDriver, "cuTensorMapEncodeTiled unavailable (no driver)");
  COMOE_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0, kBadArg,
                "tensor base must be 16-byte aligned");
  COMOE_REQUIRE(cols % 64 == 0 && rows > 0 && slots > 0 && slot_stride % 8 == 0 &&
                    slot_stride >= rows * cols,
                kUnsupportedShape, "slot tensor map %llux%llux%llu (stride %llu) unsupported",
                (unsigned long long)slots, (unsigned long long)rows, (unsigned long long)cols,
                (unsigned long long)slot_stride);
  cuuint64_t dims[3] = {cols, rows, slots};
  cuuint64_t strides[2] = {cols * 2, slot_stride * 2};
  cuuint32_t box[3] = {64, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  COMOE_REQUIRE(r == CUDA_SUCCESS, kCudaError, "cuTensorMapEncodeTiled(3d) failed (%d)", (int)r);
  return kOk;
}

int make_tmap_bf16_kblk(CUtensorMap* map, const void* base, uint64_t slots, uint64_t rows,
                        uint64_t cols, uint64_t slot_stride, uint32_t box_rows,
                        uint32_t box_kblocks) {
  std::call_once(g_encode_once, load_encode);
  COMOE_REQUIRE(g_encode != nullptr, kNoDriver, "cuTensorMapEncodeTiled unavailable (no driver)");
  COMOE_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0, kBadArg,
                "tensor base must be 16-byte aligned");
  COMOE_REQUIRE(cols % 64 == 0 && rows > 0 && slots > 0 && slot_stride % 8 == 0 &&
                    slot_stride >= rows * cols && box_kblocks >= 1 && box_kblocks <= cols / 64,
                kUnsupportedShape, "k-block tensor map %llux%llux%llu unsupported",
                (unsigned long long)slots, (unsigned long long)rows, (unsigned long long)cols);
  cuuint64_t dims[4] = {64, rows, cols / 64, slots};
  cuuint64_t strides[3] = {cols * 2, 128, slot_stride * 2};
  cuuint32_t box[4] = {64, box_rows, box_kblocks, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  COMOE_REQUIRE(r == CUDA_SUCCESS, kCudaError, "cuTensorMapEncodeTiled(k-block 4d) failed (%d)",
                (int)r);
  return kOk;
}

}  // namespace comoe

extern "C" {

int comoe_version(void) { return COMOE_B200_ABI_VERSION; }

const char* comoe_last_error(void) { return comoe::g_err; }

int comoe_num_sms(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return n;
}

}  // extern "C"
