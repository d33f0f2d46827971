// Host helpers for the tcgen05 GEMM: TMA descriptor encoding and the SM
// count.  (The GEMM self-test hooks live in csrc/testing/gemm_testing.cu,
// built into libd2ft_b200_testing.so — not part of the product library.)
#include <cuda.h>

#include <mutex>
#include <vector>

#include "common.cuh"
#include "gemm_sm100.cuh"

namespace d2ft_b200 {

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  D2FT_REQUIRE(fn, kCuda, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  return fn;
}
}  // namespace

CUtensorMap make_tmap_16_3d(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1_bytes,
                            uint64_t stride2_bytes, uint32_t box_rows, bool is_bf16) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  const cuuint32_t box[3] = {64, box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  D2FT_REQUIRE(stride1_bytes % 16 == 0 && stride2_bytes % 16 == 0, kInput, "tensor map strides must be 16B multiples");
  D2FT_REQUIRE(reinterpret_cast<uintptr_t>(base) % 16 == 0, kInput, "tensor map base must be 16B aligned");
  const CUresult r =
      encode_fn()(&m, is_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  D2FT_REQUIRE(r == CUDA_SUCCESS, kCuda, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

static CUtensorMap make_tmap_store_3d(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                                      uint64_t s2, uint32_t box0, uint32_t box1, int swizzle_bytes, int esize) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {s1, s2};
  const cuuint32_t box[3] = {box0, box1, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  D2FT_REQUIRE(s1 % 16 == 0 && s2 % 16 == 0 && (box0 * esize) % 16 == 0, kInput,
               "store tensor map: 16-byte granularity");
  const CUresult r = encode_fn()(&m, esize == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 swizzle_bytes == 64   ? CU_TENSOR_MAP_SWIZZLE_64B
                                 : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                       : CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  D2FT_REQUIRE(r == CUDA_SUCCESS, kCuda, "cuTensorMapEncodeTiled (store) failed (" + std::to_string((int)r) + ")");
  return m;
}
CUtensorMap make_tmap_store_f16_3d(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1, uint64_t s2,
                                   uint32_t box0, uint32_t box1, int swizzle_bytes) {
  return make_tmap_store_3d(base, d0, d1, d2, s1, s2, box0, box1, swizzle_bytes, 2);
}
CUtensorMap make_tmap_store_f32_3d(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1, uint64_t s2,
                                   uint32_t box0, uint32_t box1, int swizzle_bytes) {
  return make_tmap_store_3d(base, d0, d1, d2, s1, s2, box0, box1, swizzle_bytes, 4);
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    D2FT_CUDA(cudaGetDevice(&dev));
    D2FT_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

}  // namespace d2ft_b200
