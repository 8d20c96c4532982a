// Library-wide plumbing of the C ABI: per-thread error text, version, SM count.
#include <cudaTypedefs.h>

#include <cstdarg>
#include <mutex>

#include "common.cuh"

namespace ut {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* where) {
  set_error("%s: CUDA error %d (%s)", where, (int)e, cudaGetErrorString(e));
  return UT_ECUDA;
}

int sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

bool make_tmap_2d(CUtensorMap* map, int dtype, const void* base, uint64_t dim0, uint64_t dim1,
                  uint64_t stride1_bytes, uint32_t box0, uint32_t box1) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!encode) {
    set_error("cuTensorMapEncodeTiled is not available from the driver");
    return false;
  }
  CUtensorMapDataType t;
  switch (dtype) {
    case UT_U8: t = CU_TENSOR_MAP_DATA_TYPE_UINT8; break;
    case UT_U16: t = CU_TENSOR_MAP_DATA_TYPE_UINT16; break;
    case UT_F16: t = CU_TENSOR_MAP_DATA_TYPE_FLOAT16; break;
    case UT_F32: t = CU_TENSOR_MAP_DATA_TYPE_FLOAT32; break;
    default: t = CU_TENSOR_MAP_DATA_TYPE_FLOAT64; break;
  }
  const cuuint64_t dims[2] = {dim0, dim1};
  const cuuint64_t strides[1] = {stride1_bytes};
  const cuuint32_t box[2] = {box0, box1};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, t, 2, const_cast<void*>(base), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) for %llu x %llu, stride %llu, box %u x %u", (int)r,
              (unsigned long long)dim0, (unsigned long long)dim1, (unsigned long long)stride1_bytes,
              box0, box1);
    return false;
  }
  return true;
}

}  // namespace ut

extern "C" {

int ut_version(void) { return 1; }

const char* ut_last_error(void) { return ut::g_err; }

int64_t ut_moment_len(int32_t bands) {
  return 1 + (int64_t)bands + (int64_t)bands * bands;
}

}  // extern "C"
