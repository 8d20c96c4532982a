// Library-wide plumbing of the C ABI: per-thread error text, version, SM count.
#include <cstdarg>

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

}  // namespace ut

extern "C" {

int ut_version(void) { return 1; }

const char* ut_last_error(void) { return ut::g_err; }

int64_t ut_moment_len(int32_t bands) {
  return 1 + (int64_t)bands + (int64_t)bands * bands;
}

}  // extern "C"
