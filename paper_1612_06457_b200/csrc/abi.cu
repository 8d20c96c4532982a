// Library-wide plumbing of the C ABI: per-thread error text, version, build stamp,
// SM count.
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

#ifndef UT_SOURCE_HASH
#define UT_SOURCE_HASH "unstamped"
#endif
// The stamp is also kept as plain bytes so the loader can read it from the file.
extern "C" __attribute__((used)) const char ut_build_stamp[] = "UT_SOURCE_HASH=" UT_SOURCE_HASH;

extern "C" {

int ut_version(void) { return 1; }

const char* ut_build_hash(void) { return ut_build_stamp + 15; }

const char* ut_last_error(void) { return ut::g_err; }

int64_t ut_moment_len(int32_t bands) {
  return 1 + (int64_t)bands + (int64_t)bands * bands;
}

}  // extern "C"
