// compose_rgb (rendering.py:206-225): three rendered code planes -> one
// interleaved RGB image, on the device.  HBM-bound: each thread moves four
// pixels (4 samples of each plane in, 12 interleaved samples out, all vector
// accesses), so traffic is 3 reads + 3 writes of the plane size.
#include <algorithm>

#include "common.cuh"

namespace ut {
namespace {

template <typename T, typename V4, typename V12>
__global__ void compose_kernel(const T* __restrict__ r, const T* __restrict__ g,
                               const T* __restrict__ b, int64_t npix, T* __restrict__ out) {
  const int64_t quads = npix >> 2;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < quads;
       q += (int64_t)gridDim.x * blockDim.x) {
    T c[3][4];
    *reinterpret_cast<V4*>(c[0]) = reinterpret_cast<const V4*>(r)[q];
    *reinterpret_cast<V4*>(c[1]) = reinterpret_cast<const V4*>(g)[q];
    *reinterpret_cast<V4*>(c[2]) = reinterpret_cast<const V4*>(b)[q];
    T o[12];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) o[3 * i + ch] = c[ch][i];
    V12* dst = reinterpret_cast<V12*>(out + 12 * q);
#pragma unroll
    for (int w = 0; w < 3; ++w) dst[w] = reinterpret_cast<const V12*>(o)[w];
  }
  // tail pixels (npix % 4), and any misaligned remainder
  for (int64_t i = (quads << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npix;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[3 * i] = r[i];
    out[3 * i + 1] = g[i];
    out[3 * i + 2] = b[i];
  }
}

}  // namespace
}  // namespace ut

using namespace ut;

extern "C" {

int ut_compose_rgb(const void* r, const void* g, const void* b, int32_t depth, int64_t npix,
                   void* out, void* stream) {
  UT_REQUIRE(depth == 8 || depth == 16, "composite depth must be 8 or 16, got %d", depth);
  UT_REQUIRE(npix >= 0, "negative pixel count");
  if (npix == 0) return UT_OK;
  UT_REQUIRE(r && g && b && out, "ut_compose_rgb: null pointer");
  const size_t es = depth / 8;
  auto aligned = [&](const void* p, size_t a) { return reinterpret_cast<uintptr_t>(p) % a == 0; };
  UT_REQUIRE(aligned(r, 4 * es) && aligned(g, 4 * es) && aligned(b, 4 * es) && aligned(out, 4 * es),
             "ut_compose_rgb: planes must be %zu-byte aligned", 4 * es);
  cudaStream_t st = as_stream(stream);
  const int64_t work = (npix + 3) / 4;
  const unsigned grid = (unsigned)std::min<int64_t>((work + 255) / 256, (int64_t)sm_count() * 16);
  if (depth == 8)
    compose_kernel<uint8_t, uint32_t, uint32_t><<<grid, 256, 0, st>>>(
        static_cast<const uint8_t*>(r), static_cast<const uint8_t*>(g), static_cast<const uint8_t*>(b),
        npix, static_cast<uint8_t*>(out));
  else
    compose_kernel<uint16_t, uint2, uint2><<<grid, 256, 0, st>>>(
        static_cast<const uint16_t*>(r), static_cast<const uint16_t*>(g), static_cast<const uint16_t*>(b),
        npix, static_cast<uint16_t*>(out));
  UT_CHECK_LAUNCH("compose_kernel");
  return UT_OK;
}

}  // extern "C"
