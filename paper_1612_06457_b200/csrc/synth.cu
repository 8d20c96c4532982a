// Seeded synthetic cubes for the BASELINE.json configs, generated in HBM.
//
// The reference has no dataset for this path; BASELINE.json defines a
// generator.  Generating the 34 GB cfg-4 cube on the host
// would take minutes, so it is produced here, per pixel, from a counter-based
// hash (splitmix64 of seed / pixel / band) and Box-Muller normals.  The class
// map is a list of integer rectangles / ellipses evaluated exactly, so the
// host (training-point sampling) and the device agree on every pixel's class.
#include "common.cuh"

namespace ut {
namespace {

constexpr int kMaxShapes = 32;
constexpr int kMaxClasses = 8;

struct Shapes {
  int64_t v[kMaxShapes][6];
  int n;
};

__host__ __device__ __forceinline__ int class_at(const Shapes& sh, int64_t y, int64_t x) {
  int c = 0;
  for (int i = 0; i < sh.n; ++i) {
    const int64_t* s = sh.v[i];
    bool in;
    if (s[0] == 0) {
      in = y >= s[2] && x >= s[3] && y < s[4] && x < s[5];
    } else {
      const int64_t dy = y - s[2], dx = x - s[3], ry = s[4], rx = s[5];
      in = (dy * rx) * (dy * rx) + (dx * ry) * (dx * ry) <= (rx * ry) * (rx * ry);
    }
    if (in) c = (int)s[1];
  }
  return c;
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <typename T> __device__ __forceinline__ T cast_sample(float v);
template <> __device__ __forceinline__ float cast_sample<float>(float v) { return v; }
template <> __device__ __forceinline__ double cast_sample<double>(float v) { return (double)v; }
template <> __device__ __forceinline__ __half cast_sample<__half>(float v) { return __float2half_rn(v); }
template <> __device__ __forceinline__ uint16_t cast_sample<uint16_t>(float v) {
  return (uint16_t)floorf(4095.0f * v + 0.5f);  // round_half_away, v >= 0
}
template <> __device__ __forceinline__ uint8_t cast_sample<uint8_t>(float v) {
  return (uint8_t)floorf(255.0f * v + 0.5f);
}

template <typename T>
__global__ void __launch_bounds__(256)
synth_kernel(T* __restrict__ out, int64_t bs, int64_t rs, int64_t rows, int64_t cols, int64_t row0,
             int bands, const double* __restrict__ means, const double* __restrict__ chol,
             int classes, Shapes sh, uint64_t seed) {
  __shared__ float L[kMaxClasses][kMaxBands][kMaxBands];
  __shared__ float mu[kMaxClasses][kMaxBands];
  for (int e = threadIdx.x; e < classes * bands * bands; e += blockDim.x) {
    const int c = e / (bands * bands), r = (e / bands) % bands, q = e % bands;
    L[c][r][q] = (float)chol[e];
  }
  for (int e = threadIdx.x; e < classes * bands; e += blockDim.x)
    mu[e / bands][e % bands] = (float)means[e];
  __syncthreads();
  const int64_t npix = rows * cols;
  for (int64_t pix = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pix < npix;
       pix += (int64_t)gridDim.x * blockDim.x) {
    const int64_t y = pix / cols, x = pix - y * cols;
    const int64_t gy = row0 + y;
    const int c = class_at(sh, gy, x);
    const uint64_t gpix = (uint64_t)gy * (uint64_t)cols + (uint64_t)x;
    float z[kMaxBands];
#pragma unroll
    for (int b = 0; b < kMaxBands; b += 2) {
      const uint64_t h = splitmix64(seed ^ (gpix * 0x100000001B3ull + (uint64_t)b));
      const float u1 = ((float)(uint32_t)(h >> 32) + 0.5f) * 2.3283064365386963e-10f;
      const float u2 = (float)(uint32_t)h * 2.3283064365386963e-10f;
      const float r = sqrtf(-2.0f * logf(u1));
      float sv, cv;
      sincospif(2.0f * u2, &sv, &cv);
      z[b] = r * cv;
      z[b + 1] = r * sv;
    }
    T* dst = out + y * rs + x;
    for (int b = 0; b < bands; ++b) {
      float v = mu[c][b];
#pragma unroll
      for (int q = 0; q < kMaxBands; ++q)
        if (q <= b) v = fmaf(L[c][b][q], z[q], v);
      v = fminf(fmaxf(v, 0.0f), 1.0f);
      dst[b * bs] = cast_sample<T>(v);
    }
  }
}

__global__ void class_of_kernel(Shapes sh, const int32_t* xy, int64_t n, int32_t* cls) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) cls[j] = class_at(sh, xy[2 * j + 1], xy[2 * j]);
}

int load_shapes(Shapes& sh, const int64_t* shapes, int nshapes) {
  UT_REQUIRE(nshapes >= 0 && nshapes <= kMaxShapes, "at most %d shapes", kMaxShapes);
  sh.n = nshapes;
  for (int i = 0; i < nshapes; ++i)
    for (int j = 0; j < 6; ++j) sh.v[i][j] = shapes[i * 6 + j];
  return UT_OK;
}

template <typename T>
int launch_synth(const ut_cube* cube, const double* means, const double* chol, int classes,
                 const Shapes& sh, uint64_t seed, cudaStream_t st) {
  const int64_t npix = cube->rows * cube->cols;
  int64_t grid = (npix + 255) / 256;
  if (grid > (int64_t)sm_count() * 16) grid = (int64_t)sm_count() * 16;
  synth_kernel<T><<<(int)grid, 256, 0, st>>>(
      static_cast<T*>(const_cast<void*>(cube->data)), cube->band_stride, cube->row_stride,
      cube->rows, cube->cols, cube->row0, cube->bands, means, chol, classes, sh, seed);
  UT_CHECK_LAUNCH("synth_kernel");
  return UT_OK;
}

}  // namespace
}  // namespace ut

using namespace ut;

extern "C" {

int ut_synth_cube(const ut_cube* cube, int64_t height, const double* means, const double* chol,
                  int32_t classes, const int64_t* shapes, int32_t nshapes, uint64_t seed,
                  void* stream) {
  UT_REQUIRE(cube && cube->bands >= 1 && cube->bands <= kMaxBands, "ut_synth_cube: bands 1..32");
  UT_REQUIRE(classes >= 1 && classes <= kMaxClasses, "ut_synth_cube: classes 1..8");
  UT_REQUIRE(cube->row0 >= 0 && cube->row0 + cube->rows <= height, "ut_synth_cube: bad shard");
  Shapes sh;
  int rc = load_shapes(sh, shapes, nshapes);
  if (rc != UT_OK) return rc;
  if (cube->rows * cube->cols == 0) return UT_OK;
  cudaStream_t st = as_stream(stream);
  switch (cube->dtype) {
    case UT_U8: return launch_synth<uint8_t>(cube, means, chol, classes, sh, seed, st);
    case UT_U16: return launch_synth<uint16_t>(cube, means, chol, classes, sh, seed, st);
    case UT_F16: return launch_synth<__half>(cube, means, chol, classes, sh, seed, st);
    case UT_F32: return launch_synth<float>(cube, means, chol, classes, sh, seed, st);
    case UT_F64: return launch_synth<double>(cube, means, chol, classes, sh, seed, st);
  }
  set_error("ut_synth_cube: unknown dtype %d", cube->dtype);
  return UT_EDATA;
}

int ut_class_of(const int64_t* shapes, int32_t nshapes, const int32_t* xy, int64_t n, int32_t* cls,
                void* stream) {
  Shapes sh;
  int rc = load_shapes(sh, shapes, nshapes);
  if (rc != UT_OK) return rc;
  if (n <= 0) return UT_OK;
  class_of_kernel<<<(int)((n + 255) / 256), 256, 0, as_stream(stream)>>>(sh, xy, n, cls);
  UT_CHECK_LAUNCH("class_of_kernel");
  return UT_OK;
}

}  // extern "C"
