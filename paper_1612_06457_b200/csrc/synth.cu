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

// Every floating-point step below is one IEEE-754 binary32 operation with
// round-to-nearest (explicit __f*_rn intrinsics, so nvcc cannot contract a
// multiply-add into an FMA), and the transcendental steps are written out as
// fixed polynomials.  oracle/synth.py restates the generator with numpy
// float32 arithmetic in the same order, so host and device produce the same
// bits for every sample (tests/test_gpu_synth.py) -- the reference arm of
// bench.py builds its sample rows on the host without this library.
#define FADD __fadd_rn
#define FMUL __fmul_rn

// Constants are binary32 values written as hex literals (oracle/synth.py uses
// the same bit patterns).
// ln(u) for u in (0, 1]: u = m 2^e with m in [sqrt(1/2), sqrt(2)),
// ln m = 2 atanh(s) = 2s + s s^2 (2/3 + s^2 (2/5 + s^2 (2/7 + s^2 2/9))),
// s = (m - 1) / (m + 1).
__device__ __forceinline__ float synth_log(float u) {
  const int bits = __float_as_int(u);
  int e = ((bits >> 23) & 0xff) - 126;
  float m = __int_as_float((bits & 0x007fffff) | (126 << 23));  // [0.5, 1)
  if (m < 0x1.6a09e6p-1f) {                                      // sqrt(1/2)
    m = FMUL(m, 2.0f);
    e -= 1;
  }
  const float f = FADD(m, -1.0f);
  const float s = __fdiv_rn(f, FADD(f, 2.0f));
  const float s2 = FMUL(s, s);
  float p = 0x1.c71c72p-3f;                    // 2/9
  p = FADD(0x1.24924ap-2f, FMUL(s2, p));       // 2/7
  p = FADD(0x1.99999ap-2f, FMUL(s2, p));       // 2/5
  p = FADD(0x1.555556p-1f, FMUL(s2, p));       // 2/3
  const float lnm = FADD(FMUL(2.0f, s), FMUL(s, FMUL(s2, p)));
  return FADD(FMUL((float)e, 0x1.62e43p-1f), lnm);  // e ln 2 + ln m
}

// sin and cos of x = a pi/2 for a in [0, 1): Taylor polynomials in x^2
// (degree 13 / 14; truncation < 1e-9).
__device__ __forceinline__ void synth_sincos_q(float a, float* s, float* c) {
  const float x = FMUL(a, 0x1.921fb6p+0f);     // pi/2
  const float x2 = FMUL(x, x);
  float ps = -0x1.612462p-33f;                 // -1/13!
  ps = FADD(0x1.ae6456p-26f, FMUL(x2, ps));    //  1/11!
  ps = FADD(-0x1.71de3ap-19f, FMUL(x2, ps));   // -1/9!
  ps = FADD(0x1.a01a02p-13f, FMUL(x2, ps));    //  1/7!
  ps = FADD(-0x1.111112p-7f, FMUL(x2, ps));    // -1/5!
  ps = FADD(0x1.555556p-3f, FMUL(x2, ps));     //  1/3!
  *s = FADD(x, -FMUL(x, FMUL(x2, ps)));
  float pc = -0x1.93974ap-37f;                 // -1/14!
  pc = FADD(0x1.1eed8ep-29f, FMUL(x2, pc));    //  1/12!
  pc = FADD(-0x1.27e4fcp-22f, FMUL(x2, pc));   // -1/10!
  pc = FADD(0x1.a01a02p-16f, FMUL(x2, pc));    //  1/8!
  pc = FADD(-0x1.6c16c2p-10f, FMUL(x2, pc));   // -1/6!
  pc = FADD(0x1.555556p-5f, FMUL(x2, pc));     //  1/4!
  pc = FADD(-0.5f, FMUL(x2, pc));              // -1/2!
  *c = FADD(1.0f, FMUL(x2, pc));
}

// Two standard normals from one 64-bit hash (Box-Muller): u1 = (2k+1) 2^-24
// from the top 23 bits, u2 = j 2^-24 from the low 24 bits (exact in binary32).
__device__ __forceinline__ void synth_normal_pair(uint64_t h, float* z0, float* z1) {
  const float u1 = FMUL((float)(uint32_t)(2u * (uint32_t)(h >> 41) + 1u), 0x1p-24f);
  const float u2 = FMUL((float)(uint32_t)(h & 0xffffffu), 0x1p-24f);
  const float r = __fsqrt_rn(FMUL(-2.0f, synth_log(u1)));
  const float t = FMUL(u2, 4.0f);
  const float q = floorf(t);
  float s, c;
  synth_sincos_q(FADD(t, -q), &s, &c);
  float sn, cs;
  switch ((int)q & 3) {
    case 0: sn = s; cs = c; break;
    case 1: sn = c; cs = -s; break;
    case 2: sn = -s; cs = -c; break;
    default: sn = -c; cs = s; break;
  }
  *z0 = FMUL(r, cs);
  *z1 = FMUL(r, sn);
}

template <typename T> __device__ __forceinline__ T cast_sample(float v);
template <> __device__ __forceinline__ float cast_sample<float>(float v) { return v; }
template <> __device__ __forceinline__ double cast_sample<double>(float v) { return (double)v; }
template <> __device__ __forceinline__ __half cast_sample<__half>(float v) { return __float2half_rn(v); }
template <> __device__ __forceinline__ uint16_t cast_sample<uint16_t>(float v) {
  return (uint16_t)floorf(FADD(FMUL(4095.0f, v), 0.5f));  // round_half_away, v >= 0
}
template <> __device__ __forceinline__ uint8_t cast_sample<uint8_t>(float v) {
  return (uint8_t)floorf(FADD(FMUL(255.0f, v), 0.5f));
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
    for (int b = 0; b < kMaxBands; b += 2)
      synth_normal_pair(splitmix64(seed ^ (gpix * 0x100000001B3ull + (uint64_t)b)), &z[b],
                        &z[b + 1]);
    T* dst = out + y * rs + x;
    for (int b = 0; b < bands; ++b) {
      float v = mu[c][b];
#pragma unroll
      for (int q = 0; q < kMaxBands; ++q)
        if (q <= b) v = FADD(v, FMUL(L[c][b][q], z[q]));
      v = fminf(fmaxf(v, 0.0f), 1.0f);
      dst[b * bs] = cast_sample<T>(v);
    }
  }
}

#undef FADD
#undef FMUL

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
