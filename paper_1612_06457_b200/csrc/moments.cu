// K1: training-pixel gather and per-class moments.
//
// Replaces annotations.assemble_matrix's Python point loop
// (annotations.py:195-215) and compute_scatter's per-class reductions
// (projection.py:187-198).
//
// One pass.  The n points are split into G <= 128 contiguous ranges (G is a
// function of n only, so results do not depend on the GPU).  CTA g stages 128
// points at a time in shared memory -- gathered straight from the cube (fused
// pipeline) or read from a B x n design matrix -- as deviations from a local
// pivot (the first point of each class in its range), with a constant-1 row
// appended, and accumulates the upper triangle of [d;1][d;1]^T per class:
// that one Gram holds the count, the shifted sums and the shifted scatter.
// Each CTA turns its Gram into (count, mean, centred M2) per class; a second
// kernel (one CTA per class) merges the G records in fixed order with the
// parallel-axis rule.  Centring on a pivot keeps the one-pass form as exact as
// the reference's two-pass form; every reduction order is fixed, so the
// result is bit-identical run to run.
#include "common.cuh"

namespace ut {
namespace {

constexpr int kChunk = 128;      // points staged per step
constexpr int kThreads = 256;
constexpr int kMaxG = 128;       // point ranges (CTAs)
constexpr int kMinPerCta = 64;
constexpr int kMaxClasses = 16;  // per launch; more classes -> several launches
constexpr int kRows = kMaxBands + 1;                    // bands + ones row
constexpr int kMaxEnt = kRows * (kRows + 1) / 2;        // 561
constexpr int kTileLd = kChunk + 1;

__host__ __device__ inline int ent_count(int b) { return (b + 1) * (b + 2) / 2; }

// ------------------------------------------------------------------ gather
template <typename T>
__global__ void gather_kernel(const T* __restrict__ data, int64_t bs, int64_t rs,
                              int64_t rows, int64_t cols, int64_t row0, int bands,
                              const int32_t* __restrict__ xy, int64_t n,
                              double* __restrict__ values, int64_t ld,
                              unsigned long long* first_bad) {
  const int64_t total = n * bands;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(e / n);
    const int64_t j = e - (int64_t)b * n;
    const int64_t x = xy[2 * j], y = xy[2 * j + 1] - row0;
    if (x < 0 || x >= cols || y < 0 || y >= rows) {
      if (b == 0) atomicMin(first_bad, (unsigned long long)j);
      values[b * ld + j] = 0.0;
      continue;
    }
    values[b * ld + j] = to_f64(data[b * bs + y * rs + x]);
  }
}

// ------------------------------------------------------------------ sources
struct MatrixSrc {
  const double* values;
  int64_t ld;
  __device__ __forceinline__ bool valid(int64_t) const { return true; }
  __device__ __forceinline__ double at(int b, int64_t j) const { return values[b * ld + j]; }
};

template <typename T>
struct CubeSrc {
  const T* data;
  int64_t bs, rs, rows, cols, row0;
  const int32_t* xy;
  __device__ __forceinline__ bool valid(int64_t j) const {
    const int64_t x = xy[2 * j], y = xy[2 * j + 1] - row0;
    return x >= 0 && x < cols && y >= 0 && y < rows;
  }
  __device__ __forceinline__ double at(int b, int64_t j) const {
    const int64_t x = xy[2 * j], y = xy[2 * j + 1] - row0;
    return to_f64(data[b * bs + y * rs + x]);
  }
};

struct Layout {
  int64_t n;
  int bands, classes, c0;   // classes [c0, c0 + classes) handled by this launch
  int G;                    // ranges
  int64_t span;             // points per range (multiple of kChunk)
};

// per-CTA records: [c][f][g] with f in [0, 1 + B + B*B): n, mean, M2 (row-major)
__host__ __device__ inline int rec_len(int b) { return 1 + b + b * b; }

struct Smem {
  double tile[kRows * kTileLd];
  double acc[kMaxClasses * kMaxEnt];
  double pivot[kMaxClasses * kMaxBands];
  int lbl[kChunk];
  int piv_idx[kMaxClasses];
  unsigned char pi[kMaxEnt], pj[kMaxEnt];
};

template <typename Src>
__global__ void __launch_bounds__(kThreads)
moments_kernel(Src src, const int32_t* __restrict__ cls, Layout L, double* __restrict__ part,
               unsigned long long* first_bad) {
  extern __shared__ __align__(16) unsigned char raw[];
  Smem& s = *reinterpret_cast<Smem*>(raw);
  const int tid = threadIdx.x;
  const int B = L.bands, C = L.classes;
  const int R = B + 1;
  const int E = ent_count(B);
  const int64_t j0 = (int64_t)blockIdx.x * L.span;
  const int64_t j1 = j0 + L.span < L.n ? j0 + L.span : L.n;
  for (int i = tid; i < R; i += blockDim.x) {
    const int base = i * R - i * (i - 1) / 2;
    for (int j = i; j < R; ++j) {
      s.pi[base + j - i] = (unsigned char)i;
      s.pj[base + j - i] = (unsigned char)j;
    }
  }
  for (int e = tid; e < C * E; e += blockDim.x) s.acc[e] = 0.0;
  if (tid < C) s.piv_idx[tid] = 0x7fffffff;
  __syncthreads();
  // local pivots: first point of each class in [j0, j1)
  for (int64_t j = j0 + tid; j < j1; j += blockDim.x) {
    const int c = cls[j] - L.c0;
    if (c >= 0 && c < C && src.valid(j)) atomicMin(&s.piv_idx[c], (int)(j - j0));
  }
  __syncthreads();
  for (int e = tid; e < C * B; e += blockDim.x) {
    const int c = e / B, b = e - c * B;
    const int pj = s.piv_idx[c];
    s.pivot[e] = (pj != 0x7fffffff) ? src.at(b, j0 + pj) : 0.0;
  }
  __syncthreads();
  for (int64_t q0 = j0; q0 < j1; q0 += kChunk) {
    // stage deviations from the class pivot; row B is the constant 1
    for (int p = tid; p < kChunk; p += blockDim.x) {
      const int64_t j = q0 + p;
      int c = -1;
      if (j < j1) {
        c = cls[j] - L.c0;
        if (c < 0 || c >= C) c = -1;
        if (!src.valid(j)) {
          if (first_bad) atomicMin(first_bad, (unsigned long long)j);
          c = -1;
        }
      }
      s.lbl[p] = c;
      s.tile[B * kTileLd + p] = (c >= 0) ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < B * kChunk; e += blockDim.x) {
      const int b = e / kChunk, p = e - b * kChunk;
      const int c = s.lbl[p];
      s.tile[b * kTileLd + p] = (c >= 0) ? src.at(b, q0 + p) - s.pivot[c * B + b] : 0.0;
    }
    __syncthreads();
    // Gram entries, one class run at a time (points are usually class-sorted)
    for (int e = tid; e < E; e += blockDim.x) {
      const double* ri = s.tile + s.pi[e] * kTileLd;
      const double* rj = s.tile + s.pj[e] * kTileLd;
      int cur = -1;
      double a = 0.0;
      for (int p = 0; p < kChunk; ++p) {
        const int c = s.lbl[p];
        if (c < 0) continue;
        if (c != cur) {
          if (cur >= 0) s.acc[cur * E + e] = a;
          cur = c;
          a = s.acc[c * E + e];
        }
        a = fma(ri[p], rj[p], a);
      }
      if (cur >= 0) s.acc[cur * E + e] = a;
    }
    __syncthreads();
  }
  // (count, mean, M2) of this range per class, written as [c][f][g]
  const int len = rec_len(B);
  const int G = L.G;
  for (int e = tid; e < C * len; e += blockDim.x) {
    const int c = e / len, f = e - c * len;
    const double* A = s.acc + c * E;
    const int one = B;  // row of ones
    auto ent = [&](int i, int j) {  // i <= j
      return A[i * R - i * (i - 1) / 2 + (j - i)];
    };
    const double n = ent(one, one);
    double v = 0.0;
    if (n > 0.0) {
      if (f == 0) {
        v = n;
      } else if (f <= B) {
        const int b = f - 1;
        v = s.pivot[c * B + b] + ent(b, one) / n;
      } else {
        const int q = f - 1 - B, i = q / B, j = q - i * B;
        const int lo = i < j ? i : j, hi = i < j ? j : i;
        v = ent(lo, hi) - ent(i, one) * ent(j, one) / n;
      }
    }
    part[((size_t)c * len + f) * G + blockIdx.x] = v;
  }
}

// One CTA per class: merge the G range records in fixed order.
__global__ void __launch_bounds__(1024)
merge_kernel(const double* __restrict__ part, Layout L, double* __restrict__ moments) {
  __shared__ double mean[kMaxBands];
  __shared__ double cnt;
  const int c = blockIdx.x;
  const int B = L.bands, G = L.G;
  const int len = rec_len(B);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double* P = part + (size_t)c * len * G;
  const double* Pn = P;  // f = 0 row: counts per range
  // counts and means (warp per field, lanes over ranges, fixed shuffle tree)
  for (int f = warp; f <= B; f += nw) {
    double acc = 0.0;
    for (int g = lane; g < G; g += 32) {
      const double n = Pn[g];
      acc += (f == 0) ? n : (n > 0.0 ? n * P[(size_t)f * G + g] : 0.0);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      if (f == 0) cnt = acc;
      else mean[f - 1] = acc;
    }
  }
  __syncthreads();
  const double n = cnt;
  if (threadIdx.x < B) mean[threadIdx.x] = n > 0.0 ? mean[threadIdx.x] / n : 0.0;
  __syncthreads();
  double* out = moments + (size_t)(L.c0 + c) * len;
  if (threadIdx.x == 0) out[0] = n;
  if (threadIdx.x < B) out[1 + threadIdx.x] = mean[threadIdx.x];
  if (G == 1) {
    for (int q = threadIdx.x; q < B * B; q += blockDim.x) out[1 + B + q] = P[(size_t)(1 + B + q)];
    return;
  }
  // M2 = sum_g [M2_g + n_g (m_g - m)(m_g - m)^T], two entries per warp step
  for (int q0 = warp * 2; q0 < B * B; q0 += nw * 2) {
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int q = q0 + u;
      if (q >= B * B) break;
      const int i = q / B, j = q - i * B;
      for (int g = lane; g < G; g += 32) {
        const double ng = Pn[g];
        if (ng > 0.0) {
          const double di = P[(size_t)(1 + i) * G + g] - mean[i];
          const double dj = P[(size_t)(1 + j) * G + g] - mean[j];
          acc[u] += P[(size_t)(1 + B + q) * G + g] + ng * (di * dj);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
      for (int o = 16; o > 0; o >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
    if (lane == 0) {
      out[1 + B + q0] = acc[0];
      if (q0 + 1 < B * B) out[1 + B + q0 + 1] = acc[1];
    }
  }
}

Layout make_layout(int64_t n, int b, int c) {
  Layout L{};
  L.n = n;
  L.bands = b;
  L.classes = c;
  int64_t G = (n + kMinPerCta - 1) / kMinPerCta;
  if (G > kMaxG) G = kMaxG;
  if (G < 1) G = 1;
  int64_t span = (n + G - 1) / G;
  span = ((span + kChunk - 1) / kChunk) * kChunk;
  L.span = span;
  L.G = (int)((n + span - 1) / span);
  if (L.G < 1) L.G = 1;
  return L;
}

size_t ws_bytes_for(int b, int c) {
  const int per = c < kMaxClasses ? c : kMaxClasses;
  return sizeof(double) * (size_t)per * rec_len(b) * kMaxG + 256;
}

bool g_smem_set[64] = {false};

template <typename Src>
int launch_moments(const Src& src, const int32_t* cls, int64_t n, int b, int classes,
                   double* moments, void* ws, size_t ws_bytes, unsigned long long* first_bad,
                   cudaStream_t st) {
  UT_REQUIRE(ws_bytes >= ws_bytes_for(b, classes), "class moments: workspace %zu < %zu",
             ws_bytes, ws_bytes_for(b, classes));
  const int bytes = (int)sizeof(Smem);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(moments_kernel<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    attr = true;
  }
  double* part = static_cast<double*>(ws);
  for (int c0 = 0; c0 < classes; c0 += kMaxClasses) {
    Layout L = make_layout(n, b, classes - c0 < kMaxClasses ? classes - c0 : kMaxClasses);
    L.c0 = c0;
    moments_kernel<Src><<<L.G, kThreads, bytes, st>>>(src, cls, L, part, first_bad);
    UT_CHECK_LAUNCH("moments_kernel");
    merge_kernel<<<L.classes, 1024, 0, st>>>(part, L, moments);
    UT_CHECK_LAUNCH("merge_kernel");
  }
  return UT_OK;
}

template <typename T>
int launch_gather(const ut_cube* cube, const int32_t* xy, int64_t n, double* values,
                  int64_t ld, unsigned long long* first_bad, cudaStream_t s) {
  const int64_t total = n * cube->bands;
  int grid = (int)((total + 255) / 256);
  if (grid > 8 * sm_count()) grid = 8 * sm_count();
  if (grid < 1) grid = 1;
  gather_kernel<T><<<grid, 256, 0, s>>>(
      static_cast<const T*>(cube->data), cube->band_stride, cube->row_stride, cube->rows,
      cube->cols, cube->row0, cube->bands, xy, n, values, ld, first_bad);
  UT_CHECK_LAUNCH("ut_gather");
  return UT_OK;
}

template <typename T>
int launch_cube_moments(const ut_cube* cube, const int32_t* xy, const int32_t* cls, int64_t n,
                        int classes, double* moments, unsigned long long* first_bad, void* ws,
                        size_t ws_bytes, cudaStream_t st) {
  CubeSrc<T> src{static_cast<const T*>(cube->data), cube->band_stride, cube->row_stride,
                 cube->rows, cube->cols, cube->row0, xy};
  return launch_moments(src, cls, n, cube->bands, classes, moments, ws, ws_bytes, first_bad, st);
}

}  // namespace
}  // namespace ut

using namespace ut;

extern "C" {

int ut_gather(const ut_cube* cube, const int32_t* xy, int64_t n, double* values, int64_t ld,
              int64_t* first_bad, void* stream) {
  UT_REQUIRE(cube && cube->bands >= 1 && cube->bands <= kMaxBands, "ut_gather: bands must be 1..32");
  UT_REQUIRE(n >= 0 && ld >= n, "ut_gather: bad n/ld");
  cudaStream_t s = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(first_bad, 0xFF, sizeof(int64_t), s);
  if (e != cudaSuccess) return cuda_status(e, "ut_gather memset");
  if (n == 0) return UT_OK;
  auto* fb = reinterpret_cast<unsigned long long*>(first_bad);
  switch (cube->dtype) {
    case UT_U8: return launch_gather<uint8_t>(cube, xy, n, values, ld, fb, s);
    case UT_U16: return launch_gather<uint16_t>(cube, xy, n, values, ld, fb, s);
    case UT_F16: return launch_gather<__half>(cube, xy, n, values, ld, fb, s);
    case UT_F32: return launch_gather<float>(cube, xy, n, values, ld, fb, s);
    case UT_F64: return launch_gather<double>(cube, xy, n, values, ld, fb, s);
  }
  set_error("ut_gather: unknown dtype %d", cube->dtype);
  return UT_EDATA;
}

size_t ut_class_moments_ws(int64_t n, int32_t bands, int32_t classes) {
  (void)n;
  return ws_bytes_for(bands, classes);
}

int ut_class_moments(const double* values, int64_t ld, const int32_t* cls, int64_t n,
                     int32_t bands, int32_t classes, double* moments, void* ws, size_t ws_bytes,
                     void* stream) {
  UT_REQUIRE(bands >= 1 && bands <= kMaxBands, "ut_class_moments: bands must be 1..32");
  UT_REQUIRE(classes >= 1, "ut_class_moments: classes must be >= 1");
  UT_REQUIRE(n >= 1, "ut_class_moments: no points");
  MatrixSrc src{values, ld};
  return launch_moments(src, cls, n, bands, classes, moments, ws, ws_bytes, nullptr,
                        as_stream(stream));
}

int ut_cube_class_moments(const ut_cube* cube, const int32_t* xy, const int32_t* cls, int64_t n,
                          int32_t classes, double* moments, int64_t* first_bad, void* ws,
                          size_t ws_bytes, void* stream) {
  UT_REQUIRE(cube && cube->bands >= 1 && cube->bands <= kMaxBands,
             "ut_cube_class_moments: bands must be 1..32");
  UT_REQUIRE(classes >= 1 && n >= 1, "ut_cube_class_moments: bad classes/points");
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(first_bad, 0xFF, sizeof(int64_t), st);
  if (e != cudaSuccess) return cuda_status(e, "ut_cube_class_moments memset");
  auto* fb = reinterpret_cast<unsigned long long*>(first_bad);
  switch (cube->dtype) {
    case UT_U8: return launch_cube_moments<uint8_t>(cube, xy, cls, n, classes, moments, fb, ws, ws_bytes, st);
    case UT_U16: return launch_cube_moments<uint16_t>(cube, xy, cls, n, classes, moments, fb, ws, ws_bytes, st);
    case UT_F16: return launch_cube_moments<__half>(cube, xy, cls, n, classes, moments, fb, ws, ws_bytes, st);
    case UT_F32: return launch_cube_moments<float>(cube, xy, cls, n, classes, moments, fb, ws, ws_bytes, st);
    case UT_F64: return launch_cube_moments<double>(cube, xy, cls, n, classes, moments, fb, ws, ws_bytes, st);
  }
  set_error("ut_cube_class_moments: unknown dtype %d", cube->dtype);
  return UT_EDATA;
}

}  // extern "C"
