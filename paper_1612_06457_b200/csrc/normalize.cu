// normalize_stack (stack.py:180-213): per-band (or global) min/max of the raw
// cube, then every sample -> round_half_away(255 (v - lo) / (hi - lo)) as uint8.
//
// Two HBM passes (the min/max is a true dependency).  Pass 1: 2-D grid
// (blockIdx.y = band), grid-stride over the band's pixels, fp64 min/max and a
// NaN flag, folded per band with 64-bit atomics on an order-preserving integer
// image of the double (order-independent, hence deterministic).  Pass 2: the
// reference's arithmetic in fp64 -- d = v - lo, t = 255 d, x = t / (hi - lo),
// floor(x + 0.5) -- with the division done as t * (1 / (hi - lo)) unless
// x + 0.5 lies within 1e-9 of an integer, where the correctly rounded quotient
// (div.rn) is used: codes are bit-identical to numpy's.  A constant band gives
// zeros (+ a flag for the host's warning); a band holding NaN gives zeros.
#include "common.cuh"

namespace ut {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ unsigned long long order_key(double d) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(d);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_key(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

struct NormWs {
  unsigned long long* mn;  // [B] order keys
  unsigned long long* mx;  // [B]
  int* nan;                // [B]
};

size_t norm_ws_layout(NormWs* ws, void* base) {
  const size_t off_mn = 0, off_mx = 8 * kMaxBands, off_nan = 16 * kMaxBands;
  const size_t total = off_nan + 4 * kMaxBands;
  if (ws && base) {
    char* p = static_cast<char*>(base);
    ws->mn = reinterpret_cast<unsigned long long*>(p + off_mn);
    ws->mx = reinterpret_cast<unsigned long long*>(p + off_mx);
    ws->nan = reinterpret_cast<int*>(p + off_nan);
  }
  return total;
}

__global__ void norm_init_kernel(NormWs ws) {
  const int b = threadIdx.x;
  if (b < kMaxBands) {
    ws.mn[b] = ~0ull;
    ws.mx[b] = 0ull;
    ws.nan[b] = 0;
  }
}

// min/max in the sample's own arithmetic (integers / float; exact), NaN-aware
template <typename T> struct MinMax {
  using A = float;
  __device__ static A lo0() { return INFINITY; }
  __device__ static A hi0() { return -INFINITY; }
  __device__ static A of(T x) { return to_f32(x); }
  __device__ static bool nan(A a) { return a != a; }
  __device__ static A mn(A a, A b) { return fminf(a, b); }
  __device__ static A mx(A a, A b) { return fmaxf(a, b); }
};
template <> struct MinMax<uint8_t> {
  using A = unsigned;
  __device__ static A lo0() { return 0xffffffffu; }
  __device__ static A hi0() { return 0u; }
  __device__ static A of(uint8_t x) { return x; }
  __device__ static bool nan(A) { return false; }
  __device__ static A mn(A a, A b) { return min(a, b); }
  __device__ static A mx(A a, A b) { return max(a, b); }
};
template <> struct MinMax<uint16_t> : MinMax<uint8_t> {
  __device__ static A of(uint16_t x) { return x; }
};
template <> struct MinMax<double> {
  using A = double;
  __device__ static A lo0() { return INFINITY; }
  __device__ static A hi0() { return -INFINITY; }
  __device__ static A of(double x) { return x; }
  __device__ static bool nan(A a) { return a != a; }
  __device__ static A mn(A a, A b) { return fmin(a, b); }
  __device__ static A mx(A a, A b) { return fmax(a, b); }
};

template <typename T>
__global__ void __launch_bounds__(kThreads)
norm_minmax_kernel(ut_cube c, NormWs ws) {
  using M = MinMax<T>;
  using A = typename M::A;
  const int b = blockIdx.y;
  const T* base = static_cast<const T*>(c.data) + (int64_t)b * c.band_stride;
  const int64_t n = c.rows * c.cols;
  A mn = M::lo0(), mx = M::hi0();
  bool nan = false;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (c.row_stride == c.cols && (reinterpret_cast<uintptr_t>(base) % 16) == 0) {
    constexpr int V = 16 / sizeof(T);
    constexpr int U = 4;  // 4 independent 16-byte loads in flight per thread
    const int64_t nv = n / V;
    const int64_t nu = nv / U * U;
    for (int64_t i0 = tid; i0 < nu / U; i0 += stride) {
      T x[U][V];
#pragma unroll
      for (int u = 0; u < U; ++u)
        *reinterpret_cast<uint4*>(x[u]) = ld_stream_u4(base + V * (i0 + u * (nu / U)));
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < V; ++j) {
          const A a = M::of(x[u][j]);
          nan |= M::nan(a);
          mn = M::mn(mn, a);
          mx = M::mx(mx, a);
        }
    }
    for (int64_t i = nu + tid; i < nv; i += stride) {
      T x[V];
      *reinterpret_cast<uint4*>(x) = ld_stream_u4(base + V * i);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const A a = M::of(x[j]);
        nan |= M::nan(a);
        mn = M::mn(mn, a);
        mx = M::mx(mx, a);
      }
    }
    for (int64_t i = nv * V + tid; i < n; i += stride) {
      const A a = M::of(base[i]);
      nan |= M::nan(a);
      mn = M::mn(mn, a);
      mx = M::mx(mx, a);
    }
  } else {
    for (int64_t r = blockIdx.x; r < c.rows; r += gridDim.x)  // a block per row
      for (int64_t col = threadIdx.x; col < c.cols; col += blockDim.x) {
        const A a = M::of(base[r * c.row_stride + col]);
        nan |= M::nan(a);
        mn = M::mn(mn, a);
        mx = M::mx(mx, a);
      }
  }
  double dmn = (double)mn, dmx = (double)mx;
  if (!(mn <= mx)) { dmn = INFINITY; dmx = -INFINITY; }  // nothing seen (or only NaN)
  for (int o = 16; o > 0; o >>= 1) {
    dmn = fmin(dmn, __shfl_xor_sync(0xffffffffu, dmn, o));
    dmx = fmax(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
  }
  nan = __any_sync(0xffffffffu, nan);
  if ((threadIdx.x & 31) == 0) {
    if (dmn <= dmx) {
      atomicMin(&ws.mn[b], order_key(dmn));
      atomicMax(&ws.mx[b], order_key(dmx));
    }
    if (nan) atomicOr(&ws.nan[b], 1);
  }
}

// lohi[2b], lohi[2b+1]: the band's (or, global scope, the cube's) min and max;
// NaN if the band (cube) holds a NaN, as numpy's min/max.  flags[b] = 1 when
// the band maps to zeros because lo == hi (the reference warns).
__global__ void norm_finish_kernel(NormWs ws, int bands, int global, double* lohi, int32_t* flags) {
  const int b = threadIdx.x;
  if (b >= bands) return;
  unsigned long long kmn = ws.mn[b], kmx = ws.mx[b];
  int nan = ws.nan[b];
  if (global) {
    for (int j = 0; j < bands; ++j) {
      kmn = min(kmn, ws.mn[j]);
      kmx = max(kmx, ws.mx[j]);
      nan |= ws.nan[j];
    }
  }
  const double lo = nan ? __longlong_as_double(0x7ff8000000000000ll) : from_key(kmn);
  const double hi = nan ? lo : from_key(kmx);
  lohi[2 * b] = lo;
  lohi[2 * b + 1] = hi;
  flags[b] = (lo == hi) ? 1 : 0;
}

__device__ __forceinline__ uint8_t norm_code(double v, double lo, double den, double rden) {
  const double t = __dmul_rn(255.0, __dadd_rn(v, -lo));
  double x = __dmul_rn(t, rden);
  double y = __dadd_rn(x, 0.5);
  const double f = y - floor(y);
  if (f < 1e-9 || f > 1.0 - 1e-9) {  // near a rounding boundary: the exact quotient
    x = __ddiv_rn(t, den);
    y = __dadd_rn(x, 0.5);
  }
  const double code = floor(y);
  // NaN (a NaN band) -> 0, like numpy's cast on x86; the range is [0, 255]
  return (code >= 0.0 && code <= 255.0) ? (uint8_t)(int)code : (uint8_t)0;
}

// exact widening: the ALU bit trick for normal floats (F2F is quarter rate),
// the conversion instruction for zeros / subnormals (rare: a branch)
template <typename T>
__device__ __forceinline__ double norm_in(T x) { return to_f64(x); }
template <> __device__ __forceinline__ double norm_in<float>(float x) {
  if ((__float_as_uint(x) & 0x7f800000u) == 0u) return (double)x;
  return widen_f64(x);
}
template <> __device__ __forceinline__ double norm_in<__half>(__half x) {
  return norm_in<float>(__half2float(x));
}

// 8/16-bit samples: the code depends on the sample value only -> a per-block
// table over [lo, hi] in shared memory, built with the exact arithmetic, then
// one table lookup per sample.
template <typename T>
__global__ void __launch_bounds__(kThreads)
norm_codes_lut_kernel(ut_cube c, const double* __restrict__ lohi, uint8_t* __restrict__ out) {
  extern __shared__ uint8_t lut[];
  const int b = blockIdx.y;
  const double lo = lohi[2 * b], hi = lohi[2 * b + 1];
  const T* base = static_cast<const T*>(c.data) + (int64_t)b * c.band_stride;
  const int64_t n = c.rows * c.cols;
  uint8_t* o = out + (int64_t)b * n;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (!(lo < hi)) {  // constant band -> zeros
    for (int64_t i = tid; i < n; i += stride) o[i] = 0;
    return;
  }
  const int ilo = (int)lo, range = (int)hi - ilo + 1;
  const double den = __dadd_rn(hi, -lo), rden = __drcp_rn(den);
  for (int j = threadIdx.x; j < range; j += blockDim.x) lut[j] = norm_code((double)(ilo + j), lo, den, rden);
  __syncthreads();
  if (c.row_stride == c.cols && (reinterpret_cast<uintptr_t>(base) % 16) == 0 &&
      (reinterpret_cast<uintptr_t>(o) % 16) == 0) {
    constexpr int V = 16 / sizeof(T);  // samples per 16-byte load
    const int64_t nv = n / 16;
    for (int64_t i = tid; i < nv; i += stride) {
      T x[16];
#pragma unroll
      for (int q = 0; q < 16 / V; ++q) *reinterpret_cast<uint4*>(x + q * V) = ld_stream_u4(base + 16 * i + q * V);
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        w[q] = (uint32_t)lut[(int)x[4 * q] - ilo] | ((uint32_t)lut[(int)x[4 * q + 1] - ilo] << 8) |
               ((uint32_t)lut[(int)x[4 * q + 2] - ilo] << 16) | ((uint32_t)lut[(int)x[4 * q + 3] - ilo] << 24);
      st_stream_u4(o + 16 * i, make_uint4(w[0], w[1], w[2], w[3]));
    }
    for (int64_t i = nv * 16 + tid; i < n; i += stride) o[i] = lut[(int)base[i] - ilo];
    return;
  }
  for (int64_t r = blockIdx.x; r < c.rows; r += gridDim.x)
    for (int64_t col = threadIdx.x; col < c.cols; col += blockDim.x)
      o[r * c.cols + col] = lut[(int)base[r * c.row_stride + col] - ilo];
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
norm_codes_kernel(ut_cube c, const double* __restrict__ lohi, uint8_t* __restrict__ out) {
  const int b = blockIdx.y;
  const double lo = lohi[2 * b], hi = lohi[2 * b + 1];
  const T* base = static_cast<const T*>(c.data) + (int64_t)b * c.band_stride;
  const int64_t n = c.rows * c.cols;
  uint8_t* o = out + (int64_t)b * n;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (!(lo != hi)) {  // constant band: zeros (NaN bands fall through: codes 0 below)
    for (int64_t i = tid; i < n; i += stride) o[i] = 0;
    return;
  }
  const double den = __dadd_rn(hi, -lo);
  const double rden = __drcp_rn(den);
  if (c.row_stride == c.cols && (reinterpret_cast<uintptr_t>(base) % 16) == 0 &&
      (reinterpret_cast<uintptr_t>(o) % 16) == 0) {
    // contiguous band: 16 samples per thread-iteration, one 16-byte store
    constexpr int V = 16 / sizeof(T);
    const int64_t nv = n / 16;
    for (int64_t i = tid; i < nv; i += stride) {
      T x[16];
#pragma unroll
      for (int q = 0; q < 16 / V; ++q)
        *reinterpret_cast<uint4*>(x + q * V) = ld_stream_u4(base + 16 * i + q * V);
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t acc = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) acc |= (uint32_t)norm_code(norm_in(x[4 * q + j]), lo, den, rden) << (8 * j);
        w[q] = acc;
      }
      st_stream_u4(o + 16 * i, make_uint4(w[0], w[1], w[2], w[3]));
    }
    for (int64_t i = nv * 16 + tid; i < n; i += stride) o[i] = norm_code(to_f64(base[i]), lo, den, rden);
    return;
  }
  for (int64_t r = blockIdx.x; r < c.rows; r += gridDim.x)
    for (int64_t col = threadIdx.x; col < c.cols; col += blockDim.x)
      o[r * c.cols + col] = norm_code(to_f64(base[r * c.row_stride + col]), lo, den, rden);
}

template <typename T>
int launch_norm(const ut_cube& c, int global, uint8_t* out, double* lohi, int32_t* flags,
                NormWs ws, cudaStream_t st) {
  const int64_t n = c.rows * c.cols;
  int64_t gx = (n + kThreads - 1) / kThreads;
  const int64_t cap = (int64_t)sm_count() * 8 / (c.bands > 0 ? c.bands : 1) + 1;
  if (gx > cap) gx = cap;
  if (gx < 1) gx = 1;
  norm_init_kernel<<<1, kMaxBands, 0, st>>>(ws);
  UT_CHECK_LAUNCH("norm_init_kernel");
  norm_minmax_kernel<T><<<dim3((unsigned)(c.row_stride == c.cols ? gx : (c.rows < cap ? c.rows : cap)), c.bands),
                          kThreads, 0, st>>>(c, ws);
  UT_CHECK_LAUNCH("norm_minmax_kernel");
  norm_finish_kernel<<<1, kMaxBands, 0, st>>>(ws, c.bands, global, lohi, flags);
  UT_CHECK_LAUNCH("norm_finish_kernel");
  int64_t gx2 = (n / 16 + kThreads - 1) / kThreads;
  if (gx2 > cap) gx2 = cap;
  if (gx2 < 1) gx2 = 1;
  if constexpr (sizeof(T) <= 2 && Sample<T>::integral) {
    constexpr int lut_bytes = 1 << (8 * sizeof(T));
    if (lut_bytes > 48 * 1024) {
      static SmemAttr attr;
      if (int rc = ensure_smem(attr, norm_codes_lut_kernel<T>, (size_t)lut_bytes,
                               "norm_codes_lut smem attribute"))
        return rc;
    }
    norm_codes_lut_kernel<T><<<dim3((unsigned)gx2, c.bands), kThreads, lut_bytes, st>>>(c, lohi, out);
    UT_CHECK_LAUNCH("norm_codes_lut_kernel");
  } else {
    norm_codes_kernel<T><<<dim3((unsigned)gx2, c.bands), kThreads, 0, st>>>(c, lohi, out);
    UT_CHECK_LAUNCH("norm_codes_kernel");
  }
  return UT_OK;
}

}  // namespace
}  // namespace ut

using namespace ut;

extern "C" {

size_t ut_normalize_ws(void) { return norm_ws_layout(nullptr, nullptr); }

int ut_normalize_stack(const ut_cube* cube, int32_t scope, void* out, double* lohi,
                       int32_t* constant, void* ws_base, size_t ws_bytes, void* stream) {
  UT_REQUIRE(cube && cube->bands >= 1 && cube->bands <= kMaxBands,
             "ut_normalize_stack: bands must be 1..32");
  UT_REQUIRE(scope == 0 || scope == 1, "unknown normalization scope %d", scope);
  UT_REQUIRE(cube->rows >= 1 && cube->cols >= 1, "ut_normalize_stack: empty stack");
  NormWs ws;
  const size_t need = norm_ws_layout(&ws, ws_base);
  UT_REQUIRE(ws_bytes >= need, "ut_normalize_stack: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t st = as_stream(stream);
  uint8_t* o = static_cast<uint8_t*>(out);
  switch (cube->dtype) {
    case UT_U8: return launch_norm<uint8_t>(*cube, scope, o, lohi, constant, ws, st);
    case UT_U16: return launch_norm<uint16_t>(*cube, scope, o, lohi, constant, ws, st);
    case UT_F16: return launch_norm<__half>(*cube, scope, o, lohi, constant, ws, st);
    case UT_F32: return launch_norm<float>(*cube, scope, o, lohi, constant, ws, st);
    case UT_F64: return launch_norm<double>(*cube, scope, o, lohi, constant, ws, st);
  }
  set_error("ut_normalize_stack: unknown dtype %d", cube->dtype);
  return UT_EDATA;
}

}  // extern "C"
