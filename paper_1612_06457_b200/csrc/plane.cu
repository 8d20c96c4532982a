// Single-plane full-range rescale: min/max reduction and linear_to_codes for
// an arbitrary float32/float64 score plane (the host ScorePlane path of
// rescale_full, rendering.py:124-130, quantize.py:36-46).  The fused pipeline
// gets its min/max from the projector (project.cu) instead.
#include "common.cuh"

namespace ut {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxGrid = 2048;

template <typename T>
__global__ void __launch_bounds__(kThreads)
minmax_kernel(const T* __restrict__ v, int64_t n, double* part, unsigned int* counter,
              double* lohi, int32_t* nonfinite) {
  __shared__ double smn[kThreads / 32], smx[kThreads / 32], sck[kThreads / 32];
  double mn = INFINITY, mx = -INFINITY, chk = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = (double)v[i];
    mn = fmin(mn, x);
    mx = fmax(mx, x);
    chk = fma(0.0, x, chk);  // NaN iff some x is NaN or Inf
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    chk += __shfl_xor_sync(0xffffffffu, chk, o);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { smn[warp] = mn; smx[warp] = mx; sck[warp] = chk; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kThreads / 32; ++w) {
      smn[0] = fmin(smn[0], smn[w]);
      smx[0] = fmax(smx[0], smx[w]);
      sck[0] += sck[w];
    }
    part[3 * blockIdx.x] = smn[0];
    part[3 * blockIdx.x + 1] = smx[0];
    part[3 * blockIdx.x + 2] = sck[0];
  }
  if (last_block_ticket(counter) && threadIdx.x == 0) {
    double a = part[0], b = part[1], c = part[2];
    for (unsigned int g = 1; g < gridDim.x; ++g) {
      a = fmin(a, part[3 * g]);
      b = fmax(b, part[3 * g + 1]);
      c += part[3 * g + 2];
    }
    lohi[0] = a;
    lohi[1] = b;
    *nonfinite = (c != 0.0) ? 1 : 0;
    *counter = 0u;
  }
}

template <typename T, typename Code>
__global__ void __launch_bounds__(kThreads)
codes_kernel(const T* __restrict__ v, int64_t n, const double* __restrict__ lohi, double top,
             Code* __restrict__ out) {
  const double lo = lohi[0], hi = lohi[1];
  const bool flat = !(lo < hi);
  const double sc = flat ? 0.0 : top / (hi - lo);
  auto code = [&](double x) -> Code {
    if (flat) return (Code)0;
    x = fmin(fmax(__dmul_rn(__dadd_rn(x, -lo), sc), 0.0), top);
    return (Code)(int)floor(x + 0.5);
  };
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // 4 values per thread and iteration where aligned: one wide load, one store
  if ((reinterpret_cast<uintptr_t>(v) % (4 * sizeof(T))) == 0 &&
      (reinterpret_cast<uintptr_t>(out) % (4 * sizeof(Code))) == 0) {
    const int64_t n4 = n / 4;
    for (int64_t i = tid; i < n4; i += stride) {
      T x[4];
      if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<uint4*>(x) = ld_stream_u4(v + 4 * i);
      } else {
        *reinterpret_cast<uint4*>(x) = ld_stream_u4(v + 4 * i);
        *reinterpret_cast<uint4*>(x + 2) = ld_stream_u4(v + 4 * i + 2);
      }
      Code c[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) c[j] = code((double)x[j]);
      if constexpr (sizeof(Code) == 1)
        *reinterpret_cast<uint32_t*>(out + 4 * i) =
            (uint32_t)c[0] | ((uint32_t)c[1] << 8) | ((uint32_t)c[2] << 16) | ((uint32_t)c[3] << 24);
      else
        *reinterpret_cast<uint2*>(out + 4 * i) =
            make_uint2((uint32_t)c[0] | ((uint32_t)c[1] << 16), (uint32_t)c[2] | ((uint32_t)c[3] << 16));
    }
    for (int64_t i = n4 * 4 + tid; i < n; i += stride) out[i] = code((double)v[i]);
    return;
  }
  for (int64_t i = tid; i < n; i += stride) out[i] = code((double)v[i]);
}

int grid_for(int64_t n) {
  int64_t g = (n + kThreads - 1) / kThreads;
  const int64_t cap = (int64_t)sm_count() * 8;
  if (g > cap) g = cap;
  if (g > kMaxGrid) g = kMaxGrid;
  return g < 1 ? 1 : (int)g;
}

}  // namespace
}  // namespace ut

using namespace ut;

extern "C" {

size_t ut_plane_minmax_ws(void) { return 256 + sizeof(double) * 3 * kMaxGrid; }

int ut_plane_minmax(const void* plane, int32_t dtype, int64_t n, double* lohi, int32_t* nonfinite,
                    void* ws, size_t ws_bytes, void* stream) {
  UT_REQUIRE(dtype == UT_F32 || dtype == UT_F64, "ut_plane_minmax: plane must be float32/float64");
  UT_REQUIRE(n >= 1, "ut_plane_minmax: empty plane");
  UT_REQUIRE(ws_bytes >= ut_plane_minmax_ws(), "ut_plane_minmax: workspace too small");
  cudaStream_t st = as_stream(stream);
  auto* counter = static_cast<unsigned int*>(ws);
  auto* part = reinterpret_cast<double*>(static_cast<char*>(ws) + 256);
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(unsigned int), st);
  if (e != cudaSuccess) return cuda_status(e, "ut_plane_minmax memset");
  const int grid = grid_for(n);
  if (dtype == UT_F32)
    minmax_kernel<float><<<grid, kThreads, 0, st>>>(static_cast<const float*>(plane), n, part,
                                                    counter, lohi, nonfinite);
  else
    minmax_kernel<double><<<grid, kThreads, 0, st>>>(static_cast<const double*>(plane), n, part,
                                                     counter, lohi, nonfinite);
  UT_CHECK_LAUNCH("minmax_kernel");
  return UT_OK;
}

int ut_linear_to_codes(const void* plane, int32_t dtype, int64_t n, const double* lohi,
                       int32_t depth, void* codes, void* stream) {
  UT_REQUIRE(dtype == UT_F32 || dtype == UT_F64, "ut_linear_to_codes: plane must be float32/float64");
  UT_REQUIRE(depth == 8 || depth == 16, "unsupported bit depth %d; expected 8 or 16", depth);
  if (n <= 0) return UT_OK;
  cudaStream_t st = as_stream(stream);
  const int grid = grid_for(n);
  const double top = depth == 8 ? 255.0 : 65535.0;
  if (dtype == UT_F32 && depth == 8)
    codes_kernel<float, uint8_t><<<grid, kThreads, 0, st>>>(static_cast<const float*>(plane), n,
                                                            lohi, top, static_cast<uint8_t*>(codes));
  else if (dtype == UT_F32)
    codes_kernel<float, uint16_t><<<grid, kThreads, 0, st>>>(
        static_cast<const float*>(plane), n, lohi, top, static_cast<uint16_t*>(codes));
  else if (depth == 8)
    codes_kernel<double, uint8_t><<<grid, kThreads, 0, st>>>(
        static_cast<const double*>(plane), n, lohi, top, static_cast<uint8_t*>(codes));
  else
    codes_kernel<double, uint16_t><<<grid, kThreads, 0, st>>>(
        static_cast<const double*>(plane), n, lohi, top, static_cast<uint16_t*>(codes));
  UT_CHECK_LAUNCH("codes_kernel");
  return UT_OK;
}

}  // extern "C"
