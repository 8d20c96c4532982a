// standardize(dm) of the reference (projection.py:152-169): recentre each band
// row of a B x N design matrix to mean 0 and divide by its sample standard
// deviation (divisor N - 1; a constant row keeps std = 1).  It feeds fit_lda
// (projection.py:240-260), which is the CVA core (K1 + K3) on the result.
//
// One CTA per band row: pass 1 sums the row (fixed order: per-thread strided
// partial sums, xor tree per warp, warps in order), pass 2 sums the squared
// deviations from the mean the same way, pass 3 writes (x - mean) / std with
// IEEE division (as numpy).  A design matrix is at most a few hundred
// thousand points, so the row is re-read from L2 by passes 2 and 3.
#include "common.cuh"

namespace ut {
namespace {

constexpr int kThreads = 512;

__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < kThreads / 32; ++w) t += red[w];
  return t;
}

__global__ void __launch_bounds__(kThreads)
standardize_kernel(const double* __restrict__ x, int64_t ldx, int64_t n, double* __restrict__ out,
                   int64_t ldo, double* __restrict__ mean, double* __restrict__ std) {
  __shared__ double red[kThreads / 32];
  const int b = blockIdx.x;
  const double* row = x + b * ldx;
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += kThreads) s += row[j];
  const double m = block_sum(s, red) / (double)n;
  double q = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += kThreads) {
    const double d = row[j] - m;
    q = fma(d, d, q);
  }
  double sd = sqrt(block_sum(q, red) / (double)(n - 1));
  if (sd == 0.0) sd = 1.0;
  double* o = out + b * ldo;
  for (int64_t j = threadIdx.x; j < n; j += kThreads) o[j] = (row[j] - m) / sd;
  if (threadIdx.x == 0) {
    mean[b] = m;
    std[b] = sd;
  }
}

}  // namespace
}  // namespace ut

using namespace ut;

extern "C" {

int ut_standardize(const double* values, int64_t ld, int32_t bands, int64_t n, double* out,
                   int64_t ld_out, double* mean, double* std, void* stream) {
  UT_REQUIRE(n >= 2, "standardization needs at least 2 points");
  UT_REQUIRE(bands >= 1 && ld >= n && ld_out >= n, "ut_standardize: bad shape");
  UT_REQUIRE(values && out && mean && std, "ut_standardize: null pointer");
  standardize_kernel<<<bands, kThreads, 0, as_stream(stream)>>>(values, ld, n, out, ld_out, mean,
                                                                 std);
  UT_CHECK_LAUNCH("standardize_kernel");
  return UT_OK;
}

}  // extern "C"
