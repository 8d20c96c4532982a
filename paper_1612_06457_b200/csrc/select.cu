// Order statistics of a score plane for rescale_percentile (rendering.py:
// 155-179, nearest_rank_percentile :146-152): the values of rank r0 and r1
// (1-based) of the ascending plane, exactly, by radix select on the
// order-preserving integer image of the float (fp32 planes: 11+11+10-bit
// digits, 3 passes; fp64 planes: 11 x 5 + 9, 6 passes).  Each pass histograms
// the next digit of the elements still sharing each rank's prefix (shared-
// memory histograms, one global merge per CTA), then one thread per rank walks
// the histogram to fix the digit.  No sort, no copy of the plane; the result
// does not depend on the launch shape.
#include "common.cuh"

namespace ut {
namespace {

constexpr int kThreads = 512;
constexpr int kBins = 2048;

template <typename T> struct Key;
template <> struct Key<float> {
  using U = uint32_t;
  static constexpr int bits = 32;
  __device__ static U of(float x) {
    const U u = __float_as_uint(x);
    return (u >> 31) ? ~u : (u | 0x80000000u);
  }
  __device__ static double value(U k) {
    const U u = (k >> 31) ? (k & 0x7fffffffu) : ~k;
    return (double)__uint_as_float(u);
  }
};
template <> struct Key<double> {
  using U = unsigned long long;
  static constexpr int bits = 64;
  __device__ static U of(double x) {
    const U u = (U)__double_as_longlong(x);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
  }
  __device__ static double value(U k) {
    const U u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)u);
  }
};

struct SelWs {
  unsigned int* hist;        // [2][kBins]
  unsigned long long* pre;   // [2] prefix of each rank
  long long* rem;            // [2] rank left inside the prefix bucket (1-based)
};

size_t sel_ws_layout(SelWs* ws, void* base) {
  const size_t off_h = 0, off_p = 2 * kBins * 4, off_r = off_p + 16;
  if (ws && base) {
    char* p = static_cast<char*>(base);
    ws->hist = reinterpret_cast<unsigned int*>(p + off_h);
    ws->pre = reinterpret_cast<unsigned long long*>(p + off_p);
    ws->rem = reinterpret_cast<long long*>(p + off_r);
  }
  return off_r + 16;
}

__global__ void sel_init_kernel(SelWs ws, long long r0, long long r1) {
  for (int i = threadIdx.x; i < 2 * kBins; i += blockDim.x) ws.hist[i] = 0u;
  if (threadIdx.x == 0) {
    ws.pre[0] = ws.pre[1] = 0ull;
    ws.rem[0] = r0;
    ws.rem[1] = r1;
  }
}

// histogram of digit (key >> shift) & (2^width - 1) over elements whose
// higher bits (key >> (shift + width)) equal the rank's prefix
template <typename T>
__global__ void __launch_bounds__(kThreads)
sel_hist_kernel(const T* __restrict__ v, int64_t n, int shift, int width, SelWs ws) {
  using K = Key<T>;
  __shared__ unsigned int h[2][kBins];
  for (int i = threadIdx.x; i < 2 * kBins; i += blockDim.x) (&h[0][0])[i] = 0u;
  __syncthreads();
  const int hs = shift + width;
  const typename K::U p0 = (typename K::U)ws.pre[0], p1 = (typename K::U)ws.pre[1];
  const typename K::U mask = ((typename K::U)1 << width) - 1;
  const bool same = p0 == p1;
  // 4 samples per lane and iteration (one 16/32-byte load); warp-aggregated
  // shared atomics (score planes concentrate in few bins of the leading digits,
  // where per-lane atomics would serialize); iterations where no lane matches a
  // prefix (later passes: almost all) skip the aggregation entirely
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  const bool vec = (reinterpret_cast<uintptr_t>(v) % (4 * sizeof(T))) == 0;
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31)) * 4; i0 < n; i0 += stride) {
    const int64_t i = i0 + 4 * lane;
    T x[4];
    if (vec && i + 4 <= n) {
      if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<uint4*>(x) = ld_stream_u4(v + i);
      } else {
        *reinterpret_cast<uint4*>(x) = ld_stream_u4(v + i);
        *reinterpret_cast<uint4*>(x + 2) = ld_stream_u4(v + i + 2);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) x[j] = i + j < n ? v[i + j] : T(0);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      unsigned b0 = 0xffffffffu, b1 = 0xffffffffu;
      if (i + j < n) {
        const typename K::U k = K::of(x[j]);
        const typename K::U hi = hs >= K::bits ? 0 : (k >> hs);
        const unsigned d = (unsigned)((k >> shift) & mask);
        if (hi == p0) b0 = d;
        if (!same && hi == p1) b1 = d;
      }
      if (__ballot_sync(0xffffffffu, b0 != 0xffffffffu)) {
        const unsigned m0 = __match_any_sync(0xffffffffu, b0);
        if (b0 != 0xffffffffu && lane == __ffs(m0) - 1) atomicAdd(&h[0][b0], (unsigned)__popc(m0));
      }
      if (!same && __ballot_sync(0xffffffffu, b1 != 0xffffffffu)) {
        const unsigned m1 = __match_any_sync(0xffffffffu, b1);
        if (b1 != 0xffffffffu && lane == __ffs(m1) - 1) atomicAdd(&h[1][b1], (unsigned)__popc(m1));
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kBins; i += blockDim.x) {
    if (h[0][i]) atomicAdd(&ws.hist[i], h[0][i]);
    if (!same && h[1][i]) atomicAdd(&ws.hist[kBins + i], h[1][i]);
  }
}

// fix the digit of each rank; clear the histogram for the next pass.  One
// block of 1024 threads: per rank, a block-wide inclusive scan of the bins.
__global__ void __launch_bounds__(1024) sel_scan_kernel(SelWs ws, int width) {
  __shared__ unsigned long long cum[2][kBins];
  __shared__ unsigned long long wsum[2][32];
  const bool same = ws.pre[0] == ws.pre[1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bins = 1 << width;
  // each thread owns bins 2 tid, 2 tid + 1 of both histograms
  unsigned long long a[2][2];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int bin = 2 * tid + q;
      const int src = (same ? 0 : r) * kBins + bin;
      a[r][q] = bin < bins ? ws.hist[src] : 0ull;
    }
  __syncthreads();
  for (int i = tid; i < 2 * kBins; i += blockDim.x) ws.hist[i] = 0u;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    unsigned long long s = a[r][0] + a[r][1], x = s;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[r][warp] = x;
    __syncthreads();
    if (warp == 0) {
      unsigned long long w = wsum[r][lane], z = w;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= o) z += y;
      }
      wsum[r][lane] = z - w;  // exclusive warp offsets
    }
    __syncthreads();
    const unsigned long long base = wsum[r][warp] + x - s;  // exclusive before bin 2 tid
    cum[r][2 * tid] = base + a[r][0];
    cum[r][2 * tid + 1] = base + a[r][0] + a[r][1];
  }
  __syncthreads();
  // the digit: first bin whose inclusive count reaches the rank (ranks read
  // into registers before any thread rewrites them)
  const long long rems[2] = {ws.rem[0], ws.rem[1]};
  __syncthreads();
  for (int r = 0; r < 2; ++r) {
    const long long rem = rems[r];
    for (int bin = tid; bin < bins; bin += blockDim.x) {
      const unsigned long long before = bin ? cum[r][bin - 1] : 0ull;
      if ((long long)before < rem && rem <= (long long)cum[r][bin]) {
        ws.rem[r] = rem - (long long)before;
        ws.pre[r] = (ws.pre[r] << width) | (unsigned long long)bin;
      }
    }
  }
}

template <typename T>
__global__ void sel_out_kernel(SelWs ws, double* out) {
  if (threadIdx.x < 2) out[threadIdx.x] = Key<T>::value((typename Key<T>::U)ws.pre[threadIdx.x]);
}

template <typename T>
int launch_select(const T* v, int64_t n, long long r0, long long r1, double* out, SelWs ws,
                  cudaStream_t st) {
  sel_init_kernel<<<1, 256, 0, st>>>(ws, r0, r1);
  UT_CHECK_LAUNCH("sel_init_kernel");
  int64_t grid = (n / 4 + kThreads - 1) / kThreads;
  const int64_t cap = (int64_t)sm_count() * 4;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  int shift = Key<T>::bits;
  while (shift > 0) {
    const int width = shift >= 11 ? 11 : shift;
    shift -= width;
    sel_hist_kernel<T><<<(int)grid, kThreads, 0, st>>>(v, n, shift, width, ws);
    UT_CHECK_LAUNCH("sel_hist_kernel");
    sel_scan_kernel<<<1, 1024, 0, st>>>(ws, width);
    UT_CHECK_LAUNCH("sel_scan_kernel");
  }
  sel_out_kernel<T><<<1, 32, 0, st>>>(ws, out);
  UT_CHECK_LAUNCH("sel_out_kernel");
  return UT_OK;
}

}  // namespace
}  // namespace ut

using namespace ut;

extern "C" {

size_t ut_plane_select_ws(void) { return sel_ws_layout(nullptr, nullptr); }

int ut_plane_select(const void* plane, int32_t dtype, int64_t n, const int64_t* ranks,
                    double* out, void* ws_base, size_t ws_bytes, void* stream) {
  UT_REQUIRE(plane && n >= 1, "ut_plane_select: empty plane");
  UT_REQUIRE(ranks && ranks[0] >= 1 && ranks[0] <= n && ranks[1] >= 1 && ranks[1] <= n,
             "ut_plane_select: ranks must lie in [1, %lld]", (long long)n);
  SelWs ws;
  const size_t need = sel_ws_layout(&ws, ws_base);
  UT_REQUIRE(ws_bytes >= need, "ut_plane_select: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t st = as_stream(stream);
  if (dtype == UT_F32)
    return launch_select<float>(static_cast<const float*>(plane), n, ranks[0], ranks[1], out, ws, st);
  if (dtype == UT_F64)
    return launch_select<double>(static_cast<const double*>(plane), n, ranks[0], ranks[1], out, ws, st);
  set_error("ut_plane_select: dtype must be float32 or float64, got %d", dtype);
  return UT_EDATA;
}

}  // extern "C"
