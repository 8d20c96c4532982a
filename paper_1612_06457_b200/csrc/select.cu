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

constexpr int kSample = 16384;              // strided sample, sorted in one block
constexpr int64_t kCandCap = 1 << 22;       // candidates kept per rank

struct SelWs {
  unsigned int* hist;        // [2][kBins]
  unsigned long long* pre;   // [2] prefix of each rank
  long long* rem;            // [2] rank left inside the prefix bucket (1-based)
  unsigned long long* lo;    // [2] candidate window [lo, hi] (keys) per rank
  unsigned long long* hi;    // [2]
  unsigned long long* below; // [2] samples with key < lo
  unsigned long long* cnt;   // [2] candidates found
  int* fallback;             // 1: the window missed -> full radix select over the plane
  unsigned long long* cand;  // [2][kCandCap] candidate keys
};

size_t sel_ws_layout(SelWs* ws, void* base) {
  const size_t off_h = 0, off_p = 2 * kBins * 4, off_r = off_p + 16, off_lo = off_r + 16,
               off_hi = off_lo + 16, off_b = off_hi + 16, off_c = off_b + 16, off_f = off_c + 16,
               off_cand = 2 * kBins * 4 + 256;
  if (ws && base) {
    char* p = static_cast<char*>(base);
    ws->hist = reinterpret_cast<unsigned int*>(p + off_h);
    ws->pre = reinterpret_cast<unsigned long long*>(p + off_p);
    ws->rem = reinterpret_cast<long long*>(p + off_r);
    ws->lo = reinterpret_cast<unsigned long long*>(p + off_lo);
    ws->hi = reinterpret_cast<unsigned long long*>(p + off_hi);
    ws->below = reinterpret_cast<unsigned long long*>(p + off_b);
    ws->cnt = reinterpret_cast<unsigned long long*>(p + off_c);
    ws->fallback = reinterpret_cast<int*>(p + off_f);
    ws->cand = reinterpret_cast<unsigned long long*>(p + off_cand);
  }
  return off_cand + sizeof(unsigned long long) * 2 * (size_t)kCandCap;
}

// gate: a kernel of the candidate path runs when *fallback == 0, one of the
// full-plane path when it is 1
__device__ __forceinline__ bool gated_off(const SelWs& ws, int want) {
  return want >= 0 && (*ws.fallback != 0) != (want != 0);
}

__global__ void sel_init_kernel(SelWs ws, long long r0, long long r1, int want) {
  if (gated_off(ws, want)) return;
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
sel_hist_kernel(const T* __restrict__ v, int64_t n, int shift, int width, SelWs ws, int want) {
  if (gated_off(ws, want)) return;
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
__global__ void __launch_bounds__(1024) sel_scan_kernel(SelWs ws, int width, int separate, int want) {
  if (gated_off(ws, want)) return;
  __shared__ unsigned long long cum[2][kBins];
  __shared__ unsigned long long wsum[2][32];
  const bool same = !separate && ws.pre[0] == ws.pre[1];
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

// ---- candidate path: sort a strided sample, bracket each rank, keep only the
// keys inside the brackets (one pass over the plane), radix-select among them
template <typename T>
__global__ void __launch_bounds__(1024)
cand_sample_kernel(const T* __restrict__ v, int64_t n, long long r0, long long r1, SelWs ws) {
  extern __shared__ unsigned long long sk[];  // kSample keys
  using K = Key<T>;
  const int tid = threadIdx.x;
  const int S = n < kSample ? (int)n : kSample;
  int P = 1;
  while (P < S) P <<= 1;  // bitonic size (pad with the largest key)
  for (int i = tid; i < P; i += blockDim.x)
    sk[i] = i < S ? (unsigned long long)K::of(v[(int64_t)((double)i * (double)n / S)]) : ~0ull;
  for (int i = tid; i < 2 * kBins; i += blockDim.x) ws.hist[i] = 0u;
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < P; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const unsigned long long a = sk[i], b = sk[ixj];
          if ((a > b) == up) { sk[i] = b; sk[ixj] = a; }
        }
      }
      __syncthreads();
    }
  if (tid < 2) {
    const long long r = tid ? r1 : r0;
    const double f = (double)r / (double)n;
    const long long q = (long long)((double)(r - 1) * S / (double)n);
    const long long d = (long long)(3.0 * sqrt((double)S * f * (1.0 - f)) + 32.0);
    const long long a = q - d, b = q + d;
    ws.lo[tid] = a <= 0 ? 0ull : sk[a];
    ws.hi[tid] = b >= S - 1 ? ~0ull : sk[b];
    ws.below[tid] = 0ull;
    ws.cnt[tid] = 0ull;
    ws.pre[tid] = 0ull;
  }
  if (tid == 0) *ws.fallback = 0;
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
cand_filter_kernel(const T* __restrict__ v, int64_t n, SelWs ws) {
  using K = Key<T>;
  constexpr int W = 64;  // per-warp staging of candidates: one global atomic per W keys
  __shared__ unsigned long long wbuf[kThreads / 32][2][W];
  const unsigned long long lo0 = ws.lo[0], hi0 = ws.hi[0], lo1 = ws.lo[1], hi1 = ws.hi[1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  unsigned long long below0 = 0, below1 = 0;
  int wc[2] = {0, 0};
  auto flush = [&](int r) {
    __syncwarp();
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&ws.cnt[r], (unsigned long long)wc[r]);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int q = lane; q < wc[r]; q += 32) {
      const unsigned long long at = base + q;
      if (at < (unsigned long long)kCandCap) ws.cand[(size_t)r * kCandCap + at] = wbuf[warp][r][q];
    }
    __syncwarp();
    wc[r] = 0;
  };
  auto push = [&](int r, bool c, unsigned long long k) {
    const unsigned m = __ballot_sync(0xffffffffu, c);
    if (!m) return;
    if (wc[r] + __popc(m) > W) flush(r);
    if (c) wbuf[warp][r][wc[r] + __popc(m & lt)] = k;
    wc[r] += __popc(m);
  };
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  const bool vec = (reinterpret_cast<uintptr_t>(v) % (4 * sizeof(T))) == 0;
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31)) * 4; i0 < n; i0 += stride) {
    const int64_t i = i0 + 4 * lane;
    T x[4];
    if (vec && i + 4 <= n) {
      *reinterpret_cast<uint4*>(x) = ld_stream_u4(v + i);
      if constexpr (sizeof(T) == 8) *reinterpret_cast<uint4*>(x + 2) = ld_stream_u4(v + i + 2);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) x[j] = i + j < n ? v[i + j] : T(0);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool ok = i + j < n;
      const unsigned long long k = (unsigned long long)K::of(x[j]);
      below0 += (ok && k < lo0);
      below1 += (ok && k < lo1);
      push(0, ok && k >= lo0 && k <= hi0, k);
      push(1, ok && k >= lo1 && k <= hi1, k);
    }
  }
  flush(0);
  flush(1);
  for (int o = 16; o > 0; o >>= 1) {
    below0 += __shfl_xor_sync(0xffffffffu, below0, o);
    below1 += __shfl_xor_sync(0xffffffffu, below1, o);
  }
  if (lane == 0) {
    if (below0) atomicAdd(&ws.below[0], below0);
    if (below1) atomicAdd(&ws.below[1], below1);
  }
}

// the ranks inside the candidate sets, or the fall back to the full select
__global__ void cand_check_kernel(SelWs ws, long long r0, long long r1) {
  if (threadIdx.x != 0) return;
  bool ok = true;
  for (int r = 0; r < 2; ++r) {
    const long long rank = r ? r1 : r0;
    const long long below = (long long)ws.below[r], cnt = (long long)ws.cnt[r];
    ok = ok && cnt <= kCandCap && below < rank && rank <= below + cnt;
    ws.rem[r] = rank - below;
    ws.pre[r] = 0ull;
  }
  *ws.fallback = ok ? 0 : 1;
}

// histogram of one digit over each rank's own candidate keys (blockIdx.y = rank)
__global__ void __launch_bounds__(kThreads)
cand_hist_kernel(SelWs ws, int shift, int width, int keybits) {
  if (gated_off(ws, 0)) return;
  __shared__ unsigned int h[kBins];
  const int r = blockIdx.y;
  for (int i = threadIdx.x; i < kBins; i += blockDim.x) h[i] = 0u;
  __syncthreads();
  const int64_t n = (int64_t)ws.cnt[r];
  const unsigned long long* keys = ws.cand + (size_t)r * kCandCap;
  const int hs = shift + width;
  const unsigned long long p = ws.pre[r];
  const unsigned long long mask = (1ull << width) - 1ull;
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); i0 < n;
       i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + lane;
    unsigned b = 0xffffffffu;
    if (i < n) {
      const unsigned long long k = keys[i];
      const unsigned long long top = hs >= keybits ? 0ull : (k >> hs);
      if (top == p) b = (unsigned)((k >> shift) & mask);
    }
    if (__ballot_sync(0xffffffffu, b != 0xffffffffu)) {
      const unsigned m = __match_any_sync(0xffffffffu, b);
      if (b != 0xffffffffu && lane == __ffs(m) - 1) atomicAdd(&h[b], (unsigned)__popc(m));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kBins; i += blockDim.x)
    if (h[i]) atomicAdd(&ws.hist[r * kBins + i], h[i]);
}

template <typename T>
__global__ void sel_out_kernel(SelWs ws, double* out) {
  if (threadIdx.x < 2) out[threadIdx.x] = Key<T>::value((typename Key<T>::U)ws.pre[threadIdx.x]);
}

template <typename T>
int launch_select(const T* v, int64_t n, long long r0, long long r1, double* out, SelWs ws,
                  cudaStream_t st) {
  int64_t grid = (n / 4 + kThreads - 1) / kThreads;
  const int64_t cap = (int64_t)sm_count() * 4;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  // candidate path: sample + sort (one block), one filtering pass, radix over the candidates
  static SmemAttr attr;
  const int sample_smem = kSample * (int)sizeof(unsigned long long);
  if (int rc = ensure_smem(attr, cand_sample_kernel<T>, (size_t)sample_smem, "cand_sample smem attribute"))
    return rc;
  cand_sample_kernel<T><<<1, 1024, sample_smem, st>>>(v, n, r0, r1, ws);
  UT_CHECK_LAUNCH("cand_sample_kernel");
  cand_filter_kernel<T><<<(int)grid, kThreads, 0, st>>>(v, n, ws);
  UT_CHECK_LAUNCH("cand_filter_kernel");
  cand_check_kernel<<<1, 32, 0, st>>>(ws, r0, r1);
  UT_CHECK_LAUNCH("cand_check_kernel");
  const int64_t cgrid = sm_count();
  for (int shift = Key<T>::bits; shift > 0;) {
    const int width = shift >= 11 ? 11 : shift;
    shift -= width;
    cand_hist_kernel<<<dim3((unsigned)cgrid, 2), kThreads, 0, st>>>(ws, shift, width, Key<T>::bits);
    UT_CHECK_LAUNCH("cand_hist_kernel");
    sel_scan_kernel<<<1, 1024, 0, st>>>(ws, width, 1, 0);
    UT_CHECK_LAUNCH("sel_scan_kernel");
  }
  // full radix select over the plane, only when a window missed (device-gated)
  sel_init_kernel<<<1, 256, 0, st>>>(ws, r0, r1, 1);
  UT_CHECK_LAUNCH("sel_init_kernel");
  for (int shift = Key<T>::bits; shift > 0;) {
    const int width = shift >= 11 ? 11 : shift;
    shift -= width;
    sel_hist_kernel<T><<<(int)grid, kThreads, 0, st>>>(v, n, shift, width, ws, 1);
    UT_CHECK_LAUNCH("sel_hist_kernel");
    sel_scan_kernel<<<1, 1024, 0, st>>>(ws, width, 0, 1);
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
