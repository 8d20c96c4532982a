// K2: one-pass fp64 moments of every pixel of a region (unsupervised PCA).
//
// Reference: fit_pca_unsupervised (projection.py:298-347) reads the cube twice
// -- a per-band mean pass (:327-329) and a 64-row centred Gram pass
// (:330-334).  Here one pass accumulates, per pixel, d = x - s with s a fixed
// per-band shift (mean of a deterministic strided sample, so |mean - s| is
// tiny and the one-pass form M2 = sum d d^T - (sum d)(sum d)^T / n loses
// nothing at the 1e-9 bar; SURVEY Appendix B.7 measured <= 5e-15).
//
// Tiles of 64 pixels are staged in shared memory as fp64 deviations; the Gram
// upper triangle is split in 4x4 register blocks, several thread groups per
// block striding over the tile's pixels.  This is fp64-issue-bound for B = 32
// (528 DFMA per pixel), HBM-bound for B <= 16.  All reductions are fixed-order.
#include "common.cuh"

namespace ut {
namespace {

constexpr int kThreads = 256;
constexpr int kTile = 64;
constexpr int kSample = 4096;
constexpr int kMaxGrid = 2048;
constexpr int kBp = kMaxBands;                 // padded band count (multiple of 4)
constexpr int kLdd = kBp + 1;                  // tile row stride (doubles)
constexpr int kMaxBlk = (kBp / 4) * (kBp / 4 + 1) / 2;  // 36
constexpr int kRec = kMaxBands + kMaxBands * kMaxBands;   // per-CTA partial: sum d, G

struct RegionWs {
  unsigned int* counter;
  double* shift;   // B
  double* part;    // [grid][kRec]
};

size_t region_ws_layout(RegionWs* ws, void* base) {
  const size_t off_shift = 256;
  const size_t off_part = off_shift + sizeof(double) * kMaxBands;
  const size_t total = off_part + sizeof(double) * (size_t)kMaxGrid * kRec;
  if (ws && base) {
    char* p = static_cast<char*>(base);
    ws->counter = reinterpret_cast<unsigned int*>(p);
    ws->shift = reinterpret_cast<double*>(p + off_shift);
    ws->part = reinterpret_cast<double*>(p + off_part);
  }
  return total;
}

struct Region {
  const void* data;
  int64_t bs, rs;
  int64_t x0, y0;
  uint32_t w;
  int64_t npix;
  int bands;
};

template <typename T>
__device__ __forceinline__ double sample_at(const Region& r, int b, int64_t pix) {
  const int64_t y = pix / r.w, x = pix - y * r.w;
  const T* p = static_cast<const T*>(r.data) + b * r.bs + (r.y0 + y) * r.rs + r.x0 + x;
  return to_f64(*p);
}

// shift_b = mean of up to 4096 pixels at a fixed stride (one CTA, fixed order)
template <typename T>
__global__ void __launch_bounds__(kThreads) shift_kernel(Region r, RegionWs ws) {
  __shared__ double red[kThreads];
  const int64_t count = r.npix < kSample ? r.npix : kSample;
  const int64_t step = r.npix / count;
  for (int b = 0; b < r.bands; ++b) {
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) acc += sample_at<T>(r, b, i * step);
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int h = kThreads / 2; h > 0; h >>= 1) {
      if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
      __syncthreads();
    }
    if (threadIdx.x == 0) ws.shift[b] = red[0] / (double)count;
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
region_kernel(Region r, RegionWs ws, double* __restrict__ moments) {
  __shared__ double tile[kTile * kLdd];
  __shared__ double shift[kMaxBands];
  __shared__ double gsum[kThreads / 32];
  const int tid = threadIdx.x;
  const int B = r.bands;
  const int nb = (B + 3) / 4;                     // 4-band blocks per dim
  const int nblk = nb * (nb + 1) / 2;
  const int groups = kThreads / nblk;             // pixel-stride groups
  const int blk = tid % nblk, grp = tid / nblk;
  const bool gram_thread = grp < groups;
  // (bi, bj) of this thread's 4x4 block, bi <= bj
  int bi = 0, bj = 0;
  {
    int rem = blk;
    while (rem >= nb - bi) { rem -= nb - bi; ++bi; }
    bj = bi + rem;
  }
  if (tid < B) shift[tid] = ws.shift[tid];
  for (int e = tid; e < kTile * kLdd; e += blockDim.x) tile[e] = 0.0;
  __syncthreads();

  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
  double dsum = 0.0;  // sum of deviations of band `tid` (tid < B)

  const int64_t ntiles = (r.npix + kTile - 1) / kTile;
  const int p_own = tid % kTile;        // staging: fixed pixel per thread
  const int b_first = tid / kTile;      // and bands b_first, b_first + 4, ...
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t pix = t * kTile + p_own;
    const bool valid = pix < r.npix;
    int64_t base = 0;
    if (valid) {
      const int64_t y = (int64_t)((uint64_t)pix / r.w), x = pix - y * r.w;
      base = (r.y0 + y) * r.rs + r.x0 + x;
    }
    const T* src = static_cast<const T*>(r.data) + base;
    for (int b = b_first; b < B; b += kThreads / kTile)
      tile[p_own * kLdd + b] = valid ? to_f64(src[b * r.bs]) - shift[b] : 0.0;
    __syncthreads();
    if (tid < B) {
      double s = 0.0;
      for (int p = 0; p < kTile; ++p) s += tile[p * kLdd + tid];
      dsum += s;
    }
    if (gram_thread) {
      for (int p = grp; p < kTile; p += groups) {
        const double* row = tile + p * kLdd;
        double u[4], v[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          u[a] = row[4 * bi + a];
          v[a] = row[4 * bj + a];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[a][c] = fma(u[a], v[c], acc[a][c]);
      }
    }
    __syncthreads();
  }

  // ---- CTA reduction of the thread-group partials (fixed order over groups)
  double* red = tile;  // reuse: needs nblk*16*groups <= kTile*kLdd doubles? use two phases
  double* part = ws.part + (size_t)blockIdx.x * kRec;
  if (tid < B) part[tid] = dsum;
  for (int g = 0; g < groups; ++g) {
    if (gram_thread && grp == g) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) red[blk * 16 + a * 4 + c] = (g == 0 ? 0.0 : red[blk * 16 + a * 4 + c]) + acc[a][c];
    }
    __syncthreads();
  }
  for (int e = tid; e < nblk * 16; e += blockDim.x) {
    int b2 = e / 16, a = (e % 16) / 4, c = e % 4;
    int i0 = 0, rem = b2;
    while (rem >= nb - i0) { rem -= nb - i0; ++i0; }
    const int j0 = i0 + rem;
    const int i = 4 * i0 + a, j = 4 * j0 + c;
    if (i < B && j < B) part[kMaxBands + i * kMaxBands + j] = red[e];
  }
  (void)gsum;
  if (last_block_ticket(ws.counter)) {
    // fixed-order sum over CTAs, then n, mean, M2 (full symmetric)
    const double n = (double)r.npix;
    for (int e = tid; e < kRec; e += blockDim.x) {
      bool used;
      if (e < kMaxBands) {
        used = e < B;
      } else {
        const int q = e - kMaxBands, i = q / kMaxBands, j = q % kMaxBands;
        used = i < B && j < B && (i / 4) <= (j / 4);
      }
      if (!used) continue;
      double s = 0.0;
      for (unsigned int g = 0; g < gridDim.x; ++g) s += ws.part[(size_t)g * kRec + e];
      ws.part[e] = s;  // CTA 0's slot holds the totals (CTA 0 already wrote its own)
    }
    __syncthreads();
    const int len = 1 + B + B * B;
    if (tid == 0) moments[0] = n;
    if (tid < B) moments[1 + tid] = shift[tid] + ws.part[tid] / n;
    for (int e = tid; e < B * B; e += blockDim.x) {
      const int i = e / B, j = e % B;
      const int lo = (i / 4) <= (j / 4) ? i : j, hi = (i / 4) <= (j / 4) ? j : i;
      const double g = ws.part[kMaxBands + lo * kMaxBands + hi];
      moments[1 + B + e] = g - ws.part[i] * ws.part[j] / n;
    }
    (void)len;
    if (tid == 0) *ws.counter = 0u;
  }
}

template <typename T>
int launch_region(const Region& r, RegionWs ws, double* moments, cudaStream_t st) {
  shift_kernel<T><<<1, kThreads, 0, st>>>(r, ws);
  UT_CHECK_LAUNCH("shift_kernel");
  static int per_sm = 0;
  if (per_sm == 0) {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, region_kernel<T>, kThreads, 0);
    per_sm = n > 0 ? n : 1;
  }
  const int64_t ntiles = (r.npix + kTile - 1) / kTile;
  int64_t grid = (int64_t)per_sm * sm_count();
  if (grid > ntiles) grid = ntiles;
  if (grid > kMaxGrid) grid = kMaxGrid;
  region_kernel<T><<<(int)grid, kThreads, 0, st>>>(r, ws, moments);
  UT_CHECK_LAUNCH("region_kernel");
  return UT_OK;
}

}  // namespace
}  // namespace ut

using namespace ut;

extern "C" {

size_t ut_region_moments_ws(int32_t bands) {
  (void)bands;
  return region_ws_layout(nullptr, nullptr);
}

int ut_region_moments(const ut_cube* cube, int64_t x0, int64_t y0, int64_t w, int64_t h,
                      double* moments, void* ws_base, size_t ws_bytes, void* stream) {
  UT_REQUIRE(cube && cube->bands >= 1 && cube->bands <= kMaxBands,
             "ut_region_moments: bands must be 1..32");
  UT_REQUIRE(w > 0 && h > 0, "empty region (%lld, %lld, %lld, %lld)", (long long)x0,
             (long long)y0, (long long)w, (long long)h);
  UT_REQUIRE(x0 >= 0 && y0 >= 0 && x0 + w <= cube->cols && y0 + h <= cube->rows,
             "region (%lld, %lld, %lld, %lld) outside %lldx%lld stack", (long long)x0,
             (long long)y0, (long long)w, (long long)h, (long long)cube->cols,
             (long long)cube->rows);
  UT_REQUIRE(w * h < (int64_t)1 << 32, "region too large for 32-bit pixel indexing");
  RegionWs ws;
  const size_t need = region_ws_layout(&ws, ws_base);
  UT_REQUIRE(ws_bytes >= need, "ut_region_moments: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(ws.counter, 0, sizeof(unsigned int), st);
  if (e != cudaSuccess) return cuda_status(e, "ut_region_moments memset");
  Region r{cube->data, cube->band_stride, cube->row_stride, x0, y0, (uint32_t)w, w * h,
           cube->bands};
  switch (cube->dtype) {
    case UT_U8: return launch_region<uint8_t>(r, ws, moments, st);
    case UT_U16: return launch_region<uint16_t>(r, ws, moments, st);
    case UT_F16: return launch_region<__half>(r, ws, moments, st);
    case UT_F32: return launch_region<float>(r, ws, moments, st);
    case UT_F64: return launch_region<double>(r, ws, moments, st);
  }
  set_error("ut_region_moments: unknown dtype %d", cube->dtype);
  return UT_EDATA;
}

}  // extern "C"
