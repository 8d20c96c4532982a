// K2: one-pass fp64 moments of every pixel of a region (unsupervised PCA).
//
// Reference: fit_pca_unsupervised (projection.py:298-347) reads the cube twice
// -- a per-band mean pass (:327-329) and a 64-row centred Gram pass
// (:330-334).  Here one pass accumulates, per pixel, d = x - s with s a fixed
// per-band shift (mean of a deterministic strided sample of 4096 pixels, so
// |mean - s| ~ sigma/64 and the one-pass form M2 = sum d d^T - (sum d)(sum d)^T/n
// loses nothing at the 1e-9 bar; SURVEY Appendix B.7 measured <= 5e-15).
//
// G = min(tiles, 592) CTAs (a constant, so results do not depend on the GPU)
// each own a contiguous run of 64-pixel tiles.  A tile is staged in shared
// memory as fp64 deviations with a constant-1 column appended (so the Gram
// also yields the sums); the next tile is prefetched into registers while the
// current one is reduced.  The upper triangle of the Gram is split into 4x4
// register blocks, several thread groups per block striding over the tile's
// pixels.  fp64-FMA-bound for B = 32 (561 DFMA per pixel), HBM-bound for
// B <= 16.  Partials are summed by a separate kernel, one warp per entry,
// lanes over CTAs, in a fixed shuffle tree: deterministic.
#include <cstdlib>

#include "common.cuh"

namespace ut {
namespace {

constexpr int kThreads = 256;
constexpr int kTile = 64;
constexpr int kSample = 4096;
constexpr int kMaxG = 592;                                  // 4 x 148
constexpr int kCols = kMaxBands + 4;                        // bands + ones, padded to 4
constexpr int kLdd = kCols + 1;                             // tile row stride (doubles)
constexpr int kNb = kCols / 4;                              // 9 blocks per dim
constexpr int kMaxBlk = kNb * (kNb + 1) / 2;                // 45
constexpr int kEnt = kCols * kCols;                         // per-CTA Gram record (padded)

struct RegionWs {
  double* shift;   // B
  double* part;    // [kEnt][G]
};

size_t region_ws_layout(RegionWs* ws, void* base) {
  const size_t off_shift = 256;
  const size_t off_part = off_shift + sizeof(double) * kMaxBands;
  const size_t total = off_part + sizeof(double) * (size_t)kMaxG * kEnt;  // >= 1056 x 592 (DMMA path)
  if (ws && base) {
    char* p = static_cast<char*>(base);
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
  int G;
  int64_t tiles_per_cta;
};

template <typename T>
__device__ __forceinline__ const T* pixel_ptr(const Region& r, int64_t pix) {
  const int64_t y = (int64_t)((uint64_t)pix / r.w), x = pix - y * r.w;
  return static_cast<const T*>(r.data) + (r.y0 + y) * r.rs + r.x0 + x;
}

// shift_b = mean of up to 4096 pixels at a fixed stride (one CTA, fixed tree)
template <typename T>
__global__ void __launch_bounds__(1024) shift_kernel(Region r, RegionWs ws) {
  __shared__ double red[1024 / 32][kMaxBands];
  const int64_t count = r.npix < kSample ? r.npix : kSample;
  const int64_t step = r.npix / count;
  double acc[kMaxBands];
#pragma unroll
  for (int b = 0; b < kMaxBands; ++b) acc[b] = 0.0;
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
    const T* p = pixel_ptr<T>(r, i * step);
#pragma unroll
    for (int b = 0; b < kMaxBands; ++b)
      if (b < r.bands) acc[b] += to_f64(p[b * r.bs]);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int b = 0; b < kMaxBands; ++b) {
    double v = acc[b];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][b] = v;
  }
  __syncthreads();
  if (threadIdx.x < r.bands) {
    double v = 0.0;
    for (int w = 0; w < 32; ++w) v += red[w][threadIdx.x];
    ws.shift[threadIdx.x] = v / (double)count;
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
region_kernel(Region r, RegionWs ws) {
  __shared__ double tile[kTile * kLdd];
  __shared__ double shift[kMaxBands];
  const int tid = threadIdx.x;
  const int B = r.bands;
  const int nb = (B + 1 + 3) / 4;                 // 4-column blocks incl. the ones column
  const int nblk = nb * (nb + 1) / 2;
  const int groups = kThreads / nblk;
  const int blk = tid % nblk, grp = tid / nblk;
  const bool gram_thread = grp < groups;
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

  const int64_t ntiles = (r.npix + kTile - 1) / kTile;
  const int64_t t0 = (int64_t)blockIdx.x * r.tiles_per_cta;
  int64_t t1 = t0 + r.tiles_per_cta;
  if (t1 > ntiles) t1 = ntiles;
  const int p_own = tid % kTile;      // staging: one pixel per thread
  const int b_first = tid / kTile;    // bands b_first, +4, +8, ...
  constexpr int kPer = (kMaxBands + 3) / 4;  // <= 8 staged values per thread
  double next[kPer];
  bool next_valid = false;
  auto load = [&](int64_t t) {
    const int64_t pix = t * kTile + p_own;
    next_valid = pix < r.npix;
    const T* src = next_valid ? pixel_ptr<T>(r, pix) : nullptr;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int b = b_first + 4 * u;
      next[u] = (next_valid && b < B) ? to_f64(src[b * r.bs]) : 0.0;
    }
  };
  if (t0 < t1) load(t0);
  for (int64_t t = t0; t < t1; ++t) {
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int b = b_first + 4 * u;
      if (b < B) tile[p_own * kLdd + b] = next_valid ? next[u] - shift[b] : 0.0;
    }
    if (b_first == 0) tile[p_own * kLdd + B] = next_valid ? 1.0 : 0.0;
    __syncthreads();
    if (t + 1 < t1) load(t + 1);      // prefetch while this tile is reduced
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
  // reduce the thread groups (fixed order) and write this CTA's partial
  double* red = tile;  // nblk * 16 <= 720 doubles <= kTile * kLdd
  for (int g = 0; g < groups; ++g) {
    if (gram_thread && grp == g) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int e = blk * 16 + a * 4 + c;
          red[e] = (g == 0 ? 0.0 : red[e]) + acc[a][c];
        }
    }
    __syncthreads();
  }
  for (int e = tid; e < nblk * 16; e += blockDim.x) {
    const int b2 = e / 16, a = (e % 16) / 4, c = e % 4;
    int i0 = 0, rem = b2;
    while (rem >= nb - i0) { rem -= nb - i0; ++i0; }
    const int j0 = i0 + rem;
    const int i = 4 * i0 + a, j = 4 * j0 + c;
    ws.part[(size_t)(i * kCols + j) * r.G + blockIdx.x] = red[e];
  }
}

// moments = [n, mean, M2]; one warp per output entry, lanes over the G partials.
__global__ void __launch_bounds__(256)
region_merge_kernel(Region r, RegionWs ws, double* __restrict__ moments) {
  const int B = r.bands, G = r.G;
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int total = 1 + B + B * B;
  if (e >= total) return;
  auto entry = [&](int i, int j) {  // Gram entry (i <= j by block) summed over CTAs
    if ((i >> 2) > (j >> 2)) { const int t = i; i = j; j = t; }
    const double* p = ws.part + (size_t)(i * kCols + j) * G;
    double a = 0.0;
    for (int g = lane; g < G; g += 32) a += p[g];
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    return a;
  };
  const double n = (double)r.npix;
  double v;
  if (e == 0) {
    v = n;
  } else if (e <= B) {
    const int b = e - 1;
    v = ws.shift[b] + entry(b, B) / n;
  } else {
    const int q = e - 1 - B, i = q / B, j = q - i * B;
    const double sij = entry(i, j), si = entry(i, B), sj = entry(j, B);
    v = sij - si * sj / n;
  }
  if (lane == 0) moments[e] = v;
}

// ---------------------------------------------------- K2 on FP64 tensor cores
// Whole-width regions (contiguous pixel range): a producer warp streams
// [B][512]-pixel tiles into a 3-stage shared-memory ring with bulk async
// copies; 8 consumer warps each take 4-pixel quads and, per 8-band group g,
// load one fragment element per lane -- x[band 8g + lane/4][pixel lane%4] --
// widen it, subtract the shift, and issue mma.sync.m8n8k4.f64 for every
// upper block (bi <= bj) of the Gram: the A fragment of group bi and the B
// fragment of group bj have the same per-lane layout, so each sample is loaded
// and widened exactly once.  Column sums ride along in the lanes.  Per-CTA
// partials [B*B + B][G] are summed by region_dmma_merge_kernel.
constexpr int kRdCons = 256;
constexpr int kRdP = 512;
constexpr int kRdStages = 3;
constexpr int kRdGroups = kMaxBands / 8;     // band groups of 8
constexpr int kRdEnt = kMaxBands * kMaxBands + kMaxBands;

template <typename T> constexpr int rd_pad() { return 16 / (int)sizeof(T); }  // 16 B: bank spread

template <typename T>
size_t rd_smem(int bands) {
  return (size_t)kRdStages * bands * (kRdP + rd_pad<T>()) * sizeof(T) +
         2 * kRdStages * sizeof(uint64_t) + 128;
}

struct RdParams {
  const void* data;   // first pixel of the region (band 0)
  int64_t bs;
  int64_t npix;
  int bands;
  int G;              // CTAs (= partial records)
  const double* shift;
  double* part;       // [kRdEnt][G]
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <typename T, int NG>
__global__ void __launch_bounds__(kRdCons + 32, 1)
region_dmma_kernel(RdParams r) {
  extern __shared__ __align__(128) unsigned char dyn[];
  __shared__ double red[kRdEnt];
  __shared__ double shift[kMaxBands];
  const int B = r.bands;
  constexpr int PS = kRdP + rd_pad<T>();
  T* stages = reinterpret_cast<T*>(dyn);
  uint64_t* full = reinterpret_cast<uint64_t*>(dyn + (size_t)kRdStages * B * PS * sizeof(T));
  uint64_t* empty = full + kRdStages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < kRdStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kRdCons / 32);
    }
    mbar_fence_init();
  }
  for (int e = tid; e < kRdEnt; e += blockDim.x) red[e] = 0.0;
  if (tid < B) shift[tid] = r.shift[tid];
  __syncthreads();
  const int64_t ntiles = (r.npix + kRdP - 1) / kRdP;
  constexpr int NB = NG * (NG + 1) / 2;  // upper 8x8 blocks
  double c0[NB], c1[NB], dsum[NG];
#pragma unroll
  for (int q = 0; q < NB; ++q) c0[q] = c1[q] = 0.0;
#pragma unroll
  for (int g = 0; g < NG; ++g) dsum[g] = 0.0;
  if (warp == kRdCons / 32) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int i = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int st = i % kRdStages;
        const uint32_t ph = (uint32_t)(i / kRdStages) & 1u;
        if (i >= kRdStages) mbar_wait(&empty[st], ph ^ 1u);
        const int64_t p0 = t * kRdP;
        const int64_t npx = (r.npix - p0) < kRdP ? (r.npix - p0) : kRdP;
        const uint32_t bytes = (uint32_t)(npx * sizeof(T));
        mbar_expect_tx(&full[st], bytes * (uint32_t)B);
        T* dst = stages + (size_t)st * B * PS;
        const T* src = static_cast<const T*>(r.data) + p0;
        for (int b = 0; b < B; ++b)
          bulk_g2s(dst + (size_t)b * PS, src + (int64_t)b * r.bs, bytes, &full[st], pol);
      }
    }
  } else {
    const int fb = lane >> 2, fp = lane & 3;  // fragment: band 8g + fb, pixel fp of the quad
    double sh[NG];
#pragma unroll
    for (int g = 0; g < NG; ++g) sh[g] = (8 * g + fb < B) ? shift[8 * g + fb] : 0.0;
    int i = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int st = i % kRdStages;
      const uint32_t ph = (uint32_t)(i / kRdStages) & 1u;
      mbar_wait(&full[st], ph);
      const int64_t p0 = t * kRdP;
      const int npx = (int)((r.npix - p0) < kRdP ? (r.npix - p0) : kRdP);
      const T* stage = stages + (size_t)st * B * PS;
      for (int qd = warp; qd * 4 < npx; qd += kRdCons / 32) {  // warp-uniform
        const int px = qd * 4 + fp;
        double f[NG];
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          const int b = 8 * g + fb;
          // branch-free masking keeps the warp converged for mma.sync.aligned
          const bool ok = b < B && px < npx;
          const long long keep = ok ? -1LL : 0LL;
          const double x = widen_f64(stage[(size_t)(ok ? b : 0) * PS + (ok ? px : 0)]) - sh[g];
          f[g] = __longlong_as_double(__double_as_longlong(x) & keep);
          dsum[g] += f[g];
        }
        __syncwarp();
        int q = 0;
#pragma unroll
        for (int bi = 0; bi < NG; ++bi)
#pragma unroll
          for (int bj = bi; bj < NG; ++bj, ++q) dmma(c0[q], c1[q], f[bi], f[bj]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    // fold this warp into the CTA record, one warp at a time (fixed order)
    for (int w = 0; w < kRdCons / 32; ++w) {
      if (warp == w) {
        const int cm = lane >> 2, cn = 2 * (lane & 3);
        int q = 0;
#pragma unroll
        for (int bi = 0; bi < NG; ++bi)
#pragma unroll
          for (int bj = bi; bj < NG; ++bj, ++q) {
            const int row = 8 * bi + cm, col = 8 * bj + cn;
            if (row < B && col < B) red[row * kMaxBands + col] += c0[q];
            if (row < B && col + 1 < B) red[row * kMaxBands + col + 1] += c1[q];
          }
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          // lanes sharing band 8g + fb differ in fp: sum them (fixed xor tree)
          double v = dsum[g];
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          if (fp == 0 && 8 * g + fb < B) red[kMaxBands * kMaxBands + 8 * g + fb] += v;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kRdCons) : "memory");
    }
  }
  __syncthreads();
  // write the upper triangle (i <= j) + sums as this CTA's partial
  for (int e = tid; e < kRdEnt; e += blockDim.x) {
    bool used;
    if (e < kMaxBands * kMaxBands) {
      const int ii = e / kMaxBands, jj = e % kMaxBands;
      used = ii < B && jj < B && (ii >> 3) <= (jj >> 3);
    } else {
      used = (e - kMaxBands * kMaxBands) < B;
    }
    if (used) r.part[(size_t)e * r.G + blockIdx.x] = red[e];
  }
}

// moments = [n, mean, M2]; one warp per output entry, lanes over the G partials.
__global__ void __launch_bounds__(256)
region_dmma_merge_kernel(RdParams r, double* __restrict__ moments) {
  const int B = r.bands, G = r.G;
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int total = 1 + B + B * B;
  if (e >= total) return;
  auto sum = [&](int idx) {
    const double* p = r.part + (size_t)idx * G;
    double a = 0.0;
    for (int g = lane; g < G; g += 32) a += p[g];
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    return a;
  };
  auto gram = [&](int i, int j) {
    if ((i >> 3) > (j >> 3)) { const int t = i; i = j; j = t; }
    return sum(i * kMaxBands + j);
  };
  const double n = (double)r.npix;
  double v;
  if (e == 0) {
    v = n;
  } else if (e <= B) {
    const int b = e - 1;
    v = r.shift[b] + sum(kMaxBands * kMaxBands + b) / n;
  } else {
    const int q = e - 1 - B, i = q / B, j = q - i * B;
    const double si = sum(kMaxBands * kMaxBands + i), sj = sum(kMaxBands * kMaxBands + j);
    v = gram(i, j) - si * sj / n;
  }
  if (lane == 0) moments[e] = v;
}

template <typename T, int NG>
int launch_region_dmma_ng(RdParams& rp, double* moments, cudaStream_t st) {
  auto kern = region_dmma_kernel<T, NG>;
  const size_t smem = rd_smem<T>(rp.bands);
  static size_t attr = 0;
  if (attr < smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "region_dmma smem attribute");
    attr = smem;
  }
  kern<<<rp.G, kRdCons + 32, smem, st>>>(rp);
  UT_CHECK_LAUNCH("region_dmma_kernel");
  const int total = 1 + rp.bands + rp.bands * rp.bands;
  region_dmma_merge_kernel<<<(total + 7) / 8, 256, 0, st>>>(rp, moments);
  UT_CHECK_LAUNCH("region_dmma_merge_kernel");
  return UT_OK;
}

template <typename T>
int launch_region_dmma(const Region& r, RegionWs ws, double* moments, cudaStream_t st) {
  shift_kernel<T><<<1, 1024, 0, st>>>(r, ws);
  UT_CHECK_LAUNCH("shift_kernel");
  RdParams rp;
  rp.data = static_cast<const T*>(r.data) + r.y0 * r.rs + r.x0;
  rp.bs = r.bs;
  rp.npix = r.npix;
  rp.bands = r.bands;
  const int64_t ntiles = (r.npix + kRdP - 1) / kRdP;
  const int64_t g = 148;  // fixed (not the device's SM count): results independent of the GPU
  rp.G = (int)(ntiles < g ? ntiles : g);
  rp.shift = ws.shift;
  rp.part = ws.part;
  switch ((r.bands + 7) / 8) {
    case 1: return launch_region_dmma_ng<T, 1>(rp, moments, st);
    case 2: return launch_region_dmma_ng<T, 2>(rp, moments, st);
    case 3: return launch_region_dmma_ng<T, 3>(rp, moments, st);
    default: return launch_region_dmma_ng<T, 4>(rp, moments, st);
  }
}

bool region_dmma_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("UT_REGION_DMMA");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <typename T>
int launch_region(Region r, RegionWs ws, double* moments, cudaStream_t st) {
  shift_kernel<T><<<1, 1024, 0, st>>>(r, ws);
  UT_CHECK_LAUNCH("shift_kernel");
  region_kernel<T><<<r.G, kThreads, 0, st>>>(r, ws);
  UT_CHECK_LAUNCH("region_kernel");
  const int total = 1 + r.bands + r.bands * r.bands;
  region_merge_kernel<<<(total + 7) / 8, 256, 0, st>>>(r, ws, moments);
  UT_CHECK_LAUNCH("region_merge_kernel");
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
  UT_REQUIRE(w * h < ((int64_t)1 << 40), "region too large");
  RegionWs ws;
  const size_t need = region_ws_layout(&ws, ws_base);
  UT_REQUIRE(ws_bytes >= need, "ut_region_moments: workspace %zu < %zu", ws_bytes, need);
  Region r{};
  r.data = cube->data;
  r.bs = cube->band_stride;
  r.rs = cube->row_stride;
  r.x0 = x0;
  r.y0 = y0;
  r.w = (uint32_t)w;
  r.npix = w * h;
  r.bands = cube->bands;
  const int64_t ntiles = (r.npix + kTile - 1) / kTile;
  const int64_t G = ntiles < kMaxG ? ntiles : kMaxG;
  r.tiles_per_cta = (ntiles + G - 1) / G;
  r.G = (int)((ntiles + r.tiles_per_cta - 1) / r.tiles_per_cta);
  cudaStream_t st = as_stream(stream);
  // whole-width regions of a contiguous cube: TMA + DMMA path
  const int64_t esz = cube->dtype == UT_U8 ? 1 : (cube->dtype == UT_F64 ? 8 : (cube->dtype == UT_F32 ? 4 : 2));
  const uintptr_t base = reinterpret_cast<uintptr_t>(cube->data) + (uintptr_t)((y0 * cube->row_stride + x0) * esz);
  const size_t rd_bytes = cube->dtype == UT_U8 ? rd_smem<uint8_t>(cube->bands)
                          : cube->dtype == UT_F64 ? rd_smem<double>(cube->bands)
                          : cube->dtype == UT_F32 ? rd_smem<float>(cube->bands)
                                                  : rd_smem<uint16_t>(cube->bands);
  const bool dmma_ok = region_dmma_enabled() && rd_bytes <= 200 * 1024 && x0 == 0 &&
                       w == cube->cols &&
                       cube->row_stride == cube->cols && base % 16 == 0 &&
                       (cube->band_stride * esz) % 16 == 0 && (r.npix * esz) % 16 == 0;
  if (dmma_ok) {
    switch (cube->dtype) {
      case UT_U8: return launch_region_dmma<uint8_t>(r, ws, moments, st);
      case UT_U16: return launch_region_dmma<uint16_t>(r, ws, moments, st);
      case UT_F16: return launch_region_dmma<__half>(r, ws, moments, st);
      case UT_F32: return launch_region_dmma<float>(r, ws, moments, st);
      case UT_F64: return launch_region_dmma<double>(r, ws, moments, st);
    }
  }
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
