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

#ifndef UT_RD_PROD_LANES   // region_dmma_kernel: lanes share the band copies (0 = one lane)
#define UT_RD_PROD_LANES 1
#endif
#ifndef UT_IM_PROD_LANES   // region_imma_kernel: lanes of each producer warp share its copies
#define UT_IM_PROD_LANES 1
#endif

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
  double* shift;   // B: the per-band shift s_b (= S_b * 2^-f_b, see shift_kernel)
  double* scale;   // B: 2^f_b (fixed-point grid of the integer path)
  double* addend;  // B: 1.5*2^52 - S_b + 0x80808080 (magic rounding constant)
  int* fexp;       // B: f_b
  int* flag;       // integer path: nonzero if a sample fell outside its fixed-point range
  double* part;    // [kEnt][G] doubles, or the integer path's int64 records
};

size_t region_ws_layout(RegionWs* ws, void* base) {
  const size_t off_shift = 256;
  const size_t off_scale = off_shift + sizeof(double) * kMaxBands;
  const size_t off_add = off_scale + sizeof(double) * kMaxBands;
  const size_t off_fexp = off_add + sizeof(double) * kMaxBands;
  const size_t off_flag = off_fexp + sizeof(int) * kMaxBands;
  const size_t off_part = 2048;
  static_assert(256 + 3 * 8 * kMaxBands + 4 * kMaxBands + 16 <= 2048, "region ws header");
  const size_t total = off_part + sizeof(double) * (size_t)kMaxG * kEnt;  // >= 1056 x 592 (DMMA path)
  if (ws && base) {
    char* p = static_cast<char*>(base);
    ws->shift = reinterpret_cast<double*>(p + off_shift);
    ws->scale = reinterpret_cast<double*>(p + off_scale);
    ws->addend = reinterpret_cast<double*>(p + off_add);
    ws->fexp = reinterpret_cast<int*>(p + off_fexp);
    ws->flag = reinterpret_cast<int*>(p + off_flag);
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

// shift_b = mean of up to 4096 pixels at a fixed stride, one CTA per band (the
// strided samples are scattered over the cube, so the loads of all bands go out
// at once); each thread keeps its <= 4 samples in registers for the spread
// pass.  Fixed reduction order: per thread, xor tree per warp, warps in order.
template <typename T>
__global__ void __launch_bounds__(1024) shift_kernel(Region r, RegionWs ws) {
  constexpr int kPer = kSample / 1024;
  __shared__ double red[32];
  __shared__ double mean_sh;
  const int b = blockIdx.x;
  const int64_t count = r.npix < kSample ? r.npix : kSample;
  const int64_t step = r.npix / count;
  double v[kPer];
  double acc = 0.0;
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int64_t i = threadIdx.x + (int64_t)u * 1024;
    v[u] = i < count ? to_f64(pixel_ptr<T>(r, i * step)[b * r.bs]) : 0.0;
    acc += v[u];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += red[w];
    mean_sh = t / (double)count;
  }
  __syncthreads();
  const double m = mean_sh;
  // spread of the sample around it: sets the integer path's fixed-point grid
  double dev = 0.0;
#pragma unroll
  for (int u = 0; u < kPer; ++u)
    if (threadIdx.x + (int64_t)u * 1024 < count) dev = fmax(dev, fabs(v[u] - m));
  for (int o = 16; o > 0; o >>= 1) dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
  __syncthreads();
  if (lane == 0) red[warp] = dev;
  __syncthreads();
  if (threadIdx.x == 0) {
    double d = 0.0;
    for (int w = 0; w < 32; ++w) d = fmax(d, red[w]);
    // Fixed-point grid 2^-f: |x - s| <= 4 * (sample spread) maps inside +-2^30, so
    // samples up to ~8x the sampled spread fit the 32-bit range (else the
    // integer path flags the region and the fp64 path redoes it); integer
    // samples keep f = 0 (exact).  S = round(s 2^f) stays < 2^49 for the magic
    // constant.  NaN / Inf in the sample make f meaningless but are flagged.
    int f = 0;
    if (!Sample<T>::integral) {
      const double spread = fmax(4.0 * d, fabs(m) * 0x1p-20);
      f = spread > 0.0 ? 30 - (ilogb(spread) + 1) : 40;
      if (m != 0.0) f = min(f, 48 - (ilogb(fabs(m)) + 1));
      f = max(-60, min(f, 60));
    }
    const double sc = ldexp(1.0, f);
    const double S = rint(m * sc);
    ws.fexp[b] = f;
    ws.scale[b] = sc;
    ws.addend[b] = (0x1.8p52 - S) + 2155905152.0;  // + 0x80808080 (balanced digits)
    ws.shift[b] = ldexp(S, -f);
    if (b == 0) *ws.flag = 0;
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
  const int* gate;    // if set: run only when *gate != 0 (redo after the integer path)
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <typename T, int NG>
__global__ void __launch_bounds__(kRdCons + 32, 1)
region_dmma_kernel(RdParams r) {
  if (r.gate && *r.gate == 0) return;
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
    // producer warp: lane 0 arms the stage, the lanes share the band copies
    const uint64_t pol = policy_evict_first();
    int i = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int st = i % kRdStages;
      const uint32_t ph = (uint32_t)(i / kRdStages) & 1u;
      if (i >= kRdStages) mbar_wait(&empty[st], ph ^ 1u);
      const int64_t p0 = t * kRdP;
      const int64_t npx = (r.npix - p0) < kRdP ? (r.npix - p0) : kRdP;
      const uint32_t bytes = (uint32_t)(npx * sizeof(T));
      if (lane == 0) mbar_expect_tx(&full[st], bytes * (uint32_t)B);
      __syncwarp();
      T* dst = stages + (size_t)st * B * PS;
      const T* src = static_cast<const T*>(r.data) + p0;
      for (int b = UT_RD_PROD_LANES ? lane : (lane == 0 ? 0 : B); b < B; b += UT_RD_PROD_LANES ? 32 : 1)
        bulk_g2s(dst + (size_t)b * PS, src + (int64_t)b * r.bs, bytes, &full[st], pol);
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
  if (r.gate && *r.gate == 0) return;
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

// --------------------------------------- K2 on INT8 tensor cores (tcgen05)
// Exact-integer Gram for whole-width regions of 8/16/32-bit samples.  Each
// sample becomes a 32-bit fixed-point deviation v = round(x 2^f_b) - S_b (f_b,
// S_b from shift_kernel; exact for integer samples and for floats within the
// grid), split into four balanced signed bytes d_0..d_3 (v = sum_i d_i 2^8i).
// Per 256-pixel tile the CTA writes the digit planes as a K-major int8 operand
//   rows r = 32 i + b  (digit i of band b), 128 rows, K = pixels,
// plus 16 rows of which row 128 is all ones, and one thread issues
//   tcgen05.mma.kind::i8  D[128 x 144] += A[128 x 32 px] . B[144 x 32 px]^T
// with A = the digit rows and B = digit rows + ones rows (same shared memory).
// D[32i + b1][32j + b2] = sum_px d_i(b1) d_j(b2) accumulates exactly in int32
// TMEM (|d| <= 128, 2^16 pixels per window); D[32i + b1][128] = sum_px d_i(b1).
// At each window end the four epilogue warps (warp % 4 = i reads TMEM lanes
// 32i..32i+31) fold T_i[b1][b2] = sum_j 2^8j D[32i+b1][32j+b2] into int64
// registers; two TMEM accumulators ping-pong so the MMAs never wait.  Partials
// (int64, [G][4][32][33]) are summed by imma_merge_kernel in int128: the Gram
// sum_px v v^T, the sums sum_px v and hence M2 = (n S - s s^T) / n are exact
// integers until one final rounding to fp64 -- independent of G and order.
// Producer warps (4): bulk-async copies of the B band rows of a tile into a 4-stage
// ring; 8 converter warps: lane = band, 16 pixels per task (4 LDS.128 ->
// widen, one DFMA with the magic constant -> balanced bytes -> byte transpose
// -> 4 STS.128 into the operand); MMA warp: TMEM allocation + issue.
constexpr int kImP = 256;                 // pixels per tile
#ifndef UT_IM_SIN   // measured on B200 (8192 x 16384 x 32 f32): 4 / 64 / 8 best of
#define UT_IM_SIN 4  // {3,4,5} x {64,128}; 32-pixel buffers (1 MMA per commit) are slower
#define UT_IM_OPP 64
#define UT_IM_SOP 8
#endif
#ifndef UT_IM_SLEEP  // suspend-time hint (ns) of the ring waits; 0 = spin on try_wait
#define UT_IM_SLEEP 0
#endif
#ifndef UT_IM_EPI_SLEEP  // ns between polls of the epilogue warps' accumulator waits; 0 = spin
#define UT_IM_EPI_SLEEP 0
#endif
#ifndef UT_IM_DSUM   // independent fp64 accumulators of the converters' sample sums
#define UT_IM_DSUM 1
#endif
constexpr int kImStagesIn = UT_IM_SIN;    // input ring: [32][256 + pad] sample rows per stage
constexpr int kImOpP = UT_IM_OPP;         // pixels per operand buffer (MMAs of K = 32)
constexpr int kImStagesOp = UT_IM_SOP;    // operand ring
constexpr int kImProd = 4;                // producer warps (one thread's bulk copies issue slowly)
constexpr int kImConv = kImP / 16;        // converter warps: one 16-pixel chunk of every tile
#ifndef UT_IM_EPI_DED  // 1: four dedicated epilogue warps (converters never stop for a flush)
#define UT_IM_EPI_DED 1
#endif
constexpr int kImThreads = (kImProd + 1 + kImConv + (UT_IM_EPI_DED ? 4 : 0)) * 32;
constexpr int kImEpi = 8;                 // epilogue warps 8..11 (converters; warp % 4 = digit)
static_assert(kImEpi >= kImProd + 1 && kImEpi + 4 <= kImProd + 1 + kImConv, "epilogue warps");
constexpr int kImBars = 2 * kImStagesIn + 2 * kImStagesOp + 4;
constexpr int kImRows = 144;              // 128 digit rows + 16 (row 128 = ones)
constexpr int kImChunk = kImRows * 16;    // bytes per 16-pixel K chunk (LBO)
constexpr int kImOpBytes = kImChunk * (kImOpP / 16);
constexpr int kImWindowTiles = 32768 / kImP;  // int32 sums of u8 x u8 exact for 2^15 pixels
constexpr int kImMaxWindows = 200;            // per CTA: int64 records stay below 2^63
constexpr int kImRec = 4 * kMaxBands * (kMaxBands + 1) + kMaxBands;  // 8-byte words per CTA

template <typename T> constexpr int im_ps() { return kImP + 16 / (int)sizeof(T); }  // bank skew

template <typename T>
constexpr size_t im_smem() {
  return (size_t)kImStagesIn * kMaxBands * im_ps<T>() * sizeof(T) +
         (size_t)kImStagesOp * kImOpBytes + kImBars * sizeof(uint64_t);
}

struct ImParams {
  const void* data;   // first pixel of the region (band 0)
  int64_t bs;
  int64_t npix;
  int bands;
  int G;
  const double* scale;
  const double* addend;
  int* flag;
  int dbg;            // dev probes: 1 = no MMA, 2 = no conversion
  long long* part;    // [G]: int64 [4][32][33] digit-row records, then fp64 [32] sums of x - s
};

__device__ __forceinline__ void im_wait(uint64_t* bar, uint32_t parity) {
  if (UT_IM_SLEEP > 0) mbar_wait_sleep(bar, parity, UT_IM_SLEEP);
  else mbar_wait(bar, parity);
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  // K-major, no swizzle: 8-row x 16-byte core matrices; rows of a core matrix
  // 16 B apart, core matrices along M/N (SBO) 128 B apart, along K (LBO) one
  // 16-pixel chunk (kImChunk) apart.  Version 1 (sm_100).
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((kImChunk >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((128 >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// kind::i8 instruction descriptor: s32 accumulate, unsigned A and B, both K-major,
// N = 144, M = 128.
#ifndef UT_IM_PROBE_N    // dev probe (timing only): N of the MMA; B starts at row 144 - N
#define UT_IM_PROBE_N kImRows
#endif
constexpr uint32_t kImIdesc = (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(UT_IM_PROBE_N >> 3) << 17) |
                              ((uint32_t)(128 >> 4) << 24);

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma_i8(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem),
      "l"(ad), "l"(bd), "r"(kImIdesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc_ld16(uint32_t taddr, int* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tc_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Widening for the converters: fp32 (and fp16 via fp32) through F2F, which
// runs on its own pipe (~16/clk/SM) -- the ALU pipe is the converters' limit;
// 8/16-bit integers through the fp64 magic-number trick.
template <typename T> __device__ __forceinline__ double im_widen(T x) { return widen_f64(x); }
template <> __device__ __forceinline__ double im_widen<float>(float x) { return (double)x; }
template <> __device__ __forceinline__ double im_widen<__half>(__half x) { return (double)__half2float(x); }

// byte transpose of a 4x4 block: out[i] = byte i of (a, b, c, d)
__device__ __forceinline__ void transpose4(uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                           uint32_t* out) {
  const uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(a, b, 0x7362);
  const uint32_t t2 = __byte_perm(c, d, 0x5140), t3 = __byte_perm(c, d, 0x7362);
  out[0] = __byte_perm(t0, t2, 0x5410);
  out[1] = __byte_perm(t0, t2, 0x7632);
  out[2] = __byte_perm(t1, t3, 0x5410);
  out[3] = __byte_perm(t1, t3, 0x7632);
}

#ifdef UT_K2_PROBE  // dev builds: %globaltimer at entry / exit of every CTA
__device__ unsigned long long g_k2_probe[2 * 160];
#endif

template <typename T>
__global__ void __launch_bounds__(kImThreads, 1)
region_imma_kernel(ImParams r) {
#ifdef UT_K2_PROBE
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_k2_probe[2 * blockIdx.x] = t;
  }
#endif
  extern __shared__ __align__(128) unsigned char dyn_im[];
  constexpr int PS = im_ps<T>();
  const int B = r.bands;
  T* in = reinterpret_cast<T*>(dyn_im);                          // [stage][32][PS]
  unsigned char* op = dyn_im + (size_t)kImStagesIn * kMaxBands * PS * sizeof(T);
  uint64_t* bars = reinterpret_cast<uint64_t*>(op + (size_t)kImStagesOp * kImOpBytes);
  uint64_t* in_full = bars;
  uint64_t* in_empty = in_full + kImStagesIn;
  uint64_t* op_full = in_empty + kImStagesIn;
  uint64_t* op_empty = op_full + kImStagesOp;
  uint64_t* acc_full = op_empty + kImStagesOp;    // [2]
  uint64_t* acc_empty = acc_full + 2;             // [2]
  __shared__ uint32_t tmem_base;
  __shared__ int bad_any;
  __shared__ double xsum[kImConv][kMaxBands];
  constexpr int CPB = kImOpP / 16;                // chunks (converter warps) per operand buffer
  constexpr int H = kImP / kImOpP;                // operand buffers per tile
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < kImStagesIn; ++i) {
      mbar_init(&in_full[i], kImProd);
      mbar_init(&in_empty[i], kImConv);
    }
    for (int i = 0; i < kImStagesOp; ++i) {
      mbar_init(&op_full[i], CPB);
      mbar_init(&op_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);
    }
    mbar_fence_init();
    bad_any = 0;
  }
  // operand buffers: rows of absent bands and rows 129..143 stay zero; row 128 is all ones
  for (int e = tid; e < kImStagesOp * kImOpBytes / 16; e += blockDim.x) {
    const int row = e % kImRows;
    const uint32_t v = row == 128 ? 0x01010101u : 0u;
    reinterpret_cast<uint4*>(op)[e] = make_uint4(v, v, v, v);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == kImProd) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  const int64_t ntiles = (r.npix + kImP - 1) / kImP;
  const int nloc = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / r.G + 1) : 0;

  if (warp < kImProd) {
    // ------------------------------------------------- producers (bands p, p+4, ...)
#if UT_IM_PROD_LANES   // the producer warps' lanes share the band copies
    {
      const uint64_t pol = policy_evict_first();
      const int nb = B > warp ? (B - 1 - warp) / kImProd + 1 : 0;
      for (int i = 0; i < nloc; ++i) {
        const int st = i % kImStagesIn;
        if (i >= kImStagesIn) im_wait(&in_empty[st], ((i / kImStagesIn) - 1) & 1);
        const int64_t p0 = ((int64_t)blockIdx.x + (int64_t)i * r.G) * kImP;
        const int64_t npx = (r.npix - p0) < kImP ? (r.npix - p0) : kImP;
        const uint32_t bytes = (uint32_t)(npx * sizeof(T));
        if (lane == 0) mbar_expect_tx(&in_full[st], bytes * (uint32_t)nb);
        __syncwarp();
        T* dst = in + (size_t)st * kMaxBands * PS;
        const T* src = static_cast<const T*>(r.data) + p0;
        for (int b = warp + kImProd * lane; b < B; b += kImProd * 32)
          bulk_g2s(dst + (size_t)b * PS, src + (int64_t)b * r.bs, bytes, &in_full[st], pol);
      }
    }
#else
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const int nb = B > warp ? (B - 1 - warp) / kImProd + 1 : 0;
      for (int i = 0; i < nloc; ++i) {
        const int st = i % kImStagesIn;
        if (i >= kImStagesIn) im_wait(&in_empty[st], ((i / kImStagesIn) - 1) & 1);
        const int64_t p0 = ((int64_t)blockIdx.x + (int64_t)i * r.G) * kImP;
        const int64_t npx = (r.npix - p0) < kImP ? (r.npix - p0) : kImP;
        const uint32_t bytes = (uint32_t)(npx * sizeof(T));
        mbar_expect_tx(&in_full[st], bytes * (uint32_t)nb);
        T* dst = in + (size_t)st * kMaxBands * PS;
        const T* src = static_cast<const T*>(r.data) + p0;
        for (int b = warp; b < B; b += kImProd)
          bulk_g2s(dst + (size_t)b * PS, src + (int64_t)b * r.bs, bytes, &in_full[st], pol);
      }
    }
#endif
  } else if (warp == kImProd) {
    // -------------------------------------------------------------- MMA issue
    if (lane == 0) {
      const uint32_t op0 = smem_u32(op);
      for (int u = 0; u < H * nloc; ++u) {
        const int o = u % kImStagesOp;
        im_wait(&op_full[o], (u / kImStagesOp) & 1);
        const int w = u / (H * kImWindowTiles), a = w & 1;
        const bool first = (u % (H * kImWindowTiles)) == 0;
        const bool last = (u % (H * kImWindowTiles)) == H * kImWindowTiles - 1 || u == H * nloc - 1;
        if (first && w >= 2) mbar_wait(&acc_empty[a], ((w >> 1) - 1) & 1);
        tc_fence_after();
        if (r.dbg & 1) {
          mbar_arrive(&op_empty[o]);
          if (last) mbar_arrive(&acc_full[a]);
          continue;
        }
        const uint32_t base = op0 + (uint32_t)(o * kImOpBytes);
#pragma unroll
        for (int kk = 0; kk < kImOpP / 32; ++kk) {
          const uint64_t d = umma_desc(base + (uint32_t)(kk * 2 * kImChunk));
          const uint64_t db = umma_desc(base + (uint32_t)(kk * 2 * kImChunk) + (uint32_t)((kImRows - UT_IM_PROBE_N) * 16));
          tc_mma_i8(tmem + (uint32_t)(a * 256), d, db, (first && kk == 0) ? 0u : 1u);
        }
        tc_commit(&op_empty[o]);
        if (last) tc_commit(&acc_full[a]);
      }
    }
  } else {
    // -------------------------------------------------- converters + epilogue
    // warp cw converts chunk cw (pixels 16 cw .. 16 cw + 15) of every tile; lane = band
    const int cw = warp - kImProd - 1;
    const bool ded = UT_IM_EPI_DED && warp >= kImProd + 1 + kImConv;  // dedicated epilogue
    const bool epi = ded || (!UT_IM_EPI_DED && warp >= kImEpi && warp < kImEpi + 4);
    const int b = lane;
    const double scale = b < B ? r.scale[b] : 0.0;
    const double addend = b < B ? r.addend[b] : 0.0;
    double dsum[UT_IM_DSUM];  // fp64 sums of the samples: the mean does not see the grid
#pragma unroll
    for (int q = 0; q < UT_IM_DSUM; ++q) dsum[q] = 0.0;
    uint32_t bad = 0;
    // epilogue thread: digit row 32 i + b, 32 Gram columns + the ones column
    long long* rec = r.part + (size_t)blockIdx.x * kImRec +
                     ((size_t)(warp & 3) * kMaxBands + b) * (kMaxBands + 1);
    if (epi)
      for (int q = 0; q <= kMaxBands; ++q) rec[q] = 0;
    auto flush = [&](int w) {  // fold window w's TMEM accumulator into rec (int64)
      const int a = w & 1;
#if UT_IM_EPI_SLEEP > 0
      while (!mbar_test(&acc_full[a], (w >> 1) & 1)) __nanosleep(UT_IM_EPI_SLEEP);
#else
      mbar_wait(&acc_full[a], (w >> 1) & 1);
#endif
      tc_fence_after();
      const uint32_t t0 = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(a * 256);
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        long long s16[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) s16[q] = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          int v[16];
          tc_ld16(t0 + 32 * j + 16 * g, v);
          tc_wait_ld();
#pragma unroll
          for (int q = 0; q < 16; ++q) s16[q] += (long long)(unsigned)v[q] * (1LL << (8 * j));
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) rec[16 * g + q] += s16[q];
      }
      {
        int v[16];
        tc_ld16(t0 + 128, v);
        tc_wait_ld();
        rec[kMaxBands] += (long long)(unsigned)v[0];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[a]);
    };
    if (ded) {
      for (int w = 0; nloc > 0 && w <= (nloc - 1) / kImWindowTiles; ++w) flush(w);
    }
    for (int i = 0; i < (ded ? 0 : nloc); ++i) {
      const int u = H * i + cw / CPB;
      const int st = i % kImStagesIn, o = u % kImStagesOp;
      im_wait(&in_full[st], (i / kImStagesIn) & 1);
      if (u >= kImStagesOp) im_wait(&op_empty[o], ((u / kImStagesOp) - 1) & 1);
      const int64_t p0 = ((int64_t)blockIdx.x + (int64_t)i * r.G) * kImP;
      const int npx = (int)((r.npix - p0) < kImP ? (r.npix - p0) : kImP);
      const T* stage = in + (size_t)st * kMaxBands * PS;
      if (b < B && !(r.dbg & 2)) {
        // digit d of band b -> row 32 d + b of the chunk
        uint4* dst = reinterpret_cast<uint4*>(op + (size_t)o * kImOpBytes + (cw % CPB) * kImChunk + b * 16);
        const int valid = npx - 16 * cw;
        if (valid <= 0) {  // chunk past the end: v = 0, i.e. every biased digit 0x80
#pragma unroll
          for (int d = 0; d < 4; ++d) dst[32 * d] = make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);
        } else {
          constexpr int V = 16 / sizeof(T);
          T x[16];
#pragma unroll
          for (int q = 0; q < 16 / V; ++q) {
#if defined(UT_IM_PROBE) && (UT_IM_PROBE & 1)   // dev probe: no shared-memory reads of the input
            uint4 fake;
            fake.x = fake.y = fake.z = fake.w = 0x3f000000u + (uint32_t)(i & 255) * 8u + (uint32_t)q;
            *reinterpret_cast<uint4*>(x + q * V) = fake;
#else
            *reinterpret_cast<uint4*>(x + q * V) =
                *reinterpret_cast<const uint4*>(stage + (size_t)b * PS + 16 * cw + q * V);
#endif
          }
          uint32_t wd[16];
          if (valid >= 16) {  // the common case: no masks
#pragma unroll
            for (int p = 0; p < 16; ++p) {
              const double xw = im_widen(x[p]);
              const double t = fma(xw, scale, addend);
#if !(defined(UT_IM_PROBE) && (UT_IM_PROBE & 4))   // dev probe 4: no range check, no sample sums
              bad |= (uint32_t)__double2hiint(t) ^ 0x43380000u;
              dsum[p % UT_IM_DSUM] += xw;
#endif
              wd[p] = (uint32_t)__double2loint(t);
            }
          } else {
#pragma unroll
            for (int p = 0; p < 16; ++p) {
              const double xw = im_widen(x[p]);
              const double t = fma(xw, scale, addend);
              const bool ok = p < valid;
              bad |= ok ? ((uint32_t)__double2hiint(t) ^ 0x43380000u) : 0u;
              wd[p] = ok ? (uint32_t)__double2loint(t) : 0x80808080u;  // v = 0 past the end
              dsum[p % UT_IM_DSUM] += ok ? xw : 0.0;
            }
          }
          uint32_t o0[4], o1[4], o2[4], o3[4];
          transpose4(wd[0], wd[1], wd[2], wd[3], o0);
          transpose4(wd[4], wd[5], wd[6], wd[7], o1);
          transpose4(wd[8], wd[9], wd[10], wd[11], o2);
          transpose4(wd[12], wd[13], wd[14], wd[15], o3);
#if defined(UT_IM_PROBE) && (UT_IM_PROBE & 2)   // dev probe: no operand stores
          if ((o0[0] ^ o1[1] ^ o2[2] ^ o3[3]) == 0x12345678u) dst[0] = make_uint4(o0[1], o1[2], o2[3], o3[0]);
#else
#pragma unroll
#ifdef UT_IM_PROBE_SKIPD0   // dev probe (timing only): three stored digits
          for (int d = 1; d < 4; ++d) dst[32 * d] = make_uint4(o0[d], o1[d], o2[d], o3[d]);
#else
          for (int d = 0; d < 4; ++d) dst[32 * d] = make_uint4(o0[d], o1[d], o2[d], o3[d]);
#endif
#endif
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&in_empty[st]);
        mbar_arrive(&op_full[o]);
      }
      if (epi && !UT_IM_EPI_DED && (i % kImWindowTiles) == 0 && i >= kImWindowTiles)
        flush(i / kImWindowTiles - 1);
    }
    if (epi && !UT_IM_EPI_DED && nloc > 0) flush((nloc - 1) / kImWindowTiles);
    if (bad) atomicOr(&bad_any, 1);
    double ds = dsum[0];
#pragma unroll
    for (int q = 1; q < UT_IM_DSUM; ++q) ds += dsum[q];
    if (!ded) xsum[cw][b] = ds;
  }
  tc_fence_before();
  __syncthreads();
#ifdef UT_K2_PROBE
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_k2_probe[2 * blockIdx.x + 1] = t;
  }
#endif
  if (tid == 0 && bad_any) atomicOr(r.flag, 1);
  if (tid < kMaxBands) {  // fixed order over the converter warps
    double v = 0.0;
    for (int w = 0; w < kImConv; ++w) v += xsum[w][tid];
    reinterpret_cast<double*>(r.part + (size_t)blockIdx.x * kImRec + 4 * kMaxBands * (kMaxBands + 1))[tid] = v;
  }
  if (warp == kImProd) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// int128 helpers (exact sums of the integer path)
__device__ __forceinline__ __int128 shfl_xor_i128(__int128 v, int o) {
  const long long lo = (long long)(unsigned long long)v, hi = (long long)(v >> 64);
  const long long l2 = __shfl_xor_sync(0xffffffffu, lo, o), h2 = __shfl_xor_sync(0xffffffffu, hi, o);
  return ((__int128)h2 << 64) | (__int128)(unsigned long long)l2;
}
__device__ __forceinline__ double i128_to_f64(__int128 v) {
  // on the magnitude: two's-complement low words of small negatives are ~2^64
  const bool neg = v < 0;
  const unsigned __int128 m = neg ? (unsigned __int128)(-v) : (unsigned __int128)v;
  const double d = fma((double)(unsigned long long)(m >> 64), 0x1p64, (double)(unsigned long long)m);
  return neg ? -d : d;
}

// moments = [n, mean, M2] from the integer partials; one warp per entry.
__global__ void __launch_bounds__(256)
imma_merge_kernel(ImParams r, const int* __restrict__ fexp,
                  double* __restrict__ moments) {
  if (*r.flag) return;  // the fp64 path redoes this region
  const int B = r.bands, G = r.G;
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int total = 1 + B + B * B;
  if (e >= total) return;
  constexpr int ld = kMaxBands + 1;
  auto sum = [&](int b1, int q) {  // sum_g sum_i 2^8i part[g][i][b1][q]
    __int128 a = 0;
    for (int g = lane; g < G; g += 32) {
      const long long* p = r.part + (size_t)g * kImRec + (size_t)b1 * ld + q;
#pragma unroll
      for (int i = 0; i < 4; ++i) a += (__int128)p[(size_t)i * kMaxBands * ld] * (__int128)(1LL << (8 * i));
    }
    for (int o = 16; o > 0; o >>= 1) a += shfl_xor_i128(a, o);
    return a;
  };
  const long long n = r.npix;
  double v;
  if (e == 0) {
    v = (double)n;
  } else if (e <= B) {
    const int b = e - 1;
    // mean = sum x / n from the fp64 sums (exact to rounding even where
    // samples fall between grid points)
    double a = 0.0;
    for (int g = lane; g < G; g += 32)
      a += reinterpret_cast<const double*>(r.part + (size_t)g * kImRec + 4 * kMaxBands * ld)[b];
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    v = a / (double)n;
  } else {
    const int q = e - 1 - B, i = q / B, j = q - i * B;
    // every processed pixel slot (padding included) carries w = v + K, K = 0x80808080
    const __int128 np = (__int128)((n + kImP - 1) / kImP) * kImP;
    const __int128 K = 0x80808080LL;
    const __int128 wij = sum(i, j), wi = sum(i, kMaxBands), wj = sum(j, kMaxBands);
    const __int128 si = wi - np * K, sj = wj - np * K;      // sum v
    const __int128 sij = wij - K * (wi + wj) + np * K * K;  // sum v v
    const __int128 num = (__int128)n * sij - si * sj;       // n * M2 * 2^(fi + fj), exact
    v = ldexp(i128_to_f64(num) / (double)n, -(fexp[i] + fexp[j]));
  }
  if (lane == 0) moments[e] = v;
}

static_assert(148 * kImRec <= kMaxG * kEnt, "integer partials must fit the region workspace");

template <typename T>
int launch_region_imma(const Region& r, RegionWs ws, double* moments, int G, cudaStream_t st) {
  shift_kernel<T><<<r.bands, 1024, 0, st>>>(r, ws);
  UT_CHECK_LAUNCH("shift_kernel");
  ImParams ip;
  ip.data = static_cast<const T*>(r.data) + r.y0 * r.rs + r.x0;
  ip.bs = r.bs;
  ip.npix = r.npix;
  ip.bands = r.bands;
  ip.G = G;
  ip.scale = ws.scale;
  ip.addend = ws.addend;
  ip.flag = ws.flag;
  {
    const char* e = getenv("UT_IMMA_DEBUG");
    ip.dbg = e ? atoi(e) : 0;
  }
  ip.part = reinterpret_cast<long long*>(ws.part);
  auto kern = region_imma_kernel<T>;
  constexpr size_t smem = im_smem<T>();
  static SmemAttr attr;
  if (int rc = ensure_smem(attr, kern, smem, "region_imma smem attribute")) return rc;
  kern<<<G, kImThreads, smem, st>>>(ip);
  UT_CHECK_LAUNCH("region_imma_kernel");
  const int total = 1 + r.bands + r.bands * r.bands;
  imma_merge_kernel<<<(total + 7) / 8, 256, 0, st>>>(ip, ws.fexp, moments);
  UT_CHECK_LAUNCH("imma_merge_kernel");
  return UT_OK;
}

template <typename T, int NG>
int launch_region_dmma_ng(RdParams& rp, double* moments, cudaStream_t st) {
  auto kern = region_dmma_kernel<T, NG>;
  const size_t smem = rd_smem<T>(rp.bands);
  static SmemAttr attr;
  if (int rc = ensure_smem(attr, kern, smem, "region_dmma smem attribute")) return rc;
  kern<<<rp.G, kRdCons + 32, smem, st>>>(rp);
  UT_CHECK_LAUNCH("region_dmma_kernel");
  const int total = 1 + rp.bands + rp.bands * rp.bands;
  region_dmma_merge_kernel<<<(total + 7) / 8, 256, 0, st>>>(rp, moments);
  UT_CHECK_LAUNCH("region_dmma_merge_kernel");
  return UT_OK;
}

// gate: nullptr, or the integer path's flag (then ws.shift is already set and
// the kernels run only if the integer path flagged the region)
template <typename T>
int launch_region_dmma(const Region& r, RegionWs ws, double* moments, cudaStream_t st,
                       const int* gate = nullptr) {
  if (!gate) {
    shift_kernel<T><<<r.bands, 1024, 0, st>>>(r, ws);
    UT_CHECK_LAUNCH("shift_kernel");
  }
  RdParams rp;
  rp.gate = gate;
  rp.data = static_cast<const T*>(r.data) + r.y0 * r.rs + r.x0;
  rp.bs = r.bs;
  rp.npix = r.npix;
  rp.bands = r.bands;
  const int64_t ntiles = (r.npix + kRdP - 1) / kRdP;
  // fixed by the band count (not the device's SM count): results independent of the
  // GPU.  Up to 16 bands two CTAs fit an SM (3 stages x 16 bands x 2 KB = 99 KB each):
  // twice the warps hide the LDS -> F2F -> DMMA latency (cfg 2: K2' 114 -> see DESIGN)
#ifndef UT_RD_G2
#define UT_RD_G2 1
#endif
  const int64_t g = (UT_RD_G2 && rd_smem<T>(r.bands) <= 100 * 1024) ? 296 : 148;
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

// The integer path pays per sample (conversion) where the fp64 tensor-core path
// pays per band pair: it wins from ~17 bands up (B200: 32 bands 9.0 vs 14.9 ms
// at 16384^2 f32; 16 bands the fp64 path is HBM-bound already).  Read per call
// (tests switch it): UT_REGION_IMMA=0 disables it, UT_IMMA_MIN_BANDS moves the cut.
bool region_imma_enabled(int bands) {
  const char* e = getenv("UT_REGION_IMMA");
  if (e && e[0] == '0') return false;
  const char* m = getenv("UT_IMMA_MIN_BANDS");
  return bands >= (m ? atoi(m) : 17);
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
  shift_kernel<T><<<r.bands, 1024, 0, st>>>(r, ws);
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

namespace {
thread_local int g_region_path = -1;  // path of this thread's last ut_region_moments
}

extern "C" {

#ifdef UT_K2_PROBE
int ut_debug_k2_probe(unsigned long long* host) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(host, g_k2_probe, sizeof(g_k2_probe)) == cudaSuccess ? 0 : 3;
}
#endif

int32_t ut_region_last_path(void) { return g_region_path; }

int64_t ut_region_flag_offset(void) {
  RegionWs ws;
  char* base = reinterpret_cast<char*>(4096);
  region_ws_layout(&ws, base);
  return reinterpret_cast<char*>(ws.flag) - base;
}

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
  // 8/16/32-bit samples: exact integer Gram on the int8 tensor cores, with the
  // fp64 tensor-core path queued behind it, gated on the integer path's range flag
  const int G_im = sm_count() < 148 ? sm_count() : 148;   // part[] holds 148 records
  const bool imma_ok = dmma_ok && region_imma_enabled(cube->bands) && cube->dtype != UT_F64 &&
                       (r.npix + kImP - 1) / kImP <= (int64_t)G_im * kImMaxWindows * kImWindowTiles;
  g_region_path = imma_ok ? UT_REGION_PATH_IMMA : dmma_ok ? UT_REGION_PATH_DMMA : UT_REGION_PATH_DFMA;
  if (imma_ok) {
    int rc = UT_OK;
    switch (cube->dtype) {
      case UT_U8: rc = launch_region_imma<uint8_t>(r, ws, moments, G_im, st); break;
      case UT_U16: rc = launch_region_imma<uint16_t>(r, ws, moments, G_im, st); break;
      case UT_F16: rc = launch_region_imma<__half>(r, ws, moments, G_im, st); break;
      default: rc = launch_region_imma<float>(r, ws, moments, G_im, st); break;
    }
    if (rc != UT_OK) return rc;
    switch (cube->dtype) {
      case UT_U8: return launch_region_dmma<uint8_t>(r, ws, moments, st, ws.flag);
      case UT_U16: return launch_region_dmma<uint16_t>(r, ws, moments, st, ws.flag);
      case UT_F16: return launch_region_dmma<__half>(r, ws, moments, st, ws.flag);
      default: return launch_region_dmma<float>(r, ws, moments, st, ws.flag);
    }
  }
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
