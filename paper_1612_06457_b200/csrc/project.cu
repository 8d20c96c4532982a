// K4 + K5: per-pixel projection fused with the global min/max, and the
// full-range uint8/uint16 stretch.
//
// Reference: project_stack / _project_rows (projection.py:371-439),
// rescale_full (rendering.py:124-130), linear_to_codes / round_half_away
// (quantize.py:13-46).
//
// K4 streams the band-sequential cube once (HBM-bound: B*s bytes per pixel),
// each thread owning VEC adjacent pixels and issuing one 4/8/16-byte
// L1-bypassing load per band, eight bands in flight.  Per pixel it forms
// score_k = sum_b w_bk (x_b - m_b) in fixed band order, writes the fp32 score
// planes with streaming stores, and keeps a running min/max per component; the
// CTA partials are merged in fixed order by the last CTA to finish, so the
// result is deterministic and needs no init kernel.  The min is stored negated
// ([-min.., max..]) so a MAX all-reduce merges row shards.
//
// K5 re-reads the fp32 planes and applies the reference's arithmetic exactly
// in fp64: code = floor(clip((v - lo) * (top / (hi - lo)), 0, top) + 0.5).
#include <cstdlib>

#include "common.cuh"

#ifndef UT_PROD_LANES   // project_tma_kernel: the producer warp's lanes share the band copies
#define UT_PROD_LANES 1     // (cfg 3: K4 0.531 -> 0.443 ms; 0 = one lane issues them all)
#endif
#ifndef UT_DMMA_DYNAMIC     // project_dmma_kernel: tiles by global ticket (1) or static round-robin (0)
#define UT_DMMA_DYNAMIC 1
#endif
#ifndef UT_DMMA_PROD_LANES  // project_dmma_kernel: its two producer warps each issue from one
#define UT_DMMA_PROD_LANES 0  // lane (all lanes measured 0.4% slower on the cfg 4 step)
#endif

namespace ut {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxGroup = 8;      // components per pass over the cube
constexpr int kMaxGroups = 4;     // 4 * 8 = 32 >= B >= K
constexpr int kMaxGrid = 4096;
constexpr int kBandUnroll = 8;

struct ProjParams {
  const void* data;
  int64_t bs, rs, rows, cols, npix;
  int bands;
  int k0, ktotal;          // this pass covers components [k0, k0 + KG) of ktotal
  int comps[kMaxGroup];    // column of coef for each component of this pass
  const double* coef;
  int ld_coef;
  const double* mean;
  const double* std;       // nullable
  float* scores;           // plane (k0 + k) at scores + (k0 + k) * npix
  float* minmax;           // 2 * ktotal
  int* nonfinite;
  float* part;             // [grid][2 * KG]
  unsigned int* counter;
  unsigned int* tiles;     // tile tickets of the dynamically scheduled kernels (zero between launches)
};

template <int BYTES> struct Ld;
template <> struct Ld<16> {
  using U = uint4;
  __device__ __forceinline__ static U load(const void* p) { return ld_stream_u4(p); }
};
template <> struct Ld<8> {
  using U = uint2;
  __device__ __forceinline__ static U load(const void* p) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
  }
};
template <> struct Ld<4> {
  using U = uint32_t;
  __device__ __forceinline__ static U load(const void* p) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
  }
};

// Centred sample in the accumulation type.  In the fp32 path the mean is split
// as hi + lo (hi = fp32(mean)); the lo part is folded into a per-component
// fp64-computed bias so the centring error is only the rounding of x - hi.
template <typename T> __device__ __forceinline__ float centred_f32(T x, float hi, double mean) {
  return to_f32(x) - hi;
}
template <> __device__ __forceinline__ float centred_f32<double>(double x, float, double mean) {
  return (float)(x - mean);
}

// Scores are always stored as fp32.
template <int VEC> __device__ __forceinline__ void store_scores(float* dst, const float* v) {
  if constexpr (VEC == 4) {
    st_stream_u4(dst, make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]),
                                 __float_as_uint(v[2]), __float_as_uint(v[3])));
  } else if constexpr (VEC == 8) {
    st_stream_u4(dst, make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]),
                                 __float_as_uint(v[2]), __float_as_uint(v[3])));
    st_stream_u4(dst + 4, make_uint4(__float_as_uint(v[4]), __float_as_uint(v[5]),
                                     __float_as_uint(v[6]), __float_as_uint(v[7])));
  } else if constexpr (VEC == 16) {
#pragma unroll
    for (int i = 0; i < 16; i += 4)
      st_stream_u4(dst + i, make_uint4(__float_as_uint(v[i]), __float_as_uint(v[i + 1]),
                                       __float_as_uint(v[i + 2]), __float_as_uint(v[i + 3])));
  } else if constexpr (VEC == 2) {
    asm volatile("st.global.cs.v2.f32 [%0], {%1,%2};" ::"l"(dst), "f"(v[0]), "f"(v[1]) : "memory");
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) dst[i] = v[i];
  }
}

template <typename T, int VEC, int KG, bool F64>
struct Proj {
  using Acc = typename std::conditional<F64, double, float>::type;
  static constexpr int LB = VEC * (int)sizeof(T);  // load bytes per band
  static_assert(LB >= 1, "");

  // shared: weights [B][KG], shifts [B], bias [KG]
  struct Smem {
    Acc w[kMaxBands][KG];
    float hi[kMaxBands];
    double mean[kMaxBands];
    Acc bias[KG];
    float red[16][2 * KG + 1];  // up to 16 warps (TMA kernel: 9)
  };

  __device__ static void setup(const ProjParams& p, Smem& s) {
    for (int e = threadIdx.x; e < p.bands * KG; e += blockDim.x) {
      const int b = e / KG, k = e - b * KG;
      double w = p.coef[(int64_t)b * p.ld_coef + p.comps[k]];
      if (p.std) w = w / p.std[b];
      s.w[b][k] = (Acc)w;
    }
    for (int b = threadIdx.x; b < p.bands; b += blockDim.x) {
      s.mean[b] = p.mean[b];
      s.hi[b] = (float)p.mean[b];
    }
    __syncthreads();
    if (threadIdx.x < KG) {
      const int k = threadIdx.x;
      double bias = 0.0;
      if (F64) {
        // fp64 path: score = bias + sum_b w_b x_b with bias = -sum_b w_b m_b
        // (no per-sample centring; the cancellation this leaves is ~1e-16 of
        // sum |w m|, far below the 1e-6 plane bar)
        for (int b = 0; b < p.bands; ++b) bias -= (double)s.w[b][k] * s.mean[b];
      } else if (!std::is_same<T, double>::value) {
        // bias = -sum_b w_f (mean_b - hi_b): exact hi/lo split of the mean
        // (fp64 samples are centred on the full mean in fp64 instead)
        for (int b = 0; b < p.bands; ++b)
          bias -= (double)s.w[b][k] * (s.mean[b] - (double)s.hi[b]);
      }
      s.bias[k] = (Acc)bias;
    }
    __syncthreads();
  }

  // One VEC-pixel group starting at pixel index `base` (vectorized, contiguous planes).
  __device__ static void group_vec(const ProjParams& p, const Smem& s, int64_t base, float* mn,
                                   float* mx, float& chk) {
    const char* src = static_cast<const char*>(p.data) + base * (int64_t)sizeof(T);
    const int64_t bstride = p.bs * (int64_t)sizeof(T);
    Acc acc[KG][VEC];
#pragma unroll
    for (int k = 0; k < KG; ++k)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[k][v] = s.bias[k];
    for (int b0 = 0; b0 < p.bands; b0 += kBandUnroll) {
      typename Ld<LB>::U raw[kBandUnroll];
#pragma unroll
      for (int u = 0; u < kBandUnroll; ++u)
        if (b0 + u < p.bands) raw[u] = Ld<LB>::load(src + (int64_t)(b0 + u) * bstride);
#pragma unroll
      for (int u = 0; u < kBandUnroll; ++u) {
        const int b = b0 + u;
        if (b < p.bands) {
          const T* xs = reinterpret_cast<const T*>(&raw[u]);
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            Acc d;
            if constexpr (F64) d = widen_f64(xs[v]);
            else d = centred_f32<T>(xs[v], s.hi[b], s.mean[b]);
#pragma unroll
            for (int k = 0; k < KG; ++k) acc[k][v] = fma(s.w[b][k], d, acc[k][v]);
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < KG; ++k) {
      float out[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        out[v] = (float)acc[k][v];
        mn[k] = fminf(mn[k], out[v]);
        mx[k] = fmaxf(mx[k], out[v]);
        chk = nan_guard(chk, out[v]);
      }
      store_scores<VEC>(p.scores + (int64_t)(p.k0 + k) * p.npix + base, out);
    }
  }

  // One VEC-pixel group read from a shared-memory stage [bands][P] (TMA path).
  __device__ static void group_smem(const ProjParams& p, const Smem& s, const T* stage, int P,
                                    int lp, int64_t base, float* mn, float* mx, float& chk) {
    Acc acc[KG][VEC];
#pragma unroll
    for (int k = 0; k < KG; ++k)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[k][v] = s.bias[k];
    using U = typename Ld<LB>::U;
#pragma unroll 4
    for (int b = 0; b < p.bands; ++b) {
      const U raw = *reinterpret_cast<const U*>(stage + (size_t)b * P + lp);
      const T* xs = reinterpret_cast<const T*>(&raw);
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        Acc d;
        if constexpr (F64) d = widen_f64(xs[v]);
        else d = centred_f32<T>(xs[v], s.hi[b], s.mean[b]);
#pragma unroll
        for (int k = 0; k < KG; ++k) acc[k][v] = fma(s.w[b][k], d, acc[k][v]);
      }
    }
#pragma unroll
    for (int k = 0; k < KG; ++k) {
      float out[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        out[v] = (float)acc[k][v];
        mn[k] = fminf(mn[k], out[v]);
        mx[k] = fmaxf(mx[k], out[v]);
        chk = nan_guard(chk, out[v]);
      }
      store_scores<VEC>(p.scores + (int64_t)(p.k0 + k) * p.npix + base, out);
    }
  }

  // One pixel with general strides (tails, views, misaligned inputs).
  __device__ static void pixel_any(const ProjParams& p, const Smem& s, int64_t pix, float* mn,
                                   float* mx, float& chk) {
    const int64_t row = pix / p.cols, col = pix - row * p.cols;
    const T* src = static_cast<const T*>(p.data) + row * p.rs + col;
    Acc acc[KG];
#pragma unroll
    for (int k = 0; k < KG; ++k) acc[k] = s.bias[k];
    for (int b = 0; b < p.bands; ++b) {
      const T x = src[(int64_t)b * p.bs];
      Acc d;
      if constexpr (F64) d = widen_f64(x);
      else d = centred_f32<T>(x, s.hi[b], s.mean[b]);
#pragma unroll
      for (int k = 0; k < KG; ++k) acc[k] = fma(s.w[b][k], d, acc[k]);
    }
#pragma unroll
    for (int k = 0; k < KG; ++k) {
      const float o = (float)acc[k];
      mn[k] = fminf(mn[k], o);
      mx[k] = fmaxf(mx[k], o);
      chk = nan_guard(chk, o);
      p.scores[(int64_t)(p.k0 + k) * p.npix + pix] = o;
    }
  }

  __device__ static void finish(const ProjParams& p, Smem& s, float* mn, float* mx, float chk) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < KG; ++k) {
      for (int o = 16; o > 0; o >>= 1) {
        mn[k] = fminf(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], o));
        mx[k] = fmaxf(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], o));
      }
    }
    for (int o = 16; o > 0; o >>= 1) chk += __shfl_xor_sync(0xffffffffu, chk, o);
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        s.red[warp][k] = -mn[k];
        s.red[warp][KG + k] = mx[k];
      }
      s.red[warp][2 * KG] = chk;
    }
    __syncthreads();
    if (threadIdx.x <= 2 * KG) {
      const int f = threadIdx.x;
      float r = s.red[0][f];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
        r = (f == 2 * KG) ? r + s.red[w][f] : fmaxf(r, s.red[w][f]);
      p.part[(int64_t)blockIdx.x * (2 * KG + 1) + f] = r;
    }
    if (last_block_ticket(p.counter)) {
      if (threadIdx.x <= 2 * KG) {
        const int f = threadIdx.x;
        float r = p.part[f];
        for (unsigned int g = 1; g < gridDim.x; ++g) {
          const float o = p.part[(int64_t)g * (2 * KG + 1) + f];
          r = (f == 2 * KG) ? r + o : fmaxf(r, o);
        }
        if (f == 2 * KG) {
          if (r != 0.0f) atomicOr(p.nonfinite, 1);  // NaN or Inf seen
        } else if (f < KG) {
          p.minmax[p.k0 + f] = r;
        } else {
          p.minmax[p.ktotal + p.k0 + (f - KG)] = r;
        }
      }
      if (threadIdx.x == 0) {
        *p.counter = 0u;
        *p.tiles = 0u;   // every CTA has left its tile loop
      }
    }
  }
};

template <typename T, int VEC, int KG, bool F64, bool VECTOR>
__global__ void __launch_bounds__(kThreads)
project_kernel(ProjParams p) {
  using P = Proj<T, VEC, KG, F64>;
  __shared__ typename P::Smem s;
  P::setup(p, s);
  float mn[KG], mx[KG], chk = 0.0f;
#pragma unroll
  for (int k = 0; k < KG; ++k) {
    mn[k] = INFINITY;
    mx[k] = -INFINITY;
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if constexpr (VECTOR) {
    const int64_t groups = p.npix / VEC;
    for (int64_t g = tid; g < groups; g += stride) P::group_vec(p, s, g * VEC, mn, mx, chk);
    for (int64_t pix = groups * VEC + tid; pix < p.npix; pix += stride)
      P::pixel_any(p, s, pix, mn, mx, chk);
  } else {
    for (int64_t pix = tid; pix < p.npix; pix += stride) P::pixel_any(p, s, pix, mn, mx, chk);
  }
  P::finish(p, s, mn, mx, chk);
}

// ---------------------------------------------------------------- K4 (TMA)
// Warp-specialized, persistent: warp 4 streams [bands][P]-sample tiles of the
// cube into a 3-stage shared-memory ring with bulk async copies (one per band
// per tile, completing on a transaction-count mbarrier); warps 0-3 consume
// them.  Decouples HBM latency from the FMA stream at one CTA per SM.
constexpr int kTmaStages = 3;
constexpr int kTmaStageBytes = 64 * 1024;

struct TmaShape {
  int P;       // pixels per tile
  int R;       // VEC-groups per consumer thread per tile
  size_t smem; // dynamic shared bytes
};

template <typename T, int VEC, int CONS>
TmaShape tma_shape(int bands) {
  const int unit = CONS * VEC;  // pixels when each consumer takes one group
  int R = kTmaStageBytes / (unit * bands * (int)sizeof(T));
  if (R < 1) R = 1;
  if (R > 8) R = 8;
  TmaShape sh;
  sh.P = unit * R;
  sh.R = R;
  sh.smem = (size_t)kTmaStages * sh.P * bands * sizeof(T) + 2 * kTmaStages * sizeof(uint64_t) + 128;
  return sh;
}

// CONS consumer threads + one producer warp.
template <typename T, int VEC, int KG, bool F64, int CONS>
__global__ void __launch_bounds__(CONS + 32, 1)
project_tma_kernel(ProjParams p, int P, int R) {
  using Pj = Proj<T, VEC, KG, F64>;
  __shared__ typename Pj::Smem s;
  extern __shared__ __align__(128) unsigned char dyn[];
  const int B = p.bands;
  T* stages = reinterpret_cast<T*>(dyn);
  uint64_t* full = reinterpret_cast<uint64_t*>(dyn + (size_t)kTmaStages * P * B * sizeof(T));
  uint64_t* empty = full + kTmaStages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < kTmaStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], CONS / 32);
    }
    mbar_fence_init();
  }
  Pj::setup(p, s);  // contains __syncthreads (all threads)
  float mn[KG], mx[KG], chk = 0.0f;
#pragma unroll
  for (int k = 0; k < KG; ++k) {
    mn[k] = INFINITY;
    mx[k] = -INFINITY;
  }
  const int64_t ntiles = (p.npix + P - 1) / P;
  if (warp == CONS / 32) {
    // producer warp: lane 0 arms the stage, every lane issues some band copies
    const uint64_t pol = policy_evict_first();
    int i = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int st = i % kTmaStages;
      const uint32_t ph = (uint32_t)(i / kTmaStages) & 1u;
      if (i >= kTmaStages) mbar_wait(&empty[st], ph ^ 1u);
      const int64_t p0 = t * P;
      const int64_t npx = (p.npix - p0) < P ? (p.npix - p0) : P;
      const uint32_t bytes = (uint32_t)(npx * sizeof(T));
      if (lane == 0) mbar_expect_tx(&full[st], bytes * (uint32_t)B);
      __syncwarp();
      T* dst = stages + (size_t)st * P * B;
      const T* src = static_cast<const T*>(p.data) + p0;
      for (int b = UT_PROD_LANES ? lane : (lane == 0 ? 0 : B); b < B; b += UT_PROD_LANES ? 32 : 1)
        bulk_g2s(dst + (size_t)b * P, src + (int64_t)b * p.bs, bytes, &full[st], pol);
    }
  } else {
    int i = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int st = i % kTmaStages;
      const uint32_t ph = (uint32_t)(i / kTmaStages) & 1u;
      mbar_wait(&full[st], ph);
      const int64_t p0 = t * P;
      const int64_t npx = (p.npix - p0) < P ? (p.npix - p0) : P;
      const T* stage = stages + (size_t)st * P * B;
      for (int r = 0; r < R; ++r) {
        const int lp = (r * CONS + tid) * VEC;
        if (lp + VEC <= npx) Pj::group_smem(p, s, stage, P, lp, p0 + lp, mn, mx, chk);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }
  Pj::finish(p, s, mn, mx, chk);
}

// ------------------------------------------------------- K4 (TMA + DMMA)
// fp64 projection on the FP64 tensor cores: scores (8 x px) = W^T (8 x 4) x
// X (4 x px) + bias, one mma.sync.m8n8k4.f64 per 4 bands x 8 pixels.  M = the
// (<= 8) components of this pass, K = bands, N = pixels.  The A fragments (the
// weights) stay in registers for the whole kernel; every sample is read from
// the shared-memory stage and widened to fp64 exactly once (B fragments).  Same
// producer / 3-stage bulk-copy ring as project_tma_kernel; 8 consumer warps
// per CTA, two CTAs per SM, each warp owning 32 pixels (4 MMA column groups) of
// a 256-pixel tile (4/8-byte samples).
constexpr int kDmmaCons = 256;
#ifndef UT_DMMA_F2F
#define UT_DMMA_F2F 4  // all groups on F2F: K4 7.0 -> 6.28 ms at cfg4 (ALU was the busier pipe)
#endif
#ifndef UT_DMMA_PROD
#define UT_DMMA_PROD 2
#endif
constexpr int kDmmaProd = UT_DMMA_PROD;  // producer warps: one thread's bulk copies issue ~80 clk apart
// 8-pixel MMA column groups per warp per tile: 64 pixels for 4/8-byte samples,
// 128 for 1/2-byte samples (keeps each band's bulk copy >= 2 KB)
template <typename T> constexpr int dmma_groups() { return sizeof(T) >= 4 ? 4 : 16; }
template <typename T> constexpr int dmma_p() { return (kDmmaCons / 32) * dmma_groups<T>() * 8; }
template <typename T> constexpr int dmma_pad() { return 32 / (int)sizeof(T); }  // 32 B

template <typename T>
size_t dmma_smem(int bands) {
  const int ps = dmma_p<T>() + dmma_pad<T>();
  return (size_t)kTmaStages * bands * ps * sizeof(T) + 2 * kTmaStages * sizeof(uint64_t) + 128;
}

__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

#ifdef UT_K4_PROBE  // dev builds: %globaltimer at entry / main-loop end of every CTA
__device__ unsigned long long g_k4_probe[2 * 1024];
#endif

template <typename T, int KG>
__global__ void __launch_bounds__(kDmmaCons + 32 * kDmmaProd, 2)
project_dmma_kernel(ProjParams p) {
#ifdef UT_K4_PROBE
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_k4_probe[2 * blockIdx.x] = t;
  }
#endif
  using Pj = Proj<T, 1, KG, true>;
  __shared__ typename Pj::Smem s;
  extern __shared__ __align__(128) unsigned char dyn[];
  const int B = p.bands;
  constexpr int kDmmaGroups = dmma_groups<T>();
  constexpr int kDmmaP = dmma_p<T>();
  constexpr int PS = kDmmaP + dmma_pad<T>();  // padded stage row (bank spread)
  T* stages = reinterpret_cast<T*>(dyn);
  uint64_t* full = reinterpret_cast<uint64_t*>(dyn + (size_t)kTmaStages * B * PS * sizeof(T));
  uint64_t* empty = full + kTmaStages;
#if UT_DMMA_DYNAMIC
  // Tiles are handed out by a global ticket counter: CTAs on SMs that stream faster
  // (the per-CTA finish times of the static round-robin spread over 16% under
  // sustained load, profiles/r2/probes/k4_cta_spread.txt) take more tiles, so all
  // CTAs finish together.  Producer warp 0 draws the ticket of a stage (the next one
  // is in flight during the copies) and publishes it; the other producer and the
  // consumers read it from shared memory.  Scores, min/max (max-merged) and the
  // NaN flag do not depend on which CTA ran a tile.
  __shared__ long long tile_of[kTmaStages];
  __shared__ uint64_t pub[kTmaStages];
#endif
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < kTmaStages; ++i) {
      mbar_init(&full[i], kDmmaProd);
      mbar_init(&empty[i], kDmmaCons / 32);
#if UT_DMMA_DYNAMIC
      mbar_init(&pub[i], 1);
#endif
    }
    mbar_fence_init();
  }
  Pj::setup(p, s);  // fp64 weights and bias in shared memory (all threads)
  const int64_t ntiles = (p.npix + kDmmaP - 1) / kDmmaP;
  float mn[KG], mx[KG], chk = 0.0f;
#pragma unroll
  for (int k = 0; k < KG; ++k) {
    mn[k] = INFINITY;
    mx[k] = -INFINITY;
  }
  if (warp >= kDmmaCons / 32) {
    // producers: warp pw issues the rows of bands pw, pw + kDmmaProd, ...
    const int pw = warp - kDmmaCons / 32;
#if UT_DMMA_PROD_LANES   // every lane of the producer warp issues some of the band copies
    {
      const uint64_t pol = policy_evict_first();
      const int nb = B > pw ? (B - 1 - pw) / kDmmaProd + 1 : 0;
      int i = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int st = i % kTmaStages;
        const uint32_t ph = (uint32_t)(i / kTmaStages) & 1u;
        if (i >= kTmaStages) mbar_wait(&empty[st], ph ^ 1u);
        const int64_t p0 = t * kDmmaP;
        const int64_t npx = (p.npix - p0) < kDmmaP ? (p.npix - p0) : kDmmaP;
        const uint32_t bytes = (uint32_t)(npx * sizeof(T));
        if (lane == 0) mbar_expect_tx(&full[st], bytes * (uint32_t)nb);
        __syncwarp();
        T* dst = stages + (size_t)st * B * PS;
        const T* src = static_cast<const T*>(p.data) + p0;
        for (int b = pw + kDmmaProd * lane; b < B; b += kDmmaProd * 32)
          bulk_g2s(dst + (size_t)b * PS, src + (int64_t)b * p.bs, bytes, &full[st], pol);
      }
    }
#elif UT_DMMA_DYNAMIC
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const int nb = B > pw ? (B - 1 - pw) / kDmmaProd + 1 : 0;
      unsigned int ticket = 0u;
      if (pw == 0) ticket = atomicAdd(p.tiles, 1u);
      for (int i = 0;; ++i) {
        const int st = i % kTmaStages;
        const uint32_t ph = (uint32_t)(i / kTmaStages) & 1u;
        int64_t t;
        if (pw == 0) {
          if (i >= kTmaStages) mbar_wait(&empty[st], ph ^ 1u);
          t = (int64_t)ticket < ntiles ? (int64_t)ticket : -1;
          tile_of[st] = t;
          mbar_arrive(&pub[st]);
          if (t >= 0) ticket = atomicAdd(p.tiles, 1u);   // in flight during this tile's copies
        } else {
          mbar_wait(&pub[st], ph);
          t = tile_of[st];
        }
        if (t < 0) {   // no tiles left: wake the consumers and stop
          mbar_arrive(&full[st]);
          break;
        }
        const int64_t p0 = t * kDmmaP;
        const int64_t npx = (p.npix - p0) < kDmmaP ? (p.npix - p0) : kDmmaP;
        const uint32_t bytes = (uint32_t)(npx * sizeof(T));
        mbar_expect_tx(&full[st], bytes * (uint32_t)nb);
        T* dst = stages + (size_t)st * B * PS;
        const T* src = static_cast<const T*>(p.data) + p0;
        for (int b = pw; b < B; b += kDmmaProd)
          bulk_g2s(dst + (size_t)b * PS, src + (int64_t)b * p.bs, bytes, &full[st], pol);
      }
    }
#else
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const int nb = B > pw ? (B - 1 - pw) / kDmmaProd + 1 : 0;
      int i = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int st = i % kTmaStages;
        const uint32_t ph = (uint32_t)(i / kTmaStages) & 1u;
        if (i >= kTmaStages) mbar_wait(&empty[st], ph ^ 1u);
        const int64_t p0 = t * kDmmaP;
        const int64_t npx = (p.npix - p0) < kDmmaP ? (p.npix - p0) : kDmmaP;
        const uint32_t bytes = (uint32_t)(npx * sizeof(T));
        mbar_expect_tx(&full[st], bytes * (uint32_t)nb);
        T* dst = stages + (size_t)st * B * PS;
        const T* src = static_cast<const T*>(p.data) + p0;
        for (int b = pw; b < B; b += kDmmaProd)
          bulk_g2s(dst + (size_t)b * PS, src + (int64_t)b * p.bs, bytes, &full[st], pol);
      }
    }
#endif
  } else {
    // A fragments: A[m = lane/4][k = lane%4] = w[band 4q + lane%4][comp lane/4]
    const int am = lane >> 2, ak = lane & 3;
    double afrag[kMaxBands / 4];
#pragma unroll
    for (int q = 0; q < kMaxBands / 4; ++q) {
      const int b = 4 * q + ak;
      afrag[q] = (am < KG && b < B) ? (double)s.w[b][am] : 0.0;
    }
    const double bias = am < KG ? (double)s.bias[am] : 0.0;
    const int nq = (B + 3) / 4;
    float lmn = INFINITY, lmx = -INFINITY;  // this lane's component am
#if UT_DMMA_DYNAMIC && !UT_DMMA_PROD_LANES
    for (int i = 0;; ++i) {
      const int st = i % kTmaStages;
      const uint32_t ph = (uint32_t)(i / kTmaStages) & 1u;
      mbar_wait(&full[st], ph);
      const int64_t t = tile_of[st];
      if (t < 0) break;
#else
    int i = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int st = i % kTmaStages;
      const uint32_t ph = (uint32_t)(i / kTmaStages) & 1u;
      mbar_wait(&full[st], ph);
#endif
      const int64_t p0 = t * kDmmaP;
      const int64_t npx = (p.npix - p0) < kDmmaP ? (p.npix - p0) : kDmmaP;
      const T* stage = stages + (size_t)st * B * PS;
      const int wp0 = warp * (kDmmaGroups * 8);  // this warp's first pixel in the tile
      double c0[kDmmaGroups], c1[kDmmaGroups];
#pragma unroll
      for (int g = 0; g < kDmmaGroups; ++g) c0[g] = c1[g] = 0.0;
      // B fragment of group g: B[k = lane%4][n = lane/4] = x[band 4q + lane%4][pixel
      // wp0 + G n + g] (G = kDmmaGroups): a lane's G samples of a band are
      // consecutive, one vector load (16 B for fp32) instead of G scalar loads, and
      // its G scores of a component come out consecutive as well
      const int bk = lane & 3, bn = lane >> 2;
      __syncwarp();  // mma.sync.aligned: the whole warp, converged
#pragma unroll
      for (int q = 0; q < kMaxBands / 4; ++q) {
        if (q < nq) {  // warp-uniform
          const int b = 4 * q + bk;
          // lanes past the last band read band 0 (no branch: a divergent select
          // could split the warp around the mma); their A-fragment weights are
          // zero, so they add nothing -- a NaN / Inf there is a NaN / Inf of
          // this pixel's band 0, which its own term propagates as well and the
          // nonfinite guard reports
          const T* row = stage + (size_t)(b < B ? b : 0) * PS + wp0 + kDmmaGroups * bn;
          T xs[kDmmaGroups];
#pragma unroll
          for (int v = 0; v < (int)(kDmmaGroups * sizeof(T)) / 16; ++v)
            reinterpret_cast<uint4*>(xs)[v] = reinterpret_cast<const uint4*>(row)[v];
          double x[kDmmaGroups];
#pragma unroll
          for (int g = 0; g < kDmmaGroups; ++g)
            // the first UT_DMMA_F2F groups widen on the conversion pipe (F2F),
            // the rest with ALU bit operations
            x[g] = (g < UT_DMMA_F2F) ? to_f64(xs[g]) : widen_f64(xs[g]);
#pragma unroll
          for (int g = 0; g < kDmmaGroups; ++g) dmma_884(c0[g], c1[g], afrag[q], x[g]);
        }
      }
      // C[m = lane/4][n = 2 (lane%4) + h], h = 0, 1 (c0 / c1) -> scores of component m
      // at pixels wp0 + G n + g, g = 0 .. G - 1 (consecutive)
      if (am < KG) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int lp = wp0 + kDmmaGroups * (2 * (lane & 3) + h);
          float o[kDmmaGroups];
#pragma unroll
          for (int g = 0; g < kDmmaGroups; ++g) o[g] = (float)((h ? c1[g] : c0[g]) + bias);
          float* dst = p.scores + (int64_t)(p.k0 + am) * p.npix + p0 + lp;
          if (lp + kDmmaGroups <= npx) {
#pragma unroll
            for (int g = 0; g < kDmmaGroups; ++g) {
              lmn = fminf(lmn, o[g]);
              lmx = fmaxf(lmx, o[g]);
              chk = nan_guard(chk, o[g]);
            }
            store_scores<kDmmaGroups>(dst, o);
          } else {
#pragma unroll
            for (int g = 0; g < kDmmaGroups; ++g)
              if (lp + g < npx) {
                lmn = fminf(lmn, o[g]);
                lmx = fmaxf(lmx, o[g]);
                chk = nan_guard(chk, o[g]);
                dst[g] = o[g];
              }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
#pragma unroll
    for (int k = 0; k < KG; ++k)
      if (k == am) {
        mn[k] = lmn;
        mx[k] = lmx;
      }
  }
#ifdef UT_K4_PROBE
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_k4_probe[2 * blockIdx.x + 1] = t;
  }
#endif
  Pj::finish(p, s, mn, mx, chk);
}

template <typename T, int KG>
int launch_dmma(ProjParams& p, cudaStream_t st) {
  auto kern = project_dmma_kernel<T, KG>;
  const size_t smem = dmma_smem<T>(p.bands);
  static SmemAttr attr;
  if (int rc = ensure_smem(attr, kern, smem, "project_dmma smem attribute")) return rc;
  const int64_t ntiles = (p.npix + dmma_p<T>() - 1) / dmma_p<T>();
  int64_t grid = 2 * (int64_t)sm_count();  // two CTAs (2 x 8 consumer warps) per SM
  if (grid > ntiles) grid = ntiles;
  if (grid < 1) grid = 1;
  kern<<<(int)grid, kDmmaCons + 32 * kDmmaProd, smem, st>>>(p);
  UT_CHECK_LAUNCH("project_dmma_kernel");
  return UT_OK;
}

bool dmma_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("UT_PROJECT_DMMA");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

bool tma_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("UT_PROJECT_TMA");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <typename T, int VEC, int KG, bool F64, int CONS>
int launch_tma(ProjParams& p, cudaStream_t st) {
  auto kern = project_tma_kernel<T, VEC, KG, F64, CONS>;
  const TmaShape sh = tma_shape<T, VEC, CONS>(p.bands);
  static SmemAttr attr;
  if (int rc = ensure_smem(attr, kern, sh.smem, "project_tma smem attribute")) return rc;
  const int64_t ntiles = (p.npix + sh.P - 1) / sh.P;
  int64_t grid = sm_count();
  if (grid > ntiles) grid = ntiles;
  if (grid < 1) grid = 1;
  kern<<<(int)grid, CONS + 32, sh.smem, st>>>(p, sh.P, sh.R);
  UT_CHECK_LAUNCH("project_tma_kernel");
  return UT_OK;
}

template <typename T, int VEC, int KG, bool F64, bool VECTOR>
int launch_one(ProjParams& p, cudaStream_t st) {
  auto kern = project_kernel<T, VEC, KG, F64, VECTOR>;
  static int per_sm = 0;  // resident CTAs per SM for this instantiation
  if (per_sm == 0) {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kThreads, 0);
    per_sm = n > 0 ? n : 1;
  }
  const int64_t units = VECTOR ? (p.npix + VEC - 1) / VEC : p.npix;
  int64_t grid = (int64_t)per_sm * sm_count();
  const int64_t need = (units + kThreads - 1) / kThreads;
  if (grid > need) grid = need;
  if (grid > kMaxGrid) grid = kMaxGrid;
  if (grid < 1) grid = 1;
  kern<<<(int)grid, kThreads, 0, st>>>(p);
  UT_CHECK_LAUNCH("project_kernel");
  return UT_OK;
}

template <typename T, int KG, bool F64>
int launch_kg(ProjParams& p, bool vector_ok, cudaStream_t st) {
  // pixels per thread: one 16-byte load per band, capped so KG*VEC <= 32 accumulators
  constexpr int V16 = 16 / (int)sizeof(T);
  constexpr int VCAP = (32 / KG) >= 16 ? 16 : (32 / KG) >= 8 ? 8 : (32 / KG) >= 4 ? 4 : 2;
  constexpr int VEC = V16 < VCAP ? V16 : VCAP;
  constexpr int LB = VEC * (int)sizeof(T);
  const bool aligned = vector_ok &&
                       (reinterpret_cast<uintptr_t>(p.data) % LB == 0) &&
                       ((p.bs * (int64_t)sizeof(T)) % LB == 0) &&
                       (reinterpret_cast<uintptr_t>(p.scores) % 16 == 0) &&
                       (p.npix % 4 == 0);
  // TMA path: every bulk copy 16-byte aligned (plane starts, tile starts, and
  // the last partial tile); the npix % VEC tail would be skipped, so require 0.
  const bool tma_ok = aligned && tma_enabled() && (p.npix % VEC == 0) &&
                      ((p.npix * (int64_t)sizeof(T)) % 16 == 0) &&
                      (reinterpret_cast<uintptr_t>(p.data) % 16 == 0) &&
                      ((p.bs * (int64_t)sizeof(T)) % 16 == 0);
  if (tma_ok) {
    // fp64 accumulation is FMA-pipe heavy: 8 consumer warps, 2-4 pixels each;
    // fp32: 4 consumer warps with 16-byte groups.
    if constexpr (F64) {
      // even pixel count: scores are stored as aligned float2 pairs
      // DMMA pads the components to M = 8: worth it from 4 components up, and for
      // 4/8-byte samples (2-byte samples make the tile compute-bound)
      if (dmma_enabled() && sizeof(T) >= 4 && KG >= 4 && dmma_smem<T>(p.bands) <= 227 * 1024 &&
          (p.npix % 2) == 0)
        return launch_dmma<T, KG>(p, st);
      constexpr int VT = (16 / (int)sizeof(T)) < 2 ? 1 : ((8 / (int)sizeof(T)) < 2 ? 2 : 8 / (int)sizeof(T));
      // (wide fp64 cubes: one 512-pixel stage of > 18 bands would not fit three times
      // into shared memory -- those take the direct-load kernel below)
      if ((p.npix % VT) == 0 && tma_shape<T, VT, 256>(p.bands).smem <= 227 * 1024)
        return launch_tma<T, VT, KG, F64, 256>(p, st);
    } else if (tma_shape<T, VEC, 128>(p.bands).smem <= 227 * 1024) {
      return launch_tma<T, VEC, KG, F64, 128>(p, st);
    }
  }
  if (aligned) return launch_one<T, VEC, KG, F64, true>(p, st);
  return launch_one<T, 1, KG, F64, false>(p, st);
}

template <typename T, bool F64>
int launch_t(ProjParams& p, int kg, bool vector_ok, cudaStream_t st) {
  switch (kg) {
    case 1: return launch_kg<T, 1, F64>(p, vector_ok, st);
    case 2: return launch_kg<T, 2, F64>(p, vector_ok, st);
    case 3: return launch_kg<T, 3, F64>(p, vector_ok, st);
    case 4: return launch_kg<T, 4, F64>(p, vector_ok, st);
    case 5: return launch_kg<T, 5, F64>(p, vector_ok, st);
    case 6: return launch_kg<T, 6, F64>(p, vector_ok, st);
    case 7: return launch_kg<T, 7, F64>(p, vector_ok, st);
    case 8: return launch_kg<T, 8, F64>(p, vector_ok, st);
  }
  set_error("project: bad component group %d", kg);
  return UT_EDATA;
}

template <bool F64>
int launch_prec(ProjParams& p, int dtype, int kg, bool vector_ok, cudaStream_t st) {
  switch (dtype) {
    case UT_U8: return launch_t<uint8_t, F64>(p, kg, vector_ok, st);
    case UT_U16: return launch_t<uint16_t, F64>(p, kg, vector_ok, st);
    case UT_F16: return launch_t<__half, F64>(p, kg, vector_ok, st);
    case UT_F32: return launch_t<float, F64>(p, kg, vector_ok, st);
    case UT_F64: return launch_t<double, F64>(p, kg, vector_ok, st);
  }
  set_error("project: unknown dtype %d", dtype);
  return UT_EDATA;
}

// ------------------------------------------------------------------ K5
template <int DEPTH>
__global__ void __launch_bounds__(kThreads)
stretch_kernel(const float* __restrict__ scores, const float* __restrict__ minmax, int k,
               int ld_mm, int64_t npix, void* __restrict__ codes_raw, bool vec16) {
  using Code = typename std::conditional<DEPTH == 8, uint8_t, uint16_t>::type;
  constexpr double top = DEPTH == 8 ? 255.0 : 65535.0;
  __shared__ double lo_s[kMaxBands], sc_s[kMaxBands];
  __shared__ float lof_s[kMaxBands], scf_s[kMaxBands];
  __shared__ int flat_s[kMaxBands];
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    const double lo = -(double)minmax[c], hi = (double)minmax[ld_mm + c];
    lo_s[c] = lo;
    flat_s[c] = (lo == hi) || !(lo < hi);  // constant plane (rendering.py:128-129)
    sc_s[c] = flat_s[c] ? 0.0 : top / (hi - lo);
    lof_s[c] = (float)lo;
    scf_s[c] = (float)sc_s[c];
  }
  __syncthreads();
  Code* codes = static_cast<Code*>(codes_raw);
  const int64_t total = (int64_t)k * npix;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // Exact reference arithmetic in fp64: floor(clip((v - lo) * s, 0, top) + 0.5).
  // For 8-bit codes an fp32 evaluation is used first: its error is < 1e-4 code
  // units (|x| <= 255.5), so unless x lies within 2e-4 of a tie (k + 0.5),
  // round-to-nearest with saturation gives the same code; the rare near-tie
  // values are recomputed in fp64, so the result is bit-exact.
  struct Plane {
    double lo, sc;
    float lof, scf;
    bool flat;
  };
  auto plane_of = [&](int c) {
    Plane q;
    q.lo = lo_s[c];
    q.sc = sc_s[c];
    q.lof = lof_s[c];
    q.scf = scf_s[c];
    q.flat = flat_s[c] != 0;
    return q;
  };
  auto code_exact = [&](float v, const Plane& q) -> Code {
    double x = ((double)v - q.lo) * q.sc;
    x = fmin(fmax(x, 0.0), top);
    return (Code)(int)floor(x + 0.5);
  };
  auto code_of = [&](float v, const Plane& q) -> Code {
    if (q.flat) return (Code)0;
    return code_exact(v, q);
  };
  // 16 codes of one plane: fp32 fast path, exact fp64 redo if any is near a tie
  auto codes16 = [&](const float* v, const Plane& q, Code* out) {
    if (q.flat) {
#pragma unroll
      for (int i = 0; i < 16; ++i) out[i] = (Code)0;
      return;
    }
    if constexpr (DEPTH == 8) {
      bool tie = false;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float x = (v[i] - q.lof) * q.scf;
        tie |= fabsf(x - rintf(x)) >= 0.5f - 2e-4f;
        unsigned short u;
        asm("cvt.rni.sat.u8.f32 %0, %1;" : "=h"(u) : "f"(x));
        out[i] = (Code)u;
      }
      if (!tie) return;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = code_exact(v[i], q);
  };
  if (vec16) {
    // plane c = blockIdx.y; 16 consecutive scores per thread per step, two
    // steps' loads issued together (npix % 16 == 0)
    const int c = blockIdx.y;
    const Plane pl = plane_of(c);
    const float* src = scores + (int64_t)c * npix;
    Code* dst = codes + (int64_t)c * npix;
    const int64_t chunks = npix / 16;
    const int64_t step = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < chunks; q += 2 * step) {
      float v[2][16];
      const bool two = q + step < chunks;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1 && !two) break;
        const float* p = src + (q + h * step) * 16;
#pragma unroll
        for (int i = 0; i < 16; i += 4) {
          const uint4 u = ld_stream_u4(p + i);
          v[h][i] = __uint_as_float(u.x);
          v[h][i + 1] = __uint_as_float(u.y);
          v[h][i + 2] = __uint_as_float(u.z);
          v[h][i + 3] = __uint_as_float(u.w);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1 && !two) break;
        Code out[16];
        codes16(v[h], pl, out);
        Code* o = dst + (q + h * step) * 16;
        st_stream_u4(o, *reinterpret_cast<const uint4*>(out));
        if constexpr (DEPTH == 16) st_stream_u4(o + 8, *reinterpret_cast<const uint4*>(out + 8));
      }
    }
  } else {
    for (int64_t e = tid; e < total; e += stride)
      codes[e] = code_of(scores[e], plane_of((int)(e / npix)));
  }
}

// K5 on a bulk-copy ring: the fp32 score planes stream through shared memory
// (cp.async.bulk, 4 x 16 KB stages, one producer warp) so the loads in flight
// do not cost registers; 8 consumer warps turn 16 scores each per tile into
// codes with the same arithmetic as stretch_kernel (fp32 fast path, fp64 redo
// near ties, bit-exact) and store them straight to global memory.
#ifndef UT_K5_P
#define UT_K5_P 8192      // measured (cfg4, 5 planes): 4096 x 4: 1.11 ms, x 6: 1.08, 8192 x 2: 1.09, 8192 x 3: 1.01
#define UT_K5_STAGES 3
#endif
constexpr int kK5P = UT_K5_P;            // scores per tile (32 KB)
constexpr int kK5Stages = UT_K5_STAGES;
constexpr int kK5Cons = 256;      // consumer threads, 16 scores each per pass
static_assert(kK5P % (kK5Cons * 16) == 0, "a tile is whole consumer passes");

template <int DEPTH>
struct StretchPlane {
  using Code = typename std::conditional<DEPTH == 8, uint8_t, uint16_t>::type;
  static constexpr double top = DEPTH == 8 ? 255.0 : 65535.0;
  double lo, sc;
  float lof, scf;
  bool flat;
  __device__ __forceinline__ Code exact(float v) const {
    double x = ((double)v - lo) * sc;
    x = fmin(fmax(x, 0.0), top);
    return (Code)(int)floor(x + 0.5);
  }
  __device__ __forceinline__ void codes16(const float* v, Code* out) const {
    if (flat) {
#pragma unroll
      for (int i = 0; i < 16; ++i) out[i] = (Code)0;
      return;
    }
    if constexpr (DEPTH == 8) {
      bool tie = false;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float x = (v[i] - lof) * scf;
        tie |= fabsf(x - rintf(x)) >= 0.5f - 2e-4f;
        unsigned short u;
        asm("cvt.rni.sat.u8.f32 %0, %1;" : "=h"(u) : "f"(x));
        out[i] = (Code)u;
      }
      if (!tie) return;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = exact(v[i]);
  }
};

template <int DEPTH>
__global__ void __launch_bounds__(kK5Cons + 32, 2)
stretch_tma_kernel(const float* __restrict__ scores, const float* __restrict__ minmax, int k,
                   int ld_mm, int64_t npix, void* __restrict__ codes_raw) {
  using SP = StretchPlane<DEPTH>;
  using Code = typename SP::Code;
  extern __shared__ __align__(128) unsigned char k5dyn[];
  float* stages = reinterpret_cast<float*>(k5dyn);
  uint64_t* full = reinterpret_cast<uint64_t*>(k5dyn + (size_t)kK5Stages * kK5P * sizeof(float));
  uint64_t* empty = full + kK5Stages;
  __shared__ SP planes[kMaxBands];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int c = tid; c < k; c += blockDim.x) {
    SP q;
    const double lo = -(double)minmax[c], hi = (double)minmax[ld_mm + c];
    q.lo = lo;
    q.flat = (lo == hi) || !(lo < hi);  // constant plane (rendering.py:128-129)
    q.sc = q.flat ? 0.0 : SP::top / (hi - lo);
    q.lof = (float)lo;
    q.scf = (float)q.sc;
    planes[c] = q;
  }
  if (tid == 0) {
    for (int i = 0; i < kK5Stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kK5Cons / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t tpp = (npix + kK5P - 1) / kK5P;   // tiles per plane
  const int64_t ntiles = tpp * k;
  if (warp == kK5Cons / 32) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int i = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int st = i % kK5Stages;
        if (i >= kK5Stages) mbar_wait(&empty[st], ((i / kK5Stages) - 1) & 1);
        const int64_t c = t / tpp, off = (t - c * tpp) * kK5P;
        const int64_t n = (npix - off) < kK5P ? (npix - off) : kK5P;
        const uint32_t bytes = (uint32_t)(n * sizeof(float));
        mbar_expect_tx(&full[st], bytes);
        bulk_g2s(stages + (size_t)st * kK5P, scores + c * npix + off, bytes, &full[st], pol);
      }
    }
  } else {
    Code* codes = static_cast<Code*>(codes_raw);
    int i = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int st = i % kK5Stages;
      mbar_wait(&full[st], (i / kK5Stages) & 1);
      const int64_t c = t / tpp, off = (t - c * tpp) * kK5P;
      const int64_t n = (npix - off) < kK5P ? (npix - off) : kK5P;
#pragma unroll
      for (int r = 0; r < kK5P / (kK5Cons * 16); ++r) {
        const int lp = (r * kK5Cons + tid) * 16;
        if (lp + 16 <= n) {
          const float* src = stages + (size_t)st * kK5P + lp;
          float v[16];
#pragma unroll
          for (int q = 0; q < 16; q += 4)
            *reinterpret_cast<float4*>(v + q) = *reinterpret_cast<const float4*>(src + q);
          Code out[16];
          planes[c].codes16(v, out);
          Code* o = codes + c * npix + off + lp;
          st_stream_u4(o, *reinterpret_cast<const uint4*>(out));
          if constexpr (DEPTH == 16) st_stream_u4(o + 8, *reinterpret_cast<const uint4*>(out + 8));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }
}

constexpr size_t kK5Smem = (size_t)kK5Stages * kK5P * sizeof(float) + 2 * kK5Stages * sizeof(uint64_t);

template <int DEPTH>
int launch_stretch_tma(const float* scores, const float* minmax, int k, int ld_mm, int64_t npix,
                       void* codes, cudaStream_t st) {
  auto kern = stretch_tma_kernel<DEPTH>;
  static SmemAttr attr;
  if (int rc = ensure_smem(attr, kern, (size_t)kK5Smem, "stretch_tma smem attribute")) return rc;
  const int64_t ntiles = ((npix + kK5P - 1) / kK5P) * k;
  int64_t grid = 2 * (int64_t)sm_count();
  if (grid > ntiles) grid = ntiles;
  kern<<<(unsigned)grid, kK5Cons + 32, kK5Smem, st>>>(scores, minmax, k, ld_mm, npix, codes);
  UT_CHECK_LAUNCH("stretch_tma_kernel");
  return UT_OK;
}

bool k5_tma_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("UT_K5_TMA");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

}  // namespace
}  // namespace ut

using namespace ut;

extern "C" {

#ifdef UT_K4_PROBE
int ut_debug_k4_probe(unsigned long long* host) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(host, g_k4_probe, sizeof(g_k4_probe)) == cudaSuccess ? 0 : 3;
}
#endif

size_t ut_project_ws(void) {
  return 256 + sizeof(float) * (size_t)kMaxGroups * kMaxGrid * (2 * kMaxGroup + 1);
}

int ut_project_minmax(const ut_cube* cube, const double* coef, int32_t ld_coef,
                      const int32_t* components, int32_t k, const double* mean,
                      const double* std, int32_t precision, float* scores, float* minmax,
                      int32_t* nonfinite, void* ws, size_t ws_bytes, void* stream) {
  UT_REQUIRE(cube && cube->bands >= 1 && cube->bands <= kMaxBands,
             "ut_project_minmax: bands must be 1..32");
  UT_REQUIRE(k >= 1 && k <= kMaxGroup * kMaxGroups, "ut_project_minmax: k must be 1..32");
  UT_REQUIRE(ws_bytes >= ut_project_ws(), "ut_project_minmax: workspace too small");
  UT_REQUIRE(cube->rows >= 1 && cube->cols >= 1, "ut_project_minmax: empty cube");
  for (int i = 0; i < k; ++i)
    UT_REQUIRE(components[i] >= 0 && components[i] < ld_coef,
               "component %d out of range", components[i]);
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(ws, 0, 256, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(nonfinite, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return cuda_status(e, "ut_project_minmax memset");
  const bool vector_ok = cube->row_stride == cube->cols;
  ProjParams p{};
  p.data = cube->data;
  p.bs = cube->band_stride;
  p.rs = cube->row_stride;
  p.rows = cube->rows;
  p.cols = cube->cols;
  p.npix = cube->rows * cube->cols;
  p.bands = cube->bands;
  p.ktotal = k;
  p.coef = coef;
  p.ld_coef = ld_coef;
  p.mean = mean;
  p.std = std;
  p.scores = scores;
  p.minmax = minmax;
  p.nonfinite = nonfinite;
  char* base = static_cast<char*>(ws);
  for (int g = 0, k0 = 0; k0 < k; ++g, k0 += kMaxGroup) {
    const int kg = (k - k0) < kMaxGroup ? (k - k0) : kMaxGroup;
    p.k0 = k0;
    for (int i = 0; i < kg; ++i) p.comps[i] = components[k0 + i];
    p.counter = reinterpret_cast<unsigned int*>(base) + g;
    p.tiles = reinterpret_cast<unsigned int*>(base) + 16 + g;
    p.part = reinterpret_cast<float*>(base + 256) + (size_t)g * kMaxGrid * (2 * kMaxGroup + 1);
    const int rc = precision ? launch_prec<true>(p, cube->dtype, kg, vector_ok, st)
                             : launch_prec<false>(p, cube->dtype, kg, vector_ok, st);
    if (rc != UT_OK) return rc;
  }
  return UT_OK;
}

int ut_stretch(const float* scores, const float* minmax, int32_t k, int32_t ld_minmax, int64_t npix,
               int32_t depth, void* codes, void* stream) {
  UT_REQUIRE(k >= 1 && k <= kMaxBands, "ut_stretch: k must be 1..32");
  UT_REQUIRE(ld_minmax >= k, "ut_stretch: ld_minmax must be >= k");
  UT_REQUIRE(depth == 8 || depth == 16, "unsupported bit depth %d; expected 8 or 16", depth);
  if (npix <= 0) return UT_OK;
  cudaStream_t st = as_stream(stream);
  const bool vec16 = (npix % 16 == 0) && (reinterpret_cast<uintptr_t>(scores) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(codes) % 16 == 0);
  if (vec16 && k5_tma_enabled())
    return depth == 8 ? launch_stretch_tma<8>(scores, minmax, k, ld_minmax, npix, codes, st)
                      : launch_stretch_tma<16>(scores, minmax, k, ld_minmax, npix, codes, st);
  dim3 grid;
  if (vec16) {
    const int64_t chunks = npix / 16;
    int64_t gx = (chunks + 2 * kThreads - 1) / (2 * kThreads);
    int64_t cap = ((int64_t)sm_count() * 8 + k - 1) / k;
    if (gx > cap) gx = cap;
    grid = dim3((unsigned)(gx < 1 ? 1 : gx), (unsigned)k);
  } else {
    int64_t g = ((int64_t)k * npix + kThreads - 1) / kThreads;
    const int64_t cap = (int64_t)sm_count() * 8;
    grid = dim3((unsigned)(g > cap ? cap : (g < 1 ? 1 : g)));
  }
  if (depth == 8)
    stretch_kernel<8><<<grid, kThreads, 0, st>>>(scores, minmax, k, ld_minmax, npix, codes, vec16);
  else
    stretch_kernel<16><<<grid, kThreads, 0, st>>>(scores, minmax, k, ld_minmax, npix, codes, vec16);
  UT_CHECK_LAUNCH("stretch_kernel");
  return UT_OK;
}

}  // extern "C"
