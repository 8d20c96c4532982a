// K1: training-pixel gather and per-class moments.
//
// Replaces annotations.assemble_matrix's Python point loop
// (annotations.py:195-215) and compute_scatter's per-class reductions
// (projection.py:187-198).
//
// One pass.  The n points are split into G <= 1024 contiguous ranges (G is a
// function of n only, so results do not depend on the GPU).  CTA g stages 128
// points at a time in shared memory -- gathered straight from the cube (fused
// pipeline; the chunk's coordinates are staged first so all sample loads are
// independent) or read from a B x n design matrix -- as deviations from the
// class pivot (the first point of the class), with a constant-1 row appended,
// and accumulates the upper triangle of [d;1][d;1]^T per class on the fp64
// tensor cores (mma.sync.m8n8k4.f64; each warp owns up to two 8x8 blocks of the
// upper triangle): one Gram holds the count, the shifted sums and the shifted
// scatter.  A CTA writes the records of the classes it saw, contiguously, plus
// its class mask; the merge kernel (one thread per Gram entry, ranges in
// ascending order) sums the partials of the ranges that saw the class and
// finalizes mean = pivot + s/n, M2 = S - s s^T/n.  Centring on a pivot keeps the
// one-pass form as accurate as the reference's two-pass form; every reduction
// order is fixed, so results are bit-identical run to run.
#include "common.cuh"

namespace ut {
namespace {

constexpr int kChunk = 128;      // points staged per step
constexpr int kThreads = 256;
constexpr int kMaxG = 1024;      // point ranges (CTAs)
#ifndef UT_K1_MINPER
#define UT_K1_MINPER 256  // two pipelined chunks per CTA, one wave at cfg 4 (60k points): 140 -> 123 us
#endif
constexpr int kMinPerCta = UT_K1_MINPER;  // points per CTA at least (multiple of kChunk)
#ifndef UT_K1_SMALL_G
#define UT_K1_SMALL_G 296
#endif
constexpr int kSmallG = UT_K1_SMALL_G;  // up to this many 128-point CTAs, no 2-chunk minimum
constexpr int kMaxClasses = 16;  // per launch; more classes -> several launches
constexpr int kRows = kMaxBands + 1;                    // bands + ones row
constexpr int kTileLd = kChunk + 4;   // row stride = 4 mod 16 doubles: a fragment load (8 rows x 4 points) is conflict-free
constexpr int kWarps = kThreads / 32;

__host__ __device__ inline int ent_count(int b) { return (b + 1) * (b + 2) / 2; }
__host__ __device__ inline int row_groups(int b) { return (b + 1 + 7) / 8; }   // 8-row groups incl. the ones row
// upper-triangle entry (i <= j) of the (B+1) x (B+1) Gram, R = B + 1
__host__ __device__ inline int ent_index(int i, int j, int R) { return i * R - i * (i - 1) / 2 + (j - i); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

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
// A source yields sample (b, j) of point j.  The cube source first stages the
// chunk's (x, y) in shared memory so every sample load is independent.
struct MatrixSrc {
  const double* values;
  int64_t ld;
  using Coord = int64_t;
  using Raw = double;
  __device__ __forceinline__ Coord coord(int64_t j) const { return j; }
  __device__ __forceinline__ bool valid_at(Coord) const { return true; }
  __device__ __forceinline__ double sample(int b, Coord j) const { return values[b * ld + j]; }
  __device__ __forceinline__ Raw raw(int b, Coord j) const { return values[b * ld + j]; }
  __device__ __forceinline__ static double widen(Raw v) { return v; }
  __device__ __forceinline__ bool valid(int64_t) const { return true; }
  __device__ __forceinline__ void stage_xy(int64_t, int, int2*) const {}
  __device__ __forceinline__ double at(int b, int64_t j, const int2*, int) const {
    return values[b * ld + j];
  }
  __device__ __forceinline__ double at_global(int b, int64_t j) const { return values[b * ld + j]; }
};

// One gathered sample: read-only path, no L1 allocation, 64-byte L2 fetch hint --
// every sample of a training pixel sits in another band plane, so nothing near it
// is used (cfg 4 fit: K1 118 -> 112 us in A/B runs).
#ifndef UT_K1_L2HINT
#define UT_K1_L2HINT 1
#endif
template <typename T>
__device__ __forceinline__ T ld_gather(const T* p) {
#if UT_K1_L2HINT
  T out;
  if constexpr (sizeof(T) == 1) {
    uint16_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::64B.u8 %0, [%1];" : "=h"(v) : "l"(p));
    const uint8_t w = (uint8_t)v;
    memcpy(&out, &w, 1);
  } else if constexpr (sizeof(T) == 2) {
    uint16_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::64B.b16 %0, [%1];" : "=h"(v) : "l"(p));
    memcpy(&out, &v, 2);
  } else if constexpr (sizeof(T) == 4) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::64B.b32 %0, [%1];" : "=r"(v) : "l"(p));
    memcpy(&out, &v, 4);
  } else {
    unsigned long long v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::64B.b64 %0, [%1];" : "=l"(v) : "l"(p));
    memcpy(&out, &v, 8);
  }
  return out;
#else
  return *p;
#endif
}

template <typename T>
struct CubeSrc {
  const T* data;
  int64_t bs, rs, rows, cols, row0;
  const int32_t* xy;
  using Coord = int2;  // (x, local y)
  using Raw = T;
  __device__ __forceinline__ Raw raw(int b, Coord c) const {
    return ld_gather(data + (b * bs + (int64_t)c.y * rs + c.x));
  }
  __device__ __forceinline__ static double widen(Raw v) { return to_f64(v); }
  __device__ __forceinline__ Coord coord(int64_t j) const {
    const int2 v = reinterpret_cast<const int2*>(xy)[j];
    return make_int2(v.x, (int)(v.y - row0));
  }
  __device__ __forceinline__ bool valid_at(Coord c) const {
    return c.x >= 0 && c.x < cols && c.y >= 0 && c.y < rows;
  }
  __device__ __forceinline__ double sample(int b, Coord c) const {
    return to_f64(data[b * bs + (int64_t)c.y * rs + c.x]);
  }
  __device__ __forceinline__ bool valid(int64_t j) const {
    const int64_t x = xy[2 * j], y = xy[2 * j + 1] - row0;
    return x >= 0 && x < cols && y >= 0 && y < rows;
  }
  // local (x, y - row0) of points [q0, q0 + count) -> sxy[p]
  __device__ __forceinline__ void stage_xy(int64_t q0, int count, int2* sxy) const {
    for (int p = threadIdx.x; p < count; p += blockDim.x) {
      const int2 v = reinterpret_cast<const int2*>(xy)[q0 + p];
      sxy[p] = make_int2(v.x, (int)(v.y - row0));
    }
  }
  __device__ __forceinline__ double at(int b, int64_t, const int2* sxy, int p) const {
    const int2 v = sxy[p];
    return to_f64(data[b * bs + (int64_t)v.y * rs + v.x]);
  }
  __device__ __forceinline__ double at_global(int b, int64_t j) const {
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

__host__ __device__ inline int rec_len(int b) { return 1 + b + b * b; }

// Shared memory, sized for the launch's B and C (dynamic):
//   tile[8 NG x kTileLd] | acc[C x E] | pivot[C x B] | lbl[kChunk] | mask
// (NG = row groups of 8; the rows past the ones row stay zero)
struct Smem {
  double* tile;
  double* acc;
  double* pivot;
  int* lbl;
  unsigned* mask_p;
};

__host__ __device__ inline size_t smem_bytes(int b, int c) {
  const int E = ent_count(b);
  size_t off = sizeof(double) * ((size_t)8 * row_groups(b) * kTileLd + (size_t)c * E + (size_t)c * b);
  off += sizeof(int) * kChunk + 16;
  return (off + 15) & ~(size_t)15;
}

__device__ inline Smem carve(unsigned char* raw, int b, int c) {
  const int E = ent_count(b);
  Smem s;
  double* d = reinterpret_cast<double*>(raw);
  s.tile = d;
  s.acc = d + (size_t)8 * row_groups(b) * kTileLd;
  s.pivot = s.acc + (size_t)c * E;
  int* ip = reinterpret_cast<int*>(s.pivot + (size_t)c * b);
  s.lbl = ip;
  s.mask_p = reinterpret_cast<unsigned*>(ip + kChunk);
  return s;
}

// pivot[c] = first point of class c (global index), or -1
__global__ void __launch_bounds__(1024)
pivot_kernel(const int32_t* __restrict__ cls, int64_t n, int c0, int classes, int32_t* pivots) {
  __shared__ int first[kMaxClasses];
  if (threadIdx.x < classes) first[threadIdx.x] = 0x7fffffff;
  __syncthreads();
  unsigned seen = 0u;  // each thread's first hit per class is its minimum
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const int c = cls[j] - c0;
    if (c >= 0 && c < classes && !((seen >> c) & 1u)) {
      atomicMin(&first[c], (int)j);
      seen |= 1u << c;
    }
  }
  __syncthreads();
  if (threadIdx.x < classes)
    pivots[threadIdx.x] = first[threadIdx.x] == 0x7fffffff ? -1 : first[threadIdx.x];
}

// Per-range Gram of [x - pivot_c ; 1] per class -> part[g][c][e] (raw sums) for
// the classes range g saw, cmask[g] = those classes.
template <typename Src>
__global__ void __launch_bounds__(kThreads)
moments_kernel(Src src, const int32_t* __restrict__ cls, const int32_t* __restrict__ pivots,
               Layout L, double* __restrict__ part, uint32_t* __restrict__ cmask,
               double* __restrict__ pivval, unsigned long long* first_bad) {
  extern __shared__ __align__(16) unsigned char raw[];
  const Smem s = carve(raw, L.bands, L.classes);
  const int tid = threadIdx.x;
  const int B = L.bands, C = L.classes;
  const int R = B + 1;
  const int E = ent_count(B);
  const int64_t j0 = (int64_t)blockIdx.x * L.span;
  const int64_t j1 = j0 + L.span < L.n ? j0 + L.span : L.n;
  // Staging: thread -> point p = tid % 128, bands tid/128, +2, +4, ...  The
  // gather is random-access and latency-bound, so it is software-pipelined:
  // coordinates / labels are loaded two chunks ahead and raw samples one chunk
  // ahead (kept unconverted in registers), while the current chunk's Gram runs.
  constexpr int kPer = kMaxBands / (kThreads / kChunk);  // 16 bands per thread
  const int sp = tid % kChunk, sb = tid / kChunk;
  typename Src::Raw nv[kPer];
  unsigned seen = 0u;              // classes of the chunks so far
  int nl = -1;                     // label of the chunk in nv
  typename Src::Coord ncc{};       // coordinates two chunks ahead
  int nnl = -1;
  auto load_coord = [&](int64_t q0) {
    const int64_t j = q0 + sp;
    nnl = -1;
    if (j < j1) {
      ncc = src.coord(j);
      int c = cls[j] - L.c0;
      if (c < 0 || c >= C) c = -1;
      nnl = c;
    }
  };
  auto load_samples = [&](int64_t q0) {  // uses the coordinates loaded for q0
    const int64_t j = q0 + sp;
    int c = nnl;
    if (j < j1 && c >= 0 && !src.valid_at(ncc)) {
      if (first_bad && sb == 0) atomicMin(first_bad, (unsigned long long)j);
      c = -1;
    }
    nl = (j < j1) ? c : -1;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int b = sb + u * (kThreads / kChunk);
      nv[u] = (nl >= 0 && b < B) ? src.raw(b, ncc) : typename Src::Raw(0);
    }
  };
  // the first chunk's gather is issued before the set-up below (pivot
  // loads, tables) so their latencies overlap
  if (j0 < j1) {
    load_coord(j0);
    load_samples(j0);
    if (j0 + kChunk < j1) load_coord(j0 + kChunk);
  }
  const int NG = row_groups(B), NB = NG * (NG + 1) / 2;
  const int lane = tid & 31, warp = tid >> 5, fb = lane >> 2, fp = lane & 3;
  for (int e = tid; e < 8 * NG * kTileLd; e += blockDim.x) s.tile[e] = 0.0;
  for (int e = tid; e < C * E; e += blockDim.x) s.acc[e] = 0.0;
  for (int e = tid; e < C * B; e += blockDim.x) {
    const int c = e / B, b = e - c * B;
    const int pj = pivots[c];
    const double v = (pj >= 0 && src.valid(pj)) ? src.at_global(b, pj) : 0.0;
    s.pivot[e] = v;
    if (blockIdx.x == 0) pivval[e] = v;   // for the merge
  }
  __syncthreads();
  for (int64_t q0 = j0; q0 < j1; q0 += kChunk) {
    if (tid == 0) *s.mask_p = 0u;
    __syncthreads();
    // deviations from the class pivot; row B is the constant 1 (0 for padding)
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int b = sb + u * (kThreads / kChunk);
      if (b < B)
        s.tile[b * kTileLd + sp] = (nl >= 0) ? Src::widen(nv[u]) - s.pivot[nl * B + b] : 0.0;
    }
    if (sb == 0) {
      s.lbl[sp] = nl;
      s.tile[B * kTileLd + sp] = (nl >= 0) ? 1.0 : 0.0;
      if (nl >= 0) atomicOr(s.mask_p, 1u << nl);
    }
    __syncthreads();
    if (q0 + kChunk < j1) load_samples(q0 + kChunk);
    if (q0 + 2 * kChunk < j1) load_coord(q0 + 2 * kChunk);
    const unsigned mask = *s.mask_p;
    seen |= mask;
    // Gram of the chunk on the fp64 tensor cores.  Warp w owns the upper 8x8
    // blocks w, w + 8 (< NB); a lane's A element is tile[8 bi + fb][k + fp], its
    // B element tile[8 bj + fb][k + fp]; two accumulator pairs over alternate
    // 4-point steps.  One class in the chunk (class-sorted points): one pass,
    // padding / foreign points are zero rows.  Mixed chunk: one pass per class
    // present, the B element masked to the class's points.
    const bool single = (mask & (mask - 1u)) == 0u;
    for (unsigned rest = mask; rest != 0u; rest &= rest - 1u) {
      const int c = __ffs(rest) - 1;
      for (int q = warp; q < NB; q += kWarps) {   // warp-uniform
        int bi = 0, rem = q;
        while (rem >= NG - bi) { rem -= NG - bi; ++bi; }
        const int bj = bi + rem;
        const double* ra = s.tile + (8 * bi + fb) * kTileLd + fp;
        const double* rb = s.tile + (8 * bj + fb) * kTileLd + fp;
        double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
        if (single) {
#pragma unroll 4
          for (int k = 0; k < kChunk; k += 8) {
            dmma(c0, c1, ra[k], rb[k]);
            dmma(d0, d1, ra[k + 4], rb[k + 4]);
          }
        } else {
#pragma unroll 4
          for (int k = 0; k < kChunk; k += 8) {
            const double b0 = s.lbl[k + fp] == c ? rb[k] : 0.0;
            const double b1 = s.lbl[k + 4 + fp] == c ? rb[k + 4] : 0.0;
            dmma(c0, c1, ra[k], b0);
            dmma(d0, d1, ra[k + 4], b1);
          }
        }
        c0 += d0;
        c1 += d1;
        // the lane holds Gram[8 bi + fb][8 bj + 2 fp, + 1]; each upper entry has one owner
        const int i = 8 * bi + fb, j = 8 * bj + 2 * fp;
        if (i < R && j < R && i <= j) s.acc[c * E + ent_index(i, j, R)] += c0;
        if (i < R && j + 1 < R && i <= j + 1) s.acc[c * E + ent_index(i, j + 1, R)] += c1;
      }
    }
    __syncthreads();
  }
  // the records of the classes this range saw, contiguous per range
  double* rec = part + (size_t)blockIdx.x * C * E;
  for (int e = tid; e < C * E; e += blockDim.x)
    if ((seen >> (e / E)) & 1u) rec[e] = s.acc[e];
  if (tid == 0) cmask[blockIdx.x] = seen;
}

// CTA (x, c): threads 0..127 own Gram entries e = 128 x + tid of class c, threads
// 128..128+B the ones-column entries (i, B) every finalization needs.  Each sums
// its entry over the ranges that saw the class, in ascending range order, and the
// CTA finalizes count / mean = pivot + s/n / M2 = S - s s^T / n for its entries.
constexpr int kMergeEnt = 128;
constexpr int kMergeThreads = kMergeEnt + 64;
static_assert(kRows <= 64, "ones-column threads");

__global__ void __launch_bounds__(kMergeThreads)
merge_kernel(const double* __restrict__ part, const uint32_t* __restrict__ cmask,
             const double* __restrict__ pivval, Layout L, double* __restrict__ moments) {
  __shared__ int act[kMaxG];
  __shared__ int nact_sh;
  __shared__ double ones[kRows];
  const int B = L.bands, G = L.G, C = L.classes;
  const int R = B + 1, E = ent_count(B), len = rec_len(B);
  const int tid = threadIdx.x, c = blockIdx.y;
  // ranges that saw class c, ascending (one warp compacts)
  if (tid < 32) {
    int n = 0;
    for (int g0 = 0; g0 < G; g0 += 32) {
      const int g = g0 + tid;
      const bool has = g < G && ((cmask[g] >> c) & 1u);
      const unsigned bal = __ballot_sync(0xffffffffu, has);
      if (has) act[n + __popc(bal & ((1u << tid) - 1u))] = g;
      n += __popc(bal);
    }
    if (tid == 0) nact_sh = n;
  }
  __syncthreads();
  const int nact = nact_sh;
  int e = -1;
  if (tid < kMergeEnt) {
    const int t = blockIdx.x * kMergeEnt + tid;
    if (t < E) e = t;
  } else if (tid - kMergeEnt < R) {
    e = ent_index(tid - kMergeEnt, B, R);
  }
  double sum = 0.0;
  if (e >= 0) {
    const double* p = part + (size_t)c * E + e;
    const size_t stride = (size_t)C * E;
    int a = 0;
    for (; a + 4 <= nact; a += 4) {   // loads first, adds in range order
      const double v0 = p[act[a] * stride], v1 = p[act[a + 1] * stride];
      const double v2 = p[act[a + 2] * stride], v3 = p[act[a + 3] * stride];
      sum += v0;
      sum += v1;
      sum += v2;
      sum += v3;
    }
    for (; a < nact; ++a) sum += p[act[a] * stride];
  }
  if (tid >= kMergeEnt && tid - kMergeEnt < R) ones[tid - kMergeEnt] = sum;
  __syncthreads();
  if (tid >= kMergeEnt || e < 0) return;
  // e -> (i, j), i <= j
  int i = 0, rem = e;
  while (rem >= R - i) { rem -= R - i; ++i; }
  const int j = i + rem;
  const double n = ones[B];
  double* out = moments + (size_t)(L.c0 + c) * len;
  if (j == B) {
    if (i == B) {
      out[0] = n > 0.0 ? n : 0.0;
    } else {
      out[1 + i] = n > 0.0 ? pivval[c * B + i] + sum / n : 0.0;
    }
  } else {
    const double v = n > 0.0 ? sum - ones[i] * ones[j] / n : 0.0;
    out[1 + B + i * B + j] = v;
    out[1 + B + j * B + i] = v;
  }
}

Layout make_layout(int64_t n, int b, int c) {
  Layout L{};
  L.n = n;
  L.bands = b;
  L.classes = c;
  // Small point sets (a row shard's share at 4-8 GPUs): one 128-point chunk
  // per CTA, more CTAs in flight for the latency-bound gather (cfg 4 at 8
  // shards, 4590 points: 75 -> 63 us).  Larger sets keep two pipelined chunks
  // per CTA so they run in one wave.  G stays a function of n only.
  int64_t G = (n + kChunk - 1) / kChunk;
  if (G > kSmallG) G = (n + kMinPerCta - 1) / kMinPerCta;
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
  return sizeof(double) * (size_t)per * ent_count(b) * kMaxG + 256 + sizeof(int32_t) * 64 +
         sizeof(uint32_t) * kMaxG + sizeof(double) * kMaxClasses * kMaxBands;
}

template <typename Src>
int launch_moments(const Src& src, const int32_t* cls, int64_t n, int b, int classes,
                   const int32_t* given_pivots, double* moments, void* ws, size_t ws_bytes,
                   unsigned long long* first_bad, cudaStream_t st) {
  UT_REQUIRE(ws_bytes >= ws_bytes_for(b, classes), "class moments: workspace %zu < %zu",
             ws_bytes, ws_bytes_for(b, classes));
  static SmemAttr attr;
  const int full = (int)smem_bytes(b, classes < kMaxClasses ? classes : kMaxClasses);
  if (int rc = ensure_smem(attr, moments_kernel<Src>, (size_t)full, "moments smem attribute")) return rc;
  int32_t* pivots = reinterpret_cast<int32_t*>(ws);
  double* part = reinterpret_cast<double*>(static_cast<char*>(ws) + 256 + sizeof(int32_t) * 64);
  const int per = classes < kMaxClasses ? classes : kMaxClasses;
  uint32_t* cmask = reinterpret_cast<uint32_t*>(part + (size_t)per * ent_count(b) * kMaxG);
  double* pivval = reinterpret_cast<double*>(cmask + kMaxG);
  for (int c0 = 0; c0 < classes; c0 += kMaxClasses) {
    Layout L = make_layout(n, b, classes - c0 < kMaxClasses ? classes - c0 : kMaxClasses);
    L.c0 = c0;
    const int32_t* piv = given_pivots ? given_pivots + c0 : pivots;
    if (!given_pivots) {
      pivot_kernel<<<1, 1024, 0, st>>>(cls, n, c0, L.classes, pivots);
      UT_CHECK_LAUNCH("pivot_kernel");
    }
    moments_kernel<Src><<<L.G, kThreads, smem_bytes(b, L.classes), st>>>(src, cls, piv, L, part,
                                                                        cmask, pivval, first_bad);
    UT_CHECK_LAUNCH("moments_kernel");
    const dim3 mgrid((unsigned)((ent_count(b) + kMergeEnt - 1) / kMergeEnt), (unsigned)L.classes);
    merge_kernel<<<mgrid, kMergeThreads, 0, st>>>(part, cmask, pivval, L, moments);
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
                        int classes, const int32_t* pivots, double* moments,
                        unsigned long long* first_bad, void* ws, size_t ws_bytes,
                        cudaStream_t st) {
  CubeSrc<T> src{static_cast<const T*>(cube->data), cube->band_stride, cube->row_stride,
                 cube->rows, cube->cols, cube->row0, xy};
  return launch_moments(src, cls, n, cube->bands, classes, pivots, moments, ws, ws_bytes,
                        first_bad, st);
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
                     int32_t bands, int32_t classes, const int32_t* pivots, double* moments,
                     void* ws, size_t ws_bytes, void* stream) {
  UT_REQUIRE(bands >= 1 && bands <= kMaxBands, "ut_class_moments: bands must be 1..32");
  UT_REQUIRE(classes >= 1, "ut_class_moments: classes must be >= 1");
  UT_REQUIRE(n >= 1, "ut_class_moments: no points");
  MatrixSrc src{values, ld};
  return launch_moments(src, cls, n, bands, classes, pivots, moments, ws, ws_bytes, nullptr,
                        as_stream(stream));
}

int ut_cube_class_moments(const ut_cube* cube, const int32_t* xy, const int32_t* cls, int64_t n,
                          int32_t classes, const int32_t* pivots, double* moments,
                          int64_t* first_bad, void* ws, size_t ws_bytes, void* stream) {
  UT_REQUIRE(cube && cube->bands >= 1 && cube->bands <= kMaxBands,
             "ut_cube_class_moments: bands must be 1..32");
  UT_REQUIRE(classes >= 1 && n >= 1, "ut_cube_class_moments: bad classes/points");
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(first_bad, 0xFF, sizeof(int64_t), st);
  if (e != cudaSuccess) return cuda_status(e, "ut_cube_class_moments memset");
  auto* fb = reinterpret_cast<unsigned long long*>(first_bad);
  switch (cube->dtype) {
    case UT_U8: return launch_cube_moments<uint8_t>(cube, xy, cls, n, classes, pivots, moments, fb, ws, ws_bytes, st);
    case UT_U16: return launch_cube_moments<uint16_t>(cube, xy, cls, n, classes, pivots, moments, fb, ws, ws_bytes, st);
    case UT_F16: return launch_cube_moments<__half>(cube, xy, cls, n, classes, pivots, moments, fb, ws, ws_bytes, st);
    case UT_F32: return launch_cube_moments<float>(cube, xy, cls, n, classes, pivots, moments, fb, ws, ws_bytes, st);
    case UT_F64: return launch_cube_moments<double>(cube, xy, cls, n, classes, pivots, moments, fb, ws, ws_bytes, st);
  }
  set_error("ut_cube_class_moments: unknown dtype %d", cube->dtype);
  return UT_EDATA;
}

}  // extern "C"
