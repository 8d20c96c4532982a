// K1: training-pixel gather and per-class moments.
//
// Replaces annotations.assemble_matrix's Python point loop
// (annotations.py:195-215) and compute_scatter's per-class reductions
// (projection.py:187-198).  Both are tiny next to the projector (N <= 60k
// points) but were 139 ms + 30 ms on the host at cfg 4.
//
// Determinism: every reduction runs in a fixed order -- points in input order
// inside a 128-point chunk, chunks in index order in the finishing CTA -- so
// the result is bit-identical run to run and independent of the grid size.
#include "common.cuh"

namespace ut {
namespace {

constexpr int kChunk = 128;     // points per CTA
constexpr int kThreads = 256;
constexpr int kMaxClasses = 64;

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

struct MomentWs {
  unsigned int* counter;  // 2 counters (pass A, pass B)
  double* part_a;         // [chunks][C][1+B]  count, sums
  double* sums;           // [C][1+B]          count, mean (after pass A)
  double* part_b;         // [chunks][C][npairs]
};

__host__ __device__ inline int npairs_of(int b) { return b * (b + 1) / 2; }

size_t moment_ws_bytes(int64_t n, int b, int c, MomentWs* ws, void* base) {
  const int64_t chunks = (n + kChunk - 1) / kChunk;
  size_t off = 256;  // counters
  const size_t a = off;
  off += sizeof(double) * chunks * c * (1 + b);
  const size_t s = off;
  off += sizeof(double) * c * (1 + b);
  const size_t pb = off;
  off += sizeof(double) * chunks * c * npairs_of(b);
  if (ws && base) {
    char* p = static_cast<char*>(base);
    ws->counter = reinterpret_cast<unsigned int*>(p);
    ws->part_a = reinterpret_cast<double*>(p + a);
    ws->sums = reinterpret_cast<double*>(p + s);
    ws->part_b = reinterpret_cast<double*>(p + pb);
  }
  return off;
}

// Stage one chunk: vals[b][p] (padded stride kChunk+1), labels lbl[p] (-1 pad).
__device__ __forceinline__ void stage_chunk(const double* __restrict__ values, int64_t ld,
                                            const int32_t* __restrict__ cls, int64_t n,
                                            int bands, int64_t j0, double* vals, int* lbl) {
  for (int e = threadIdx.x; e < bands * kChunk; e += blockDim.x) {
    const int b = e / kChunk, p = e - b * kChunk;
    const int64_t j = j0 + p;
    vals[b * (kChunk + 1) + p] = (j < n) ? values[b * ld + j] : 0.0;
  }
  for (int p = threadIdx.x; p < kChunk; p += blockDim.x) {
    const int64_t j = j0 + p;
    lbl[p] = (j < n) ? cls[j] : -1;
  }
}

__global__ void __launch_bounds__(kThreads)
class_sums_kernel(const double* __restrict__ values, int64_t ld, const int32_t* __restrict__ cls,
                  int64_t n, int bands, int classes, MomentWs ws) {
  __shared__ double vals[kMaxBands * (kChunk + 1)];
  __shared__ int lbl[kChunk];
  const int64_t j0 = (int64_t)blockIdx.x * kChunk;
  stage_chunk(values, ld, cls, n, bands, j0, vals, lbl);
  __syncthreads();
  const int rec = 1 + bands;
  double* out = ws.part_a + (size_t)blockIdx.x * classes * rec;
  for (int e = threadIdx.x; e < classes * rec; e += blockDim.x) {
    const int c = e / rec, f = e - c * rec;
    double s = 0.0;
    if (f == 0) {
      for (int p = 0; p < kChunk; ++p) s += (lbl[p] == c) ? 1.0 : 0.0;
    } else {
      const double* row = vals + (f - 1) * (kChunk + 1);
      for (int p = 0; p < kChunk; ++p)
        if (lbl[p] == c) s += row[p];
    }
    out[e] = s;
  }
  if (last_block_ticket(ws.counter)) {
    for (int e = threadIdx.x; e < classes * rec; e += blockDim.x) {
      double s = 0.0;
      for (unsigned int g = 0; g < gridDim.x; ++g) s += ws.part_a[(size_t)g * classes * rec + e];
      ws.sums[e] = s;  // raw sums for now
    }
    __syncthreads();
    for (int e = threadIdx.x; e < classes * rec; e += blockDim.x) {
      const int c = e / rec, f = e - c * rec;
      if (f > 0) {
        const double cnt = ws.sums[c * rec];
        ws.sums[e] = cnt > 0.0 ? ws.sums[e] / cnt : 0.0;
      }
    }
    if (threadIdx.x == 0) ws.counter[0] = 0u;
  }
}

__global__ void __launch_bounds__(kThreads)
class_scatter_kernel(const double* __restrict__ values, int64_t ld,
                     const int32_t* __restrict__ cls, int64_t n, int bands, int classes,
                     MomentWs ws, double* __restrict__ moments) {
  __shared__ double vals[kMaxBands * (kChunk + 1)];
  __shared__ int lbl[kChunk];
  __shared__ unsigned char pi[kMaxBands * (kMaxBands + 1) / 2];
  __shared__ unsigned char pj[kMaxBands * (kMaxBands + 1) / 2];
  const int64_t j0 = (int64_t)blockIdx.x * kChunk;
  const int rec = 1 + bands;
  const int np = npairs_of(bands);
  stage_chunk(values, ld, cls, n, bands, j0, vals, lbl);
  for (int i = threadIdx.x; i < bands; i += blockDim.x) {
    int base = i * bands - i * (i - 1) / 2;  // pairs (i, j>=i) enumerated row by row
    for (int j = i; j < bands; ++j) {
      pi[base + j - i] = (unsigned char)i;
      pj[base + j - i] = (unsigned char)j;
    }
  }
  __syncthreads();
  // centre each staged point on its class mean (two-pass, projection.py:195)
  for (int e = threadIdx.x; e < bands * kChunk; e += blockDim.x) {
    const int b = e / kChunk, p = e - b * kChunk;
    const int c = lbl[p];
    if (c >= 0) vals[b * (kChunk + 1) + p] -= ws.sums[c * rec + 1 + b];
  }
  __syncthreads();
  double* out = ws.part_b + (size_t)blockIdx.x * classes * np;
  for (int e = threadIdx.x; e < classes * np; e += blockDim.x) out[e] = 0.0;
  __syncthreads();
  // each thread owns pairs; class runs are flushed to this CTA's partial record
  for (int pr = threadIdx.x; pr < np; pr += blockDim.x) {
    const double* ri = vals + pi[pr] * (kChunk + 1);
    const double* rj = vals + pj[pr] * (kChunk + 1);
    int cur = -1;
    double acc = 0.0;
    for (int p = 0; p < kChunk; ++p) {
      const int c = lbl[p];
      if (c < 0) continue;
      if (c != cur) {
        if (cur >= 0) out[cur * np + pr] = acc;
        cur = c;
        acc = out[c * np + pr];
      }
      acc += ri[p] * rj[p];
    }
    if (cur >= 0) out[cur * np + pr] = acc;
  }
  if (last_block_ticket(ws.counter + 1)) {
    const int len = 1 + bands + bands * bands;
    for (int e = threadIdx.x; e < classes * np; e += blockDim.x) {
      const int c = e / np, pr = e - c * np;
      double s = 0.0;
      for (unsigned int g = 0; g < gridDim.x; ++g) s += ws.part_b[(size_t)g * classes * np + e];
      double* m = moments + (size_t)c * len + 1 + bands;
      m[pi[pr] * bands + pj[pr]] = s;
      m[pj[pr] * bands + pi[pr]] = s;
    }
    for (int e = threadIdx.x; e < classes * rec; e += blockDim.x) {
      const int c = e / rec, f = e - c * rec;
      moments[(size_t)c * len + f] = ws.sums[e];
    }
    if (threadIdx.x == 0) ws.counter[1] = 0u;
  }
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
  return moment_ws_bytes(n > 0 ? n : 1, bands, classes, nullptr, nullptr);
}

int ut_class_moments(const double* values, int64_t ld, const int32_t* cls, int64_t n,
                     int32_t bands, int32_t classes, double* moments, void* ws_base,
                     size_t ws_bytes, void* stream) {
  UT_REQUIRE(bands >= 1 && bands <= kMaxBands, "ut_class_moments: bands must be 1..32");
  UT_REQUIRE(classes >= 1 && classes <= kMaxClasses, "ut_class_moments: classes must be 1..64");
  UT_REQUIRE(n >= 1, "ut_class_moments: no points");
  MomentWs ws;
  const size_t need = moment_ws_bytes(n, bands, classes, &ws, ws_base);
  UT_REQUIRE(ws_bytes >= need, "ut_class_moments: workspace %zu < %zu bytes", ws_bytes, need);
  cudaStream_t s = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(ws.counter, 0, 2 * sizeof(unsigned int), s);
  if (e != cudaSuccess) return cuda_status(e, "ut_class_moments memset");
  const int chunks = (int)((n + kChunk - 1) / kChunk);
  class_sums_kernel<<<chunks, kThreads, 0, s>>>(values, ld, cls, n, bands, classes, ws);
  UT_CHECK_LAUNCH("class_sums_kernel");
  class_scatter_kernel<<<chunks, kThreads, 0, s>>>(values, ld, cls, n, bands, classes, ws, moments);
  UT_CHECK_LAUNCH("class_scatter_kernel");
  return UT_OK;
}

}  // extern "C"
