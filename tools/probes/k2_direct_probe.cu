// Dev probe for the K2 next-round plan (item 1): can
// converter warps stream a band-planar fp32 cube straight from global memory
// (lane = 4 pixels, one LDG.128 per lane, 512 coalesced bytes per band and
// warp) fast enough without the bulk-copy ring?  Each CTA walks 256-pixel x
// 32-band tiles like K2; a warp task is (band, 128-pixel half), four per warp
// per tile, with D tiles of loads kept in flight in registers.  Optionally the
// samples go through K2's conversion (widen, magic-constant DFMA, 4x4 byte
// transpose) and one STS.32 per digit into a padded operand buffer, so the
// probe also prices the shared-memory stores of the plan (no MMA).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 k2_direct_probe.cu -o k2_direct_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kBands = 32;
constexpr int kTileP = 256;
constexpr int kWarps = 16;
constexpr int kChunkPad = 144 * 16 + 16;  // padded LBO of the operand chunks

__device__ __forceinline__ void transpose4(uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                           uint32_t* out) {
  const uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(a, b, 0x7362);
  const uint32_t t2 = __byte_perm(c, d, 0x5140), t3 = __byte_perm(c, d, 0x7362);
  out[0] = __byte_perm(t0, t2, 0x5410);
  out[1] = __byte_perm(t0, t2, 0x7632);
  out[2] = __byte_perm(t1, t3, 0x5410);
  out[3] = __byte_perm(t1, t3, 0x7632);
}

template <int D, bool CONVERT>
__global__ void __launch_bounds__(kWarps * 32, 1)
probe(const float* __restrict__ cube, int64_t npix, int64_t ntiles, double* out) {
  extern __shared__ __align__(16) unsigned char op[];  // 16 chunks x padded rows
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // task j of this warp in a tile: band = (4 warp + j) / 2, half = (4 warp + j) % 2
  uint4 buf[D][4];
  auto issue = [&](int slot, int64_t t) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int task = 4 * warp + j, b = task >> 1, h = task & 1;
      const float* src = cube + (int64_t)b * npix + t * kTileP + 128 * h + 4 * lane;
      buf[slot][j] = __ldg(reinterpret_cast<const uint4*>(src));
    }
  };
  double acc = 0.0;
  uint32_t bad = 0;
  int64_t t = blockIdx.x;
#pragma unroll
  for (int s = 0; s < D; ++s)
    if (t + (int64_t)s * gridDim.x < ntiles) issue(s, t + (int64_t)s * gridDim.x);
  int slot = 0;
  for (; t < ntiles; t += gridDim.x) {
#pragma unroll
    for (int s = 0; s < D; ++s) {
      if (s != slot) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint4 v = buf[s][j];
        const float x[4] = {__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z),
                            __uint_as_float(v.w)};
        if (CONVERT) {
          uint32_t wd[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double tt = fma((double)x[q], 1073741824.0, 6755399441055744.0 + 2155905152.0);
            bad |= (uint32_t)__double2hiint(tt) ^ 0x43380000u;
            wd[q] = (uint32_t)__double2loint(tt);
            acc += (double)x[q];
          }
          uint32_t dg[4];
          transpose4(wd[0], wd[1], wd[2], wd[3], dg);
          const int task = 4 * warp + j, b = task >> 1, h = task & 1;
          const int px = 128 * h + 4 * lane;       // pixel in the tile
          const int chunk = (px & 255) >> 4;       // 16 chunks of 16 pixels
          unsigned char* base = op + chunk * kChunkPad + (px & 15);
#pragma unroll
          for (int d = 0; d < 4; ++d)
            *reinterpret_cast<uint32_t*>(base + (32 * d + b) * 16) = dg[d];
        } else {
          acc += (double)(x[0] + x[1] + x[2] + x[3]);
        }
      }
      const int64_t nt = t + (int64_t)D * gridDim.x;
      if (nt < ntiles) issue(s, nt);
    }
    slot = slot + 1 == D ? 0 : slot + 1;
  }
  if (acc == 12345.0 || bad == 0xdeadbeef) out[blockIdx.x] = acc;
}

template <int D, bool C>
float run(const float* cube, int64_t npix, int ctas_per_sm, int sms, double* out) {
  const int64_t ntiles = npix / kTileP;
  const size_t smem = C ? 16 * kChunkPad : 16;
  cudaFuncSetAttribute(probe<D, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = ctas_per_sm * sms;
  probe<D, C><<<grid, kWarps * 32, smem>>>(cube, npix, ntiles, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) probe<D, C><<<grid, kWarps * 32, smem>>>(cube, npix, ntiles, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  const int64_t npix = 16384LL * 16384LL;
  const size_t bytes = (size_t)npix * kBands * sizeof(float);
  float* cube = nullptr;
  double* out = nullptr;
  if (cudaMalloc(&cube, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&out, 4096 * sizeof(double));
  cudaMemset(cube, 0x3c, bytes);  // ~0.0115f everywhere (finite)
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto report = [&](const char* name, int ctas, float ms) {
    printf("%-28s ctas/SM=%d  %.3f ms  %.0f GB/s\n", name, ctas, ms, bytes / (ms * 1e6));
  };
  for (int c = 1; c <= 2; ++c) {
    report("load only, D=1", c, run<1, false>(cube, npix, c, sms, out));
    report("load only, D=2", c, run<2, false>(cube, npix, c, sms, out));
    report("load only, D=4", c, run<4, false>(cube, npix, c, sms, out));
    report("load+convert+STS, D=2", c, run<2, true>(cube, npix, c, sms, out));
    report("load+convert+STS, D=4", c, run<4, true>(cube, npix, c, sms, out));
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
