// Shared helpers for the sm_100a kernels of the CVA / PCA hot path.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cfloat>
#include <type_traits>
#include <cstdio>

#include "../../include/undertext_b200.h"

namespace ut {

constexpr int kMaxBands = 32;

// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);

// Dynamic shared memory above 48 KB must be opted into per kernel AND per device
// (cudaFuncSetAttribute applies to the current device only): a per-call-site
// cache keyed by device ordinal, so a process driving several GPUs sets it on each.
struct SmemAttr {
  size_t bytes[64] = {};
};
template <typename K>
inline int ensure_smem(SmemAttr& a, K kern, size_t bytes, const char* what) {
  int dev = 0;
  cudaGetDevice(&dev);
  size_t* slot = (dev >= 0 && dev < 64) ? &a.bytes[dev] : nullptr;
  if (slot && *slot >= bytes) return UT_OK;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();   // do not leave it for the next launch check to report
    return cuda_status(e, what);
  }
  if (slot) *slot = bytes;
  return UT_OK;
}

#define UT_CHECK_LAUNCH(where)                                   \
  do {                                                           \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return ::ut::cuda_status(_e, where);  \
  } while (0)

#define UT_REQUIRE(cond, ...)         \
  do {                                \
    if (!(cond)) {                    \
      ::ut::set_error(__VA_ARGS__);   \
      return UT_EDATA;                \
    }                                 \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();

// ---------------------------------------------------------------- samples
template <typename T> struct Sample;
template <> struct Sample<uint8_t>  { static constexpr int code = UT_U8;  static constexpr bool integral = true; };
template <> struct Sample<uint16_t> { static constexpr int code = UT_U16; static constexpr bool integral = true; };
template <> struct Sample<__half>   { static constexpr int code = UT_F16; static constexpr bool integral = false; };
template <> struct Sample<float>    { static constexpr int code = UT_F32; static constexpr bool integral = false; };
template <> struct Sample<double>   { static constexpr int code = UT_F64; static constexpr bool integral = false; };

__device__ __forceinline__ float to_f32(uint8_t v) { return (float)v; }
__device__ __forceinline__ float to_f32(uint16_t v) { return (float)v; }
__device__ __forceinline__ float to_f32(__half v) { return __half2float(v); }
__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(double v) { return (float)v; }

__device__ __forceinline__ double to_f64(uint8_t v) { return (double)v; }
__device__ __forceinline__ double to_f64(uint16_t v) { return (double)v; }
__device__ __forceinline__ double to_f64(__half v) { return (double)__half2float(v); }
__device__ __forceinline__ double to_f64(float v) { return (double)v; }
__device__ __forceinline__ double to_f64(double v) { return v; }

// Widening to fp64 without the quarter-rate F2F/I2F conversions (measured on
// B200: 15 conversions/clk/SM vs 62-64 DFMA/clk/SM), so the fp64 projector's
// conversions run on the ALU pipe next to the DFMA stream:
//  * float: re-bias the exponent and shift the mantissa (exact for normal
//    numbers; +-0 and subnormals land within 6e-39 of their value; Inf/NaN
//    become values >= 2^128, which overflow the fp32 score and trip the
//    NaN/Inf guard);
//  * 8/16-bit integers: the 2^52 magic-number trick (exact).
__device__ __forceinline__ double widen_f64(float x) {
  const int u = __float_as_int(x);
  const int hi = ((u >> 3) & (int)0x8fffffff) + 0x38000000;
  return __hiloint2double(hi, (int)((unsigned)u << 29));
}
__device__ __forceinline__ double widen_f64(uint16_t x) {
  return __hiloint2double(0x43300000, (int)x) - 4503599627370496.0;
}
__device__ __forceinline__ double widen_f64(uint8_t x) {
  return __hiloint2double(0x43300000, (int)x) - 4503599627370496.0;
}
__device__ __forceinline__ double widen_f64(__half x) { return widen_f64(__half2float(x)); }
__device__ __forceinline__ double widen_f64(double x) { return x; }

// Streaming 128-bit global loads: read once, do not pollute L1.
__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream_u4(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

// Unpack a 16-byte vector into V = 16/sizeof(T) samples.
template <typename T> struct Vec {
  static constexpr int V = 16 / sizeof(T);
  __device__ __forceinline__ static void unpack_f32(const uint4& u, float* out) {
    const T* t = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int i = 0; i < V; ++i) out[i] = to_f32(t[i]);
  }
  __device__ __forceinline__ static void unpack_f64(const uint4& u, double* out) {
    const T* t = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int i = 0; i < V; ++i) out[i] = to_f64(t[i]);
  }
};

// chk stays 0 unless some v is NaN or +-Inf (0 * v is then NaN).
__device__ __forceinline__ float nan_guard(float acc, float v) { return fmaf(0.0f, v, acc); }

// Block-wide "last CTA finishes" ticket: returns true in exactly one CTA, after
// every CTA's preceding global writes are visible.  *counter must be 0 on entry
// of the launch; the last CTA resets it.
__device__ __forceinline__ bool last_block_ticket(unsigned int* counter) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int t = atomicAdd(counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// ------------------------------------------------ mbarrier / bulk async copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n"
      "}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// One non-blocking test of the phase (for waits that back off with nanosleep).
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n"
      "}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// The same wait with a suspend-time hint: a warp whose phase is not complete
// sleeps in the barrier unit (up to `ns`) instead of spinning on try_wait, so
// waiting warps stop competing for issue slots with the working ones.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n"
      "}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(ns)
      : "memory");
}
// One bulk (TMA-engine) copy global -> shared, completing on `bar` (tx bytes).
// 16-byte aligned addresses and size.  Evict-first L2 policy: streamed once.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// Bulk prefetch of a global range into L2 (no shared memory, no completion).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

}  // namespace ut
