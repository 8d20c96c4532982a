// Throughput probe: fp64 DFMA vs DMMA (mma.sync m8n8k4 f64) vs F2F.F64.F32 on one GPU.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int s = u & 3;
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c0[s]), "+d"(c1[s]) : "d"(a), "d"(b));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c0[0] + c1[0] + c0[1] + c1[1] + c0[2] + c1[2] + c0[3] + c1[3];
}

__global__ void f2f_loop(double* out, const float* in, int iters) {
  float x = in[threadIdx.x];
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc0 += (double)x; x += 1.0f;
      acc1 += (double)(x * 0.5f);
      acc2 += (double)(x * 0.25f);
      acc3 += (double)(x * 0.125f);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  float* in;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaMalloc(&in, 4096);
  cudaMemset(in, 0, 4096);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(a);
    dfma_loop<<<sms * 4, 256>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double fma = (double)sms * 4 * 256 * iters * 64;
    printf("DFMA: %.2f TFMA/s (%.1f FMA/clk/SM @1.965GHz)\n", fma / ms / 1e9, fma / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(a);
    dmma_loop<<<sms * 4, 256>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double mfma = (double)sms * 4 * (256 / 32) * iters * 16 * 256;
    printf("DMMA: %.2f TFMA/s (%.1f FMA/clk/SM)\n", mfma / ms / 1e9, mfma / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(a);
    f2f_loop<<<sms * 4, 256>>>(out, in, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double cv = (double)sms * 4 * 256 * iters * 32;
    printf("F2F+DADD: %.2f Tconv/s (%.1f conv/clk/SM)\n", cv / ms / 1e9, cv / (ms * 1e-3) / sms / 1.965e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
