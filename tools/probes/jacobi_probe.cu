#define UT_JACOBI_PROBE
// Time jacobi_team<32> on a 6x6 / 32x32 matrix in a minimal kernel (isolates
// the Jacobi round cost from the large cva_solve kernel).
#include "../../paper_1612_06457_b200/csrc/eig.cu"
#include "../../paper_1612_06457_b200/csrc/abi.cu"

namespace ut { namespace {
template <int NT>
__global__ void probe(int n, int reps, double* out, long long* cycles) {
  __shared__ Smem s;
  long long t0 = clock64();
  int code = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < n * n; e += NT) {
      const int i = e / n, j = e % n;
      s.a[i * LD + j] = (i == j ? 10.0 + i : 0.0) + 1.0 / (1.0 + i + j);
    }
    if (NT == 32) __syncwarp(); else asm volatile("bar.sync 1, %0;" ::"n"(NT));
    code |= jacobi_team<NT>(s, s.a, s.v, n);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = s.a[0]; out[1] = code; cycles[0] = (t1 - t0) / reps; }
}
}}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 64); cudaMalloc(&cyc, 64);
  for (int n : {6, 16, 32}) {
    ut::probe<32><<<1, 32>>>(n, 10, out, cyc);
    long long c; double o[2];
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(o, out, 16, cudaMemcpyDeviceToHost);
    printf("team32 n=%d: %lld cycles per solve (%.1f us @1.965GHz) code=%g\n", n, c, c / 1965.0, o[1]);
    long long jp[8];
    cudaMemcpyFromSymbol(jp, ut::g_jprobe, sizeof(jp));
    printf("   phases A, syncA, B, syncB, C, syncC (cycles, summed): %lld %lld %lld %lld %lld %lld\n", jp[0], jp[1], jp[2], jp[3], jp[4], jp[5]);
    long long z[8] = {0}; cudaMemcpyToSymbol(ut::g_jprobe, z, sizeof(z));
    ut::probe<128><<<1, 128>>>(n, 10, out, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(o, out, 16, cudaMemcpyDeviceToHost);
    printf("team128 n=%d: %lld cycles per solve (%.1f us) code=%g\n", n, c, c / 1965.0, o[1]);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
