// K3: single-CTA fp64 solvers for the B x B (B <= 32) problems of the path.
//
//  * ut_gen_eig_sym  -- solve_gen_eig_sym (eigen.py:75-113): symmetry check,
//    ridge (eigen.py:63-72), Cholesky, C = L^-1 A L^-T, symmetric eigensolve,
//    V = L^-T U, descending sort, sign normalization (eigen.py:40-52).
//  * ut_cva_solve    -- combine per-shard class moments, build the symmetrized
//    within / between scatter (projection.py:187-200), then the solve above.
//  * ut_pca_solve    -- combine region moments, std / correlation
//    (projection.py:335-337), eigh + sort + sign (projection.py:263-270).
//
// The reference diagonalizes with LAPACK syevd (tridiagonal QR); here a cyclic
// parallel-order Jacobi runs in shared memory on 1024 threads (one per matrix
// element).  Jacobi is at least as accurate (it has high relative accuracy),
// and every step is in a fixed order, so the result is deterministic.
#include "common.cuh"

namespace ut {
namespace {

constexpr int N = kMaxBands;    // 32
constexpr int LD = N + 1;       // padded row stride in shared memory
constexpr int kThreads = N * N; // 1024

struct Smem {
  double a[N * LD];   // working matrix (A, then C, then Jacobi iterate)
  double m[N * LD];   // M (then L, the Cholesky factor)
  double x[N * LD];   // scratch for the triangular solves
  double v[N * LD];   // eigenvectors
  double cs[N / 2], sn[N / 2], npp[N / 2], nqq[N / 2];
  int pp[N / 2], qq[N / 2];
  double red[kThreads / 32];
  double scal[4];
  int flag;
  int order[N];
};

__device__ __forceinline__ double block_max(Smem& s, double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) s.red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = s.red[0];
  for (int w = 1; w < kThreads / 32; ++w) r = fmax(r, s.red[w]);
  __syncthreads();
  return r;
}

// max|X| and max|X - X^T| -> asymmetric beyond rtol 1e-10 (eigen.py:55-60)
__device__ bool is_asym(Smem& s, const double* x, int n) {
  const int i = threadIdx.x / N, j = threadIdx.x % N;
  double mag = 0.0, dif = 0.0;
  if (i < n && j < n) {
    mag = fabs(x[i * LD + j]);
    dif = fabs(x[i * LD + j] - x[j * LD + i]);
  }
  const double top = block_max(s, mag);
  const double gap = block_max(s, dif);
  return top != 0.0 && gap > 1e-10 * top;
}

// In-place cyclic Jacobi on s.a (n x n) with eigenvectors accumulated in s.v.
// Parallel (round-robin) ordering: n/2 disjoint rotations per round.
__device__ int jacobi(Smem& s, int n) {
  const int tid = threadIdx.x;
  const int i = tid / N, j = tid % N;
  if (i < n && j < n) s.v[i * LD + j] = (i == j) ? 1.0 : 0.0;
  const int m = n + (n & 1);
  const int half = m / 2;
  // absolute floor: off-diagonals below 1e-22 * ||A||_F are treated as zero
  double fro = 0.0;
  if (i < n && j < n) fro = s.a[i * LD + j] * s.a[i * LD + j];
  for (int o = 16; o > 0; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
  __syncthreads();
  if ((tid & 31) == 0) s.red[tid >> 5] = fro;
  __syncthreads();
  if (tid == 0) {
    double f = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) f += s.red[w];
    s.scal[0] = 1e-22 * sqrt(f);
  }
  __syncthreads();
  const double floor_abs = s.scal[0];
  if (n < 2) return 0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) s.flag = 0;
    __syncthreads();
    for (int r = 0; r < m - 1; ++r) {
      if (tid < half) {
        const int k = tid;
        int p, q;
        if (k == 0) {
          p = m - 1;
          q = r;
        } else {
          p = (r + k) % (m - 1);
          q = (r - k + (m - 1)) % (m - 1);
        }
        if (p > q) { const int t = p; p = q; q = t; }
        double c = 1.0, sn = 0.0, npp = 0.0, nqq = 0.0;
        int act = 0;
        if (q < n) {
          const double apq = s.a[p * LD + q];
          const double app = s.a[p * LD + p], aqq = s.a[q * LD + q];
          const double thr = fmax(0.5 * DBL_EPSILON * sqrt(fabs(app) * fabs(aqq)), floor_abs);
          if (fabs(apq) > thr) {
            const double theta = (aqq - app) / (2.0 * apq);
            double t;
            if (fabs(theta) > 1e150) {
              t = 0.5 / theta;
            } else {
              t = 1.0 / (fabs(theta) + sqrt(1.0 + theta * theta));
              if (theta < 0.0) t = -t;
            }
            c = 1.0 / sqrt(1.0 + t * t);
            sn = t * c;
            npp = app - t * apq;
            nqq = aqq + t * apq;
            act = 1;
          }
        }
        s.pp[k] = act ? p : -1;
        s.qq[k] = q;
        s.cs[k] = c;
        s.sn[k] = sn;
        s.npp[k] = npp;
        s.nqq[k] = nqq;
        if (act) s.flag = 1;
      }
      __syncthreads();
      // rows p, q  <- J^T A
      if (tid < half * N) {
        const int k = tid / N, col = tid % N;
        const int p = s.pp[k];
        if (p >= 0 && col < n) {
          const int q = s.qq[k];
          const double c = s.cs[k], sn = s.sn[k];
          const double ap = s.a[p * LD + col], aq = s.a[q * LD + col];
          s.a[p * LD + col] = c * ap - sn * aq;
          s.a[q * LD + col] = sn * ap + c * aq;
        }
      }
      __syncthreads();
      // columns p, q <- A J ; V <- V J
      if (tid < half * N) {
        const int k = tid / N, row = tid % N;
        const int p = s.pp[k];
        if (p >= 0 && row < n) {
          const int q = s.qq[k];
          const double c = s.cs[k], sn = s.sn[k];
          const double ap = s.a[row * LD + p], aq = s.a[row * LD + q];
          s.a[row * LD + p] = c * ap - sn * aq;
          s.a[row * LD + q] = sn * ap + c * aq;
          const double vp = s.v[row * LD + p], vq = s.v[row * LD + q];
          s.v[row * LD + p] = c * vp - sn * vq;
          s.v[row * LD + q] = sn * vp + c * vq;
        }
      }
      __syncthreads();
      if (tid < half) {
        const int p = s.pp[tid];
        if (p >= 0) {
          const int q = s.qq[tid];
          s.a[p * LD + p] = s.npp[tid];
          s.a[q * LD + q] = s.nqq[tid];
          s.a[p * LD + q] = 0.0;
          s.a[q * LD + p] = 0.0;
        }
      }
      __syncthreads();
    }
    const int rotated = s.flag;
    __syncthreads();
    if (!rotated) return 0;
  }
  return UT_INFO_NO_CONVERGE;
}

// Cholesky of s.m in place (lower).  Returns false if a pivot is not > 0.
__device__ bool cholesky(Smem& s, int n) {
  const int tid = threadIdx.x;
  const int i = tid / N, j = tid % N;
  for (int k = 0; k < n; ++k) {
    if (tid == 0) {
      const double d = s.m[k * LD + k];
      s.flag = (d > 0.0) ? 1 : 0;  // also rejects NaN
      if (d > 0.0) s.m[k * LD + k] = sqrt(d);
    }
    __syncthreads();
    if (!s.flag) return false;
    if (tid > k && tid < n) s.m[tid * LD + k] /= s.m[k * LD + k];
    __syncthreads();
    if (i > k && i < n && j > k && j <= i) s.m[i * LD + j] -= s.m[i * LD + k] * s.m[j * LD + k];
    __syncthreads();
  }
  if (i < n && j < n && j > i) s.m[i * LD + j] = 0.0;
  __syncthreads();
  return true;
}

// x <- L^-1 x (forward substitution, all columns in parallel)
__device__ void solve_lower(Smem& s, double* x, int n) {
  const int tid = threadIdx.x;
  const int i = tid / N, j = tid % N;
  for (int p = 0; p < n; ++p) {
    if (tid < n) x[p * LD + tid] /= s.m[p * LD + p];
    __syncthreads();
    if (i > p && i < n && j < n) x[i * LD + j] -= s.m[i * LD + p] * x[p * LD + j];
    __syncthreads();
  }
}

// x <- L^-T x (backward substitution)
__device__ void solve_upper_t(Smem& s, double* x, int n) {
  const int tid = threadIdx.x;
  const int i = tid / N, j = tid % N;
  for (int p = n - 1; p >= 0; --p) {
    if (tid < n) x[p * LD + tid] /= s.m[p * LD + p];
    __syncthreads();
    if (i < p && j < n) x[i * LD + j] -= s.m[p * LD + i] * x[p * LD + j];
    __syncthreads();
  }
}

// Descending order of the diagonal of s.a (stable on ties by index).
__device__ void sort_desc(Smem& s, int n) {
  const int tid = threadIdx.x;
  if (tid < n) {
    const double me = s.a[tid * LD + tid];
    int rank = 0;
    for (int o = 0; o < n; ++o) {
      const double other = s.a[o * LD + o];
      rank += (other > me) || (other == me && o < tid);
    }
    s.order[rank] = tid;
  }
  __syncthreads();
}

// Write eigenvalues/vectors in sorted order, sign-normalized (eigen.py:40-52:
// the first entry of largest magnitude is made positive).
__device__ void emit(Smem& s, const double* vec, int n, double* evals, double* evecs) {
  const int tid = threadIdx.x;
  const int i = tid / N, j = tid % N;
  if (tid < n) {
    const int src = s.order[tid];
    evals[tid] = s.a[src * LD + src];
    int lead = 0;
    double best = -1.0;
    for (int r = 0; r < n; ++r) {
      const double mag = fabs(vec[r * LD + src]);
      if (mag > best) { best = mag; lead = r; }
    }
    s.order[tid] = (vec[lead * LD + src] < 0.0) ? -(src + 1) : (src + 1);
  }
  __syncthreads();
  if (i < n && j < n) {
    const int code = s.order[j];
    const int src = (code < 0 ? -code : code) - 1;
    const double val = vec[i * LD + src];
    evecs[i * n + j] = code < 0 ? -val : val;
  }
}

// Generalized (M != null) or standard symmetric eigenproblem on s.a / s.m.
// Returns an info code; on NOT_PD, aux gets the eigenvalues of M'.
__device__ int solve_pair(Smem& s, int n, bool generalized, double ridge, double* evals,
                          double* evecs, double* aux) {
  const int tid = threadIdx.x;
  const int i = tid / N, j = tid % N;
  if (generalized) {
    if (is_asym(s, s.a, n)) return UT_INFO_ASYM_A;
    if (is_asym(s, s.m, n)) return UT_INFO_ASYM_M;
    // ridge: M' = M + ridge * (tr M / B) I, or ridge * I if tr M <= 0
    if (tid == 0) {
      double tr = 0.0;
      for (int k = 0; k < n; ++k) tr += s.m[k * LD + k];
      s.scal[1] = ridge * (tr > 0.0 ? tr / n : 1.0);
    }
    __syncthreads();
    if (tid < n) s.m[tid * LD + tid] += s.scal[1];
    __syncthreads();
    // keep M' for the failure report
    if (i < n && j < n) s.x[i * LD + j] = s.m[i * LD + j];
    __syncthreads();
    if (!cholesky(s, n)) {
      if (i < n && j < n) s.a[i * LD + j] = 0.5 * (s.x[i * LD + j] + s.x[j * LD + i]);
      __syncthreads();
      jacobi(s, n);
      sort_desc(s, n);
      if (tid < n) aux[tid] = s.a[s.order[tid] * LD + s.order[tid]];
      return UT_INFO_NOT_PD;
    }
    // C = L^-1 A L^-T: X = L^-1 A; C = L^-1 X^T; symmetrize (eigen.py:107-109)
    solve_lower(s, s.a, n);
    if (i < n && j < n) s.x[i * LD + j] = s.a[j * LD + i];
    __syncthreads();
    solve_lower(s, s.x, n);
    if (i < n && j < n) s.a[i * LD + j] = 0.5 * (s.x[i * LD + j] + s.x[j * LD + i]);
    __syncthreads();
  } else {
    if (i < n && j < n) s.x[i * LD + j] = 0.5 * (s.a[i * LD + j] + s.a[j * LD + i]);
    __syncthreads();
    if (i < n && j < n) s.a[i * LD + j] = s.x[i * LD + j];
    __syncthreads();
  }
  const int info = jacobi(s, n);
  sort_desc(s, n);
  if (generalized) {
    // V = L^-T U (eigen.py:112)
    if (i < n && j < n) s.x[i * LD + j] = s.v[i * LD + j];
    __syncthreads();
    solve_upper_t(s, s.x, n);
    emit(s, s.x, n, evals, evecs);
  } else {
    emit(s, s.v, n, evals, evecs);
  }
  return info;
}

__global__ void __launch_bounds__(kThreads, 1)
gen_eig_kernel(const double* __restrict__ A, const double* __restrict__ M, int n, double ridge,
               double* evals, double* evecs, double* aux, int32_t* info) {
  __shared__ Smem s;
  const int i = threadIdx.x / N, j = threadIdx.x % N;
  if (i < n && j < n) {
    s.a[i * LD + j] = A[i * n + j];
    if (M) s.m[i * LD + j] = M[i * n + j];
  }
  __syncthreads();
  const int code = solve_pair(s, n, M != nullptr, ridge, evals, evecs, aux);
  if (threadIdx.x == 0) *info = code;
}

// moments: [groups][classes][1 + B + B*B] = count, mean, M2 (centred)
__global__ void __launch_bounds__(kThreads, 1)
cva_solve_kernel(const double* __restrict__ mom, int groups, int n, int classes, double ridge,
                 ut_cva_out out) {
  __shared__ Smem s;
  const int tid = threadIdx.x;
  const int i = tid / N, j = tid % N;
  const int len = 1 + n + n * n;
  // per class: pooled count / mean (parallel-axis rule across groups)
  for (int e = tid; e < classes * (1 + n); e += blockDim.x) {
    const int c = e / (1 + n), f = e - c * (1 + n);
    double cnt = 0.0;
    for (int g = 0; g < groups; ++g) cnt += mom[((size_t)g * classes + c) * len];
    if (f == 0) {
      out.counts[c] = cnt;
    } else if (groups == 1) {
      out.class_means[c * n + f - 1] = mom[(size_t)c * len + f];
    } else {
      double acc = 0.0;
      for (int g = 0; g < groups; ++g) {
        const double* r = mom + ((size_t)g * classes + c) * len;
        if (r[0] > 0.0) acc += r[0] * r[f];
      }
      out.class_means[c * n + f - 1] = cnt > 0.0 ? acc / cnt : 0.0;
    }
  }
  __syncthreads();
  // grand mean = sum_c n_c m_c / N
  if (tid < n) {
    double tot = 0.0, acc = 0.0;
    for (int c = 0; c < classes; ++c) {
      tot += out.counts[c];
      acc += out.counts[c] * out.class_means[c * n + tid];
    }
    out.grand_mean[tid] = acc / tot;
  }
  __syncthreads();
  // within = sum_c [sum_g M2_gc + n_gc (m_gc - m_c)(m_gc - m_c)^T]
  // between = sum_c n_c (m_c - m)(m_c - m)^T     (projection.py:196-198)
  if (i < n && j < n) {
    double w = 0.0, b = 0.0;
    for (int c = 0; c < classes; ++c) {
      const double* mc = out.class_means + c * n;
      double wc = 0.0;
      for (int g = 0; g < groups; ++g) {
        const double* r = mom + ((size_t)g * classes + c) * len;
        wc += r[1 + n + i * n + j];
        if (groups > 1 && r[0] > 0.0) wc += r[0] * ((r[1 + i] - mc[i]) * (r[1 + j] - mc[j]));
      }
      w += wc;
      const double gi = mc[i] - out.grand_mean[i], gj = mc[j] - out.grand_mean[j];
      b += out.counts[c] * (gi * gj);
    }
    s.m[i * LD + j] = w;
    s.a[i * LD + j] = b;
  }
  __syncthreads();
  // symmetrize both (projection.py:199-200) and publish the scatter pair
  double wsym = 0.0, bsym = 0.0;
  if (i < n && j < n) {
    wsym = 0.5 * (s.m[i * LD + j] + s.m[j * LD + i]);
    bsym = 0.5 * (s.a[i * LD + j] + s.a[j * LD + i]);
  }
  __syncthreads();
  if (i < n && j < n) {
    s.m[i * LD + j] = wsym;
    s.a[i * LD + j] = bsym;
    out.within[i * n + j] = wsym;
    out.between[i * n + j] = bsym;
  }
  __syncthreads();
  const int code = solve_pair(s, n, true, ridge, out.evals, out.evecs, out.aux);
  if (tid == 0) *out.info = code;
}

// moments: [groups][1 + B + B*B] = n, mean, M2
__global__ void __launch_bounds__(kThreads, 1)
pca_solve_kernel(const double* __restrict__ mom, int groups, int n, ut_pca_out out) {
  __shared__ Smem s;
  const int tid = threadIdx.x;
  const int i = tid / N, j = tid % N;
  const int len = 1 + n + n * n;
  if (tid == 0) {
    double tot = 0.0;
    for (int g = 0; g < groups; ++g) tot += mom[(size_t)g * len];
    s.scal[2] = tot;
  }
  __syncthreads();
  const double tot = s.scal[2];
  if (tid < n) {
    double mean;
    if (groups == 1) {
      mean = mom[1 + tid];
    } else {
      double acc = 0.0;
      for (int g = 0; g < groups; ++g) {
        const double* r = mom + (size_t)g * len;
        if (r[0] > 0.0) acc += r[0] * r[1 + tid];
      }
      mean = acc / tot;
    }
    out.mean[tid] = mean;
  }
  __syncthreads();
  if (i < n && j < n) {
    double g2 = 0.0;
    for (int g = 0; g < groups; ++g) {
      const double* r = mom + (size_t)g * len;
      g2 += r[1 + n + i * n + j];
      if (groups > 1 && r[0] > 0.0)
        g2 += r[0] * ((r[1 + i] - out.mean[i]) * (r[1 + j] - out.mean[j]));
    }
    s.x[i * LD + j] = g2;
  }
  __syncthreads();
  // std = sqrt(diag / (n-1)), 0 -> 1; corr = scatter / (n-1) / outer(std, std)
  if (tid < n) {
    double sd = sqrt(s.x[tid * LD + tid] / (tot - 1.0));
    if (sd == 0.0) sd = 1.0;
    out.std[tid] = sd;
    s.v[tid] = sd;
  }
  __syncthreads();
  if (i < n && j < n) {
    const double c = s.x[i * LD + j] / (tot - 1.0) / (s.v[i] * s.v[j]);
    s.a[i * LD + j] = c;
  }
  __syncthreads();
  if (i < n && j < n) out.corr[i * n + j] = 0.5 * (s.a[i * LD + j] + s.a[j * LD + i]);
  __syncthreads();
  const int code = solve_pair(s, n, false, 0.0, out.evals, out.evecs, nullptr);
  if (tid == 0) *out.info = code;
}

}  // namespace
}  // namespace ut

using namespace ut;

extern "C" {

int ut_gen_eig_sym(const double* A, const double* M, int32_t bands, double ridge, double* evals,
                   double* evecs, double* aux, int32_t* info, void* stream) {
  UT_REQUIRE(bands >= 1 && bands <= kMaxBands, "ut_gen_eig_sym: size must be 1..32");
  UT_REQUIRE(!M || aux, "ut_gen_eig_sym: aux required for the generalized problem");
  gen_eig_kernel<<<1, kThreads, 0, as_stream(stream)>>>(A, M, bands, ridge, evals, evecs,
                                                            aux, info);
  UT_CHECK_LAUNCH("gen_eig_kernel");
  return UT_OK;
}

int ut_cva_solve(const double* moments, int32_t groups, int32_t bands, int32_t classes,
                 double ridge, const ut_cva_out* out, void* stream) {
  UT_REQUIRE(bands >= 1 && bands <= kMaxBands, "ut_cva_solve: bands must be 1..32");
  UT_REQUIRE(groups >= 1 && classes >= 1, "ut_cva_solve: bad groups/classes");
  UT_REQUIRE(out, "ut_cva_solve: null output");
  cva_solve_kernel<<<1, kThreads, 0, as_stream(stream)>>>(moments, groups, bands, classes,
                                                              ridge, *out);
  UT_CHECK_LAUNCH("cva_solve_kernel");
  return UT_OK;
}

int ut_pca_solve(const double* moments, int32_t groups, int32_t bands, const ut_pca_out* out,
                 void* stream) {
  UT_REQUIRE(bands >= 1 && bands <= kMaxBands, "ut_pca_solve: bands must be 1..32");
  UT_REQUIRE(groups >= 1 && out, "ut_pca_solve: bad arguments");
  pca_solve_kernel<<<1, kThreads, 0, as_stream(stream)>>>(moments, groups, bands, *out);
  UT_CHECK_LAUNCH("pca_solve_kernel");
  return UT_OK;
}

}  // extern "C"
