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
// The reference diagonalizes with LAPACK syevd; here a cyclic Jacobi with
// parallel (round-robin) ordering runs in shared memory on a team of 128
// threads (3 named-barrier phases per round).  Cholesky and the triangular
// solves run on one warp (lane = row or column).  Everything is fixed-order,
// so results are deterministic.
//
// CVA low-rank path: S_b = H H^T with H = [sqrt(n_c) (m_c - m)] (B x C), rank
// <= C-1.  With W' = L L^T and G = L^-1 H, the nonzero eigenpairs of
// L^-1 S_b L^-T = G G^T are those of the C x C matrix G^T G (u = G w /
// sqrt(lambda)), so only a C x C Jacobi is needed and the B x B one is skipped.
// Used when the caller wants at most C-1 leading pairs and they are clearly
// non-zero; otherwise the full path runs.
#include "common.cuh"

namespace ut {
namespace {

constexpr int N = kMaxBands;     // 32
constexpr int LD = N + 1;        // padded row stride in shared memory
constexpr int kThreads = N * N;  // 1024 (combine steps use all of them)
#ifndef UT_JACOBI_TEAM
#define UT_JACOBI_TEAM 512  // measured: 128 -> 391 us, 256 -> 305, 512 -> 286, 1024 -> 301 (B = 32 PCA fit)
#endif
constexpr int kTeam = UT_JACOBI_TEAM;  // Jacobi team
constexpr int kMaxC = 32;        // classes handled by the low-rank path

#ifdef UT_PHASES  // dev builds: per-phase %globaltimer stamps of thread 0
__device__ unsigned long long g_eig_phase[32];
#define EPH(i)                                                     \
  do {                                                             \
    if (threadIdx.x == 0) {                                        \
      unsigned long long _t;                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));       \
      g_eig_phase[(i)] = _t;                                       \
    }                                                              \
  } while (0)
#define EPV(i, v)                                     \
  do {                                                \
    if (threadIdx.x == 0) g_eig_phase[(i)] = (v);     \
  } while (0)
#else
#define EPH(i) \
  do {         \
  } while (0)
#define EPV(i, v) \
  do {            \
  } while (0)
#endif

struct Smem {
  double a[N * LD];   // working matrix (A, then C, then Jacobi iterate)
  double m[N * LD];   // M (then L)
  double x[N * LD];   // scratch
  double v[N * LD];   // eigenvectors
  double h[N * LD];   // H, then G = L^-1 H (B x C)
  double cs[N / 2], sn[N / 2], npp[N / 2], nqq[N / 2];
  int pp[N / 2], qq[N / 2], rr[N / 2];
  double red[kThreads / 32];
  double scal[4];
  int flag;
  int order[N];
  int code[N];
  double qd[N], qe[N], qc[N], qs[N];  // tridiagonal QL: diagonal, off-diagonal, rotations
  double hu[N];                        // Householder vector
};

template <int NT> __device__ __forceinline__ void team_sync() {
  if constexpr (NT == 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  }
}

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

// Cyclic Jacobi on a (n x n, stride LD) with eigenvectors in v, run by threads
// [0, NT) of the CTA (the caller parks the others at a __syncthreads).
#ifdef UT_JACOBI_PROBE
__device__ long long g_jprobe[8];
#define JP(i) long long _jp##i = clock64();
#define JACC(i, a, b) if (t == 0) g_jprobe[i] += (_jp##b - _jp##a);
#else
#define JP(i)
#define JACC(i, a, b)
#endif

template <int NT>
__device__ int jacobi_team(Smem& s, double* a, double* v, int n) {
  const int t = threadIdx.x;
  for (int e = t; e < n * n; e += NT) {
    const int i = e / n, j = e - i * n;
    v[i * LD + j] = (i == j) ? 1.0 : 0.0;
  }
  // absolute floor: off-diagonals below 1e-14 * ||A||_F count as zero.  They
  // move eigenvalues by at most that much (<< the 1e-9 * lambda_max bar), and
  // rounding noise of a few eps * ||A|| in rank-deficient matrices (the CVA
  // null space) would otherwise keep the sweeps going.
  double fro = 0.0;
  for (int e = t; e < n * n; e += NT) {
    const int i = e / n, j = e - i * n;
    fro += a[i * LD + j] * a[i * LD + j];
  }
  for (int o = 16; o > 0; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
  if ((t & 31) == 0) s.red[t >> 5] = fro;
  team_sync<NT>();
  double f = 0.0;
  for (int w = 0; w < NT / 32; ++w) f += s.red[w];
  team_sync<NT>();
  const double floor2 = 1e-28 * f;  // (1e-14 ||A||_F)^2
  if (n < 2) return 0;
  const int m = n + (n & 1);
  const int half = m / 2;
  for (int sweep = 0; sweep < 40; ++sweep) {
    int rotated = 0;
    for (int r = 0; r < m - 1; ++r) {
      JP(0)
      // phase A: rotation of pair k (Rutishauser's formulas; round-robin pairs)
      if (t < half) {
        const int k = t;
        int p, q;
        if (k == 0) {
          p = m - 1;
          q = r;
        } else {
          p = r + k;
          if (p >= m - 1) p -= m - 1;
          q = r - k + (m - 1);
          if (q >= m - 1) q -= m - 1;
        }
        if (p > q) { const int tmp = p; p = q; q = tmp; }
        double c = 1.0, sn = 0.0;
        int act = 0;
        if (q < n) {
          const double apq = a[p * LD + q];
          const double app = a[p * LD + p], aqq = a[q * LD + q];
          // |a_pq| > max(eps/2 sqrt(|a_pp a_qq|), floor), squared (no sqrt)
          const double apq2 = apq * apq;
          if (apq2 > 0.25 * DBL_EPSILON * DBL_EPSILON * fabs(app * aqq) && apq2 > floor2) {
            // The angle is evaluated in fp32 with fast intrinsics when the
            // operands are in range (short latency chain); the rotation is then
            // made orthogonal to fp64 accuracy and applied as a full
            // similarity, so the angle's precision only sets how far a_pq drops
            // per step, not the result.
            const double dd = aqq - app, d2 = 2.0 * apq;
            double tt;
            const double mag = fmax(fabs(dd), fabs(d2));
            if (mag < 1e30 && fabs(d2) > 1e-30 && fabs(d2) > 1e-12 * fabs(dd)) {
              const float theta = __fdividef((float)dd, (float)d2);
              const float tf = __frcp_rn(fabsf(theta) + __fsqrt_rn(fmaf(theta, theta, 1.0f)));
              tt = (double)(theta < 0.0f ? -tf : tf);
            } else {  // out of fp32 range: Rutishauser in fp64
              const double theta = dd / d2;
              if (fabs(theta) > 1e150) {
                tt = 0.5 / theta;
              } else {
                tt = 1.0 / (fabs(theta) + sqrt(1.0 + theta * theta));
                if (theta < 0.0) tt = -tt;
              }
            }
            const double x = fma(tt, tt, 1.0);
            double rr = (double)rsqrtf((float)x);  // 1/sqrt(1 + t^2): fp32 guess,
            rr = rr * fma(-0.5 * x, rr * rr, 1.5);  // two Newton steps in fp64
            rr = rr * fma(-0.5 * x, rr * rr, 1.5);
            c = rr;
            sn = tt * rr;
            act = 1;
          }
        }
        s.pp[k] = act ? p : -1;
        s.rr[k] = p;
        s.qq[k] = q;
        s.cs[k] = c;
        s.sn[k] = sn;
        rotated |= act;
      }
      JP(1)
      team_sync<NT>();
      JP(2)
      // phase B: every 2x2 block (pairs k1, k2) <- J_k1^T A J_k2 in one step
      // (the blocks partition A, so each thread owns its block), and V <- V J
      for (int e = t; e < half * half; e += NT) {
        const int k1 = e / half, k2 = e - k1 * half;
        const int p1 = s.pp[k1], p2 = s.pp[k2];
        if (p1 < 0 && p2 < 0) continue;
        const int q1 = s.qq[k1], q2 = s.qq[k2];
        if (p1 >= 0 && p2 >= 0) {
          const double c1 = s.cs[k1], s1 = s.sn[k1], c2 = s.cs[k2], s2 = s.sn[k2];
          const double x00 = a[p1 * LD + p2], x01 = a[p1 * LD + q2];
          const double x10 = a[q1 * LD + p2], x11 = a[q1 * LD + q2];
          const double y00 = c1 * x00 - s1 * x10, y01 = c1 * x01 - s1 * x11;
          const double y10 = s1 * x00 + c1 * x10, y11 = s1 * x01 + c1 * x11;
          a[p1 * LD + p2] = c2 * y00 - s2 * y01;
          a[p1 * LD + q2] = s2 * y00 + c2 * y01;
          a[q1 * LD + p2] = c2 * y10 - s2 * y11;
          a[q1 * LD + q2] = s2 * y10 + c2 * y11;
        } else if (p1 >= 0) {  // rows of pair k1 only; columns of pair k2 (< n)
          const double c1 = s.cs[k1], s1 = s.sn[k1];
          for (int side = 0; side < 2; ++side) {
            const int col = side ? s.qq[k2] : s.rr[k2];
            if (col >= n) continue;
            const double x0 = a[p1 * LD + col], x1 = a[q1 * LD + col];
            a[p1 * LD + col] = c1 * x0 - s1 * x1;
            a[q1 * LD + col] = s1 * x0 + c1 * x1;
          }
        } else {  // columns of pair k2 only
          const double c2 = s.cs[k2], s2 = s.sn[k2];
          for (int side = 0; side < 2; ++side) {
            const int row = side ? s.qq[k1] : s.rr[k1];
            if (row >= n) continue;
            const double x0 = a[row * LD + p2], x1 = a[row * LD + q2];
            a[row * LD + p2] = c2 * x0 - s2 * x1;
            a[row * LD + q2] = s2 * x0 + c2 * x1;
          }
        }
      }
      for (int e = t; e < half * n; e += NT) {
        const int k = e / n, row = e - k * n;
        const int p = s.pp[k];
        if (p >= 0) {
          const int q = s.qq[k];
          const double c = s.cs[k], sn = s.sn[k];
          const double vp = v[row * LD + p], vq = v[row * LD + q];
          v[row * LD + p] = c * vp - sn * vq;
          v[row * LD + q] = sn * vp + c * vq;
        }
      }
      JP(3) JP(4)
      JP(5)
      team_sync<NT>();
      JP(6)
      JACC(0, 0, 1) JACC(1, 1, 2) JACC(2, 2, 3) JACC(3, 3, 4) JACC(4, 4, 5) JACC(5, 5, 6)
    }
    // any rotation this sweep?  (team-wide OR through shared memory)
    const int warp_any = __any_sync(0xffffffffu, rotated);
    if ((t & 31) == 0) s.red[t >> 5] = warp_any ? 1.0 : 0.0;
    team_sync<NT>();
    double any = 0.0;
    for (int w = 0; w < NT / 32; ++w) any += s.red[w];
    team_sync<NT>();
    if (any == 0.0) {
      EPV(NT == 32 ? 30 : 31, (unsigned long long)(sweep + 1));
      return 0;
    }
  }
  return UT_INFO_NO_CONVERGE;
}

// Symmetric eigensolver for n <= 32 run by warp 0 (lane = row): Householder
// reduction to tridiagonal form with the transformations accumulated in v
// (Golub & Van Loan, Alg. 8.3.1), then the implicit QL iteration with
// Wilkinson-type shifts on the tridiagonal matrix (the classic tql2 scheme),
// its Givens rotations applied to the rows of v.  Same contract as
// jacobi_team: on return the eigenvalues are on the diagonal of a (off-
// diagonals zeroed) and the eigenvectors are the columns of v.  The scalar
// QL recurrence runs on lane 0; each QL step's rotation sequence is then
// applied by all lanes to their row of v.  O(n^3) work in ~n^2 warp steps,
// instead of ~9 sweeps x 31 rounds x 2 block barriers of the parallel Jacobi
// at n = 32.  Returns 0, or UT_INFO_NO_CONVERGE (the caller falls back).
__device__ int ql_warp(Smem& s, double* a, double* v, int n) {
  const int lane = threadIdx.x & 31;
  for (int c = 0; c < n; ++c)
    if (lane < n) v[lane * LD + c] = (lane == c) ? 1.0 : 0.0;
  __syncwarp();
  // ---- Householder: zero column k below the subdiagonal, k = 0 .. n-3
  for (int k = 0; k + 2 < n; ++k) {
    const double x = (lane > k && lane < n) ? a[lane * LD + k] : 0.0;
    double ss = x * x;
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const double x1 = __shfl_sync(0xffffffffu, x, k + 1);
    const double alpha = sqrt(ss);
    const double beta = x1 > 0.0 ? -alpha : alpha;
    const double h = ss - beta * x1;  // |u|^2 / 2, u = x - beta e_{k+1}
    if (!(h > 0.0)) continue;         // column already reduced (or all zero)
    const double u = (lane == k + 1) ? x1 - beta : x;
    if (lane < N) s.hu[lane] = u;
    __syncwarp();
    // p = A u / h on the trailing block (rows, columns k+1..n-1)
    double pr = 0.0;
    if (lane > k && lane < n)
      for (int c = k + 1; c < n; ++c) pr += a[lane * LD + c] * s.hu[c];
    pr /= h;
    double up = (lane > k && lane < n) ? u * pr : 0.0;
    for (int o = 16; o > 0; o >>= 1) up += __shfl_xor_sync(0xffffffffu, up, o);
    const double q = pr - (up / (2.0 * h)) * u;  // q = p - K u, K = u^T p / (2h)
    __syncwarp();
    if (lane < N) s.qs[lane] = q;
    __syncwarp();
    if (lane > k && lane < n)
      for (int c = k + 1; c < n; ++c) a[lane * LD + c] -= u * s.qs[c] + q * s.hu[c];
    // column / row k: (beta, 0, ..., 0)
    if (lane > k && lane < n) {
      const double val = (lane == k + 1) ? beta : 0.0;
      a[lane * LD + k] = val;
      a[k * LD + lane] = val;
    }
    // v <- v H, H = I - u u^T / h (lane = row of v)
    if (lane < n) {
      double w = 0.0;
      for (int c = k + 1; c < n; ++c) w += v[lane * LD + c] * s.hu[c];
      w /= h;
      for (int c = k + 1; c < n; ++c) v[lane * LD + c] -= w * s.hu[c];
    }
    __syncwarp();
  }
  // ---- tridiagonal: d = diag, e[i] = a[i+1][i] (e[n-1] = 0)
  if (lane < n) {
    s.qd[lane] = a[lane * LD + lane];
    s.qe[lane] = lane + 1 < n ? a[(lane + 1) * LD + lane] : 0.0;
  }
  __syncwarp();
  int info = 0;
  double f = 0.0, tst1 = 0.0;
  const double eps = DBL_EPSILON;
  for (int l = 0; l < n; ++l) {
    // lane 0 owns the scalar recurrence (d, e in shared memory)
    int m = l, iter = 0;
    if (lane == 0) {
      tst1 = fmax(tst1, fabs(s.qd[l]) + fabs(s.qe[l]));
      while (m < n - 1 && !(fabs(s.qe[m]) <= eps * tst1)) ++m;
    }
    m = __shfl_sync(0xffffffffu, m, 0);
    while (m > l) {
      int nrot = 0;
      if (lane == 0) {
        ++iter;
        double g = s.qd[l];
        double p = (s.qd[l + 1] - g) / (2.0 * s.qe[l]);
        double r = hypot(p, 1.0);
        if (p < 0.0) r = -r;
        s.qd[l] = s.qe[l] / (p + r);
        s.qd[l + 1] = s.qe[l] * (p + r);
        const double dl1 = s.qd[l + 1];
        double hh = g - s.qd[l];
        for (int i = l + 2; i < n; ++i) s.qd[i] -= hh;
        f += hh;
        p = s.qd[m];
        double c = 1.0, c2 = 1.0, c3 = 1.0, sn = 0.0, s2 = 0.0;
        const double el1 = s.qe[l + 1];
        for (int i = m - 1; i >= l; --i) {
          // r = |(p, e_i)| and its reciprocal from one rsqrt (entries are the
          // matrix's scale here: no over/underflow guard needed, unlike the
          // shift above)
          const double ei = s.qe[i], di = s.qd[i];
          c3 = c2;
          c2 = c;
          s2 = sn;
          g = c * ei;
          hh = c * p;
          const double r2 = fma(p, p, ei * ei);
          const double rr = rsqrt(r2);
          s.qe[i + 1] = sn * (r2 * rr);
          sn = ei * rr;
          c = p * rr;
          p = c * di - sn * g;
          s.qd[i + 1] = hh + sn * (c * g + sn * di);
          s.qc[nrot] = c;   // rotation of columns (i, i + 1) of v
          s.qs[nrot] = sn;
          ++nrot;
        }
        p = -sn * s2 * c3 * el1 * s.qe[l] / dl1;
        s.qe[l] = sn * p;
        s.qd[l] = c * p;
        if (fabs(s.qe[l]) <= eps * tst1) m = l;  // converged: leave the loop
        if (iter > 60) {
          info = UT_INFO_NO_CONVERGE;
          m = l;
        }
      }
      nrot = __shfl_sync(0xffffffffu, nrot, 0);
      const int mm = __shfl_sync(0xffffffffu, m, 0);
      __syncwarp();
      if (lane < n) {
        // apply the step's rotations (i = m0-1 down to l) to row `lane` of v
        int i = l + nrot - 1;
        for (int t = 0; t < nrot; ++t, --i) {
          const double c = s.qc[t], sn = s.qs[t];
          const double hv = v[lane * LD + i + 1], vi = v[lane * LD + i];
          v[lane * LD + i + 1] = sn * vi + c * hv;
          v[lane * LD + i] = c * vi - sn * hv;
        }
      }
      __syncwarp();
      m = mm;
    }
    if (lane == 0) {
      s.qd[l] += f;
      s.qe[l] = 0.0;
    }
    __syncwarp();
  }
  info = __shfl_sync(0xffffffffu, info, 0);
  if (lane < n)
    for (int c = 0; c < n; ++c) a[lane * LD + c] = (lane == c) ? s.qd[c] : 0.0;
  __syncwarp();
  return info;
}

#ifndef UT_EIG_QL
#define UT_EIG_QL 1   // 0: parallel Jacobi only (the round-1 solver)
#endif

// Eigen-decomposition of the symmetric a (n x n) into (diag a, v), whole CTA
// calls it.  use_ql: warp 0 runs the Householder + QL solver (if that ever fails
// to converge, the parallel Jacobi team redoes it from the saved matrix in s.x);
// otherwise the parallel Jacobi team.  Measured on B200 (tools/probes/
// solve_speed.py): the generalized CVA problem at B = 32 (C = L^-1 S_b L^-T,
// rank C - 1, a cluster of null eigenvalues) 296 -> 218 us with QL, while the
// B = 32 PCA correlation matrix is faster with Jacobi (9 sweeps: ~250 us vs
// ~300 us for the serial QL chain) and the 6 x 6 low-rank problem is a tie.
// Returns an info code (uniform across the CTA).
__device__ int sym_eig(Smem& s, double* a, double* v, int n, bool use_ql) {
  const int tid = threadIdx.x;
  if (UT_EIG_QL && use_ql) {
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int i = e / n, j = e - i * n;
      s.x[i * LD + j] = a[i * LD + j];
    }
    __syncthreads();
    if (tid < 32) {
      const int code = ql_warp(s, a, v, n);
      if (tid == 0) s.flag = code;
    }
    __syncthreads();
    if (s.flag == 0) return 0;
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int i = e / n, j = e - i * n;
      a[i * LD + j] = s.x[i * LD + j];
    }
    __syncthreads();
  }
  if (tid < kTeam) {
    const int code = jacobi_team<kTeam>(s, a, v, n);
    if (tid == 0) s.flag = code;
  }
  __syncthreads();
  return s.flag;
}

// Cholesky of m (lower, in place) by warp 0; false if a pivot is not > 0.
__device__ bool chol_warp(double* m, int n) {
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < n; ++k) {
    __syncwarp();
    const double d = m[k * LD + k];
    if (!(d > 0.0)) return false;  // also rejects NaN (uniform across lanes)
    const double lkk = sqrt(d);
    __syncwarp();
    if (lane == k) m[k * LD + k] = lkk;
    if (lane > k && lane < n) m[lane * LD + k] /= lkk;
    __syncwarp();
    if (lane > k && lane < n) {
      const double lik = m[lane * LD + k];
      for (int j = k + 1; j <= lane; ++j) m[lane * LD + j] -= lik * m[j * LD + k];
    }
  }
  __syncwarp();
  if (lane < n)
    for (int j = lane + 1; j < n; ++j) m[lane * LD + j] = 0.0;
  __syncwarp();
  return true;
}

// X <- L^-1 X for columns [0, cols) (lane = column), warp 0
__device__ void fsolve_warp(const double* L, double* X, int n, int cols) {
  const int lane = threadIdx.x & 31;
  if (lane < cols) {
    for (int p = 0; p < n; ++p) {
      double acc = X[p * LD + lane];
      for (int q = 0; q < p; ++q) acc -= L[p * LD + q] * X[q * LD + lane];
      X[p * LD + lane] = acc / L[p * LD + p];
    }
  }
  __syncwarp();
}

// X[:, col] <- L^-T X[:, col] (lane -> column cols_of[lane]), warp 0
__device__ void bsolve_warp(const double* L, double* X, int n, int cols, const int* cols_of) {
  const int lane = threadIdx.x & 31;
  if (lane < cols) {
    const int c = cols_of ? cols_of[lane] : lane;
    for (int p = n - 1; p >= 0; --p) {
      double acc = X[p * LD + c];
      for (int q = p + 1; q < n; ++q) acc -= L[q * LD + p] * X[q * LD + c];
      X[p * LD + c] = acc / L[p * LD + p];
    }
  }
  __syncwarp();
}

// order[r] = index of the r-th largest diagonal entry of a (stable on ties)
__device__ void sort_desc(Smem& s, const double* a, int n) {
  const int tid = threadIdx.x;
  if (tid < n) {
    const double me = a[tid * LD + tid];
    int rank = 0;
    for (int o = 0; o < n; ++o) {
      const double other = a[o * LD + o];
      rank += (other > me) || (other == me && o < tid);
    }
    s.order[rank] = tid;
  }
  __syncthreads();
}

// Write nval sorted eigenvalues and `cols` sign-normalized vectors of length b
// (first largest-|entry| made positive, eigen.py:40-52); vector r is column
// s.order[r] of vec.  evecs columns >= cols are written as zeros.
__device__ void emit(Smem& s, const double* a, const double* vec, int b, int nval, int cols,
                     double* evals, double* evecs) {
  const int tid = threadIdx.x;
  const int i = tid / N, j = tid % N;
  if (tid < nval) {
    const int src = s.order[tid];
    evals[tid] = a[src * LD + src];
    int c = src + 1;
    if (tid < cols) {
      int lead = 0;
      double best = -1.0;
      for (int r = 0; r < b; ++r) {
        const double mag = fabs(vec[r * LD + src]);
        if (mag > best) { best = mag; lead = r; }
      }
      if (vec[lead * LD + src] < 0.0) c = -c;
    }
    s.code[tid] = c;
  }
  __syncthreads();
  if (i < b && j < b) {
    double val = 0.0;
    if (j < cols) {
      const int cj = s.code[j];
      const int src = (cj < 0 ? -cj : cj) - 1;
      val = vec[i * LD + src];
      if (cj < 0) val = -val;
    }
    evecs[i * b + j] = val;
  }
  __syncthreads();
}

__device__ void ridge_into_m(Smem& s, int n, double ridge) {
  // M' = M + ridge * (tr M / B) I, or ridge * I if tr M <= 0 (eigen.py:63-72)
  if (threadIdx.x == 0) {
    double tr = 0.0;
    for (int k = 0; k < n; ++k) tr += s.m[k * LD + k];
    s.scal[1] = ridge * (tr > 0.0 ? tr / n : 1.0);
  }
  __syncthreads();
  if (threadIdx.x < n) s.m[threadIdx.x * LD + threadIdx.x] += s.scal[1];
  __syncthreads();
}

// Full path.  Generalized (M in s.m) or standard symmetric problem on s.a.
// Returns an info code; on NOT_PD, aux gets the eigenvalues of M'.
__device__ int solve_full(Smem& s, int n, bool generalized, double ridge, bool checks,
                          double* evals, double* evecs, double* aux) {
  const int tid = threadIdx.x;
  const int i = tid / N, j = tid % N;
  if (generalized) {
    if (checks) {
      if (is_asym(s, s.a, n)) return UT_INFO_ASYM_A;
      if (is_asym(s, s.m, n)) return UT_INFO_ASYM_M;
    }
    ridge_into_m(s, n, ridge);
    if (i < n && j < n) s.x[i * LD + j] = s.m[i * LD + j];  // keep M' for the report
    __syncthreads();
    if (tid < 32) {
      const bool ok = chol_warp(s.m, n);
      if (tid == 0) s.flag = ok ? 1 : 0;
    }
    __syncthreads();
    if (!s.flag) {
      if (i < n && j < n) s.a[i * LD + j] = 0.5 * (s.x[i * LD + j] + s.x[j * LD + i]);
      __syncthreads();
      sym_eig(s, s.a, s.v, n, false);
      sort_desc(s, s.a, n);
      if (tid < n) aux[tid] = s.a[s.order[tid] * LD + s.order[tid]];
      return UT_INFO_NOT_PD;
    }
    // C = L^-1 A L^-T: X = L^-1 A; C = L^-1 X^T; symmetrize (eigen.py:107-109)
    if (tid < 32) fsolve_warp(s.m, s.a, n, n);
    __syncthreads();
    if (i < n && j < n) s.x[i * LD + j] = s.a[j * LD + i];
    __syncthreads();
    if (tid < 32) fsolve_warp(s.m, s.x, n, n);
    __syncthreads();
    if (i < n && j < n) s.a[i * LD + j] = 0.5 * (s.x[i * LD + j] + s.x[j * LD + i]);
    __syncthreads();
  } else {
    if (i < n && j < n) s.x[i * LD + j] = 0.5 * (s.a[i * LD + j] + s.a[j * LD + i]);
    __syncthreads();
    if (i < n && j < n) s.a[i * LD + j] = s.x[i * LD + j];
    __syncthreads();
  }
  const int info = sym_eig(s, s.a, s.v, n, generalized);
  sort_desc(s, s.a, n);
  if (generalized) {
    // V = L^-T U (eigen.py:112)
    if (i < n && j < n) s.x[i * LD + j] = s.v[i * LD + j];
    __syncthreads();
    if (tid < 32) bsolve_warp(s.m, s.x, n, n, nullptr);
    __syncthreads();
    emit(s, s.a, s.x, n, n, n, evals, evecs);
  } else {
    emit(s, s.a, s.v, n, n, n, evals, evecs);
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
  const int code = solve_full(s, n, M != nullptr, ridge, true, evals, evecs, aux);
  if (threadIdx.x == 0) *info = code;
}

// Low-rank CVA solve without triangular solves.  With W' the ridged within
// scatter and S_b = H H^T, the nonzero eigenpairs of W'^-1 S_b come from the
// C x C symmetric matrix T = H^T X, X = W'^-1 H:  T w = lambda w  ->
// v = X w / sqrt(lambda), which is W'-orthonormal (v^T W' v = w^T T w / lambda).
// X is formed by Gauss-Jordan elimination of [W' | H] -- W' is SPD, so no
// pivoting is needed (growth factor <= 1) -- with all (row, column) updates of
// a step in parallel: 2 barriers per step instead of the long serial chains of
// Cholesky + two triangular solves.  Requires want <= C_live - 1 and clearly
// nonzero wanted eigenvalues; returns false otherwise (caller: full path).
// Expects W (unridged, symmetrized) in s.m and H in s.h.
__device__ bool cva_low_rank_gj(Smem& s, int n, int C, double ridge, int want,
                                ut_cva_out& out) {
  const int tid = threadIdx.x, nt = blockDim.x;
  EPH(5);
  ridge_into_m(s, n, ridge);
  // Whole CTA, one barrier per step: every (row i != k, column j > k) entry of
  // [W' | H] is updated in parallel with its own factor m[i][k] / m[k][k];
  // row k is left unnormalized and the pivots are divided out at the end.
  const int wl = n + C;  // columns of [W' | H]
  for (int k = 0; k < n; ++k) {
    const double piv = s.m[k * LD + k];
    if (!(piv > 0.0)) {  // uniform: W' not positive definite
      if (tid == 0) s.flag = 0;
      __syncthreads();
      return false;
    }
    // warp i owns row i (n <= 32 rows, 32 warps): the factor is warp-uniform
    // and the lanes walk the columns > k with no index division
    const int i = tid >> 5;
    if (i < n && i != k) {
      const double g = s.m[i * LD + k] * __drcp_rn(piv);
      for (int q = k + 1 + (tid & 31); q < wl; q += 32) {
        if (q < n) s.m[i * LD + q] -= g * s.m[k * LD + q];
        else s.h[i * LD + (q - n)] -= g * s.h[k * LD + (q - n)];
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < n * C; e += nt) {
    const int i = e / C, c = e - i * C;
    s.h[i * LD + c] /= s.m[i * LD + i];
  }
  if (tid == 0) s.flag = 1;
  __syncthreads();
  if (!s.flag) return false;
  EPH(6);
  // now s.h = X = W'^-1 H.  T = H^T X (H from the outputs), symmetrized
  for (int e = tid; e < C * C; e += nt) {
    const int c1 = e / C, c2 = e - c1 * C;
    double acc = 0.0;
    const double cnt = out.counts[c1];
    if (cnt > 0.0) {
      const double sq = sqrt(cnt);
      for (int p = 0; p < n; ++p)
        acc += sq * (out.class_means[c1 * n + p] - out.grand_mean[p]) * s.h[p * LD + c2];
    }
    s.v[c1 * LD + c2] = acc;  // scratch
  }
  __syncthreads();
  for (int e = tid; e < C * C; e += nt) {
    const int c1 = e / C, c2 = e - c1 * C;
    s.a[c1 * LD + c2] = 0.5 * (s.v[c1 * LD + c2] + s.v[c2 * LD + c1]);
  }
  __syncthreads();
  EPH(7);
  if (tid < 32) {
    const int code = jacobi_team<32>(s, s.a, s.v, C);
    if (tid == 0) s.flag = code;
  }
  __syncthreads();
  EPH(8);
  if (s.flag != 0) return false;
  sort_desc(s, s.a, C);
  const double lmax = s.a[s.order[0] * LD + s.order[0]];
  const double lw = s.a[s.order[want - 1] * LD + s.order[want - 1]];
  if (!(lmax > 0.0) || !(lw > 1e-12 * lmax)) return false;
  // v_r = X w_r / sqrt(lambda_r) into column order[r] of s.m (free now)
  for (int e = tid; e < n * want; e += nt) {
    const int i = e / want, r = e - i * want;
    const int src = s.order[r];
    double acc = 0.0;
    for (int c = 0; c < C; ++c) acc += s.h[i * LD + c] * s.v[c * LD + src];
    s.m[i * LD + src] = acc / sqrt(s.a[src * LD + src]);
  }
  __syncthreads();
  EPH(9);
  if (tid < n) out.evals[tid] = 0.0;  // the null space: exact zeros
  __syncthreads();
  emit(s, s.a, s.m, n, C, want, out.evals, out.evecs);
  EPH(10);
  return true;
}

// moments: [groups][classes][1 + B + B*B] = count, mean, M2 (centred)
__global__ void __launch_bounds__(kThreads, 1)
cva_solve_kernel(const double* __restrict__ mom, int groups, int n, int classes, double ridge,
                 int want, ut_cva_out out) {
  __shared__ Smem s;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int len = 1 + n + n * n;
  EPH(0);
  // per class: pooled count / mean (parallel-axis rule across groups)
  for (int e = tid; e < classes * (1 + n); e += nt) {
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
  EPH(1);
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
  EPH(2);
  // within = sum_c [sum_g M2_gc + n_gc (m_gc - m_c)(m_gc - m_c)^T]
  // between = sum_c n_c (m_c - m)(m_c - m)^T     (projection.py:196-198)
  for (int e = tid; e < n * n; e += nt) {
    const int i = e / n, j = e - i * n;
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
    s.x[i * LD + j] = w;
    s.v[i * LD + j] = b;
  }
  // H = [sqrt(n_c) (m_c - m)] for the low-rank path
  for (int e = tid; e < n * classes && classes <= kMaxC; e += nt) {
    const int i = e / classes, c = e - i * classes;
    const double cnt = out.counts[c];
    s.h[i * LD + c] =
        cnt > 0.0 ? sqrt(cnt) * (out.class_means[c * n + i] - out.grand_mean[i]) : 0.0;
  }
  __syncthreads();
  EPH(3);
  // symmetrize both (projection.py:199-200) and publish the scatter pair
  for (int e = tid; e < n * n; e += nt) {
    const int i = e / n, j = e - i * n;
    const double w = 0.5 * (s.x[i * LD + j] + s.x[j * LD + i]);
    const double b = 0.5 * (s.v[i * LD + j] + s.v[j * LD + i]);
    s.m[i * LD + j] = w;
    s.a[i * LD + j] = b;
    out.within[e] = w;
    out.between[e] = b;
  }
  __syncthreads();
  EPH(4);
  int live = 0;
  for (int c = 0; c < classes; ++c) live += out.counts[c] > 0.0;
  if (classes <= kMaxC && classes <= n && want >= 1 && want <= live - 1) {
    if (cva_low_rank_gj(s, n, classes, ridge, want, out)) {
      if (tid == 0) *out.info = 0;
      return;
    }
    __syncthreads();  // fall back: restore W and S_b
    for (int e = tid; e < n * n; e += nt) {
      const int i = e / n, j = e - i * n;
      s.m[i * LD + j] = out.within[e];
      s.a[i * LD + j] = out.between[e];
    }
    __syncthreads();
  }
  const int code = solve_full(s, n, true, ridge, false, out.evals, out.evecs, out.aux);
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
    s.scal[3] = tot;
  }
  __syncthreads();
  const double tot = s.scal[3];
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
  if (i < n && j < n) s.a[i * LD + j] = s.x[i * LD + j] / (tot - 1.0) / (s.v[i] * s.v[j]);
  __syncthreads();
  if (i < n && j < n) out.corr[i * n + j] = 0.5 * (s.a[i * LD + j] + s.a[j * LD + i]);
  __syncthreads();
  const int code = solve_full(s, n, false, 0.0, false, out.evals, out.evecs, nullptr);
  if (tid == 0) *out.info = code;
}

}  // namespace
}  // namespace ut

using namespace ut;

extern "C" {

#ifdef UT_PHASES
int ut_debug_eig_phases(unsigned long long* host) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(host, g_eig_phase, sizeof(g_eig_phase)) == cudaSuccess ? 0 : 3;
}
#endif

int ut_gen_eig_sym(const double* A, const double* M, int32_t bands, double ridge, double* evals,
                   double* evecs, double* aux, int32_t* info, void* stream) {
  UT_REQUIRE(bands >= 1 && bands <= kMaxBands, "ut_gen_eig_sym: size must be 1..32");
  UT_REQUIRE(!M || aux, "ut_gen_eig_sym: aux required for the generalized problem");
  gen_eig_kernel<<<1, kThreads, 0, as_stream(stream)>>>(A, M, bands, ridge, evals, evecs, aux,
                                                        info);
  UT_CHECK_LAUNCH("gen_eig_kernel");
  return UT_OK;
}

int ut_cva_solve(const double* moments, int32_t groups, int32_t bands, int32_t classes,
                 double ridge, int32_t want, const ut_cva_out* out, void* stream) {
  UT_REQUIRE(bands >= 1 && bands <= kMaxBands, "ut_cva_solve: bands must be 1..32");
  UT_REQUIRE(groups >= 1 && classes >= 1, "ut_cva_solve: bad groups/classes");
  UT_REQUIRE(out, "ut_cva_solve: null output");
  cva_solve_kernel<<<1, kThreads, 0, as_stream(stream)>>>(moments, groups, bands, classes, ridge,
                                                          want, *out);
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
