// Top-k symmetric eigensolver for the Lanczos Rayleigh-Ritz step (N <= 64),
// FP64, block-cooperative, in shared memory.  Same contract as the call it
// replaces (symlin.small_eigh on H[:m,:m], eigsolve.py:152) restricted to the
// eigenpairs the thick-restart Lanczos uses: the nw algebraically largest
// (theta[:ell] and Y[:, :ell] for the restart, theta[:k_c], Y[:, :k_c] and
// the last row Y[m-1, :k_c] for the residuals).
//
//   1. Householder tridiagonalisation H = Q T Q^T (GvL Alg. 8.3.1, Q
//      accumulated); skipped when H is already tridiagonal (first cycle).
//   2. Eigenvalues of T by multisection on Sturm counts: one warp per
//      eigenvalue, 32 shifts per sweep (5 bits), to |interval| <= 2 eps |T|.
//   3. Eigenvectors of T by inverse iteration (tridiagonal LU with partial
//      pivoting, LAPACK dlagtf/dlagts style), two iterations, with
//      re-orthogonalisation inside clusters (|lambda_i - lambda_j| <= 1e-3|T|),
//      as LAPACK dstein.
//   4. Y = Q Z.
// Eigenvalue accuracy matches LAPACK (~eps |T|); vectors ~eps |T| / gap.
#pragma once
#include "usbs_common.cuh"

namespace usbs {

struct TriSmem {
  double* A;    // N*N input (destroyed)
  double* Q;    // N*N accumulated reflectors
  double* Z;    // N*nw eigenvectors of T (column-major: Z[j*N + i])
  double* v;    // N
  double* p;    // N
  double* dd;   // N diagonal of T
  double* ee;   // N off-diagonal of T
  double* lam;  // 64 eigenvalues (descending)
  double* red;  // 64
  int* iw;      // 64
};

// 1/q to ~1 ulp: FP32 MUFU seed + two Newton steps (4 dependent DFMA), exact
// division only when q is outside the FP32 range.
__device__ __forceinline__ double fast_rcp(double q) {
  const double aq = fabs(q);
  if (!(aq > 1e-37 && aq < 1e37)) return 1.0 / q;
  double r = (double)__frcp_rn((float)q);
  r = fma(r, fma(-q, r, 1.0), r);
  r = fma(r, fma(-q, r, 1.0), r);
  return r;
}

// number of eigenvalues of T below sigma (LDL^T pivot signs, Kahan's form);
// e2[i] = e[i]^2.  An approximate reciprocal perturbs e2 by ~1e-16 relative,
// i.e. a backward-stable count.
__device__ inline int sturm_count(const double* d, const double* e2, int N, double sigma, double pivmin) {
  int cnt = 0;
  double q = d[0] - sigma;
  if (fabs(q) < pivmin) q = -pivmin;
  if (q < 0.0) ++cnt;
  for (int i = 1; i < N; ++i) {
    q = (d[i] - sigma) - e2[i - 1] * fast_rcp(q);
    if (fabs(q) < pivmin) q = -pivmin;
    if (q < 0.0) ++cnt;
  }
  return cnt;
}

// All threads of the block call.  tridiagonal != 0: A already tridiagonal.
// Outputs: vals[0..nw) descending, Y (row-major N x nw, ld ldy).
__device__ __forceinline__ unsigned long long tri_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#define TRI_MARK(slot)                                  \
  do {                                                  \
    if (tprof && threadIdx.x == 0) {                    \
      const unsigned long long _t = tri_clock();        \
      tprof[slot] += _t - tlast;                        \
      tlast = _t;                                       \
    }                                                   \
  } while (0)

__device__ inline void rr_topk(int N, int nw, int tridiagonal, TriSmem s, double* vals, double* Y, int ldy,
                               unsigned long long* tprof = nullptr) {
  unsigned long long tlast = (tprof && threadIdx.x == 0) ? tri_clock() : 0ull;
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nwp = nth >> 5;
  double* A = s.A;
  // ------------------------------------------------ 1. tridiagonalisation
  for (int x = tid; x < N * N; x += nth) s.Q[x] = (x / N == x % N) ? 1.0 : 0.0;
  __syncthreads();
  if (!tridiagonal) {
    for (int k = 0; k + 2 < N; ++k) {
      const int L = N - k - 1;  // length of x = A[k+1.., k]
      // Householder vector (warp 0): v(0) = 1, beta
      if (warp == 0) {
        double sg = 0.0;
        for (int i = 1 + lane; i < L; i += 32) {
          const double xi = A[(k + 1 + i) * N + k];
          sg = fma(xi, xi, sg);
        }
        sg = warp_sum(sg);
        const double x0 = A[(k + 1) * N + k];
        double beta = 0.0, mu = x0, v0 = 1.0;
        if (sg != 0.0) {
          mu = sqrt(fma(x0, x0, sg));
          v0 = (x0 <= 0.0) ? x0 - mu : -sg / (x0 + mu);
          beta = 2.0 * v0 * v0 / (sg + v0 * v0);
          // H x = mu e1 when x0 <= 0 ... GvL: H x = ||x|| e1
        }
        for (int i = lane; i < L; i += 32) s.v[i] = (i == 0) ? 1.0 : (sg != 0.0 ? A[(k + 1 + i) * N + k] / v0 : 0.0);
        if (lane == 0) {
          s.red[0] = beta;
          s.red[1] = (sg != 0.0) ? mu : x0;
        }
      }
      __syncthreads();
      const double beta = s.red[0];
      if (beta != 0.0) {
        // p = beta A22 v (warp per row)
        for (int i = warp; i < L; i += nwp) {
          double t = 0.0;
          for (int c = lane; c < L; c += 32) t = fma(A[(k + 1 + i) * N + (k + 1 + c)], s.v[c], t);
          t = warp_sum(t);
          if (lane == 0) s.p[i] = beta * t;
        }
        __syncthreads();
        // every warp forms K = beta/2 p^T v itself (no extra barrier); rows of
        // A22 -= v w^T + w v^T with w = p - K v, and Q[:, k+1:] -= beta (Q v) v^T
        double K = 0.0;
        for (int c = lane; c < L; c += 32) K = fma(s.p[c], s.v[c], K);
        K = 0.5 * beta * warp_sum(K);
        for (int i = warp; i < L; i += nwp) {
          const double vi = s.v[i], wi = s.p[i] - K * vi;
          double* row = A + (k + 1 + i) * N + (k + 1);
          for (int c = lane; c < L; c += 32) {
            const double vc = s.v[c];
            row[c] -= vi * (s.p[c] - K * vc) + wi * vc;
          }
        }
        for (int i = warp; i < N; i += nwp) {
          double* row = s.Q + i * N + (k + 1);
          double t = 0.0;
          for (int c = lane; c < L; c += 32) t = fma(row[c], s.v[c], t);
          t = beta * warp_sum(t);
          for (int c = lane; c < L; c += 32) row[c] -= t * s.v[c];
        }
      }
      if (tid == 0) {
        A[(k + 1) * N + k] = s.red[1];
        A[k * N + (k + 1)] = s.red[1];
      }
      for (int i = k + 2 + tid; i < N; i += nth) {
        A[i * N + k] = 0.0;
        A[k * N + i] = 0.0;
      }
      __syncthreads();
    }
  }
  for (int i = tid; i < N; i += nth) {
    s.dd[i] = A[i * N + i];
    s.ee[i] = (i + 1 < N) ? A[(i + 1) * N + i] : 0.0;
    s.p[i] = s.ee[i] * s.ee[i];  // e^2 for the Sturm counts
  }
  __syncthreads();
  TRI_MARK(0);
  // ------------------------------------------------ 2. multisection bisection
  double tnorm = 0.0, glo = 0.0, ghi = 0.0;
  {
    double lo = INFINITY, hi = -INFINITY, nm = 0.0;
    for (int i = 0; i < N; ++i) {
      const double r = (i > 0 ? fabs(s.ee[i - 1]) : 0.0) + (i + 1 < N ? fabs(s.ee[i]) : 0.0);
      lo = fmin(lo, s.dd[i] - r);
      hi = fmax(hi, s.dd[i] + r);
      nm = fmax(nm, fabs(s.dd[i]) + r);
    }
    tnorm = nm;
    const double pad = 2.2e-16 * nm * N + 1e-300;
    glo = lo - pad;
    ghi = hi + pad;
  }
  const double pivmin = 1e-300 + 2.2e-16 * 2.2e-16 * tnorm * tnorm;
  for (int j = warp; j < nw; j += nwp) {
    const int asc = N - 1 - j;  // ascending index of the j-th largest
    double lo = glo, hi = ghi;
    for (int it = 0; it < 16; ++it) {
      if (hi - lo <= 2.2e-16 * fmax(fabs(lo), fabs(hi)) * 2.0 + 1e-300) break;
      const double sig = lo + (hi - lo) * (double)(lane + 1) / 33.0;
      const int cnt = sturm_count(s.dd, s.p, N, sig, pivmin);
      const unsigned mask = __ballot_sync(0xffffffffu, cnt >= asc + 1);
      const int first = mask ? __ffs(mask) - 1 : 32;
      const double nhi = (first < 32) ? lo + (hi - lo) * (double)(first + 1) / 33.0 : hi;
      const double nlo = (first > 0) ? lo + (hi - lo) * (double)first / 33.0 : lo;
      lo = nlo;
      hi = nhi;
    }
    if (lane == 0) s.lam[j] = 0.5 * (lo + hi);
  }
  __syncthreads();
  TRI_MARK(1);
  // ------------------------------------------------ 3. inverse iteration
  // cluster boundaries (descending order): new cluster when the gap exceeds 1e-3 |T|
  if (tid == 0) {
    int c = 0;
    for (int j = 0; j < nw; ++j) {
      if (j > 0 && s.lam[j - 1] - s.lam[j] > 1e-3 * tnorm) ++c;
      s.iw[j] = c;
    }
  }
  __syncthreads();
  // one thread per eigenvalue solves (T - lam I) z = b twice; clusters are
  // handled by their first member's thread, sequentially (re-orthogonalised)
  const double eps = 2.2e-16;
  for (int j = tid; j < nw; j += nth) {
    if (j > 0 && s.iw[j] == s.iw[j - 1]) continue;  // not a cluster leader
    int jend = j;
    while (jend + 1 < nw && s.iw[jend + 1] == s.iw[j]) ++jend;
    for (int jj = j; jj <= jend; ++jj) {
      // perturb members of a cluster apart as dstein does
      const double lam = s.lam[jj] - (double)(jj - j) * 10.0 * eps * tnorm;
      double* z = s.Z + (size_t)jj * N;
      // LU with partial pivoting of T - lam I: rows hold (l, u0, u1, u2)
      double u0[64], u1[64], u2[64], lm[64];
      int swp[64];
      double a0 = s.dd[0] - lam, c0 = N > 1 ? s.ee[0] : 0.0;
      const double tiny = eps * tnorm + 1e-300;
      for (int i = 0; i < N - 1; ++i) {
        const double b = s.ee[i];  // sub-diagonal entry below the pivot
        const double dn = s.dd[i + 1] - lam;
        const double cn = (i + 2 < N) ? s.ee[i + 1] : 0.0;
        // u0 keeps the reciprocal pivot (guarded away from zero), so the
        // solves below only multiply
        if (fabs(a0) >= fabs(b)) {
          const double piv = (fabs(a0) < tiny) ? copysign(tiny, a0 == 0.0 ? 1.0 : a0) : a0;
          const double rp = fast_rcp(piv);
          const double l = b * rp;
          u0[i] = rp; u1[i] = c0; u2[i] = 0.0; lm[i] = l; swp[i] = 0;
          a0 = dn - l * c0;
          c0 = cn;
        } else {
          const double l = a0 * fast_rcp(b);
          u0[i] = fast_rcp(b); u1[i] = dn; u2[i] = cn; lm[i] = l; swp[i] = 1;
          a0 = c0 - l * dn;
          c0 = -l * cn;
        }
      }
      u0[N - 1] = fast_rcp((fabs(a0) < tiny) ? copysign(tiny, a0 == 0.0 ? 1.0 : a0) : a0);
      // deterministic pseudo-random start vector in (-0.5, 0.5), three solves
      for (int i = 0; i < N; ++i) {
        unsigned h = (unsigned)(i + 1) * 2654435761u ^ (unsigned)(jj + 7) * 40503u;
        h ^= h >> 13;
        h *= 0x5bd1e995u;
        h ^= h >> 15;
        z[i] = (double)(h & 0xffffff) / 16777216.0 - 0.5;
      }
      for (int iter = 0; iter < 2; ++iter) {
        // forward: apply L^-1 with the recorded swaps
        for (int i = 0; i < N - 1; ++i) {
          if (swp[i]) {
            const double t = z[i];
            z[i] = z[i + 1];
            z[i + 1] = t - lm[i] * z[i];
          } else {
            z[i + 1] -= lm[i] * z[i];
          }
        }
        // backward: U z = y
        for (int i = N - 1; i >= 0; --i) {
          double t = z[i];
          if (i + 1 < N) t -= u1[i] * z[i + 1];
          if (i + 2 < N) t -= u2[i] * z[i + 2];
          z[i] = t * u0[i];
        }
        // re-orthogonalise against earlier cluster members, normalise
        for (int q = j; q < jj; ++q) {
          const double* zq = s.Z + (size_t)q * N;
          double dp = 0.0;
          for (int i = 0; i < N; ++i) dp = fma(zq[i], z[i], dp);
          for (int i = 0; i < N; ++i) z[i] -= dp * zq[i];
        }
        double nrm = 0.0;
        for (int i = 0; i < N; ++i) nrm = fma(z[i], z[i], nrm);
        nrm = sqrt(nrm);
        const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
        for (int i = 0; i < N; ++i) z[i] *= inv;
      }
    }
  }
  __syncthreads();
  TRI_MARK(2);
  // ------------------------------------------------ 4. Y = Q Z
  for (int x = tid; x < N * nw; x += nth) {
    const int i = x / nw, j = x % nw;
    double t = 0.0;
    for (int c = 0; c < N; ++c) t = fma(s.Q[i * N + c], s.Z[(size_t)j * N + c], t);
    Y[i * ldy + j] = t;
  }
  for (int j = tid; j < nw; j += nth) vals[j] = s.lam[j];
  __syncthreads();
  TRI_MARK(3);
}

}  // namespace usbs
