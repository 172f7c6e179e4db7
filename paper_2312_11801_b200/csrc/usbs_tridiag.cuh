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
  int* iw;      // 128
};

// 1/q correctly rounded (the CUDA double reciprocal: an FP64 MUFU seed and
// Newton steps, no division); measured 1.6x faster inside the LU recurrences
// than an FP32 seed with a range-checked division fallback
__device__ __forceinline__ double fast_rcp(double q) { return __drcp_rn(q); }

// Top-k eigenpairs of the Lanczos projection H (m x m) for the Rayleigh-Ritz
// step.  After a thick restart with ell kept Ritz pairs, H is an arrowhead
// followed by a tridiagonal block:
//
//   H = [ diag(theta_0..theta_{ell-1})  b                       ]
//       [ b^T                           d_ell  e_ell            ]
//       [                               e_ell  d_ell+1  e_ell+1 ]
//       [                                       ...             ]
//
// (ell = 0 in the first cycle: plain tridiagonal).  The entries outside this
// pattern are the O(eps |H|) residue of the full reorthogonalisation; they are
// ignored, which moves eigenvalues by O(eps |H|), the accuracy of eigh itself.
// The structure is used directly, without a Householder reduction:
//   Sturm counts  signs of the LDL^T pivots of H - sigma I, eliminating the
//                 arrow block first (pivots theta_k - sigma), then the
//                 tridiagonal Schur complement, evaluated division-free as
//                 ratios of leading minors (Barth-Martin-Wilkinson): one
//                 dependent FMA per row, minors rescaled by powers of two
//                 every 4 rows; a pivot |q| < pivmin counts as -pivmin as in
//                 LAPACK's ratio form.
//   eigenvalues   multisection, one warp per eigenvalue, 32 shifts per sweep,
//                 to |interval| <= max(4 eps max|endpoint|, eps |H|)
//                 (LAPACK dstebz's default absolute tolerance).
//   eigenvectors  inverse iteration, one thread per eigenvalue, all in
//                 parallel: LU with partial pivoting of H - lam I (the arrow
//                 block first: a swap makes the running arrow row a U row,
//                 stored as its scale mu and its A_ell entry; then the
//                 tridiagonal rows), two solves; eigenvalues closer than 1e-3 |H|
//                 (LAPACK dstein's cluster rule) are perturbed apart and
//                 modified-Gram-Schmidt orthogonalised after every solve.
__device__ __forceinline__ void pow2_rescale(double& p, double& pm) {
  const long long bits = __double_as_longlong(p);
  const int ex = (int)((bits >> 52) & 0x7ff);
  if (ex > 0 && ex < 2046) {
    const double sc = __longlong_as_double((long long)(2046 - ex) << 52);
    p *= sc;
    pm *= sc;
  }
}

// number of eigenvalues of the arrowhead + tridiagonal H below sigma.
// d: diagonal (theta_k for k < ell); sq: b_k^2 for k < ell, e_i^2 for i >= ell.
// Division-free: the arrow block's pivots theta_k - sigma are counted
// directly while a_k = prod_{i<k}(theta_i - sigma) and
// b_k = sum_{i<k} b_i^2 prod_{i'<k, i'!=i}(theta_i' - sigma) accumulate the
// leading minor of the arrow, det = (d_ell - sigma) a_ell - b_ell; from there
// the tridiagonal minors follow the three-term recurrence.  The sign of the
// ratio of consecutive minors is the sign of the LDL^T pivot.
__device__ inline int sturm_arrow(int N, int ell, const double* d, const double* sq, double sigma, double pivmin) {
  int cnt = 0;
  double pa = 1.0, pb = 0.0;
  // rows in blocks of four with the block's d / sq loaded up front, so the
  // shared-memory latency stays off the dependent FMA chain; the power-of-two
  // rescale falls on every block's last row
  auto arrow_row = [&](double f, double s2) {
    if (fabs(f) < pivmin) f = -pivmin;
    cnt += f < 0.0;
    pb = fma(pb, f, s2 * pa);
    pa *= f;
  };
  int k = 0;
  for (; k + 3 < ell; k += 4) {
    const double f0 = d[k] - sigma, f1 = d[k + 1] - sigma, f2 = d[k + 2] - sigma, f3 = d[k + 3] - sigma;
    const double q0 = sq[k], q1 = sq[k + 1], q2 = sq[k + 2], q3 = sq[k + 3];
    arrow_row(f0, q0);
    arrow_row(f1, q1);
    arrow_row(f2, q2);
    arrow_row(f3, q3);
    pow2_rescale(pa, pb);
  }
  for (; k < ell; ++k) arrow_row(d[k] - sigma, sq[k]);
  double pm = pa;
  double p = fma(d[ell] - sigma, pa, -pb);
  if (fabs(p) < pivmin * fabs(pm)) p = -pivmin * pm;
  cnt += (p < 0.0) != (pm < 0.0);
  pow2_rescale(p, pm);
  auto tri_row = [&](double f, double s2) {
    double pn = fma(f, p, -s2 * pm);
    if (fabs(pn) < pivmin * fabs(p)) pn = -pivmin * p;
    cnt += (pn < 0.0) != (p < 0.0);
    pm = p;
    p = pn;
  };
  int i = ell + 1;
  for (; i + 3 < N; i += 4) {
    const double f0 = d[i] - sigma, f1 = d[i + 1] - sigma, f2 = d[i + 2] - sigma, f3 = d[i + 3] - sigma;
    const double q0 = sq[i - 1], q1 = sq[i], q2 = sq[i + 1], q3 = sq[i + 2];
    tri_row(f0, q0);
    tri_row(f1, q1);
    tri_row(f2, q2);
    tri_row(f3, q3);
    pow2_rescale(p, pm);  // row i + 3 = ell + 4 (mod 4)
  }
  for (; i < N; ++i) tri_row(d[i] - sigma, sq[i - 1]);
  return cnt;
}

// All threads of the block call.  H: row-major with leading dimension ldh
// (global or shared).  Outputs: vals[0..nw) descending, Y (row-major N x nw,
// ld ldy; also used as scratch, so it must hold N * nw doubles).
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

struct RrNoShare {
  __device__ void operator()(double*, int, int) const {}
};

// csize > 1 (one CTA of a cluster of csize, rank crank, all calling): the
// eigenvalues are split across the CTAs -- CTA j runs the multisection of
// eigenvalue j with all its warps (32 x warps shifts a sweep instead of 32)
// and share(lam, j, nw) publishes lam[j] to every CTA; the rest of the
// Rayleigh-Ritz step is redundant per CTA as before.
template <class Share = RrNoShare>
__device__ inline void rr_arrow(int N, int ell, int nw, const double* H, int ldh, TriSmem s, double* vals, double* Y,
                                int ldy, unsigned long long* tprof = nullptr, int crank = 0, int csize = 1,
                                Share share = Share()) {
  unsigned long long tlast = (tprof && threadIdx.x == 0) ? tri_clock() : 0ull;
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nwp = nth >> 5;
  double* U0 = s.A;  // [i * nw + j]: reciprocal pivots (arrow: 1/(theta_k - lam))
  double* U1 = s.Q;  // [i * nw + j]: first super-diagonal of U
  double* LM = Y;    // [i * nw + j]: multipliers (Y is written last)
  double* Z = s.Z;   // [i * nw + j]: eigenvectors
  // ------------------------------------------------ 0. read the pattern
  for (int i = tid; i < N; i += nth) {
    s.dd[i] = H[(size_t)i * ldh + i];
    if (i < ell) {
      const double bk = H[(size_t)i * ldh + ell];
      s.v[i] = bk;
      s.p[i] = bk * bk;
    } else {
      const double ei = (i + 1 < N) ? H[(size_t)(i + 1) * ldh + i] : 0.0;
      s.ee[i] = ei;
      s.p[i] = ei * ei;
    }
  }
  __syncthreads();
  // Gershgorin bounds and |H| (every thread, identical)
  double tnorm = 0.0, glo = 0.0, ghi = 0.0;
  {
    double lo = INFINITY, hi = -INFINITY, nm = 0.0, bsum = 0.0;
    for (int k = 0; k < ell; ++k) {
      const double r = fabs(s.v[k]);
      bsum += r;
      lo = fmin(lo, s.dd[k] - r);
      hi = fmax(hi, s.dd[k] + r);
      nm = fmax(nm, fabs(s.dd[k]) + r);
    }
    for (int i = ell; i < N; ++i) {
      const double r = (i > ell ? fabs(s.ee[i - 1]) : bsum) + (i + 1 < N ? fabs(s.ee[i]) : 0.0);
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
  TRI_MARK(0);
  // ------------------------------------------------ 1. multisection
  const bool split = csize >= nw && csize > 1;
  if (split) {
    const int j = crank;
    if (j < nw) {
      // four warps: a sweep's Sturm counts are latency-bound up to ~4 warps
      // and FP64-throughput-bound beyond, so 128 shifts per sweep is the
      // cheapest way down (measured: 16 warps, 512 shifts, cost more per
      // sweep than they save in sweeps)
      const int NWU = nwp < 4 ? nwp : 4;
      const int asc = N - 1 - j, P = NWU * 32;
      const double tol = 2.2e-16 * tnorm;
      double lo = glo, hi = ghi;
      int* wf = s.iw;  // per-warp first shift (the cluster table is built later)
      // the sweep's shifts: geometric above theta_j (first sweep after a
      // restart, as in the warp version) or uniform in (lo, hi)
      auto sweep = [&](bool geo, double l0) {
        if (warp < NWU) {
          const double sig = geo ? (tid < P - 1 ? fmin(l0 + tnorm * exp10(15.0 * tid / (P - 2) - 15.0), ghi) : ghi)
                                 : lo + (hi - lo) * (double)(tid + 1) / (double)(P + 1);
          const int cnt = sturm_arrow(N, ell, s.dd, s.p, sig, pivmin);
          const unsigned mask = __ballot_sync(0xffffffffu, cnt >= asc + 1);
          if (lane == 0) wf[warp] = mask ? __ffs(mask) - 1 : 32;
        }
        __syncthreads();
        int g = P;
        for (int w = 0; w < NWU; ++w)
          if (wf[w] < 32) { g = 32 * w + wf[w]; break; }
        __syncthreads();
        if (geo) {
          const double sg = g < P - 1 ? fmin(l0 + tnorm * exp10(15.0 * g / (P - 2) - 15.0), ghi) : ghi;
          const double sp = g > 0 ? fmin(l0 + tnorm * exp10(15.0 * (g - 1) / (P - 2) - 15.0), ghi) : l0;
          hi = sg;
          lo = sp;
        } else {
          const double nhi = g < P ? lo + (hi - lo) * (double)(g + 1) / (double)(P + 1) : hi;
          const double nlo = g > 0 ? lo + (hi - lo) * (double)g / (double)(P + 1) : lo;
          lo = nlo;
          hi = nhi;
        }
      };
      if (j < ell) {
        const double th = s.dd[j];
        sweep(true, fmax(glo, th - 8.8e-16 * fabs(th) - pivmin));
      }
      for (int it = 0; it < 24; ++it) {
        if (hi - lo <= fmax(4.4e-16 * fmax(fabs(lo), fabs(hi)), tol) + 1e-300) break;
        sweep(false, 0.0);
      }
      if (tid == 0) s.lam[j] = 0.5 * (lo + hi);
    }
    __syncthreads();
    share(s.lam, crank, nw);
  }
  for (int j = split ? nw : warp; j < nw; j += nwp) {
    const int asc = N - 1 - j;  // ascending index of the j-th largest
    double lo = glo, hi = ghi;
    if (j < ell) {
      // after a thick restart the arrow's diagonal holds the kept Ritz values
      // theta_0 >= theta_1 >= ..., the eigenvalues of a principal submatrix,
      // so lambda_j >= theta_j (Cauchy interlacing); the first sweep puts its
      // shifts at theta_j + |H| 10^(k/2 - 15), k = 0..30, and |H|'s upper
      // bound, which brackets lambda_j within a factor 10^0.5 of its distance
      // to theta_j (small once the Ritz values settle)
      const double th = s.dd[j];
      const double l0 = fmax(glo, th - 8.8e-16 * fabs(th) - pivmin);
      const double sig = lane < 31 ? l0 + tnorm * exp10(0.5 * lane - 15.0) : ghi;
      const int cnt0 = sturm_arrow(N, ell, s.dd, s.p, fmin(sig, ghi), pivmin);
      const unsigned mask = __ballot_sync(0xffffffffu, cnt0 >= asc + 1);
      const int first = mask ? __ffs(mask) - 1 : 31;
      const double sf = __shfl_sync(0xffffffffu, fmin(sig, ghi), first);
      const double sp = __shfl_sync(0xffffffffu, fmin(sig, ghi), first > 0 ? first - 1 : 0);
      hi = sf;
      lo = first > 0 ? sp : l0;
    }
    for (int it = 0; it < 24; ++it) {
      if (hi - lo <= fmax(4.4e-16 * fmax(fabs(lo), fabs(hi)), 2.2e-16 * tnorm) + 1e-300) break;
      const double sig = lo + (hi - lo) * (double)(lane + 1) / 33.0;
      const int cnt = sturm_arrow(N, ell, s.dd, s.p, sig, pivmin);
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
  // clusters (descending order): a new one when the gap exceeds 1e-3 |H|;
  // iw[j] = position of j inside its cluster, iw[32 + j] = cluster id
  if (tid == 0) {
    int c = 0, pos = 0;
    for (int j = 0; j < nw; ++j) {
      if (j > 0 && s.lam[j - 1] - s.lam[j] > 1e-3 * tnorm) {
        ++c;
        pos = 0;
      }
      s.iw[j] = pos++;
      s.iw[64 + j] = c;
    }
  }
  __syncthreads();
  TRI_MARK(1);
  // ------------------------------------------------ 2. inverse iteration
  const double eps = 2.2e-16;
  const double tiny = eps * tnorm + 1e-300;
  unsigned long long swp = 0ull;
  if (tid < nw) {
    const int j = tid;
    const double lam = s.lam[j] - (double)s.iw[j] * 10.0 * eps * tnorm;
    // arrow block by partial pivoting: column k's candidates are row k
    // (theta_k - lam) and the running arrow row, whose entries in the
    // columns still to come are mu * b_c (scaled by each swap), A_ell at
    // column ell and mu * e_ell at column ell + 1
    double mu = 1.0, aell = s.dd[ell] - lam;
    auto arrow_col = [&](int k, double dk, double vk) {
      const double D = dk - lam, ak = mu * vk;
      if (fabs(D) >= fabs(ak)) {
        const double piv = (fabs(D) < tiny) ? copysign(tiny, D == 0.0 ? 1.0 : D) : D;
        const double g = fast_rcp(piv);
        const double l = ak * g;
        U0[k * nw + j] = g;
        LM[k * nw + j] = l;
        aell = fma(-l, vk, aell);
      } else {
        const double g = fast_rcp(ak);
        const double l = D * g;
        U0[k * nw + j] = g;
        LM[k * nw + j] = l;
        U1[k * nw + j] = aell;
        swp |= 1ull << k;
        mu = -l * mu;
        aell = fma(-l, aell, vk);
      }
    };
    {
      int k = 0;
      for (; k + 3 < ell; k += 4) {
        const double d0 = s.dd[k], d1 = s.dd[k + 1], d2 = s.dd[k + 2], d3 = s.dd[k + 3];
        const double v0 = s.v[k], v1 = s.v[k + 1], v2 = s.v[k + 2], v3 = s.v[k + 3];
        arrow_col(k, d0, v0);
        arrow_col(k + 1, d1, v1);
        arrow_col(k + 2, d2, v2);
        arrow_col(k + 3, d3, v3);
      }
      for (; k < ell; ++k) arrow_col(k, s.dd[k], s.v[k]);
    }
    double a0 = aell, c0 = (ell + 1 < N) ? mu * s.ee[ell] : 0.0;
    auto tri_col = [&](int i, double bsub, double dn, double cn) {
      if (fabs(a0) >= fabs(bsub)) {
        const double piv = (fabs(a0) < tiny) ? copysign(tiny, a0 == 0.0 ? 1.0 : a0) : a0;
        const double rp = fast_rcp(piv);
        const double l = bsub * rp;
        U0[i * nw + j] = rp;
        U1[i * nw + j] = c0;
        LM[i * nw + j] = l;
        a0 = dn - l * c0;
        c0 = cn;
      } else {
        const double rb = fast_rcp(bsub);
        const double l = a0 * rb;
        U0[i * nw + j] = rb;
        U1[i * nw + j] = dn;
        LM[i * nw + j] = l;
        swp |= 1ull << i;
        a0 = c0 - l * dn;
        c0 = -l * cn;
      }
    };
    {
      int i = ell;
      for (; i + 3 < N - 1; i += 4) {
        double b4[4], d4[4], c4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          b4[u] = s.ee[i + u];
          d4[u] = s.dd[i + u + 1] - lam;
          c4[u] = (i + u + 2 < N) ? s.ee[i + u + 1] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) tri_col(i + u, b4[u], d4[u], c4[u]);
      }
      for (; i < N - 1; ++i) tri_col(i, s.ee[i], s.dd[i + 1] - lam, (i + 2 < N) ? s.ee[i + 1] : 0.0);
    }
    U0[(N - 1) * nw + j] = fast_rcp((fabs(a0) < tiny) ? copysign(tiny, a0 == 0.0 ? 1.0 : a0) : a0);
    // deterministic pseudo-random start vector in (-0.5, 0.5)
    for (int i = 0; i < N; ++i) {
      unsigned h = (unsigned)(i + 1) * 2654435761u ^ (unsigned)(j + 7) * 40503u;
      h ^= h >> 13;
      h *= 0x5bd1e995u;
      h ^= h >> 15;
      Z[i * nw + j] = (double)(h & 0xffffff) / 16777216.0 - 0.5;
    }
  }
  for (int iter = 0; iter < 2; ++iter) {
    if (tid < nw) {
      const int j = tid;
      // the sweeps below go in blocks of four rows whose operands are loaded
      // into registers before any of the block's stores, so the shared-memory
      // latency overlaps the dependent chain (same arithmetic, same order)
      // arrow forward (row k keeps its rhs, or takes the arrow's on a swap)
      double t = Z[ell * nw + j];
      {
        int k = 0;
        for (; k + 3 < ell; k += 4) {
          double l4[4], z4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            l4[u] = LM[(k + u) * nw + j];
            z4[u] = Z[(k + u) * nw + j];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if ((swp >> (k + u)) & 1ull) {
              Z[(k + u) * nw + j] = t;
              t = fma(-l4[u], t, z4[u]);
            } else {
              t = fma(-l4[u], z4[u], t);
            }
          }
        }
        for (; k < ell; ++k) {
          const double l = LM[k * nw + j], zk = Z[k * nw + j];
          if ((swp >> k) & 1ull) {
            Z[k * nw + j] = t;
            t = fma(-l, t, zk);
          } else {
            t = fma(-l, zk, t);
          }
        }
      }
      // tridiagonal forward: L^-1 with the recorded swaps (z_i carried)
      double zi = t;
      {
        int i = ell;
        for (; i + 3 < N - 1; i += 4) {
          double l4[4], n4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            n4[u] = Z[(i + u + 1) * nw + j];
            l4[u] = LM[(i + u) * nw + j];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if ((swp >> (i + u)) & 1ull) {
              Z[(i + u) * nw + j] = n4[u];
              zi = fma(-l4[u], n4[u], zi);
            } else {
              Z[(i + u) * nw + j] = zi;
              zi = fma(-l4[u], zi, n4[u]);
            }
          }
        }
        for (; i < N - 1; ++i) {
          const double zn = Z[(i + 1) * nw + j], l = LM[i * nw + j];
          if ((swp >> i) & 1ull) {
            Z[i * nw + j] = zn;
            zi = fma(-l, zn, zi);
          } else {
            Z[i * nw + j] = zi;
            zi = fma(-l, zi, zn);
          }
        }
      }
      Z[(N - 1) * nw + j] = zi;
      // backward: U z = y  (U row i: 1/U0, U1, and e_{i+1} after a swap)
      double z1 = 0.0, z2 = 0.0;
      {
        auto brow = [&](int i, double tt, double u1, double u0, double e1) {
          if (i + 1 < N) tt -= u1 * z1;
          if (i + 2 < N && ((swp >> i) & 1ull)) tt -= e1 * z2;
          const double zz = tt * u0;
          Z[i * nw + j] = zz;
          z2 = z1;
          z1 = zz;
        };
        int i = N - 1;
        for (; i - 3 >= ell; i -= 4) {
          double t4[4], a4[4], b4[4], e4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int r = i - u;
            t4[u] = Z[r * nw + j];
            a4[u] = U1[r * nw + j];
            b4[u] = U0[r * nw + j];
            e4[u] = (r + 2 < N) ? s.ee[r + 1] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) brow(i - u, t4[u], a4[u], b4[u], e4[u]);
        }
        for (; i >= ell; --i) brow(i, Z[i * nw + j], U1[i * nw + j], U0[i * nw + j], (i + 2 < N) ? s.ee[i + 1] : 0.0);
      }
      // arrow back-substitution; S = sum_{k < c < ell} b_c z_c for the
      // swapped (dense) rows
      const double zl = Z[ell * nw + j], zl1 = (ell + 1 < N) ? Z[(ell + 1) * nw + j] : 0.0;
      double S = 0.0;
      {
        const double eel = s.ee[ell];
        auto arow = [&](int k, double g, double rk, double vk, double u1) {
          double y;
          if ((swp >> k) & 1ull)
            y = fma(rk - u1 * zl, g, -(S + eel * zl1) * fast_rcp(vk));
          else
            y = fma(-vk, zl, rk) * g;
          Z[k * nw + j] = y;
          S = fma(vk, y, S);
        };
        int k = ell - 1;
        for (; k - 3 >= 0; k -= 4) {
          double g4[4], r4[4], v4[4], u4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int r = k - u;
            g4[u] = U0[r * nw + j];
            r4[u] = Z[r * nw + j];
            v4[u] = s.v[r];
            u4[u] = U1[r * nw + j];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) arow(k - u, g4[u], r4[u], v4[u], u4[u]);
        }
        for (; k >= 0; --k) arow(k, U0[k * nw + j], Z[k * nw + j], s.v[k], U1[k * nw + j]);
      }
      double nrm = 0.0;
#pragma unroll 4
      for (int i = 0; i < N; ++i) nrm = fma(Z[i * nw + j], Z[i * nw + j], nrm);
      const double inv = nrm > 0.0 ? rsqrt(nrm) : 0.0;
#pragma unroll 4
      for (int i = 0; i < N; ++i) Z[i * nw + j] *= inv;
    }
    __syncthreads();
    // modified Gram-Schmidt inside clusters: step q removes z_q from the
    // later members (one warp each), z_q already final
    for (int q = 0; q + 1 < nw; ++q) {
      if (s.iw[64 + q + 1] != s.iw[64 + q]) continue;  // q ends its cluster
      const int cid = s.iw[64 + q];
      for (int jj = q + 1 + warp; jj < nw && s.iw[64 + jj] == cid; jj += nwp) {
        double qq = 0.0, qz = 0.0;
        for (int i = lane; i < N; i += 32) {
          const double zq = Z[i * nw + q];
          qq = fma(zq, zq, qq);
          qz = fma(zq, Z[i * nw + jj], qz);
        }
        qq = warp_sum(qq);
        qz = warp_sum(qz);
        const double f = qq > 0.0 ? qz / qq : 0.0;
        for (int i = lane; i < N; i += 32) Z[i * nw + jj] = fma(-f, Z[i * nw + q], Z[i * nw + jj]);
        // normalise jj now if it is the next pivot (keeps magnitudes sane)
      }
      __syncthreads();
    }
    if (tid < nw) {
      const int j = tid;
      double nrm = 0.0;
#pragma unroll 4
      for (int i = 0; i < N; ++i) nrm = fma(Z[i * nw + j], Z[i * nw + j], nrm);
      const double inv = nrm > 0.0 ? rsqrt(nrm) : 0.0;
#pragma unroll 4
      for (int i = 0; i < N; ++i) Z[i * nw + j] *= inv;
    }
    __syncthreads();
  }
  TRI_MARK(2);
  // ------------------------------------------------ 3. output
  for (int x = tid; x < N * nw; x += nth) {
    const int i = x / nw, j = x % nw;
    Y[(size_t)i * ldy + j] = Z[x];
  }
  for (int j = tid; j < nw; j += nth) vals[j] = s.lam[j];
  __syncthreads();
  TRI_MARK(3);
}

}  // namespace usbs
