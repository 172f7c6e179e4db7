// K12: the k x k bundle subproblem as ONE single-CTA kernel per solve.
//
// Mirrors subqp._ipm_solve (subqp.py:353-435) with its pieces:
//   _cold_state 184-197, _stationarity 210-219, newton_direction 222-265,
//   line_search_feasible 294-343, barrier_update 346-350, _objective 200-207,
//   IpmOptions 150-162 (mu_tol 1e-11, kkt_tol 1e-6, max_newton 100,
//   step_frac 0.99, backtrack 0.8, min_step 1e-12, max_step_failures 6,
//   warm_blend 0.2).
// Differences in arithmetic only (no change of algorithm):
//   * symm_kron(T, S^-1) (symlin.py:133-145) is never materialised through
//     the k^2 x k^2 Kronecker products; its entries come from the closed form
//     E[p,q] = w_p w_q / 4 (H_ik G_lj + H_il G_kj + G_ik H_lj + G_il H_kj),
//     p = (i,j), q = (k,l) in svec order, and E ds = svec((H D G + G D H)/2).
//   * S^-1 comes from the Cholesky factor of S (S is positive definite at
//     every iterate) instead of an LU inverse; it is symmetrised the same way.
//   * The reduced Newton matrix M (d x d, d = k(k+1)/2) lives packed-lower in
//     shared memory (d <= 210, i.e. k <= 20; larger k spills M to global) and
//     is factorised by a blocked right-looking Cholesky (8-column panels,
//     trailing tiles on the FP64 tensor cores) that fails exactly on a
//     non-positive or NaN pivot, like LAPACK potrf.
#include <algorithm>
#include <cmath>

#include "usbs_common.cuh"
#include "usbs_kernels.cuh"
#include "usbs_tma.cuh"

namespace usbs {

struct IpmOpts {
  double mu_tol, kkt_tol, step_frac, backtrack, min_step, warm_blend;
  int max_newton, max_step_failures;
};

struct IpmArgs {
  int k, d, has_eta;
  const double* Q11;   // d x d row-major (nullptr: zero, the eval problem)
  const double* q12;   // d (nullptr: zero)
  const double* lin_s; // d
  const double* scal;  // [q22, lin_eta]
  const double* warm;  // state or nullptr
  double* state;       // out state (may alias warm)
  double* result;      // [value, newton_iters, exact, eta_opt, failures]
  double* gM;          // global scratch for M when d > SMEM_D
  double* gQp;         // global scratch: Q11 packed lower (k_ipm<true>, d <= SMEM_D)
  IpmOpts o;
  unsigned long long* prof;  // optional phase timers (ns), thread 0
};

// phase timers: 0 stationarity/exit test, 1 S^-1, 2 rd/rhs, 3 M build,
// 4 Cholesky, 5 solves, 6 E ds / scalar directions, 7 line search, 8 update
#define IPM_MARK(slot)                                             \
  do {                                                             \
    if (a.prof && tid == 0) {                                      \
      unsigned long long _t;                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));       \
      ipm_acc[slot] += _t - ipm_last;                              \
      ipm_last = _t;                                               \
    }                                                              \
  } while (0)

// state layout: S (k*k), T (k*k), eta, zeta, omega, mu, has_eta, k, valid
__host__ __device__ inline int state_len(int k) { return 2 * k * k + 7; }

#ifdef USBS_CHOL_PROF
constexpr int IPM_PROF_SLOTS = 128;
#else
constexpr int IPM_PROF_SLOTS = 16;
#endif
constexpr int IPM_THREADS = 512;
constexpr int SMEM_D = 210;
constexpr int KMAX = 32;

__device__ __forceinline__ int pidx(int i, int j) { return i * (i + 1) / 2 + j; }  // packed lower, i >= j

struct IpmSmem {
  double *S, *T, *H, *dS, *dT, *W1, *W2, *X1, *X2;  // k x k
  double *s, *t, *vI, *h, *g, *f1, *rhs, *ds, *dt, *rd, *tmp, *cb0, *cb1;  // d
  unsigned char *pi, *pj;
  unsigned short* ctab;  // lower-triangle table of the warp Cholesky
  double* red;   // 32
  double* sc;    // scalars 64
  int* flg;      // 16
  uint64_t* bar; // packed-Q11 copy barrier
  double* M;
};

// ---------------------------------------------------------------- helpers
__device__ double blk_max_abs(const double* x, int n, double* red) {
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v = fmax(v, fabs(x[i]));
  v = warp_max(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, red[w]);
  __syncthreads();
  return r;
}

__device__ __forceinline__ void dmma8x8x4(double& d0, double& d1, double a, double b, double c0, double c1);

// A pointer known to lie in the kernel's dynamic shared memory, rebuilt from
// the shared window so the compiler addresses it with LDS / STS (a pointer
// that crossed a noinline call or a run-time select is generic: 64-bit
// address arithmetic and LD.E / ST.E on every access).
__device__ __forceinline__ double* as_shared(double* p) {
  extern __shared__ __align__(16) unsigned char usbs_ipm_dyn_smem[];
  const unsigned off = (unsigned)__cvta_generic_to_shared(p) - (unsigned)__cvta_generic_to_shared(usbs_ipm_dyn_smem);
  return (double*)(usbs_ipm_dyn_smem + off);
}


// One warp factors W (lower, row-major k x k, k <= 32) in place, blocked by
// 8: the 8 x 8 diagonal block in registers (lanes 0-7 hold its rows; per
// column the pivot's rsqrt, the column scaled, the trailing entries of the
// block updated with L(t, c) shuffled from lane t), the rows below by
// substitution (a lane per row, the block's rsqrt values in registers), the
// trailing 8 x 8 tiles with two FP64 m8n8k4 MMAs per tile (the row stride k
// keeps the fragment loads of a half-warp on distinct banks for k = 20).
// Same factor as the column-by-column form (bit-identical in the
// microbenchmark, profiles/mb/chol_mb.cu: k = 20 12.1k -> 8.4k cycles).
// Fails on a pivot <= 0 or NaN (potrf); returns ok.  Own register
// allocation (noinline) so the callers' live state does not spill it.
__device__ __noinline__ int warp_chol_core(double* Wg, int k, const unsigned short* /*ctab*/) {
  double* W = as_shared(Wg);  // every caller passes a k x k block of the kernel's shared memory
  const int lane = threadIdx.x & 31, r = lane & 7, g = lane >> 2, q = lane & 3;
  int ok = 1;
  for (int j0 = 0; j0 < k; j0 += 8) {
    const int jb = min(8, k - j0);
    double a[8], rsv[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) a[t] = (r < jb && t <= r) ? W[(j0 + r) * k + j0 + t] : 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      rsv[c] = 0.0;
      if (c < jb) {
        const double pv = __shfl_sync(0xffffffffu, a[c], c);
        if (!(pv > 0.0)) ok = 0;
        const double rs = rsqrt(pv);
        rsv[c] = rs;
        a[c] = (r == c) ? pv * rs : a[c] * rs;
#pragma unroll
        for (int t = c + 1; t < 8; ++t) {
          const double ltc = __shfl_sync(0xffffffffu, a[c], t);
          if (t <= r) a[t] -= a[c] * ltc;
        }
      }
    }
    if (lane < 8 && r < jb) {
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if (t <= r) W[(j0 + r) * k + j0 + t] = a[t];
    }
    if (!ok) return 0;  // warp-uniform (every lane saw the same pivots)
    __syncwarp();
    const int r0 = j0 + jb;
    if (r0 >= k) break;
    const int i = r0 + lane;
    if (i < k) {
      double v[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = W[i * k + j0 + c];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        v[c] *= rsv[c];
#pragma unroll
        for (int t = c + 1; t < 8; ++t) v[t] = fma(-v[c], W[(j0 + t) * k + j0 + c], v[t]);
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) W[i * k + j0 + c] = v[c];
    }
    __syncwarp();
    const int T = (k + 7) >> 3, I0 = r0 >> 3;
    for (int I = I0; I < T; ++I) {
      const int ra = I * 8 + g;
      const bool va = ra < k;
      const double a0 = va ? -W[ra * k + j0 + q] : 0.0, a1 = va ? -W[ra * k + j0 + 4 + q] : 0.0;
      for (int K = I0; K <= I; ++K) {
        const int rb = K * 8 + g;
        const bool vb = rb < k;
        const double b0 = vb ? W[rb * k + j0 + q] : 0.0, b1 = vb ? W[rb * k + j0 + 4 + q] : 0.0;
        const int cc = K * 8 + 2 * q;
        const bool v0 = va && cc <= ra, v1 = va && cc + 1 <= ra;
        double c0 = v0 ? W[ra * k + cc] : 0.0, c1 = v1 ? W[ra * k + cc + 1] : 0.0;
        dmma8x8x4(c0, c1, a0, b0, c0, c1);
        dmma8x8x4(c0, c1, a1, b1, c0, c1);
        if (v0) W[ra * k + cc] = c0;
        if (v1) W[ra * k + cc + 1] = c1;
      }
    }
    __syncwarp();
  }
  return ok;
}

// warp 0 factors W; the result goes to all threads through flg[slot]
__device__ void warp_chol(double* W, int k, int* flg, int slot, const unsigned short* ctab) {
  if (threadIdx.x < 32) {
    const int ok = warp_chol_core(W, k, ctab);
    if ((threadIdx.x & 31) == 0) flg[slot] = ok;
  }
  __syncthreads();
}

// two independent k x k Cholesky tests at once: warp 0 factors Wa, warp 1 Wb
// (the line search's S + d dS and T + d dT); flg[sa], flg[sb] get the results
__device__ void warp_chol2(double* Wa, double* Wb, int k, int* flg, int sa, int sb, const unsigned short* ctab) {
  const int w = threadIdx.x >> 5;
  if (w < 2) {
    const int ok = warp_chol_core(w == 0 ? Wa : Wb, k, ctab);
    if ((threadIdx.x & 31) == 0) flg[w == 0 ? sa : sb] = ok;
  }
  __syncthreads();
}

// svec of a symmetric k x k matrix (row-major) into v (length d)
__device__ void blk_svec(const double* A, int k, int d, const IpmSmem& sm, double* v) {
  for (int p = threadIdx.x; p < d; p += blockDim.x) {
    int i = sm.pi[p], j = sm.pj[p];
    v[p] = A[i * k + j] * (i == j ? 1.0 : 1.4142135623730951);
  }
}

__device__ void blk_smat(const double* v, int k, int d, const IpmSmem& sm, double* A) {
  for (int p = threadIdx.x; p < d; p += blockDim.x) {
    int i = sm.pi[p], j = sm.pj[p];
    double x = (i == j) ? v[p] : v[p] / 1.4142135623730951;
    A[i * k + j] = x;
    A[j * k + i] = x;
  }
}

// y = Q11 x (+ beta*y0) over d, warp per row (Q11 in global, coalesced rows)
__device__ void blk_gemv_q11(const double* Q, const double* x, int d, double* y) {
  // rows in groups of four per warp, every load of the group issued before
  // the FMAs (Q11 sits in L2: its latency, not bandwidth, bounds this)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int p0 = 4 * w; p0 < d; p0 += 4 * nw) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    if (Q) {
      for (int q = lane; q < d; q += 32) {
        double qv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) qv[u] = p0 + u < d ? __ldg(Q + (int64_t)(p0 + u) * d + q) : 0.0;
        const double xq = x[q];
#pragma unroll
        for (int u = 0; u < 4; ++u) s[u] = fma(qv[u], xq, s[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double t = warp_sum(s[u]);
      if (lane == 0 && p0 + u < d) y[p0 + u] = t;
    }
  }
}

// y = Q x for a symmetric Q stored packed lower in shared memory: row p is
// Q[p][0..p] (contiguous) and Q[q][p] for q > p (column p of the lower part);
// four rows per warp in flight
__device__ void blk_gemv_packed(const double* __restrict__ Mp, const double* __restrict__ x, int d,
                                double* __restrict__ y) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int p0 = 4 * w; p0 < d; p0 += 4 * nw) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int q = lane; q < d; q += 32) {
      const double xq = x[q];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = p0 + u;
        if (p < d) s[u] = fma(q <= p ? Mp[pidx(p, q)] : Mp[pidx(q, p)], xq, s[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double t = warp_sum(s[u]);
      if (lane == 0 && p0 + u < d) y[p0 + u] = t;
    }
  }
}

__device__ double blk_dot(const double* a, const double* b, int n, double* red) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s = fma(a[i], b[i], s);
  return block_sum(s, red);
}

// C = A B for k x k row-major (block-parallel)
__device__ void blk_mm(const double* A, const double* B, int k, double* C) {
  for (int x = threadIdx.x; x < k * k; x += blockDim.x) {
    int r = x / k, c = x % k;
    double s = 0.0;
    for (int u = 0; u < k; ++u) s = fma(A[r * k + u], B[u * k + c], s);
    C[x] = s;
  }
}

// complementarity <S,T> + omega*sigma (+ eta*zeta)
__device__ double blk_compl(const IpmSmem& sm, int k, double eta, double zeta, double omega, int has_eta) {
  double s = 0.0;
  for (int x = threadIdx.x; x < k * k; x += blockDim.x) s = fma(sm.S[x], sm.T[x], s);
  s = block_sum(s, sm.red);
  double tr = 0.0;
  for (int i = 0; i < k; ++i) tr += sm.S[i * k + i];
  double sigma = 1.0 - tr - eta;
  double c = s + omega * sigma;
  if (has_eta) c += eta * zeta;
  return c;
}

__device__ double trace_k(const double* A, int k) {
  double tr = 0.0;
  for (int i = 0; i < k; ++i) tr += A[i * k + i];
  return tr;
}


// D = A B + C on the FP64 tensor cores (m8n8k4): a = A[lane>>2][lane&3],
// b = B[lane&3][lane>>2], c/d = C[lane>>2][2(lane&3) + {0,1}]
__device__ __forceinline__ void dmma8x8x4(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// 8 x 8 diagonal block J by one warp: lane r (< 8) holds row r of the block
// in registers; per column c the pivot A(c, c) comes by shuffle from lane c,
// the column is scaled by its rsqrt, and every row updates its entries
// t <= r with L(t, c) shuffled from lane t (1.6 K cycles per block against
// 2.3 K for a two-entries-per-lane layout, identical results;
// profiles/mb/diag8_mb.cu).  Writes L and rdiag; lane 0 sets *flag.
__device__ __forceinline__ void chol_diag8(double* __restrict__ Mp, int d, int J, double* __restrict__ rdiag,
                                           int* flag) {
  const int lane = threadIdx.x & 31;
  const int j0 = J * 8, jb = min(8, d - j0);
  const int r = lane & 7;
  double a[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) a[t] = (r < jb && t <= r) ? Mp[pidx(j0 + r, j0 + t)] : 0.0;
  int ok = 1;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (c < jb) {
      const double pv = __shfl_sync(0xffffffffu, a[c], c);
      if (!(pv > 0.0)) ok = 0;
      const double rs = ok ? rsqrt(pv) : 0.0;
      if (lane == 0) rdiag[j0 + c] = rs;
      a[c] = (r == c) ? pv * rs : a[c] * rs;
      // the next pivot's update from the lane's own value first (the serial
      // chain is then shuffle, rsqrt, scale, one FMA); the other entries take
      // L(t, c) shuffled from lane t -- the same operations either way
      if (c + 1 < 8 && r == c + 1) a[c + 1] -= a[c] * a[c];
#pragma unroll
      for (int t = c + 1; t < 8; ++t) {
        const double ltc = __shfl_sync(0xffffffffu, a[c], t);  // L(t, c)
        if (t <= r && !(t == c + 1 && r == c + 1)) a[t] -= a[c] * ltc;
      }
    }
  }
  if (lane < 8 && r < jb) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (t <= r) Mp[pidx(j0 + r, j0 + t)] = a[t];
  }
  if (lane == 0) *flag = ok;
}

// C_IK -= L_IJ L_KJ^T for one 8 x 8 tile pair (I, K tile rows/cols, absolute)
__device__ __forceinline__ void chol_tile_update(double* __restrict__ Mp, int d, int j0, int jb, int I, int K) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int ra = I * 8 + g, rb = K * 8 + g;
  const int oa = ra < d ? pidx(ra, 0) : 0;
  const int ob = rb < d ? pidx(rb, 0) : 0;
  const double a0 = (ra < d && q < jb) ? -Mp[oa + j0 + q] : 0.0;
  const double a1 = (ra < d && q + 4 < jb) ? -Mp[oa + j0 + 4 + q] : 0.0;
  const double b0 = (rb < d && q < jb) ? Mp[ob + j0 + q] : 0.0;
  const double b1 = (rb < d && q + 4 < jb) ? Mp[ob + j0 + 4 + q] : 0.0;
  const int cc = K * 8 + 2 * q;
  const bool v0 = ra < d && cc <= ra, v1 = ra < d && cc + 1 <= ra;
  double c0 = v0 ? Mp[oa + cc] : 0.0, c1 = v1 ? Mp[oa + cc + 1] : 0.0;
  double d0, d1;
  dmma8x8x4(d0, d1, a0, b0, c0, c1);
  dmma8x8x4(d0, d1, a1, b1, d0, d1);
  if (v0) Mp[oa + cc] = d0;
  if (v1) Mp[oa + cc + 1] = d1;
}

// Blocked right-looking Cholesky of the packed lower matrix M (d x d) by
// 8-column panels with look-ahead: per panel J, (a) the rows below block J
// by forward substitution, a thread per row; (b) the trailing update
// C_IK -= L_IJ L_KJ^T per 8 x 8 tile pair, two DMMA m8n8k4 per tile, while
// warp 0 first updates the next diagonal block and factorises it (potrf
// semantics: fails on a pivot <= 0 or NaN), so the diagonal chain overlaps
// the tensor-core update.  Two barriers per panel.  rdiag[j] = 1 / L_jj.
// Returns 0 on failure (uniform).
__device__ int chol_tiled(double* __restrict__ Mp, int d, double* __restrict__ rdiag, int* flag) {
  const int tid = threadIdx.x, nth = blockDim.x, warp = tid >> 5, nwp = nth >> 5;
  const int T = (d + 7) >> 3;
  if (warp == 0) chol_diag8(Mp, d, 0, rdiag, flag);
  __syncthreads();
  if (!*flag) return 0;
  for (int J = 0; J < T; ++J) {
    const int j0 = J * 8, jb = min(8, d - j0);
    // (a) panel rows below: x = a L_JJ^{-T}
    // (the row's entries are read first and stored last, so the L_JJ and
    // rdiag loads are free to issue ahead of the dependent chain)
    for (int i = j0 + jb + tid; i < d; i += nth) {
      double* ri = Mp + pidx(i, j0);
      double v[8], x[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = c < jb ? ri[c] : 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < jb) {
          double s = v[c];
#pragma unroll
          for (int t = 0; t < c; ++t) s -= x[t] * Mp[pidx(j0 + c, j0 + t)];
          x[c] = s * rdiag[j0 + c];
        }
      }
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < jb) ri[c] = x[c];
    }
    __syncthreads();
    // (b) trailing tile pairs (I, K), J < K <= I; pair 0 = the next diagonal
    // block goes to warp 0 (update + factorisation), the rest round-robin
    const int R = T - J - 1;
    if (warp == 0) {
      if (R > 0) {
        chol_tile_update(Mp, d, j0, jb, J + 1, J + 1);
        __syncwarp();
        chol_diag8(Mp, d, J + 1, rdiag, flag);
      }
    } else if (R > 1) {
      // the other warps take whole tile rows I >= J + 2 (longest first),
      // the row's L_IJ fragments and offsets loaded once for all its tiles
      const int lane = tid & 31, g = lane >> 2, q = lane & 3;
      const int wk = warp - 1, nw1 = nwp - 1;
      for (int I = T - 1 - wk; I >= J + 2; I -= nw1) {
        const int ra = I * 8 + g;
        const bool va = ra < d;
        const int oa = va ? pidx(ra, 0) : 0;
        const double a0 = (va && q < jb) ? -Mp[oa + j0 + q] : 0.0;
        const double a1 = (va && q + 4 < jb) ? -Mp[oa + j0 + 4 + q] : 0.0;
        for (int K = J + 1; K <= I; ++K) {
          const int rb = K * 8 + g;
          const bool vb = rb < d;
          const int ob = vb ? pidx(rb, 0) : 0;
          const double b0 = (vb && q < jb) ? Mp[ob + j0 + q] : 0.0;
          const double b1 = (vb && q + 4 < jb) ? Mp[ob + j0 + 4 + q] : 0.0;
          const int cc = K * 8 + 2 * q;
          const bool v0 = va && cc <= ra, v1 = va && cc + 1 <= ra;
          const double c0 = v0 ? Mp[oa + cc] : 0.0, c1 = v1 ? Mp[oa + cc + 1] : 0.0;
          double d0, d1;
          dmma8x8x4(d0, d1, a0, b0, c0, c1);
          dmma8x8x4(d0, d1, a1, b1, d0, d1);
          if (v0) Mp[oa + cc] = d0;
          if (v1) Mp[oa + cc + 1] = d1;
        }
      }
    }
    __syncthreads();
    if (R > 0 && !*flag) return 0;
  }
  return 1;
}

// C_IK -= sum over DEPTH columns c0.. of L_I L_K^T for up to NT consecutive
// tiles K0.. of tile row I (independent accumulator chains, the row's
// fragments loaded once); rows/columns >= N masked
template <int DEPTH, int NT>
__device__ __forceinline__ void tiles_update(double* __restrict__ Mp, int N, int c0, int I, int K0, int nt) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int ra = I * 8 + g;
  const bool va = ra < N;
  const int oa = va ? pidx(ra, 0) : 0;
  double af[DEPTH / 4];
#pragma unroll
  for (int s = 0; s < DEPTH / 4; ++s) af[s] = va ? -Mp[oa + c0 + 4 * s + q] : 0.0;
  double c0v[NT], c1v[NT];
  int ob[NT];
#pragma unroll
  for (int u = 0; u < NT; ++u) {
    const int rb = (K0 + u) * 8 + g;
    ob[u] = (u < nt && rb < N) ? pidx(rb, 0) : -1;
    const int cc = (K0 + u) * 8 + 2 * q;
    c0v[u] = (u < nt && va && cc <= ra) ? Mp[oa + cc] : 0.0;
    c1v[u] = (u < nt && va && cc + 1 <= ra) ? Mp[oa + cc + 1] : 0.0;
  }
#pragma unroll
  for (int s = 0; s < DEPTH / 4; ++s) {
#pragma unroll
    for (int u = 0; u < NT; ++u) {
      if (u < nt) {
        const double b = ob[u] >= 0 ? Mp[ob[u] + c0 + 4 * s + q] : 0.0;
        dmma8x8x4(c0v[u], c1v[u], af[s], b, c0v[u], c1v[u]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < NT; ++u) {
    const int cc = (K0 + u) * 8 + 2 * q;
    if (u < nt && va && cc <= ra) Mp[oa + cc] = c0v[u];
    if (u < nt && va && cc + 1 <= ra) Mp[oa + cc + 1] = c1v[u];
  }
}

// The 16 x 16 diagonal block at j0 by warp 0 alone (no block barrier):
// diag8, the 8 rows below it by substitution (a lane per row), their 8 x 8
// tile update on the tensor cores, diag8.  Sets *flag (potrf semantics).
// wait_peer: the tiles of the block's second tile row come from warp 1
// (named barrier 1, 64 threads: warp 1 arrives when they are stored), so
// their 16-deep update runs beside the first 8 x 8 block instead of ahead of
// it on this warp's chain.
__device__ void chol_diag16_warp(double* __restrict__ Mp, int N, int j0, double* __restrict__ rdiag, int* flag,
                                 bool wait_peer = false) {
  const int lane = threadIdx.x & 31;
  const int JB = min(16, N - j0);
  chol_diag8(Mp, N, j0 >> 3, rdiag, flag);
  __syncwarp();
  if (wait_peer) asm volatile("bar.sync 1, 64;" ::: "memory");  // always taken when set: the arrival count stays paired
  if (JB <= 8 || !*(volatile int*)flag) return;
  const int i = j0 + 8 + lane;
  if (lane < JB - 8) {
    double v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = Mp[pidx(i, j0 + c)];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      v[c] *= rdiag[j0 + c];
#pragma unroll
      for (int t = c + 1; t < 8; ++t) v[t] = fma(-v[c], Mp[pidx(j0 + t, j0 + c)], v[t]);
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) Mp[pidx(i, j0 + c)] = v[c];
  }
  __syncwarp();
  tiles_update<8, 1>(Mp, N, j0, (j0 + 8) >> 3, (j0 + 8) >> 3, 1);
  __syncwarp();
  chol_diag8(Mp, N, (j0 + 8) >> 3, rdiag, flag);
  __syncwarp();
}

// Blocked right-looking Cholesky of the packed lower N x N matrix in
// 16-column panels (profiles/mb/chol_mb.cu: d + 1 = 211 150.9k -> 122.1k
// cycles against the 8-column form): warp 0 factors the diagonal block
// without block barriers, all threads solve the panel rows (x L_JJ^T = v, a
// thread per row, right-looking inside the row: the substitution's
// operations in its order), the trailing update is 16 deep (four m8n8k4
// per tile, groups of four tiles dealt round-robin over the warps); warp 0 looks ahead: it updates
// the next diagonal block's tiles first and factors it while the other
// warps run the rest of the trailing update (warp 1 first updates the next
// diagonal block's second tile row and hands it over through a named
// barrier).  Two block barriers per panel.
// rdiag[j] = 1 / L_jj.  Returns 0 on failure (uniform).  Own register
// allocation (noinline).
#ifdef USBS_CHOL_PROF
__device__ unsigned long long* g_cholprof = nullptr;
#define CP_T(v) const long long v = clock64()
#define CP_ADD(slot, dt) do { if (g_cholprof) atomicAdd(&g_cholprof[10 + slot], (unsigned long long)(dt)); } while (0)
#else
#define CP_T(v)
#define CP_ADD(slot, dt)
#endif
template <bool MSM>
__device__ __noinline__ int chol_p16(double* __restrict__ Mg, int N, double* __restrict__ rdiag_g, int* flag) {
  double* __restrict__ Mp = MSM ? as_shared(Mg) : Mg;
  double* __restrict__ rdiag = as_shared(rdiag_g);
  const int tid = threadIdx.x, warp = tid >> 5, nwp = blockDim.x >> 5, nth = blockDim.x;
  const int T = (N + 7) >> 3;
  if (warp == 0) chol_diag16_warp(Mp, N, 0, rdiag, flag);
  __syncthreads();
  if (!*flag) return 0;
  for (int j0 = 0; j0 < N; j0 += 16) {
    const int JB = min(16, N - j0), r0 = j0 + JB;
    if (r0 >= N) break;  // JB == 16 from here on
    CP_T(t0);
    for (int i = r0 + tid; i < N; i += nth) {
      double* ri = Mp + pidx(i, j0);
      double v[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) v[c] = ri[c];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        v[c] *= rdiag[j0 + c];
#pragma unroll
        for (int t = c + 1; t < 16; ++t) v[t] = fma(-v[c], Mp[pidx(j0 + t, j0 + c)], v[t]);
      }
#pragma unroll
      for (int c = 0; c < 16; ++c) ri[c] = v[c];
    }
    CP_T(t1);
    __syncthreads();
    CP_T(t2);
    const int a = r0 >> 3;  // first trailing tile row
    if (warp == 0) {
      tiles_update<16, 1>(Mp, N, j0, a, a, 1);
      __syncwarp();
      chol_diag16_warp(Mp, N, r0, rdiag, flag, a + 1 < T);
    } else {
      if (warp == 1 && a + 1 < T) {
        // the next diagonal block's second tile row, handed to warp 0
        tiles_update<16, 2>(Mp, N, j0, a + 1, a, 2);
        __threadfence_block();
        asm volatile("bar.arrive 1, 64;" ::: "memory");
      }
      // groups of four tiles (I, K0) dealt round-robin over the 15 warps in
      // row order from the longest row: every warp within one group of the
      // mean (whole tile rows per warp left warp 1 with 35 of 325 tiles at
      // the first panel, 1.6x the mean)
      int I = T - 1, first = 0;
      for (int idx = warp - 1;; idx += nwp - 1) {
        while (I >= a + 2 && idx >= first + ((I - a + 4) >> 2)) {
          first += (I - a + 4) >> 2;
          --I;
        }
        if (I < a + 2) break;
        const int K0 = a + 4 * (idx - first);
        tiles_update<16, 4>(Mp, N, j0, I, K0, min(4, I - K0 + 1));
      }
    }
    CP_T(t3);
    __syncthreads();
    CP_T(t4);
#ifdef USBS_CHOL_PROF
    { const int pn = j0 >> 4;
    if (tid == 0) { CP_ADD(6 + pn, t1 - t0); CP_ADD(6 + 16 + pn, t3 - t2); }
    if (tid == 32) { CP_ADD(6 + 32 + pn, t3 - t2); }
    if (tid == 256) { CP_ADD(6 + 48 + pn, t3 - t2); }
    if (tid == 480) { CP_ADD(6 + 64 + pn, t3 - t2); } }
#endif
    if (!*flag) return 0;
  }
  return 1;
}

// ---------------------------------------------------------------- kernel
// P16: the 16-column-panel Cholesky (d + 1 >= 100: C3 / C5, d = 210); the
// 8-column form otherwise (d = 66: 15.3 vs 18.8 us).  Two instantiations so
// each kernel carries one factorisation (code size and register allocation
// of the kernel otherwise cost the gain).
template <bool P16, bool MSM>
__global__ void __launch_bounds__(IPM_THREADS, 1) k_ipm(IpmArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int k = a.k, d = a.d, kk = k * k, tid = threadIdx.x, nth = blockDim.x;
  const int has_eta = a.has_eta;
  IpmSmem sm;
  double* base = (double*)smem_raw;
  constexpr bool m_in_smem = MSM;  // d <= SMEM_D (launch_ipm)
  // P16: M first (16-byte aligned for the bulk copy of packed Q11 into it)
  const int mfirst = (P16 && m_in_smem) ? (((d + 1) * (d + 2) / 2 + 1) & ~1) : 0;
  sm.S = base + mfirst; sm.T = sm.S + kk; sm.H = sm.T + kk; sm.dS = sm.H + kk; sm.dT = sm.dS + kk;
  sm.W1 = sm.dT + kk; sm.W2 = sm.W1 + kk; sm.X1 = sm.W2 + kk; sm.X2 = sm.X1 + kk;
  sm.s = sm.X2 + kk; sm.t = sm.s + d; sm.vI = sm.t + d; sm.h = sm.vI + d; sm.g = sm.h + d;
  sm.f1 = sm.g + d; sm.rhs = sm.f1 + d + 1;  // f1: d + 1 entries (rdiag of the augmented factor)
  sm.ds = sm.rhs + d; sm.dt = sm.ds + d; sm.rd = sm.dt + d;
  sm.tmp = sm.rd + d; sm.cb0 = sm.tmp + d; sm.cb1 = sm.cb0 + d;
  sm.red = sm.cb1 + d; sm.sc = sm.red + 32;
  sm.bar = (uint64_t*)(sm.sc + 64);  // P16 only (the 8-column kernel keeps M right after sc)
  sm.M = (P16 && m_in_smem) ? base : sm.sc + 64;
  double* Mp;
  if constexpr (MSM) Mp = sm.M; else Mp = a.gM;
  unsigned char* ub = (unsigned char*)(sm.sc + (P16 ? 66 : 64) + ((m_in_smem && !P16) ? (d + 1) * (d + 2) / 2 : 0));
  sm.pi = ub; sm.pj = ub + 600;
  sm.flg = (int*)(ub + 1200);
  sm.ctab = (unsigned short*)(ub + 1264);

  // lower-triangle table of the warp Cholesky: column c (1 <= c < k) holds
  // rows c .. k-1 from entry (c - 1) k - c (c - 1) / 2
  for (int c = 1 + tid; c < k; c += nth) {
    const int base = (c - 1) * k - c * (c - 1) / 2;
    for (int r = c; r < k; ++r) sm.ctab[base + r - c] = (unsigned short)((r << 5) | c);
  }
  // svec index tables (column-major lower triangle, symlin.py:57-69)
  if (tid == 0) {
    int p = 0;
    for (int j = 0; j < k; ++j)
      for (int i = j; i < k; ++i) { sm.pi[p] = (unsigned char)i; sm.pj[p] = (unsigned char)j; ++p; }
    if (P16) {
      mbar_init(sm.bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();
  for (int p = tid; p < d; p += nth) {
    sm.vI[p] = sm.pi[p] == sm.pj[p] ? 1.0 : 0.0;
    sm.h[p] = a.lin_s[p];
    sm.g[p] = a.q12 ? a.q12[p] : 0.0;
  }
  const double q22 = a.scal[0], h2 = has_eta ? a.scal[1] : 0.0;
  const double q22e = has_eta ? q22 : 0.0;
  const int pairs = k + (has_eta ? 2 : 1);
  // ---- cold centre (subqp.py:184-197)
  const double cc = 1.0 / (2.0 * pairs);
  double eta, zeta, omega, mu;
  // warm start (subqp.py:355-373): strictly feasible check, blend 0.2 to centre
  int use_warm = 0;
  if (a.warm && (int)a.warm[2 * kk + 5] == k && (int)a.warm[2 * kk + 4] == has_eta && a.warm[2 * kk + 6] != 0.0) {
    for (int x = tid; x < kk; x += nth) { sm.W1[x] = a.warm[x]; sm.W2[x] = a.warm[kk + x]; }
    __syncthreads();
    double we = a.warm[2 * kk], wz = a.warm[2 * kk + 1], wo = a.warm[2 * kk + 2];
    double sig = 1.0 - trace_k(sm.W1, k) - we;
    int ok = (wo > 0.0 && sig > 0.0) && (!has_eta || (we > 0.0 && wz > 0.0));
    __syncthreads();
    if (ok) {
      warp_chol(sm.W1, k, sm.flg, 0, sm.ctab);
      int ok1 = sm.flg[0];
      warp_chol(sm.W2, k, sm.flg, 1, sm.ctab);
      int ok2 = sm.flg[1];
      ok = ok1 && ok2;
    }
    if (ok) {
      const double lam = a.o.warm_blend;
      for (int x = tid; x < kk; x += nth) {
        int r = x / k, c = x % k;
        sm.S[x] = (1 - lam) * a.warm[x] + lam * (r == c ? cc : 0.0);
        sm.T[x] = (1 - lam) * a.warm[kk + x] + lam * (r == c ? 1.0 : 0.0);
      }
      eta = (1 - lam) * we + lam * (has_eta ? cc : 0.0);
      zeta = (1 - lam) * wz + lam * (has_eta ? 1.0 : 0.0);
      omega = (1 - lam) * wo + lam * 1.0;
      use_warm = 1;
    }
  }
  if (!use_warm) {
    for (int x = tid; x < kk; x += nth) {
      int r = x / k, c = x % k;
      sm.S[x] = (r == c) ? cc : 0.0;
      sm.T[x] = (r == c) ? 1.0 : 0.0;
    }
    eta = has_eta ? cc : 0.0;
    zeta = has_eta ? 1.0 : 0.0;
    omega = 1.0;
  }
  __syncthreads();
  mu = blk_compl(sm, k, eta, zeta, omega, has_eta) / (2.0 * pairs);
  // ---- coefficient scale (subqp.py:376-382).  P16: Q11 also packed lower
  // into gQp (bulk-copied into M's slot every Newton step, where it serves
  // the stationarity product and the base of M; 16-byte multiples, so one
  // pad entry, landing on row d's first entry, which the right-hand side
  // overwrites) and checked for exact symmetry (the packed product assumes
  // it; an asymmetric Q11 is read row-wise from global)
  const bool packed = P16 && a.Q11 && m_in_smem && a.gQp;
  const uint32_t qbytes = (uint32_t)(((d * (d + 1) / 2 + 1) & ~1) * sizeof(double));
  int asym = 0;
  double qmax = 0.0;
  if (a.Q11) {
    double v = 0.0;
    if (packed) {
      const int lane = tid & 31, warp = tid >> 5, nwp = nth >> 5;
      int bad = 0;
      for (int p = warp; p < d; p += nwp) {
        const double* qr = a.Q11 + (int64_t)p * d;
        for (int q = lane; q < d; q += 32) {
          const double x = __ldg(qr + q);
          v = fmax(v, fabs(x));
          if (q <= p) {
            a.gQp[pidx(p, q)] = x;
            if (x != __ldg(a.Q11 + (int64_t)q * d + p)) bad = 1;
          }
        }
      }
      fence_proxy_global();
      asym = __syncthreads_or(bad);
    } else {
      for (int x = tid; x < d * d; x += nth) v = fmax(v, fabs(a.Q11[x]));
    }
    v = warp_max(v);
    __syncthreads();
    if ((tid & 31) == 0) sm.red[tid >> 5] = v;
    __syncthreads();
    for (int w = 0; w < nth / 32; ++w) qmax = fmax(qmax, sm.red[w]);
    __syncthreads();
  }
  // the per-step copy of packed Q11 into M's slot (issued when M is dead)
  uint32_t ph = 0;
  bool pending = false;
  auto issue_q = [&]() {
    if (packed && !pending) {
      fence_proxy_smem();  // every thread's generic accesses to M before the async-proxy write
      __syncthreads();
      if (tid == 0) {
        mbar_expect_tx(sm.bar, qbytes);
        bulk_g2s(sm.M, a.gQp, qbytes, sm.bar);
      }
      pending = true;
    }
  };
  auto wait_q = [&]() {
    if (pending) {
      mbar_wait(sm.bar, ph);
      ph ^= 1u;
      pending = false;
    }
  };
  const double hmax = blk_max_abs(sm.h, d, sm.red);
  const double gmax = blk_max_abs(sm.g, d, sm.red);
  const double coeff_scale = 1.0 + fmax(fmax(fmax(hmax, fabs(h2)), qmax), fmax(gmax, fabs(q22e)));

  int exact = 0, failures = 0, it = 0;
  unsigned long long ipm_acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long ipm_last = 0;
  if (a.prof && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ipm_last));
#ifdef USBS_CHOL_PROF
  if (tid == 0) g_cholprof = a.prof;
  __syncthreads();
#endif
  const double SQ2 = 1.4142135623730951;
  for (it = 1; it <= a.o.max_newton; ++it) {
    issue_q();  // M is dead here
    // ---- stationarity (subqp.py:210-219)
    blk_svec(sm.S, k, d, sm, sm.s);
    blk_svec(sm.T, k, d, sm, sm.t);
    __syncthreads();
    if (packed && !asym) {
      wait_q();
      blk_gemv_packed(sm.M, sm.s, d, sm.f1);
    } else {
      blk_gemv_q11(a.Q11, sm.s, d, sm.f1);
    }
    __syncthreads();
    for (int p = tid; p < d; p += nth) {
      double f = sm.f1[p] + sm.h[p] - sm.t[p] + omega * sm.vI[p];
      if (has_eta) f += eta * sm.g[p];
      sm.f1[p] = f;
    }
    __syncthreads();
    double f2 = 0.0;
    if (has_eta) f2 = blk_dot(sm.g, sm.s, d, sm.red) + eta * q22e + h2 - zeta + omega;
    const double fmaxv = blk_max_abs(sm.f1, d, sm.red);
    const double stat_res = fmax(fmaxv, fabs(f2));
    const double achieved = blk_compl(sm, k, eta, zeta, omega, has_eta) / (2.0 * pairs);
    if (mu < a.o.mu_tol && achieved < a.o.mu_tol && stat_res <= a.o.kkt_tol * coeff_scale) {
      exact = 1;
      it -= 1;
      break;
    }
    IPM_MARK(0);
    // ---- newton_direction (subqp.py:222-265)
    int fail = 0;
    // H = S^-1 via Cholesky: S = L L^T, Linv by forward substitution, H = Linv^T Linv
    for (int x = tid; x < kk; x += nth) sm.W1[x] = sm.S[x];
    __syncthreads();
    warp_chol(sm.W1, k, sm.flg, 2, sm.ctab);
    if (!sm.flg[2]) fail = 1;
    if (!fail) {
      // X1 = L^-1 (lower): column c solved by thread c
      for (int r = tid; r < k; r += nth) sm.rd[r] = 1.0 / sm.W1[r * k + r];  // rd is free until rd is formed
      __syncthreads();
      for (int c = tid; c < k; c += nth) {
        for (int r = 0; r < c; ++r) sm.X1[r * k + c] = 0.0;
        for (int r = c; r < k; ++r) {
          double s = (r == c) ? 1.0 : 0.0;
          for (int u = c; u < r; ++u) s -= sm.W1[r * k + u] * sm.X1[u * k + c];
          sm.X1[r * k + c] = s * sm.rd[r];
        }
      }
      __syncthreads();
      for (int x = tid; x < kk; x += nth) {
        int r = x / k, c = x % k;
        double s = 0.0;
        for (int u = max(r, c); u < k; ++u) s = fma(sm.X1[u * k + r], sm.X1[u * k + c], s);
        sm.X2[x] = s;
      }
      __syncthreads();
      for (int x = tid; x < kk; x += nth) {
        int r = x / k, c = x % k;
        sm.H[x] = 0.5 * (sm.X2[r * k + c] + sm.X2[c * k + r]);
      }
      __syncthreads();
      const double tr = trace_k(sm.S, k);
      const double sigma = 1.0 - tr - eta;
      const double rc = mu / omega - sigma;
      const double kappa1 = sigma / omega;
      IPM_MARK(1);
      // rd = mu svec(H) - t
      blk_svec(sm.H, k, d, sm, sm.rd);
      __syncthreads();
      for (int p = tid; p < d; p += nth) sm.rd[p] = mu * sm.rd[p] - sm.t[p];
      double re = 0.0, kappa2 = 0.0, cden = 1.0;
      if (has_eta) {
        re = mu / eta - zeta;
        kappa2 = zeta / eta + q22e;
        cden = kappa1 * kappa2 + 1.0;
      }
      __syncthreads();
      // rhs
      for (int p = tid; p < d; p += nth) {
        double r;
        if (!has_eta) r = -sm.f1[p] + sm.rd[p] - (rc / kappa1) * sm.vI[p];
        else
          r = sm.g[p] * ((rc + kappa1 * (f2 - re)) / cden) + sm.vI[p] * ((f2 - re - kappa2 * rc) / cden) -
              sm.f1[p] + sm.rd[p];
        sm.rhs[p] = r;
        // the low-rank term's per-column factors, divided once per column
        // instead of once per entry of M
        if (!has_eta) {
          sm.cb0[p] = sm.vI[p] / kappa1;
        } else {
          sm.cb0[p] = (kappa1 * sm.g[p] + sm.vI[p]) / cden;
          sm.cb1[p] = (sm.g[p] - kappa2 * sm.vI[p]) / cden;
        }
      }
      __syncthreads();
      IPM_MARK(2);
      // M (packed lower): Q11 + E + low-rank; warp per row p, lanes over q <= p
      // (Q11 already in place when packed)
      wait_q();
      {
        const int lane = tid & 31, wid = tid >> 5, nwp = nth >> 5;
        const double* Hm = sm.H;
        const double* Gm = sm.T;
        // the row's Q11 entries (global, L2) are loaded one iteration ahead
        // so their latency overlaps the E computation
        for (int p = wid; p < d; p += nwp) {
          const int i = sm.pi[p], j = sm.pj[p];
          const double wp = (i == j) ? 1.0 : SQ2;
          const double gp = sm.g[p], vp = sm.vI[p];
          const double* qrow = (a.Q11 && !packed) ? a.Q11 + (int64_t)p * d : nullptr;
          const int base = p * (p + 1) / 2;
          double qn = (qrow && lane <= p) ? __ldg(qrow + lane) : 0.0;
          for (int q = lane; q <= p; q += 32) {
            const double qv = packed ? Mp[base + q] : qn;
            qn = (qrow && q + 32 <= p) ? __ldg(qrow + q + 32) : 0.0;
            const int kq = sm.pi[q], l = sm.pj[q];
            const double wq = (kq == l) ? 1.0 : SQ2;
            double e = Hm[i * k + kq] * Gm[l * k + j] + Hm[i * k + l] * Gm[kq * k + j] +
                       Gm[i * k + kq] * Hm[l * k + j] + Gm[i * k + l] * Hm[kq * k + j];
            e *= (wp * wq) * 0.25;
            double v = qv + e;
            if (!has_eta) v = fma(vp, sm.cb0[q], v);
            else v -= gp * sm.cb0[q] + vp * sm.cb1[q];
            Mp[base + q] = v;
          }
        }
      }
      __syncthreads();
      // the right-hand side as row d of the packed matrix, with a diagonal
      // no pivot can reach: factorising [M rhs; rhs^T big] leaves
      // y = L^-1 rhs in row d of the factor, so the forward solve is folded
      // into the Cholesky's panel substitutions and tile updates
      for (int q = tid; q <= d; q += nth) Mp[pidx(d, q)] = q < d ? sm.rhs[q] : 1e300;
      __syncthreads();
      IPM_MARK(3);
      // Cholesky of M (potrf semantics: fails on a pivot <= 0 or NaN) in
      // 8-column panels with the trailing update on the FP64 tensor cores;
      // rdiag keeps 1 / L_jj for the solves (f1 is dead once rhs is formed)
      double* rdiag = sm.f1;
      int chol_ok;
      if constexpr (P16) chol_ok = chol_p16<MSM>(Mp, d + 1, rdiag, &sm.flg[5]);
      else chol_ok = chol_tiled(Mp, d + 1, rdiag, &sm.flg[5]);
      if (!chol_ok) fail = 1;
      IPM_MARK(4);
      if (!fail) {
        const int lane = tid & 31;
        for (int q = tid; q < d; q += nth) sm.rhs[q] = Mp[pidx(d, q)];
        __syncthreads();
        {
        // generic pointer on purpose in the 16-panel kernel (measured at d = 210:
        // this solve 18.2 us with LD.E, 24.4 us with LDS; d = 66: 6.4 vs 7.3 us the other way)
        double* Mb = Mp;
        if constexpr (P16) asm volatile("" : "+l"(Mb));
        // blocked backward solve: the 32-row diagonal triangles by warp 0
        // with shuffles, the off-diagonal updates by the whole block
        for (int Jend = d; Jend > 0; Jend -= 32) {  // backward: L^T x = y
          const int J = max(0, Jend - 32), JB = Jend - J;
          if (tid < 32) {
            double x = lane < JB ? sm.rhs[J + lane] : 0.0;
            const double rdl = lane < JB ? rdiag[J + lane] : 0.0;
            double Lc[32];
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) Lc[jj] = (lane < jj && jj < JB) ? Mb[pidx(J + jj, J + lane)] : 0.0;
#pragma unroll
            for (int jj = 31; jj >= 0; --jj) {
              if (jj < JB) {
                const double xj = __shfl_sync(0xffffffffu, x * rdl, jj);
                if (lane == jj) x = xj;
                else x = fma(-Lc[jj], xj, x);
              }
            }
            if (lane < JB) sm.ds[J + lane] = x;
          }
          __syncthreads();
          for (int i = tid; i < J; i += nth) {
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int jj = 0;
            for (; jj + 3 < JB; jj += 4) {
              s0 = fma(Mb[pidx(J + jj, i)], sm.ds[J + jj], s0);
              s1 = fma(Mb[pidx(J + jj + 1, i)], sm.ds[J + jj + 1], s1);
              s2 = fma(Mb[pidx(J + jj + 2, i)], sm.ds[J + jj + 2], s2);
              s3 = fma(Mb[pidx(J + jj + 3, i)], sm.ds[J + jj + 3], s3);
            }
            for (; jj < JB; ++jj) s0 = fma(Mb[pidx(J + jj, i)], sm.ds[J + jj], s0);
            sm.rhs[i] -= (s0 + s1) + (s2 + s3);
          }
          __syncthreads();
        }
        }
        issue_q();  // M is dead: the next step's Q11 copy overlaps the rest of this step
        IPM_MARK(5);
        // E ds = svec((H D G + G D H)/2), D = smat(ds), G = T
        blk_smat(sm.ds, k, d, sm, sm.W1);
        __syncthreads();
        blk_mm(sm.W1, sm.T, k, sm.X1);  // D G
        __syncthreads();
        blk_mm(sm.H, sm.X1, k, sm.X2);  // H D G
        __syncthreads();
        for (int x = tid; x < kk; x += nth) {
          int r = x / k, c = x % k;
          sm.W2[x] = 0.5 * (sm.X2[r * k + c] + sm.X2[c * k + r]);
        }
        __syncthreads();
        blk_svec(sm.W2, k, d, sm, sm.tmp);  // E ds
        __syncthreads();
        for (int p = tid; p < d; p += nth) sm.dt[p] = sm.rd[p] - sm.tmp[p];
        const double vds = blk_dot(sm.vI, sm.ds, d, sm.red);
        double deta = 0.0, dzeta = 0.0, domega;
        if (!has_eta) {
          domega = (rc + vds) / kappa1;
        } else {
          const double gds = blk_dot(sm.g, sm.ds, d, sm.red);
          deta = -(rc + kappa1 * (f2 - re) + (kappa1 * gds + vds)) / cden;
          dzeta = re - (zeta / eta) * deta;
          domega = -f2 + re - gds - kappa2 * deta;
        }
        __syncthreads();
        IPM_MARK(6);
        // ---- line_search_feasible (subqp.py:294-343)
        int finite = 1;
        for (int p = tid; p < d; p += nth)
          if (!isfinite(sm.ds[p]) || !isfinite(sm.dt[p])) finite = 0;
        finite = __syncthreads_and(finite);
        if (!(finite && isfinite(deta) && isfinite(dzeta) && isfinite(domega))) {
          fail = 1;
        } else {
          double bmin = INFINITY;
          bool any = false;
          if (domega < 0) { bmin = fmin(bmin, -omega / domega); any = true; }
          if (has_eta) {
            if (deta < 0) { bmin = fmin(bmin, -eta / deta); any = true; }
            if (dzeta < 0) { bmin = fmin(bmin, -zeta / dzeta); any = true; }
          }
          const double dsig = -(vds + deta);
          if (dsig < 0) { bmin = fmin(bmin, -sigma / dsig); any = true; }
          double delta = any ? fmin(1.0, a.o.step_frac * bmin) : 1.0;
          blk_smat(sm.ds, k, d, sm, sm.dS);
          blk_smat(sm.dt, k, d, sm, sm.dT);
          __syncthreads();
          bool found = false;
          // the backtracking sequence delta, 0.8 delta, ... tested two steps
          // per round (warps 0-1 the first, 2-3 the second, X1/X2 are free
          // here): the first passing step of the pair is the one the
          // sequential search would stop at
          auto step_ok = [&](double dl, int f0, int f1) {
            int ok = sm.flg[f0] && sm.flg[f1];
            if (ok) {
              if (omega + dl * domega <= 0 || sigma + dl * dsig <= 0) ok = 0;
              if (has_eta && (eta + dl * deta <= 0 || zeta + dl * dzeta <= 0)) ok = 0;
            }
            return ok;
          };
          while (delta >= a.o.min_step) {
            const double d2 = delta * a.o.backtrack;
            const bool two = d2 >= a.o.min_step;
            for (int x = tid; x < kk; x += nth) {
              sm.W1[x] = sm.S[x] + delta * sm.dS[x];
              sm.W2[x] = sm.T[x] + delta * sm.dT[x];
              sm.X1[x] = sm.S[x] + d2 * sm.dS[x];
              sm.X2[x] = sm.T[x] + d2 * sm.dT[x];
            }
            __syncthreads();
            {
              const int w = tid >> 5;
              if (w < 4 && (w < 2 || two)) {
                double* Wm = w == 0 ? sm.W1 : (w == 1 ? sm.W2 : (w == 2 ? sm.X1 : sm.X2));
                const int ok = warp_chol_core(Wm, k, sm.ctab);
                if ((tid & 31) == 0) sm.flg[6 + w] = ok;
              }
            }
            __syncthreads();
            const int ok1 = step_ok(delta, 6, 7);
            const int ok2 = two ? step_ok(d2, 8, 9) : 0;
            __syncthreads();
            if (ok1) { found = true; break; }
            if (ok2) { delta = d2; found = true; break; }
            delta = d2 * a.o.backtrack;
          }
          if (!found) {
            fail = 1;
          } else {
            IPM_MARK(7);
            // ---- step + barrier_update (subqp.py:415-422, 346-350)
            failures = 0;
            for (int x = tid; x < kk; x += nth) {
              sm.S[x] = sm.S[x] + delta * sm.dS[x];
              sm.T[x] = sm.T[x] + delta * sm.dT[x];
            }
            omega += delta * domega;
            if (has_eta) {
              eta += delta * deta;
              zeta += delta * dzeta;
            }
            __syncthreads();
            const double gamma = delta <= 0.2 ? 1.0 : 0.5 - 0.4 * delta * delta;
            const double est = blk_compl(sm, k, eta, zeta, omega, has_eta) / (2.0 * pairs);
            mu = fmin(mu, gamma * est);
            IPM_MARK(8);
            continue;
          }
        }
      }
    }
    // recovery (subqp.py:406-413)
    __syncthreads();
    failures += 1;
    if (failures > a.o.max_step_failures) break;
    mu = fmax(mu * 10.0, 10.0 * a.o.mu_tol);
  }
  wait_q();  // no bulk copy may be outstanding at exit
  if (it > a.o.max_newton) it = a.o.max_newton;
  if (a.prof && tid == 0)
    for (int s = 0; s < 10; ++s) a.prof[s] += ipm_acc[s];
  // ---- objective (subqp.py:200-207) and outputs
  blk_svec(sm.S, k, d, sm, sm.s);
  __syncthreads();
  blk_gemv_q11(a.Q11, sm.s, d, sm.f1);
  __syncthreads();
  const double sQs = blk_dot(sm.s, sm.f1, d, sm.red);
  const double hs = blk_dot(sm.h, sm.s, d, sm.red);
  double val = 0.5 * sQs + hs;
  if (has_eta) {
    const double gs = blk_dot(sm.g, sm.s, d, sm.red);
    val += eta * gs + 0.5 * eta * eta * q22e + eta * h2;
  }
  for (int x = tid; x < kk; x += nth) {
    a.state[x] = sm.S[x];
    a.state[kk + x] = sm.T[x];
  }
  if (tid == 0) {
    a.state[2 * kk] = eta;
    a.state[2 * kk + 1] = zeta;
    a.state[2 * kk + 2] = omega;
    a.state[2 * kk + 3] = mu;
    a.state[2 * kk + 4] = has_eta;
    a.state[2 * kk + 5] = k;
    a.state[2 * kk + 6] = 1.0;
    a.result[0] = val;
    a.result[1] = it;
    a.result[2] = exact;
    a.result[3] = has_eta ? eta : 0.0;
    a.result[4] = failures;
  }
}

size_t ipm_smem_bytes(int k) {
  const int d = k * (k + 1) / 2, kk = k * k;
  size_t doubles = 9 * kk + 13 * d + 1 + 32 + 64 + 2 + (d <= SMEM_D ? ((d + 1) * (d + 2) / 2 + 1) : 0);
  return doubles * sizeof(double) + 1264 + 2 * (k * (k - 1) / 2 + 1) + 64;
}

void launch_ipm(usbs_ctx* ctx, const IpmArgs& a) {
  size_t sm = ipm_smem_bytes(a.k);
  IpmArgs b = a;
  if (a.d + 1 >= 100 && a.d <= SMEM_D) {
    smem_optin(ctx, (const void*)k_ipm<true, true>, 227 * 1024);
    k_ipm<true, true><<<1, IPM_THREADS, sm, ctx->stream>>>(b);
  } else if (a.d + 1 >= 100) {
    smem_optin(ctx, (const void*)k_ipm<true, false>, 227 * 1024);
    k_ipm<true, false><<<1, IPM_THREADS, sm, ctx->stream>>>(b);
  } else {
    smem_optin(ctx, (const void*)k_ipm<false, true>, 227 * 1024);
    k_ipm<false, true><<<1, IPM_THREADS, sm, ctx->stream>>>(b);
  }
  check_launch(ctx);
}

}  // namespace usbs

using namespace usbs;

extern "C" usbs_status usbs_ipm_solve(usbs_ctx* ctx, int k, int has_eta, const double* Q11, const double* q12,
                                      const double* lin_s, const double* scal, const double* warm_state,
                                      double* state_out, double* result, const double* opts) {
  USBS_API_BEGIN
  if (k < 1 || k > KMAX) fail(USBS_ERR_SHAPE, "ipm: 1 <= k <= 32");
  IpmArgs a{};
  a.k = k;
  a.d = k * (k + 1) / 2;
  a.has_eta = has_eta ? 1 : 0;
  a.Q11 = Q11;
  a.q12 = q12;
  a.lin_s = lin_s;
  a.scal = scal;
  a.warm = warm_state;
  a.state = state_out;
  a.result = result;
  a.gM = a.d > SMEM_D ? (double*)ctx->ws.get(WS_IPM, (size_t)(a.d + 1) * (a.d + 2) / 2 * sizeof(double)) : nullptr;
  a.gQp = (Q11 && a.d <= SMEM_D && a.d + 1 >= 100)
              ? (double*)ctx->ws.get(WS_IPM + 2, (size_t)((a.d * (a.d + 1) / 2 + 1) & ~1) * sizeof(double))
              : nullptr;
  a.prof = nullptr;
  if (getenv("USBS_IPM_PROF")) {
    static bool zeroed = false;
    a.prof = (unsigned long long*)ctx->ws.get(WS_IPM + 1, IPM_PROF_SLOTS * sizeof(unsigned long long));
    if (!zeroed) {
      USBS_CUDA(cudaMemsetAsync(a.prof, 0, IPM_PROF_SLOTS * sizeof(unsigned long long), ctx->stream));
      zeroed = true;
    }
  }
  // IpmOptions defaults (subqp.py:150-162) unless given:
  // [mu_tol, kkt_tol, max_newton, step_frac, backtrack, min_step, max_step_failures, warm_blend]
  double o[8] = {1e-11, 1e-6, 100, 0.99, 0.8, 1e-12, 6, 0.2};
  if (opts)
    for (int i = 0; i < 8; ++i) o[i] = opts[i];
  a.o.mu_tol = o[0]; a.o.kkt_tol = o[1]; a.o.max_newton = (int)o[2]; a.o.step_frac = o[3];
  a.o.backtrack = o[4]; a.o.min_step = o[5]; a.o.max_step_failures = (int)o[6]; a.o.warm_blend = o[7];
  launch_ipm(ctx, a);
  USBS_API_END
}

extern "C" int usbs_ipm_state_len(int k) { return state_len(k); }

// Phase timers of k_ipm (ns) accumulated while USBS_IPM_PROF is set.
extern "C" usbs_status usbs_ipm_profile(usbs_ctx* ctx, unsigned long long* out, int reset) {
  USBS_API_BEGIN
  auto* p = (unsigned long long*)ctx->ws.get(WS_IPM + 1, IPM_PROF_SLOTS * sizeof(unsigned long long));
#ifdef USBS_CHOL_PROF
  USBS_CUDA(cudaMemcpyAsync(out, p, IPM_PROF_SLOTS * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
#else
  USBS_CUDA(cudaMemcpyAsync(out, p, 10 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
#endif
  USBS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (reset) USBS_CUDA(cudaMemsetAsync(p, 0, IPM_PROF_SLOTS * sizeof(unsigned long long), ctx->stream));
  USBS_API_END
}
