// Microbenchmark (diagnostic): building blocks of the IPM's Cholesky chain.
//   1. dependent-chain latencies: SHFL, DFMA, rsqrt(double), rsqrt.approx + 2 Newton
//   2. 8 x 8 diagonal block by one warp: v1 (round-1 kernel) vs v4 (own-value
//      pivot update, approx rsqrt + Newton)
//   3. k x k (k = 20) warp Cholesky: shared-memory table form vs registers
//   4. packed d+1 = 211 blocked Cholesky: round-1 row-per-warp trailing
//      update vs balanced 4-tile groups
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chol_mb chol_mb.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#define FULL 0xffffffffu
__device__ __forceinline__ int pidx(int i, int j) { return i * (i + 1) / 2 + j; }

__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  double r = y * y;
  double e = fma(-h, r, 0.5);
  y = fma(y, e, y);
  r = y * y;
  e = fma(-h, r, 0.5);
  y = fma(y, e, y);
  return y;
}

__global__ void k_lat(double* out, long long* cyc) {
  double a = out[0], b = out[1];
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) a = fma(a, b, 1e-9);
  long long t1 = clock64();
  double s = a;
  for (int i = 0; i < 256; ++i) s = __shfl_sync(FULL, s, (threadIdx.x + 1) & 31);
  long long t2 = clock64();
  double r = 1.0 + a * 1e-3;
  for (int i = 0; i < 256; ++i) r = rsqrt(r + 1.0);
  long long t3 = clock64();
  double q = 1.0 + a * 1e-3;
  for (int i = 0; i < 256; ++i) q = rsqrt_nr(q + 1.0);
  long long t4 = clock64();
  double m = a;
  for (int i = 0; i < 256; ++i) m = m * b;
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
  }
  out[2 + threadIdx.x] = a + s + r + q + m;
}

// ---- 8 x 8 diagonal block variants (lanes 0..7 hold rows)
template <int V>
__device__ __forceinline__ void diag8(double* Mp, int j0, double* rdiag, int* flag, int d = 1 << 30) {
  const int lane = threadIdx.x & 31, r = lane & 7;
  const int jb = min(8, d - j0);
  double a[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) a[t] = (t <= r && r < jb) ? Mp[pidx(j0 + r, j0 + t)] : 0.0;
  int ok = 1;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (c >= jb) break;
    const double pv = __shfl_sync(FULL, a[c], c);
    if (!(pv > 0.0)) ok = 0;
    const double rs = V == 1 ? (ok ? rsqrt(pv) : 0.0) : rsqrt_nr(pv);
    if (lane == 0) rdiag[j0 + c] = rs;
    a[c] = (r == c) ? pv * rs : a[c] * rs;
    if (V == 1) {
#pragma unroll
      for (int t = c + 1; t < 8; ++t) {
        const double ltc = __shfl_sync(FULL, a[c], t);
        if (t <= r) a[t] -= a[c] * ltc;
      }
    } else {
      if (c + 1 < 8 && r == c + 1) a[c + 1] = fma(-a[c], a[c], a[c + 1]);
#pragma unroll
      for (int t = c + 1; t < 8; ++t) {
        const double ltc = __shfl_sync(FULL, a[c], t);
        if (t < r || (t == r && t > c + 1)) a[t] = fma(-a[c], ltc, a[t]);
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

template <int V>
__global__ void k_diag8(double* g, long long* cyc, int reps) {
  __shared__ double M[64 * 65 / 2 + 8];
  __shared__ double rd[64];
  __shared__ int flag;
  for (int i = threadIdx.x; i < 64 * 65 / 2; i += blockDim.x) M[i] = g[i];
  __syncwarp();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    for (int J = 0; J < 8; ++J) diag8<V>(M, J * 8, rd, &flag);
    __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / (reps * 8);
  __syncwarp();
  for (int i = threadIdx.x; i < 64 * 65 / 2; i += blockDim.x) g[i] = M[i];
}

// ---- k x k warp Cholesky (row-major smem W, k <= 32)
__device__ int wchol_smem(double* W, int k, const unsigned short* ctab) {
  const int lane = threadIdx.x & 31;
  const int ntab = k * (k - 1) / 2;
  int ok = 1;
  for (int j = 0; j < k; ++j) {
    const double piv = W[j * k + j];
    if (!(piv > 0.0)) { ok = 0; break; }
    const double r = rsqrt(piv);
    const int row = j + 1 + lane;
    if (row < k) W[row * k + j] *= r;
    if (lane == 0) W[j * k + j] = piv * r;
    __syncwarp();
    for (int e = j * k - (j + 1) * j / 2 + lane; e < ntab; e += 32) {
      const int rc = ctab[e], rr = rc >> 5, cc = rc & 31;
      W[rr * k + cc] -= W[rr * k + j] * W[cc * k + j];
    }
    __syncwarp();
  }
  return ok;
}

// registers, rolled over columns: lane r holds row r shifted so a[0] is the
// current column; NR = 32
template <int NR, bool FAST>
__device__ int wchol_roll(double (&a)[NR], int n) {
  const int lane = threadIdx.x & 31;
  int ok = 1;
#pragma unroll 1
  for (int c = 0; c < n; ++c) {
    const double pv = __shfl_sync(FULL, a[0], c);
    if (!(pv > 0.0)) ok = 0;
    const double rs = FAST ? rsqrt_nr(pv) : rsqrt(pv);
    if (lane == c) a[0] = pv * rs;
    else if (lane > c) a[0] *= rs;
    if (lane == c + 1) a[1] = fma(-a[0], a[0], a[1]);
#pragma unroll
    for (int t = 1; t < NR; ++t) {
      const double l = __shfl_sync(FULL, a[0], (c + t) & 31);
      if (c + t < lane || (c + t == lane && t > 1)) a[t] = fma(-a[0], l, a[t]);
    }
#pragma unroll
    for (int t = 0; t < NR - 1; ++t) a[t] = a[t + 1];
    a[NR - 1] = 0.0;
  }
  return ok;
}

// registers, fully unrolled
template <int NR, bool FAST>
__device__ int wchol_unr(double (&a)[NR], int n) {
  const int lane = threadIdx.x & 31;
  int ok = 1;
#pragma unroll
  for (int c = 0; c < NR; ++c) {
    if (c < n) {
      const double pv = __shfl_sync(FULL, a[c], c);
      if (!(pv > 0.0)) ok = 0;
      const double rs = FAST ? rsqrt_nr(pv) : rsqrt(pv);
      if (lane == c) a[c] = pv * rs;
      else if (lane > c) a[c] *= rs;
      if (c + 1 < NR && lane == c + 1) a[c + 1] = fma(-a[c], a[c], a[c + 1]);
#pragma unroll
      for (int t = c + 1; t < NR; ++t) {
        if (t < n) {
          const double l = __shfl_sync(FULL, a[c], t);
          if (t < lane || (t == lane && t > c + 1)) a[t] = fma(-a[c], l, a[t]);
        }
      }
    }
  }
  return ok;
}

// thread per lower entry, one named barrier per column (nthr threads, id 1)
__device__ int bchol(double* W, double* L, int k, int nthr) {
  const int tid = threadIdx.x;
  int ok = 1;
  const int ne = k * (k + 1) / 2;
  int er[4], et[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int e = tid + u * nthr;
    int r = (int)((sqrtf(8.0f * e + 1.0f) - 1.0f) * 0.5f);
    while (r * (r + 1) / 2 > e) --r;
    while ((r + 1) * (r + 2) / 2 <= e) ++r;
    er[u] = e < ne ? r : -1;
    et[u] = e - r * (r + 1) / 2;
  }
  for (int c = 0; c < k; ++c) {
    const double pv = W[c * k + c];
    if (!(pv > 0.0)) { ok = 0; break; }
    const double rs = rsqrt(pv);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = er[u], t = et[u];
      if (r >= 0 && t >= c) {
        if (t == c) L[r * k + c] = (r == c) ? pv * rs : W[r * k + c] * rs;
        else W[r * k + t] = fma(-(W[r * k + c] * rs), W[t * k + c] * rs, W[r * k + t]);
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(nthr));
  }
  return ok;
}

template <int NT>
__global__ void k_bchol(const double* g, double* out, long long* cyc, int k, int reps) {
  __shared__ double W[32 * 32], L[32 * 32];
  long long best = 1LL << 60;
  int okk = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int i = threadIdx.x; i < k * k; i += NT) W[i] = g[i];
    __syncthreads();
    long long t0 = clock64();
    okk += bchol(W, L, k, NT);
    __syncthreads();
    long long t1 = clock64();
    best = min(best, t1 - t0);
  }
  if (threadIdx.x == 0) { cyc[0] = best; cyc[1] = okk / NT; }
  out[threadIdx.x] = L[threadIdx.x];
}

__device__ __noinline__ int wchol_b8(double* W, int k);
template <int V>
__global__ void k_wchol(const double* g, double* out, long long* cyc, int k, int reps) {
  __shared__ double W[32 * 32];
  __shared__ unsigned short ctab[32 * 31 / 2];
  const int lane = threadIdx.x & 31;
  for (int c = 1; c < k; ++c) {
    const int base = (c - 1) * k - c * (c - 1) / 2;
    if (lane == 0)
      for (int r = c; r < k; ++r) ctab[base + r - c] = (unsigned short)((r << 5) | c);
  }
  __syncwarp();
  long long t0 = 0, tot = 0;
  int okk = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int i = lane; i < k * k; i += 32) W[i] = g[i];
    __syncwarp();
    t0 = clock64();
    if (V == 0) {
      okk += wchol_smem(W, k, ctab);
    } else if (V == 5) {
      okk += wchol_b8(W, k);
    } else {
      double a[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) a[t] = (lane < k && t <= lane) ? W[lane * k + t] : 0.0;
      int ok = V == 1 ? wchol_roll<32, false>(a, k) : V == 2 ? wchol_roll<32, true>(a, k)
             : V == 3 ? wchol_unr<32, false>(a, k) : wchol_unr<32, true>(a, k);
      okk += ok;
      out[lane] = a[0] + a[5];
    }
    __syncwarp();
    tot = rep == 0 ? clock64() - t0 : min(tot, clock64() - t0);
  }
  if (lane == 0) { cyc[0] = tot; cyc[1] = okk; }
  if (V == 0 || V == 5) for (int i = lane; i < k * k; i += 32) out[i] = W[i];
}

// ---- packed blocked Cholesky (8-column panels), variants of the trailing update
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}


// blocked warp Cholesky of a row-major k x k (k <= 32): 8 x 8 diagonal
// blocks in registers (lanes 0-7 = rows), 8-column substitutions a lane per
// row below, trailing 8 x 8 tiles on the FP64 tensor cores
__device__ __noinline__ int wchol_b8(double* W, int k) {
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
        const double pv = __shfl_sync(FULL, a[c], c);
        if (!(pv > 0.0)) ok = 0;
        const double rs = rsqrt(pv);
        rsv[c] = rs;
        a[c] = (r == c) ? pv * rs : a[c] * rs;
#pragma unroll
        for (int t = c + 1; t < 8; ++t) {
          const double ltc = __shfl_sync(FULL, a[c], t);
          if (t <= r) a[t] -= a[c] * ltc;
        }
      }
    }
    if (lane < 8 && r < jb) {
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if (t <= r) W[(j0 + r) * k + j0 + t] = a[t];
    }
    if (!ok) return 0;
    __syncwarp();
    const int r0 = j0 + jb;
    if (r0 >= k) break;
    // rows below: x L_JJ^T = v, a lane per row
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
    // trailing tiles (I, K), r0/8 <= K <= I
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
        dmma(c0, c1, a0, b0, c0, c1);
        dmma(c0, c1, a1, b1, c0, c1);
        if (v0) W[ra * k + cc] = c0;
        if (v1) W[ra * k + cc + 1] = c1;
      }
    }
    __syncwarp();
  }
  return ok;
}

__device__ __forceinline__ void tile_update(double* Mp, int d, int j0, int jb, int I, int K) {
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
  dmma(d0, d1, a0, b0, c0, c1);
  dmma(d0, d1, a1, b1, d0, d1);
  if (v0) Mp[oa + cc] = d0;
  if (v1) Mp[oa + cc + 1] = d1;
}

template <int V>  // V 0: round-1 trailing (rows per warp); 1: balanced groups of 4 tiles
__device__ int chol_tiled(double* Mp, int d, double* rdiag, int* flag) {
  const int tid = threadIdx.x, nth = blockDim.x, warp = tid >> 5, nwp = nth >> 5, lane = tid & 31;
  const int T = (d + 7) >> 3;
  if (warp == 0) diag8<V == 0 ? 1 : 4>(Mp, 0, rdiag, flag, d);
  __syncthreads();
  if (!*flag) return 0;
  for (int J = 0; J < T; ++J) {
    const int j0 = J * 8, jb = min(8, d - j0);
    for (int i = j0 + jb + tid; i < d; i += nth) {
      double* ri = Mp + pidx(i, j0);
      double v[8], x[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = c < jb ? ri[c] : 0.0;
      if (V == 0) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (c < jb) {
            double s = v[c];
#pragma unroll
            for (int t = 0; t < c; ++t) s -= x[t] * Mp[pidx(j0 + c, j0 + t)];
            x[c] = s * rdiag[j0 + c];
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (c < jb) {
            x[c] = v[c] * rdiag[j0 + c];
#pragma unroll
            for (int t = c + 1; t < 8; ++t) v[t] = fma(-x[c], Mp[pidx(j0 + t, j0 + c)], v[t]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < jb) ri[c] = x[c];
    }
    __syncthreads();
    const int R = T - J - 1;
    if (warp == 0) {
      if (R > 0) {
        tile_update(Mp, d, j0, jb, J + 1, J + 1);
        __syncwarp();
        diag8<V == 0 ? 1 : 4>(Mp, (J + 1) * 8, rdiag, flag, d);
      }
    } else if (R > 1) {
      const int g = lane >> 2, q = lane & 3, nw1 = nwp - 1;
      if (V == 0) {
        for (int I = T - warp; I >= J + 2; I -= nw1) {
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
            dmma(d0, d1, a0, b0, c0, c1);
            dmma(d0, d1, a1, b1, d0, d1);
            if (v0) Mp[oa + cc] = d0;
            if (v1) Mp[oa + cc + 1] = d1;
          }
        }
      } else {
        // tiles (I, K), J+2 <= I < T, J+1 <= K <= I minus (J+1, J+1): groups of
        // up to 4 consecutive K in one row, dealt round-robin over warps 1..
        const int I0 = J + 1;
        int gbase = 0;
        for (int I = J + 2; I < T; ++I) {
          const int len = I - I0 + 1, ng = (len + 3) >> 2;
          int gi = (warp - 1 - gbase) % nw1;
          if (gi < 0) gi += nw1;
          for (; gi < ng; gi += nw1) {
            const int K0 = I0 + 4 * gi, nt = min(4, I - K0 + 1);
            const int ra = I * 8 + g;
            const bool va = ra < d;
            const int oa = va ? pidx(ra, 0) : 0;
            const double a0 = (va && q < jb) ? -Mp[oa + j0 + q] : 0.0;
            const double a1 = (va && q + 4 < jb) ? -Mp[oa + j0 + 4 + q] : 0.0;
            double c0[4], c1[4], b0[4], b1[4];
            bool v0[4], v1[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int rb = (K0 + u) * 8 + g;
              const bool vb = u < nt && rb < d;
              const int ob = vb ? pidx(rb, 0) : 0;
              b0[u] = (vb && q < jb) ? Mp[ob + j0 + q] : 0.0;
              b1[u] = (vb && q + 4 < jb) ? Mp[ob + j0 + 4 + q] : 0.0;
              const int cc = (K0 + u) * 8 + 2 * q;
              v0[u] = u < nt && va && cc <= ra;
              v1[u] = u < nt && va && cc + 1 <= ra;
              c0[u] = v0[u] ? Mp[oa + cc] : 0.0;
              c1[u] = v1[u] ? Mp[oa + cc + 1] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) dmma(c0[u], c1[u], a0, b0[u], c0[u], c1[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) dmma(c0[u], c1[u], a1, b1[u], c0[u], c1[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int cc = (K0 + u) * 8 + 2 * q;
              if (v0[u]) Mp[oa + cc] = c0[u];
              if (v1[u]) Mp[oa + cc + 1] = c1[u];
            }
          }
          gbase += ng;
        }
      }
    }
    __syncthreads();
    if (R > 0 && !*flag) return 0;
  }
  return 1;
}


// 8-wide TRSM of rows i >= r0 against the factored 8 x 8 block at j0
// (right-looking inside the row: the same operations as the left-looking
// form, in the same order), a thread per row
__device__ __forceinline__ void trsm8(double* Mp, int N, int j0, int r0, const double* rdiag) {
  const int jb = min(8, N - j0);
  for (int i = r0 + threadIdx.x; i < N; i += blockDim.x) {
    double* ri = Mp + pidx(i, j0);
    double v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = c < jb ? ri[c] : 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c < jb) {
        v[c] *= rdiag[j0 + c];
#pragma unroll
        for (int t = c + 1; t < 8; ++t) v[t] = fma(-v[c], Mp[pidx(j0 + t, j0 + c)], v[t]);
      }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c < jb) ri[c] = v[c];
  }
}

// C_IK -= sum over the DEPTH/8 column tiles s of L_Is L_Ks^T for up to NT
// consecutive tiles K0.. of row I (columns c0 .. c0 + DEPTH - 1 of L)
template <int DEPTH, int NT>
__device__ __forceinline__ void tiles_update(double* Mp, int N, int c0, int I, int K0, int nt) {
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
        dmma(c0v[u], c1v[u], af[s], b, c0v[u], c1v[u]);
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

// Recursive 32/8 blocked Cholesky: 32-column panels factored 8 columns at a
// time (diag8 + trsm8 + 8-deep updates inside the panel only), then ONE
// 32-deep trailing update of the rest (4x fewer passes over the trailing
// tiles than 8-column panels).  Warp 0 runs the diagonal chain ahead.
__device__ long long g_ph[8];
#define PH(i) do { if (tid == 0 || tid == 32) { long long _n = clock64(); atomicAdd((unsigned long long*)&g_ph[(i) + (tid == 32 ? 4 : 0)], (unsigned long long)(_n - _t)); _t = _n; } } while (0)
__device__ int chol_r32(double* Mp, int N, double* rdiag, int* flag) {
  const int tid = threadIdx.x, warp = tid >> 5, nwp = blockDim.x >> 5;
  const int T = (N + 7) >> 3;
  long long _t = clock64();
  if (warp == 0) diag8<4>(Mp, 0, rdiag, flag, N);
  __syncthreads();
  if (!*flag) return 0;
  for (int P0 = 0; P0 < T; P0 += 4) {
    const int P1 = min(T, P0 + 4);
    for (int J = P0; J < P1; ++J) {
      trsm8(Mp, N, J * 8, J * 8 + 8, rdiag);
      PH(0);
      __syncthreads();
      PH(1);
      if (J + 1 < P1) {
        // in-panel update by column tile J: tiles (I, K), J+1 <= K < P1, K <= I
        if (warp == 0) {
          tiles_update<8, 1>(Mp, N, J * 8, J + 1, J + 1, 1);
          __syncwarp();
          diag8<4>(Mp, (J + 1) * 8, rdiag, flag, N);
        } else {
          // workers: warps not sharing warp 0's SMSP (warp % 4 != 0)
          if (warp & 3) {
            const int wk = warp - 1 - (warp >> 2), nwk = nwp - (nwp >> 2);
            for (int I = J + 1 + wk; I < T; I += nwk) {
              const int K0 = (I == J + 1) ? J + 2 : J + 1;  // (J+1, J+1) is warp 0's
              const int nt = min(P1 - 1, I) - K0 + 1;
              if (nt > 0) tiles_update<8, 3>(Mp, N, J * 8, I, K0, nt);
            }
          }
        }
        PH(2);
        __syncthreads();
        PH(1);
        if (!*flag) return 0;
      }
    }
    if (P1 >= T) break;
    // trailing update by the whole panel (depth 8 (P1 - P0) = 32): tiles
    // (I, K), P1 <= K <= I < T, in groups of up to 4 consecutive K per row;
    // warp 0 takes (P1, P1) and factors it
    if (warp == 0) {
      tiles_update<32, 1>(Mp, N, P0 * 8, P1, P1, 1);
      __syncwarp();
      diag8<4>(Mp, P1 * 8, rdiag, flag, N);
    } else if (warp & 3) {
      const int wk = warp - 1 - (warp >> 2), nwk = nwp - (nwp >> 2);
      int gbase = 0;
      for (int I = P1; I < T; ++I) {
        const int Ks = (I == P1) ? P1 + 1 : P1;
        const int len = I - Ks + 1, ng = (len + 3) >> 2;
        if (len <= 0) continue;
        int gi = (wk - gbase) % nwk;
        if (gi < 0) gi += nwk;
        for (; gi < ng; gi += nwk) {
          const int K0 = Ks + 4 * gi;
          tiles_update<32, 4>(Mp, N, P0 * 8, I, K0, min(4, I - K0 + 1));
        }
        gbase += ng;
      }
    }
    PH(3);
    __syncthreads();
    PH(1);
    if (!*flag) return 0;
  }
  return 1;
}


// 16-column panels: warp 0 factors the 16 x 16 diagonal block without block
// barriers (diag8, an 8-row substitution, one DMMA tile update, diag8), all
// threads solve the panel rows (16-column right-looking row solves), the
// trailing update is 16 deep; warp 0 looks ahead (updates and factors the
// next diagonal block while the other warps run the trailing update)
__device__ void diag16_warp(double* Mp, int N, int j0, double* rdiag, int* flag) {
  const int lane = threadIdx.x & 31;
  const int JB = min(16, N - j0);
  diag8<4>(Mp, j0, rdiag, flag, N);
  __syncwarp();
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
  diag8<4>(Mp, j0 + 8, rdiag, flag, N);
  __syncwarp();
}

__device__ int chol_p16(double* Mp, int N, double* rdiag, int* flag) {
  const int tid = threadIdx.x, warp = tid >> 5, nwp = blockDim.x >> 5, nth = blockDim.x;
  const int T = (N + 7) >> 3;
  if (warp == 0) diag16_warp(Mp, N, 0, rdiag, flag);
  __syncthreads();
  if (!*flag) return 0;
  for (int j0 = 0; j0 < N; j0 += 16) {
    const int JB = min(16, N - j0), r0 = j0 + JB;
    if (r0 >= N) break;
    // panel rows below: x L_JJ^T = v, 16 columns, a thread per row
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
    __syncthreads();
    const int a = r0 >> 3;  // first trailing tile row
    if (warp == 0) {
      // rows a, a+1 of the trailing update (the next diagonal block), then its factorisation
      tiles_update<16, 1>(Mp, N, j0, a, a, 1);
      if (a + 1 < T) tiles_update<16, 2>(Mp, N, j0, a + 1, a, 2);
      __syncwarp();
      diag16_warp(Mp, N, r0, rdiag, flag);
    } else {
      // rows a+2 .. T-1 (all their tiles K = a .. I), longest first, in
      // groups of four tiles
      for (int I = T - warp; I >= a + 2; I -= nwp - 1)
        for (int K0 = a; K0 <= I; K0 += 4) tiles_update<16, 4>(Mp, N, j0, I, K0, min(4, I - K0 + 1));
    }
    __syncthreads();
    if (!*flag) return 0;
  }
  return 1;
}


// generic W-column panels (W = 8 nb): warp 0 factors the W x W diagonal
// block as nb diag8 steps with in-warp substitutions and DMMA tile updates
template <int W>
__device__ void diagW_warp(double* Mp, int N, int j0, double* rdiag, int* flag) {
  const int lane = threadIdx.x & 31;
  const int JB = min(W, N - j0);
  for (int s = 0; s * 8 < JB; ++s) {
    const int c0 = j0 + 8 * s;
    diag8<4>(Mp, c0, rdiag, flag, N);
    __syncwarp();
    if (!*(volatile int*)flag) return;
    const int rb = c0 + 8, re = j0 + JB;  // rows of the block below sub-block s
    if (rb >= re) break;
    for (int i = rb + lane; i < re; i += 32) {
      double v[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = Mp[pidx(i, c0 + c)];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        v[c] *= rdiag[c0 + c];
#pragma unroll
        for (int t = c + 1; t < 8; ++t) v[t] = fma(-v[c], Mp[pidx(c0 + t, c0 + c)], v[t]);
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) Mp[pidx(i, c0 + c)] = v[c];
    }
    __syncwarp();
    const int a = rb >> 3, e = (re + 7) >> 3;
    for (int I = a; I < e; ++I) tiles_update<8, 4>(Mp, re, c0, I, a, I - a + 1);
    __syncwarp();
  }
}

template <int W>
__device__ int chol_pw(double* Mp, int N, double* rdiag, int* flag) {
  const int tid = threadIdx.x, warp = tid >> 5, nwp = blockDim.x >> 5, nth = blockDim.x;
  const int T = (N + 7) >> 3;
  if (warp == 0) diagW_warp<W>(Mp, N, 0, rdiag, flag);
  __syncthreads();
  if (!*flag) return 0;
  for (int j0 = 0; j0 < N; j0 += W) {
    const int JB = min(W, N - j0), r0 = j0 + JB;
    if (r0 >= N) break;
    for (int i = r0 + tid; i < N; i += nth) {
      double* ri = Mp + pidx(i, j0);
      double v[W];
#pragma unroll
      for (int c = 0; c < W; ++c) v[c] = ri[c];
#pragma unroll
      for (int c = 0; c < W; ++c) {
        v[c] *= rdiag[j0 + c];
#pragma unroll
        for (int t = c + 1; t < W; ++t) v[t] = fma(-v[c], Mp[pidx(j0 + t, j0 + c)], v[t]);
      }
#pragma unroll
      for (int c = 0; c < W; ++c) ri[c] = v[c];
    }
    __syncthreads();
    const int a = r0 >> 3, nb = W / 8;
    const int ad = min(T, a + nb);  // tile rows of the next diagonal block
    if (warp == 0) {
      for (int I = a; I < ad; ++I) tiles_update<W, 4>(Mp, N, j0, I, a, I - a + 1);
      __syncwarp();
      diagW_warp<W>(Mp, N, r0, rdiag, flag);
    } else {
      for (int I = T - warp; I >= ad; I -= nwp - 1)
        for (int K0 = a; K0 <= I; K0 += 4) tiles_update<W, 4>(Mp, N, j0, I, K0, min(4, I - K0 + 1));
    }
    __syncthreads();
    if (!*flag) return 0;
  }
  return 1;
}

template <int V>
__global__ void __launch_bounds__(512, 1) k_chol(const double* g, double* out, long long* cyc, int d, int reps) {
  extern __shared__ double M[];
  __shared__ double rd[256];
  __shared__ int flag;
  const int np = d * (d + 1) / 2;
  long long tot = 1LL << 60;
  for (int rep = 0; rep < reps; ++rep) {
    for (int i = threadIdx.x; i < np; i += blockDim.x) M[i] = g[i];
    __syncthreads();
    long long t0 = clock64();
    if (V == 2) chol_r32(M, d, rd, &flag);
    else if (V == 3) chol_p16(M, d, rd, &flag);
    else if (V == 4) chol_pw<16>(M, d, rd, &flag);
    else if (V == 5) chol_pw<24>(M, d, rd, &flag);
    else if (V == 6) chol_pw<32>(M, d, rd, &flag);
    else chol_tiled<V>(M, d, rd, &flag);
    __syncthreads();
    tot = min(tot, clock64() - t0);
  }
  for (int i = threadIdx.x; i < np; i += blockDim.x) out[i] = M[i];
  if (threadIdx.x == 0) cyc[0] = tot;
}

static void spd(int n, std::vector<double>& A, unsigned seed) {
  srand(seed);
  std::vector<double> B(n * (n + 5));
  for (auto& x : B) x = rand() / (double)RAND_MAX - 0.5;
  A.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0;
      for (int t = 0; t < n + 5; ++t) s += B[i * (n + 5) + t] * B[j * (n + 5) + t];
      A[i * n + j] = s / (n + 5) + (i == j ? 1e-3 : 0.0);
    }
}

static double chol_err(int n, const std::vector<double>& A, const std::vector<double>& Lp) {
  double e = 0, nrm = 0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = 0;
      for (int t = 0; t <= j; ++t) s += Lp[i * (i + 1) / 2 + t] * Lp[j * (j + 1) / 2 + t];
      e = fmax(e, fabs(s - A[i * n + j]));
      nrm = fmax(nrm, fabs(A[i * n + j]));
    }
  return e / nrm;
}

int main() {
  double *dg, *dout;
  long long* dc;
  cudaMalloc(&dg, 8 * 40000);
  cudaMalloc(&dout, 8 * 40000);
  cudaMalloc(&dc, 64);
  long long c[8];
  {
    double h[2] = {0.999, 1.0001};
    cudaMemcpy(dout, h, 16, cudaMemcpyHostToDevice);
    k_lat<<<1, 32>>>(dout, dc);
    cudaMemcpy(c, dc, 40, cudaMemcpyDeviceToHost);
    printf("latency (cycles/op): DFMA %.1f SHFL %.1f rsqrt(double) %.1f rsqrt.approx+2NR %.1f DMUL %.1f\n",
           c[0] / 256.0, c[1] / 256.0, c[2] / 256.0 - 4, c[3] / 256.0 - 4, c[4] / 256.0);
  }
  {
    std::vector<double> A;
    spd(64, A, 1);
    std::vector<double> P(64 * 65 / 2);
    for (int i = 0; i < 64; ++i)
      for (int j = 0; j <= i; ++j) P[i * (i + 1) / 2 + j] = A[i * 64 + j];
    // diag8 only factors the 8 diagonal blocks independently; cycles per block
    for (int v : {1, 4}) {
      cudaMemcpy(dg, P.data(), 8 * P.size(), cudaMemcpyHostToDevice);
      if (v == 1) k_diag8<1><<<1, 32>>>(dg, dc, 1);
      else k_diag8<4><<<1, 32>>>(dg, dc, 1);
      cudaMemcpy(dg, P.data(), 8 * P.size(), cudaMemcpyHostToDevice);
      if (v == 1) k_diag8<1><<<1, 32>>>(dg, dc, 1);
      else k_diag8<4><<<1, 32>>>(dg, dc, 1);
      cudaMemcpy(c, dc, 8, cudaMemcpyDeviceToHost);
      printf("diag8 v%d: %lld cycles per 8x8 block\n", v, c[0]);
    }
  }
  for (int k : {11, 20}) {
    std::vector<double> A;
    spd(k, A, 2);
    cudaMemcpy(dg, A.data(), 8 * A.size(), cudaMemcpyHostToDevice);
    const char* nm[6] = {"smem table", "regs rolled", "regs rolled + fast rsqrt", "regs unrolled",
                         "regs unrolled + fast rsqrt", "blocked 8 (diag regs, DMMA)"};
    std::vector<double> L0(k * k), L5(k * k);
    for (int v = 0; v < 6; ++v) {
      for (int w = 0; w < 2; ++w) {
        switch (v) {
          case 0: k_wchol<0><<<1, 32>>>(dg, dout, dc, k, 4); break;
          case 1: k_wchol<1><<<1, 32>>>(dg, dout, dc, k, 4); break;
          case 2: k_wchol<2><<<1, 32>>>(dg, dout, dc, k, 4); break;
          case 3: k_wchol<3><<<1, 32>>>(dg, dout, dc, k, 4); break;
          case 4: k_wchol<4><<<1, 32>>>(dg, dout, dc, k, 4); break;
          default: k_wchol<5><<<1, 32>>>(dg, dout, dc, k, 4); break;
        }
      }
      cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
      if (v == 0) cudaMemcpy(L0.data(), dout, 8 * k * k, cudaMemcpyDeviceToHost);
      if (v == 5) {
        cudaMemcpy(L5.data(), dout, 8 * k * k, cudaMemcpyDeviceToHost);
        double e = 0;
        for (int i = 0; i < k; ++i) for (int j = 0; j <= i; ++j) e = fmax(e, fabs(L0[i * k + j] - L5[i * k + j]));
        printf("  blocked vs table max |dL| = %.3e\n", e);
      }
      printf("wchol k=%d %-28s %6lld cycles (ok %lld)\n", k, nm[v], c[0], c[1]);
    }
    k_bchol<128><<<1, 128>>>(dg, dout, dc, k, 4);
    cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
    printf("wchol k=%d %-28s %6lld cycles (ok %lld)\n", k, "block 128 thr", c[0], c[1]);
    k_bchol<256><<<1, 256>>>(dg, dout, dc, k, 4);
    cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
    printf("wchol k=%d %-28s %6lld cycles (ok %lld)\n", k, "block 256 thr", c[0], c[1]);
  }
  for (int d : {67, 211}) {
    std::vector<double> A;
    spd(d, A, 3);
    std::vector<double> P(d * (d + 1) / 2), L(P.size());
    for (int i = 0; i < d; ++i)
      for (int j = 0; j <= i; ++j) P[i * (i + 1) / 2 + j] = A[i * d + j];
    cudaMemcpy(dg, P.data(), 8 * P.size(), cudaMemcpyHostToDevice);
    int sm = (int)(8 * P.size() + 16);
    cudaFuncSetAttribute(k_chol<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_chol<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_chol<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_chol<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_chol<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_chol<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_chol<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    for (int v = 0; v < 7; ++v) {
      if (v == 0) k_chol<0><<<1, 512, sm>>>(dg, dout, dc, d, 3);
      else if (v == 1) k_chol<1><<<1, 512, sm>>>(dg, dout, dc, d, 3);
      else if (v == 2) k_chol<2><<<1, 512, sm>>>(dg, dout, dc, d, 3);
      else if (v == 3) k_chol<3><<<1, 512, sm>>>(dg, dout, dc, d, 3);
      else if (v == 4) k_chol<4><<<1, 512, sm>>>(dg, dout, dc, d, 3);
      else if (v == 5) k_chol<5><<<1, 512, sm>>>(dg, dout, dc, d, 3);
      else k_chol<6><<<1, 512, sm>>>(dg, dout, dc, d, 3);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(c, dc, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(L.data(), dout, 8 * L.size(), cudaMemcpyDeviceToHost);
      long long ph[8];
      cudaMemcpyFromSymbol(ph, g_ph, sizeof(ph));
      cudaMemset(dc, 0, 8);
      long long z[8] = {0};
      cudaMemcpyToSymbol(g_ph, z, sizeof(z));
      if (v == 2) printf("  phases/3reps: w0 trsm %lld bar %lld inpanel %lld big %lld | w1 trsm %lld bar %lld inpanel %lld big %lld\n",
                         ph[0], ph[1], ph[2], ph[3], ph[4], ph[5], ph[6], ph[7]);
      printf("chol d=%d v%d: %lld cycles (%.1f us at 1.965 GHz), rel err %.2e %s\n", d, v, c[0], c[0] / 1965.0,
             chol_err(d, A, L), cudaGetErrorString(e));
    }
  }
  return 0;
}
