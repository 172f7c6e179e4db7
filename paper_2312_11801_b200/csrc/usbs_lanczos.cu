// K2/K3: thick-restart Lanczos with full (CGS2) reorthogonalisation as ONE
// persistent cooperative kernel per lanczos_top call.
//
// Follows eigsolve.py:83-181 step for step:
//   m = max(inner, k_c+1, 2); tol default 1e-9; q_0 = seeded unit vector
//   per step j: w = Z q_j; c = Q^T w; w -= Q c; c' = Q^T w; w -= Q c';
//               h[:j+1, j] = c + c'; beta = ||w||;
//               beta <= 1e-13 max(1, max|c+c'|) -> fresh direction (host RNG)
//   per cycle:  theta, Y = eigh(H[:m,:m]) (descending); res = |beta_m Y[m-1,:]|
//               converged iff all res[:k_c] <= tol (1 + |theta_0|)
//               thick restart: ell = max(1, min(k_c+3, m-2)),
//               Q[:, :ell] = Q[:, :m] Y[:, :ell], Q[:, ell] = q_m, H = diag(theta[:ell])
//
// Device layout: Q row-blocked (qidx: 32-row tiles, all m+1 columns of a
// tile contiguous, so a warp's 32-row chunk of every column is one streamed
// 8.4 KB region), two n-vectors W0/W1 (double
// buffered so the SpMV of step j+1 can gather w''_j / beta_j from any row
// while this step's w is being written), H (m+1)^2 row-major in global.
// Grid: G blocks (one per SM at most), each owning a contiguous row range
// balanced on nnz; 3 grid barriers per step:
//   A: q_j = w''_{j-1}/beta (own rows), w = Z q_j (row segments, split rows
//      combined in-block), partial Q^T w  --sync--
//   B: c = sum of partials; w' = w - Q c; partial Q^T w'  --sync--
//   C: c' = sum; w'' = w' - Q c'; partial ||w''||^2; H column j  --sync--
// The column reductions use a warp butterfly reduce-scatter (lane t ends with
// the 32-row sum of column t): each Q element is read once per phase.
// Rayleigh-Ritz runs redundantly in every block (identical Jacobi), so no
// extra barrier is needed before the restart.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "usbs_common.cuh"
#include "usbs_jacobi.cuh"
#include "usbs_tridiag.cuh"
#include "usbs_kernels.cuh"
#include "usbs_lanczos.cuh"

namespace cg = cooperative_groups;

namespace usbs {

// phase timers (block 0, thread 0): 0 phase A work, 1 grid barriers,
// 2 phase B work, 3 phase C work, 4 end-of-cycle, 5 Rayleigh-Ritz, 6 restart
#define LZ_MARK(slot)                                   \
  do {                                                  \
    if (a.prof && b == 0 && tid == 0) {                 \
      unsigned long long _t = gtimer();                 \
      lz_acc[slot] += _t - lz_last;                     \
      lz_last = _t;                                     \
    }                                                   \
  } while (0)

// per-block work timers (every block's thread 0): [32 + 4b + s] for the
// SpMV, the Q^T w sums, phase B and phase C; barrier waits excluded
#define BW_START()                                      \
  do {                                                  \
    if (a.prof && tid == 0) bw_last = gtimer();         \
  } while (0)
#define BW_STOP(slot)                                   \
  do {                                                  \
    if (a.prof && tid == 0) bw_acc[slot] += gtimer() - bw_last; \
  } while (0)

template <int LG>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = LG / 2; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, LG);
  return v;
}

// butterfly reduce-scatter over a warp: on exit lane l holds sum_lanes v[l]
__device__ __forceinline__ double butterfly32(double (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      double send = up ? v[i] : v[i + s];
      double keep = up ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

// Per-block column sums sum_{own rows i} Q[i,t] * x_i for t <= j (MAXQ = 32*NH),
// with x_i produced by `rowfn(i, q[], &x)` which may also update the row.
// Result: red[t] (smem) for t < 32*NH, summed over warps in fixed order.
template <int NH, typename RowFn>
__device__ __forceinline__ void column_reduce(const LzArgs& a, int j, int r0, int r1, double* wred,
                                              double* red, RowFn rowfn) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double acc[NH];
#pragma unroll
  for (int h = 0; h < NH; ++h) acc[h] = 0.0;
  for (int base = r0 + warp * 32; base < r1; base += nw * 32) {
    const int i = base + lane;
    const bool live = i < r1;
    double q[NH][32];
#pragma unroll
    for (int h = 0; h < NH; ++h)
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        const int tt = h * 32 + t;
        q[h][t] = (live && tt <= j) ? __ldcg(a.Q + qidx(i, tt, a.m + 1)) : 0.0;
      }
    double x = 0.0;
    if (live) x = rowfn(i, q);
#pragma unroll
    for (int h = 0; h < NH; ++h) {
#pragma unroll
      for (int t = 0; t < 32; ++t) q[h][t] *= x;
      acc[h] += butterfly32(q[h]);
    }
  }
#pragma unroll
  for (int h = 0; h < NH; ++h) wred[warp * (32 * NH) + h * 32 + lane] = acc[h];
  __syncthreads();
  for (int t = threadIdx.x; t < 32 * NH; t += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += wred[w * (32 * NH) + t];
    red[t] = s;
  }
  __syncthreads();
}

// out[t] = sum_{b < G} P[t*G + b] for t < cols: one warp per column, lanes
// stride over blocks (coalesced: the column's partials are contiguous), all
// loads issued before the fixed-order adds
__device__ __forceinline__ void cross_block_sum(const double* P, int G, int cols, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int t = warp; t < cols; t += nw) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int bb = lane + 32 * u;
      v[u] = bb < G ? P[(int64_t)t * G + bb] : 0.0;
    }
    double s = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
    s = warp_sum(s);
    if (lane == 0) out[t] = s;
  }
}

template <int LG, int NH>
__global__ void __launch_bounds__(NH == 1 ? 512 : 256, 1) k_lanczos(LzArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int m = a.m, M1 = m + 1;
  const int tid = threadIdx.x, nth = blockDim.x, nw = nth >> 5;
  const int b = blockIdx.x, G = gridDim.x;
  const int r0 = a.blk_row[b], r1 = a.blk_row[b + 1];
  const int e0 = a.blk_seg[b], e1 = a.blk_seg[b + 1];

  // shared memory carve-up
  double* wred = (double*)smem_raw;              // nw * 32 * NH
  double* cvec = wred + nw * 32 * NH;            // 64
  double* c2vec = cvec + 64;                     // 64
  double* red = c2vec + 64;                      // 64
  double* misc = red + 64;                       // 8
  double* thetaS = misc + 8;                     // 64
  double* Ys = thetaS + 64;                      // m*m
  JacobiSmem js;
  js.A = Ys + m * m;
  js.A2 = js.A + m * m;
  js.V = js.A2 + m * m;
  js.V2 = js.V + m * m;
  js.cself = js.V2 + m * m;
  js.cmate = js.cself + 64;
  js.red = js.cmate + 64;
  js.mate = (int*)(js.red + 32);
  js.flag = js.mate + 64;
  js.ptab = (unsigned char*)(js.flag + 4);
  // SpMV staging (after the Rayleigh-Ritz scratch, see the smem size below)
  double* sp_prod = (double*)(js.ptab + JAC_PTAB_BYTES) + 6 * 64 + 64;  // LZT_NNZ
  int* sp_rp = (int*)(sp_prod + LZT_NNZ);                             // LZT_ROWS + 1
  int* sp_long = sp_rp + LZT_ROWS + 1;                                 // LZT_ROWS
  int* sp_nl = sp_long + LZT_ROWS;                                     // 1

  int cycle = a.cycle0, ell = a.ell0, jstart = a.j0, restarts = a.restarts0, nhist = a.nhist0;
  int matvecs = a.matvecs0, wb = a.wbuf0;
  double beta = a.beta_prev;
  bool from_q = a.first_from_q != 0;
  bool pending = false;  // w''_{m-1} waits in W[wb^1] to become q_m
  int converged = 0;
  unsigned long long lz_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long lz_last = (a.prof && b == 0 && tid == 0) ? gtimer() : 0ull;
  unsigned long long bw_acc[4] = {0ull, 0ull, 0ull, 0ull}, bw_last = 0ull;
  BW_START();

  for (; cycle <= a.max_restarts; ++cycle) {
    for (int j = jstart; j < m; ++j) {
      double* Wprev = wb ? a.W1 : a.W0;
      double* Wcur = wb ? a.W0 : a.W1;
      // ------------------------------------------------------------ phase A
      const double* xsrc;
      double xs;
      if (from_q) {
        xsrc = nullptr;  // gathers read Q[:, j] through qidx
        xs = 1.0;
      } else {
        xsrc = Wprev;
        xs = 1.0 / beta;
        for (int i = r0 + tid; i < r1; i += nth) a.Q[qidx(i, j, M1)] = Wprev[i] * xs;
        if (b == 0 && tid == 0) {
          a.H[j * M1 + (j - 1)] = beta;
          a.H[(j - 1) * M1 + j] = beta;
        }
      }
      // SpMV over the block's segments (CSR-stream): a tile's nonzeros are
      // loaded coalesced, LZT_NNZ / nth per thread in flight, products staged
      // in smem and summed per row (a thread per short row, a warp per longer
      // one); a row above LZT_NNZ nonzeros is summed by the whole block.
      for (int e = e0; e < e1; ++e) {
        const int t0 = a.seg_r0[e], t1 = a.seg_r1[e];
        if (t1 < 0) {  // a piece of a long row: block-wide partial sum
          const int pc = -t1 - 1;
          const int base = a.piece_z0[pc], cnt = a.piece_z1[pc] - base;
          double acc[4] = {0.0, 0.0, 0.0, 0.0};
          for (int z0 = 0; z0 < cnt; z0 += nth * 8) {
            int cc[8];
            double vv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int z = z0 + tid + nth * u;
              cc[u] = z < cnt ? __ldcg(a.col + base + z) : -1;
              vv[u] = z < cnt ? __ldcg(a.val + base + z) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (cc[u] >= 0) acc[u & 3] = fma(vv[u], (from_q ? a.Q[qidx(cc[u], j, M1)] : Wprev[cc[u]]) * xs, acc[u & 3]);
          }
          const double tot = block_sum((acc[0] + acc[1]) + (acc[2] + acc[3]), red);
          if (tid == 0) a.piece_sum[pc] = tot;
          continue;  // block_sum ends with a barrier
        }
        const int base = a.rowptr[t0], cnt = a.rowptr[t1] - base;
        constexpr int PER = LZT_NNZ / (NH == 1 ? 512 : 256);
        int cc[PER];
        double vv[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int z = tid + u * nth;
          cc[u] = z < cnt ? __ldcg(a.col + base + z) : 0;
          vv[u] = z < cnt ? __ldcg(a.val + base + z) : 0.0;
        }
        for (int i = tid; i <= t1 - t0; i += nth) sp_rp[i] = a.rowptr[t0 + i] - base;
        if (tid == 0) sp_nl[0] = 0;
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int z = tid + u * nth;
          if (z < cnt) sp_prod[z] = vv[u] * ((from_q ? a.Q[qidx(cc[u], j, M1)] : Wprev[cc[u]]) * xs);
        }
        __syncthreads();
        for (int il = tid; il < t1 - t0; il += nth) {
          const int zb = sp_rp[il], ze = sp_rp[il + 1];
          if (ze - zb > 32) {
            sp_long[atomicAdd(sp_nl, 1)] = il;  // order irrelevant: one row, one sum
            continue;
          }
          double sacc = 0.0;
          for (int z = zb; z < ze; ++z) sacc += sp_prod[z];
          Wcur[t0 + il] = sacc;
        }
        __syncthreads();
        {
          const int lane = tid & 31, warp = tid >> 5;
          for (int q = warp; q < sp_nl[0]; q += nw) {
            const int il = sp_long[q];
            const int zb = sp_rp[il], ze = sp_rp[il + 1];
            double sacc = 0.0;
            for (int z = zb + lane; z < ze; z += 32) sacc += sp_prod[z];
            sacc = warp_sum(sacc);
            if (lane == 0) Wcur[t0 + il] = sacc;
          }
        }
        __syncthreads();
      }
      BW_STOP(0);
      // the SpMV segments are balanced on nonzeros, the rows below on rows:
      // every W row must be final before the column sums
      grid.sync();
      BW_START();
      // rows cut into pieces: their owner adds the partial sums in order
      for (int x = a.blk_split[b] + tid; x < a.blk_split[b + 1]; x += nth) {
        double tot = 0.0;
        const int f = a.split_first[x], c = a.split_cnt[x];
        for (int u = 0; u < c; ++u) tot += a.piece_sum[f + u];
        Wcur[a.split_row[x]] = tot;
      }
      if (a.blk_split[b + 1] > a.blk_split[b]) __syncthreads();
      ++matvecs;
      {
        int bad = 0;
        column_reduce<NH>(a, j, r0, r1, wred, red, [&](int i, double (&q)[NH][32]) {
          double w = Wcur[i];
          if (!isfinite(w)) bad = 1;
          return w;
        });
        if (__syncthreads_or(bad) && tid == 0) atomicOr(&a.flags[F_NONFINITE], 1);
        for (int t = tid; t <= j; t += nth) a.P1[(int64_t)t * G + b] = red[t];
      }
      BW_STOP(1);
      LZ_MARK(0);
      grid.sync();
      LZ_MARK(1);
      BW_START();
      // ------------------------------------------------------------ phase B
      if (*(volatile int*)&a.flags[F_NONFINITE]) {
        if (b == 0 && tid == 0) {
          a.flags[F_EXIT] = EXIT_NONFINITE;
          a.flags[F_MATVECS] = matvecs;
        }
        return;
      }
      cross_block_sum(a.P1, G, j + 1, cvec);
      for (int t = j + 1 + tid; t < 32 * NH; t += nth) cvec[t] = 0.0;  // the row pass reads all 32 NH
      __syncthreads();
      column_reduce<NH>(a, j, r0, r1, wred, red, [&](int i, double (&q)[NH][32]) {
        // four independent chains (q is zero above j)
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int h = 0; h < NH; ++h)
#pragma unroll
          for (int t = 0; t < 32; t += 4) {
            const int tt = h * 32 + t;
            s0 = fma(q[h][t], cvec[tt], s0);
            s1 = fma(q[h][t + 1], cvec[tt + 1], s1);
            s2 = fma(q[h][t + 2], cvec[tt + 2], s2);
            s3 = fma(q[h][t + 3], cvec[tt + 3], s3);
          }
        const double s = (s0 + s1) + (s2 + s3);
        double w = Wcur[i] - s;
        Wcur[i] = w;
        return w;
      });
      for (int t = tid; t <= j; t += nth) a.P2[(int64_t)t * G + b] = red[t];
      BW_STOP(2);
      LZ_MARK(2);
      grid.sync();
      LZ_MARK(1);
      BW_START();
      // ------------------------------------------------------------ phase C
      cross_block_sum(a.P2, G, j + 1, c2vec);
      for (int t = j + 1 + tid; t < 32 * NH; t += nth) c2vec[t] = 0.0;
      __syncthreads();
      {
        // w'' = w' - Q c' with the row's Q entries loaded unrolled (all in
        // flight at once), lane = row
        const int lane = tid & 31, warp = tid >> 5;
        double ss = 0.0;
        for (int base = r0 + warp * 32; base < r1; base += nw * 32) {
          const int i = base + lane;
          const bool live = i < r1;
          double q[NH][32];
#pragma unroll
          for (int h = 0; h < NH; ++h)
#pragma unroll
            for (int t = 0; t < 32; ++t) {
              const int tt = h * 32 + t;
              q[h][t] = (live && tt <= j) ? __ldcg(a.Q + qidx(i, tt, M1)) : 0.0;
            }
          // four independent chains, no per-column predicates (q and c2vec
          // are zero above j)
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
          for (int h = 0; h < NH; ++h)
#pragma unroll
            for (int t = 0; t < 32; t += 4) {
              const int tt = h * 32 + t;
              s0 = fma(q[h][t], c2vec[tt], s0);
              s1 = fma(q[h][t + 1], c2vec[tt + 1], s1);
              s2 = fma(q[h][t + 2], c2vec[tt + 2], s2);
              s3 = fma(q[h][t + 3], c2vec[tt + 3], s3);
            }
          s0 += s2;
          s1 += s3;
          if (live) {
            const double w = Wcur[i] - (s0 + s1);
            Wcur[i] = w;
            ss = fma(w, w, ss);
          }
        }
        ss = block_sum(ss, red);
        if (tid == 0) a.P3[b] = ss;
      }
      // coefficients, scale (identical in every block)
      for (int t = tid; t <= j; t += nth) cvec[t] += c2vec[t];
      __syncthreads();
      if (b == 0)
        for (int t = tid; t <= j; t += nth) {
          a.H[t * M1 + j] = cvec[t];
          a.H[j * M1 + t] = cvec[t];
        }
      if (tid == 0) {
        double mx = 0.0;
        for (int t = 0; t <= j; ++t) mx = fmax(mx, fabs(cvec[t]));
        misc[0] = fmax(1.0, mx);
      }
      BW_STOP(3);
      LZ_MARK(3);
      grid.sync();
      LZ_MARK(1);
      BW_START();
      if (tid < 32) {
        double s = 0.0;
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = (tid + 32 * u < G) ? a.P3[tid + 32 * u] : 0.0;
        s = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
        s = warp_sum(s);
        if (tid == 0) misc[1] = sqrt(s);
      }
      __syncthreads();
      beta = misc[1];
      const double scale = misc[0];
      wb ^= 1;  // Wcur becomes Wprev for the next step
      from_q = false;
      if (beta <= 1e-13 * scale) {
        if (b == 0 && tid == 0) {
          a.flags[F_EXIT] = EXIT_BREAKDOWN;
          a.flags[F_J] = j;
          a.flags[F_CYCLE] = cycle;
          a.flags[F_ELL] = ell;
          a.flags[F_RESTARTS] = restarts;
          a.flags[F_NHIST] = nhist;
          a.flags[F_MATVECS] = matvecs;
          a.flags[F_PENDING] = wb;
        }
        return;
      }
      pending = (j == m - 1);
    }
    // ---------------------------------------------------------- end of cycle
    if (pending) {
      double* Wprev = wb ? a.W1 : a.W0;
      const double xs = 1.0 / beta;
      for (int i = r0 + tid; i < r1; i += nth) a.Q[qidx(i, m, M1)] = Wprev[i] * xs;
      if (b == 0 && tid == 0) {
        a.H[m * M1 + (m - 1)] = beta;
        a.H[(m - 1) * M1 + m] = beta;
      }
      pending = false;
    }
    grid.sync();
    LZ_MARK(4);
    // Rayleigh-Ritz (every block, identical)
    // only the nw leading Ritz pairs are used: theta/Y[:, :ell] for the
    // restart, theta/Y[:, :k_c] for the output and the residual test
    const int ell_next = max(1, min(a.k_c + 3, m - 2));
    const int nwant = min(m, max(ell_next, a.k_c));
    {
      TriSmem ts;
      ts.A = js.A;
      ts.Q = js.V;
      ts.Z = js.A2;
      ts.v = (double*)(js.ptab + JAC_PTAB_BYTES);
      ts.p = ts.v + 64;
      ts.dd = ts.p + 64;
      ts.ee = ts.dd + 64;
      ts.lam = ts.ee + 64;
      ts.red = ts.lam + 64;
      ts.iw = (int*)(ts.red + 64);
      rr_arrow(m, ell, nwant, a.H, M1, ts, thetaS, Ys, m, (a.prof && b == 0) ? a.prof + 8 : nullptr);
    }
    LZ_MARK(5);
    const double beta_last = a.H[m * M1 + (m - 1)];
    if (tid == 0) {
      bool ok = true;
      const double tol_eff = a.tol * (1.0 + fabs(thetaS[0]));
      for (int u = 0; u < a.k_c; ++u) {
        double r = fabs(beta_last * Ys[(m - 1) * m + u]);
        if (!(r <= tol_eff)) ok = false;
      }
      misc[2] = ok ? 1.0 : 0.0;
    }
    __syncthreads();
    if (b == 0) {
      for (int u = tid; u < nwant; u += nth) {
        a.theta[u] = thetaS[u];
        a.res[u] = fabs(beta_last * Ys[(m - 1) * m + u]);
      }
      if (tid == 0) a.hist[nhist] = thetaS[0];
    }
    ++nhist;
    if (misc[2] != 0.0) { converged = 1; break; }
    if (cycle == a.max_restarts) break;
    // thick restart
    ell = max(1, min(a.k_c + 3, m - 2));
    for (int i = r0 + tid; i < r1; i += nth) {
      double qrow[64];
      for (int t = 0; t < m; ++t) qrow[t] = a.Q[qidx(i, t, M1)];
      for (int u = 0; u < ell; ++u) {
        double s = 0.0;
        for (int t = 0; t < m; ++t) s = fma(qrow[t], Ys[t * m + u], s);
        a.Q[qidx(i, u, M1)] = s;
      }
      a.Q[qidx(i, ell, M1)] = a.Q[qidx(i, m, M1)];
    }
    ++restarts;
    jstart = ell;
    from_q = true;
    grid.sync();
    // H reset after the barrier: every block has read H for its Rayleigh-Ritz;
    // only block 0 writes H, and it does so in program order from here on
    if (b == 0) {
      for (int x = tid; x < M1 * M1; x += nth) a.H[x] = 0.0;
      __syncthreads();
      for (int u = tid; u < ell; u += nth) a.H[u * M1 + u] = thetaS[u];
      __syncthreads();
    }
    LZ_MARK(6);
  }
  // ---------------------------------------------------------------- output
  if (a.prof && b == 0 && tid == 0)
    for (int s = 0; s < 8; ++s) a.prof[s] += lz_acc[s];
  if (a.prof && tid == 0)
    for (int s = 0; s < 4; ++s) a.prof[32 + 4 * b + s] += bw_acc[s];
  for (int i = r0 + tid; i < r1; i += nth) {
    double qrow[64];
    for (int t = 0; t < m; ++t) qrow[t] = a.Q[qidx(i, t, M1)];
    for (int u = 0; u < a.k_c; ++u) {
      double s = 0.0;
      for (int t = 0; t < m; ++t) s = fma(qrow[t], Ys[t * m + u], s);
      a.vecs_out[(int64_t)i * a.ldvecs + u] = s;
    }
  }
  if (b == 0 && tid == 0) {
    a.flags[F_EXIT] = EXIT_DONE;
    a.flags[F_CONV] = converged;
    a.flags[F_RESTARTS] = restarts;
    a.flags[F_NHIST] = nhist;
    a.flags[F_MATVECS] = matvecs;
  }
}

// ------------------------------------------------------------ cluster variant
// Small operators (n <= ~10^4, m <= 32): the same algorithm on ONE thread-block
// cluster of CS CTAs (one per SM).  The Lanczos basis Q and the w vectors of
// a CTA's contiguous R rows live in its shared memory for the whole call;
// the SpMV gathers remote q_j / w'' entries through distributed shared memory
// and the cross-CTA partial sums are read from the owners' smem, so a step
// costs 3 cluster barriers (~0.2 us) instead of 3 grid barriers (~1.6 us)
// and no L2 round trips for Q.  Breakdown exits spill Q to global so the
// host can reseed exactly as in the grid variant.
// leading dimension of the CTA's Q slice: R rounded up to 2 (mod 4), so
// column reads with 128-bit loads (two rows per lane) are conflict-free for
// lane = column (8 lanes cover all banks) and every column starts 16-byte
// aligned; the padding rows stay zero
__host__ __device__ inline int lz_ldq(int R) { return ((R + 1) & 3) == 2 ? R + 1 : R + 3; }

template <int LG>
__global__ void __launch_bounds__(512, 1) k_lanczos_cl(LzArgs a, int R, int hmax) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int m = a.m, M1 = m + 1;
  const int tid = threadIdx.x, nth = blockDim.x, nw = nth >> 5, lane = tid & 31, warp = tid >> 5;
  const int b = (int)cluster.block_rank(), CS = (int)cluster.num_blocks();
  const int r0 = min(a.n, b * R), r1 = min(a.n, r0 + R), nloc = r1 - r0;
  const int LDQ = lz_ldq(R), npair = (nloc + 1) >> 1;

  double* Qs = (double*)smem_raw;   // M1 * LDQ, column-major (ld LDQ), local rows
  double* W0s = Qs + (size_t)M1 * LDQ;  // LDQ
  double* W1s = W0s + LDQ;           // LDQ
  // partial-sum exchange: every CTA pushes its 32 column partials (and its
  // ||w''||^2 share) into slot [rank] of EVERY CTA's buffer before the
  // barrier, so the sums after it are local, fixed-order reads
  double* XA = W1s + LDQ;              // 16 * 32  Q^T w partials
  double* XB = XA + 16 * 32;         // 16 * 32  Q^T w' partials
  double* XC = XB + 16 * 32;         // 16 * 16  ||w''||^2 partials (CTA, warp)
  double* wred = XC + 16 * 16;       // nw * 32  (also each warp's copy of c / c')
  double* hval = wred + nw * 32;     // hmax  halo: remote x entries of this step
  double* misc = hval + hmax;        // 8
  double* thetaS = misc + 8;         // 64
  double* Ys = thetaS + 64;          // m*m
  TriSmem ts;
  ts.A = Ys + m * m;
  ts.Q = ts.A + m * m;
  ts.Z = ts.Q + m * m;
  ts.v = ts.Z + m * m;
  ts.p = ts.v + 64;
  ts.dd = ts.p + 64;
  ts.ee = ts.dd + 64;
  ts.lam = ts.ee + 64;
  ts.red = ts.lam + 64;
  ts.iw = (int*)(ts.red + 64);
  int* rp = ts.iw + 128;  // R + 1 own row pointers
  // halo slot h fetches x[li] from CTA owner: hsrc[h] = owner << 11 | li
  unsigned short* hsrc = reinterpret_cast<unsigned short*>(rp + R + 1);
  int* hcnt = reinterpret_cast<int*>(misc + 3);
  // c / R as a multiply-high: exact for c * R < 2^32 (host checks n * R)
  const unsigned rmagic = (unsigned)((0x100000000ull + (unsigned)R - 1) / (unsigned)R);

  // sum over the own rows of Q[:, lane] * x for lane <= j: warp w takes a
  // contiguous block of row pairs, 128-bit loads (LDQ = 2 mod 4: the 32
  // lanes' column reads are bank-conflict free), four independent FMA chains
  auto colsum = [&](const double* x, int j) -> double {
    const int ppw = (npair + nw - 1) / nw;
    const int p0 = min(npair, warp * ppw), p1 = min(npair, p0 + ppw);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (lane <= j) {
      const double2* qc = reinterpret_cast<const double2*>(Qs + (size_t)lane * LDQ);
      const double2* x2 = reinterpret_cast<const double2*>(x);
      int p = p0;
      for (; p + 1 < p1; p += 2) {
        const double2 q0 = qc[p], q1 = qc[p + 1], y0 = x2[p], y1 = x2[p + 1];
        a0 = fma(q0.x, y0.x, a0);
        a1 = fma(q0.y, y0.y, a1);
        a2 = fma(q1.x, y1.x, a2);
        a3 = fma(q1.y, y1.y, a3);
      }
      if (p < p1) {
        const double2 q0 = qc[p], y0 = x2[p];
        a0 = fma(q0.x, y0.x, a0);
        a1 = fma(q0.y, y0.y, a1);
      }
    }
    return (a0 + a1) + (a2 + a3);
  };
  // (Q c)[rows 2pp, 2pp+1] over columns 0..j (c in smem, broadcast within the
  // warp): columns in chunks of eight whose loads are all issued before the
  // chunk's FMAs (a branch per chunk, not per column); c is zero above j
  // (the column sums of unused columns are zero), so the chunk's tail
  // columns add exact zeros
  auto pair_sub = [&](int pp, const double* cv, int j) -> double2 {
    const double2* q2 = reinterpret_cast<const double2*>(Qs) + pp;
    const int ld2 = LDQ >> 1;
    double s0 = 0.0, s1 = 0.0, u0 = 0.0, u1 = 0.0;
    for (int t0 = 0; t0 <= j; t0 += 8) {
      double2 q[8];
      double c[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        q[u] = q2[(t0 + u) * ld2];
        c[u] = cv[t0 + u];
      }
#pragma unroll
      for (int u = 0; u < 8; u += 2) {
        s0 = fma(q[u].x, c[u], s0);
        s1 = fma(q[u].y, c[u], s1);
        u0 = fma(q[u + 1].x, c[u + 1], u0);
        u1 = fma(q[u + 1].y, c[u + 1], u1);
      }
    }
    return make_double2(s0 + u0, s1 + u1);
  };
  // row il of Q (m <= 32 columns) into registers, and its product with Y[:, u]
  auto load_qrow = [&](int il, double (&q)[32]) {
#pragma unroll
    for (int t = 0; t < 32; ++t) q[t] = t < m ? Qs[(size_t)t * LDQ + il] : 0.0;
  };
  auto qrow_dot = [&](const double (&q)[32], int u) -> double {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int t = 0; t < 32; t += 2) {
      if (t < m) s0 = fma(q[t], Ys[t * m + u], s0);
      if (t + 1 < m) s1 = fma(q[t + 1], Ys[(t + 1) * m + u], s1);
    }
    return s0 + s1;
  };

  // Q for the own rows from global (start vector / restart state / reseed);
  // the padding rows of Q and of both w buffers are zero for good
  for (int x = tid; x < (M1 + 2) * LDQ; x += nth) Qs[x] = 0.0;
  __syncthreads();
  for (int x = tid; x < M1 * nloc; x += nth) {
    const int t = x / nloc, i = x % nloc;
    Qs[(size_t)t * LDQ + i] = a.Q[qidx(r0 + i, t, M1)];
  }
  for (int i = tid; i <= nloc; i += nth) rp[i] = a.rowptr[r0 + i];
  __syncthreads();
  // SpMV operand cache (thread-per-row path): the CTA's nonzeros as value +
  // 16-bit column in the Rayleigh-Ritz scratch (Ys .. ts.Z, 4 m^2 doubles),
  // which is free between Rayleigh-Ritz calls; reloaded after each restart
  const int nz0 = rp[0], nnz_loc = rp[nloc] - nz0;
  const bool use_cache = LG == 1 && a.n <= 65536 && (int64_t)nnz_loc * 10 <= (int64_t)m * m * 32;
  // halo mode (hmax > 0, cached operands): the step's remote x entries are
  // fetched once into hval by all threads, and the cached column of a
  // nonzero is its local index (own row) or nloc + its halo slot, so the
  // SpMV itself reads only local shared memory
  const bool use_halo = use_cache && hmax > 0;
  int nhalo = 0;
  double* cv = Ys;
  unsigned short* cc = (unsigned short*)(Ys + nnz_loc);
  auto load_cache = [&]() {
    if (!use_cache) return;
    if (use_halo) {
      if (tid == 0) *hcnt = 0;
      __syncthreads();
    }
    for (int z = tid; z < nnz_loc; z += nth) {
      const int c = a.col[nz0 + z];
      cv[z] = a.val[nz0 + z];
      if (!use_halo) {
        cc[z] = (unsigned short)c;
      } else if (c >= r0 && c < r1) {
        cc[z] = (unsigned short)(c - r0);
      } else {
        const int h = atomicAdd(hcnt, 1);  // slot order is irrelevant: sums run in nonzero order
        const int owner = (int)__umulhi((unsigned)c, rmagic);
        hsrc[h] = (unsigned short)((owner << 11) | (c - owner * R));
        cc[z] = (unsigned short)(nloc + h);
      }
    }
    if (use_halo) {
      __syncthreads();
      nhalo = *hcnt;
    }
  };
  load_cache();
  cluster.sync();

  int cycle = a.cycle0, ell = a.ell0, jstart = a.j0, restarts = a.restarts0, nhist = a.nhist0;
  int matvecs = a.matvecs0, wb = a.wbuf0;
  double beta = a.beta_prev;
  bool from_q = a.first_from_q != 0;
  bool pending = false;
  int converged = 0;
  unsigned long long lz_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long lz_last = (a.prof && b == 0 && tid == 0) ? gtimer() : 0ull;

  for (; cycle <= a.max_restarts; ++cycle) {
    for (int j = jstart; j < m; ++j) {
      double* Wprev = wb ? W1s : W0s;
      double* Wcur = wb ? W0s : W1s;
      // ------------------------------------------------------------ phase A
      const double* xloc = from_q ? Qs + (size_t)j * LDQ : Wprev;
      const double xs = from_q ? 1.0 : 1.0 / beta;
      if (!from_q) {
        for (int i = tid; i < nloc; i += nth) Qs[(size_t)j * LDQ + i] = Wprev[i] * xs;
        if (b == 0 && tid == 0) {
          a.H[j * M1 + (j - 1)] = beta;
          a.H[(j - 1) * M1 + j] = beta;
        }
      }
      // x[c] lives in CTA c / R (own smem for the local band, DSMEM otherwise)
      auto gather = [&](int c) -> double {
        const int owner = (int)__umulhi((unsigned)c, rmagic), li = c - owner * R;
        const double* src = owner == b ? xloc : cluster.map_shared_rank(xloc, owner);
        return src[li];
      };
      if (use_halo) {
        for (int h = tid; h < nhalo; h += nth) {
          const unsigned sh = hsrc[h];
          hval[h] = cluster.map_shared_rank(xloc, (int)(sh >> 11))[sh & 2047u];
        }
        __syncthreads();
        // a thread per row; every operand in local shared memory (own row
        // or halo slot), the products in nonzero order as in the gather path
        for (int il = tid; il < nloc; il += nth) {
          const int z1 = rp[il + 1] - nz0;
          double acc = 0.0;
          for (int z = rp[il] - nz0; z < z1; ++z) {
            const int c = cc[z];
            const double x = c < nloc ? xloc[c] : hval[c - nloc];
            acc = fma(cv[z], x * xs, acc);
          }
          Wcur[il] = acc;
        }
      } else if constexpr (LG == 1) {
        // short rows: one thread per row, two rows in flight per thread and
        // the row's loads batched by U so the col -> gather chains overlap
        constexpr int U = 8;
        for (int il = tid; il < nloc; il += 2 * nth) {
          const int il2 = il + nth;
          const bool two = il2 < nloc;
          int z1 = rp[il];
          const int e1 = rp[il + 1];
          int z2 = two ? rp[il2] : 0;
          const int e2 = two ? rp[il2 + 1] : 0;
          double acc1 = 0.0, acc2 = 0.0;
          while (z1 < e1 || z2 < e2) {
            int c1[U], c2[U];
            double v1[U], v2[U], x1[U], x2[U];
#pragma unroll
            if (use_cache) {
              for (int u = 0; u < U; ++u) {
                const bool o1 = z1 + u < e1, o2 = z2 + u < e2;
                c1[u] = o1 ? (int)cc[z1 + u - nz0] : -1;
                v1[u] = o1 ? cv[z1 + u - nz0] : 0.0;
                c2[u] = o2 ? (int)cc[z2 + u - nz0] : -1;
                v2[u] = o2 ? cv[z2 + u - nz0] : 0.0;
              }
            } else {
#pragma unroll
              for (int u = 0; u < U; ++u) {
                const bool o1 = z1 + u < e1, o2 = z2 + u < e2;
                c1[u] = o1 ? a.col[z1 + u] : -1;
                v1[u] = o1 ? a.val[z1 + u] : 0.0;
                c2[u] = o2 ? a.col[z2 + u] : -1;
                v2[u] = o2 ? a.val[z2 + u] : 0.0;
              }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              x1[u] = c1[u] >= 0 ? gather(c1[u]) : 0.0;
              x2[u] = c2[u] >= 0 ? gather(c2[u]) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              if (c1[u] >= 0) acc1 = fma(v1[u], x1[u] * xs, acc1);
              if (c2[u] >= 0) acc2 = fma(v2[u], x2[u] * xs, acc2);
            }
            z1 += U;
            z2 += U;
          }
          Wcur[il] = acc1;
          if (two) Wcur[il2] = acc2;
        }
      } else {
        constexpr int GPW = 32 / LG;
        const int gw = lane / LG, t = lane % LG;
        for (int base = warp * GPW; base < nloc; base += nw * GPW) {
          const int il = base + gw;
          const bool ok = il < nloc;
          double acc = 0.0;
          if (ok) {
            const int rb = rp[il], re = rp[il + 1];
            for (int z = rb + t; z < re; z += LG) acc = fma(a.val[z], gather(a.col[z]) * xs, acc);
          }
          acc = group_sum<LG>(acc);
          if (ok && t == 0) Wcur[il] = acc;
        }
      }
      __syncthreads();
      LZ_MARK(7);
      ++matvecs;
      {
        // partial Q^T w over the own rows: lane = column, warp = row block
        const double acc = colsum(Wcur, j);
        wred[warp * 32 + lane] = acc;
        __syncthreads();
        if (warp == 0) {
          double s = 0.0;
          for (int w2 = 0; w2 < nw; ++w2) s += wred[w2 * 32 + lane];
          for (int d = 0; d < CS; ++d) cluster.map_shared_rank(XA, d)[b * 32 + lane] = s;
        }
      }
      LZ_MARK(0);
      cluster.sync();
      LZ_MARK(1);
      // ------------------------------------------------------------ phase B
      // c = sum over CTAs in rank order, formed by every warp (identical
      // everywhere, no block barrier); the warp's copy goes to its wred row
      double cl = 0.0;
      for (int src = 0; src < CS; ++src) cl += XA[src * 32 + lane];
      // a non-finite w entry makes every column sum non-finite (inf * 0 = NaN)
      if (!isfinite(__shfl_sync(0xffffffffu, cl, 0))) {
        if (b == 0 && tid == 0) {
          atomicOr(&a.flags[F_NONFINITE], 1);
          a.flags[F_EXIT] = EXIT_NONFINITE;
          a.flags[F_MATVECS] = matvecs;
        }
        cluster.sync();
        return;
      }
      double* cw = wred + warp * 32;
      cw[lane] = cl;
      __syncwarp();
      {
        // w' = w - Q c (lane = row pair), then partial Q^T w' (lane = column)
        for (int pp = tid; pp < npair; pp += nth) {
          const double2 qc = pair_sub(pp, cw, j);
          double2* w2 = reinterpret_cast<double2*>(Wcur) + pp;
          double2 w = *w2;
          w.x -= qc.x;
          w.y -= qc.y;
          *w2 = w;
        }
        __syncthreads();
        const double acc = colsum(Wcur, j);
        wred[warp * 32 + lane] = acc;
        __syncthreads();
        if (warp == 0) {
          double s = 0.0;
          for (int w2 = 0; w2 < nw; ++w2) s += wred[w2 * 32 + lane];
          for (int d = 0; d < CS; ++d) cluster.map_shared_rank(XB, d)[b * 32 + lane] = s;
        }
      }
      LZ_MARK(2);
      cluster.sync();
      LZ_MARK(1);
      // ------------------------------------------------------------ phase C
      // c' per warp as above; H column j = c + c' and the breakdown scale
      // max(1, max |c + c'|) in registers
      double c2l = 0.0;
      for (int src = 0; src < CS; ++src) c2l += XB[src * 32 + lane];
      const double ctl = cl + c2l;
      const double scale = fmax(1.0, warp_max(lane <= j ? fabs(ctl) : 0.0));
      cw[lane] = c2l;
      __syncwarp();
      {
        double ss = 0.0;
        for (int pp = tid; pp < npair; pp += nth) {
          const double2 qc = pair_sub(pp, cw, j);
          double2* w2 = reinterpret_cast<double2*>(Wcur) + pp;
          double2 w = *w2;
          w.x -= qc.x;
          w.y -= qc.y;
          *w2 = w;
          ss = fma(w.x, w.x, ss);
          ss = fma(w.y, w.y, ss);
        }
        // warp partials straight into slot [rank][warp] of every CTA
        ss = warp_sum(ss);
        if (lane < CS) cluster.map_shared_rank(XC, lane)[b * nw + warp] = ss;
      }
      if (b == 0 && warp == 0 && lane <= j) {
        a.H[lane * M1 + j] = ctl;
        a.H[j * M1 + lane] = ctl;
      }
      LZ_MARK(3);
      cluster.sync();
      LZ_MARK(1);
      {
        const int nx = CS * nw;
        double s = 0.0;
        for (int x = lane; x < nx; x += 32) s += XC[x];
        beta = sqrt(warp_sum(s));
      }
      wb ^= 1;
      from_q = false;
      if (beta <= 1e-13 * scale) {
        // spill Q for the host reseed (the host uses columns 0..j)
        for (int x = tid; x < M1 * nloc; x += nth) {
          const int t = x / nloc, i = x % nloc;
          a.Q[qidx(r0 + i, t, M1)] = Qs[(size_t)t * LDQ + i];
        }
        if (b == 0 && tid == 0) {
          a.flags[F_EXIT] = EXIT_BREAKDOWN;
          a.flags[F_J] = j;
          a.flags[F_CYCLE] = cycle;
          a.flags[F_ELL] = ell;
          a.flags[F_RESTARTS] = restarts;
          a.flags[F_NHIST] = nhist;
          a.flags[F_MATVECS] = matvecs;
          a.flags[F_PENDING] = wb;
        }
        cluster.sync();  // remote readers of this CTA's smem are done
        return;
      }
      pending = (j == m - 1);
      // the next phase A reads the other CTAs' Wcur (now Wprev): the barrier
      // above already orders it; P1s/P2s/P3s are rewritten only after two
      // more barriers
    }
    // ---------------------------------------------------------- end of cycle
    if (pending) {
      double* Wprev = wb ? W1s : W0s;
      const double xs = 1.0 / beta;
      for (int i = tid; i < nloc; i += nth) Qs[(size_t)m * LDQ + i] = Wprev[i] * xs;
      if (b == 0 && tid == 0) {
        a.H[m * M1 + (m - 1)] = beta;
        a.H[(m - 1) * M1 + m] = beta;
      }
      pending = false;
    }
    __threadfence();
    cluster.sync();
    LZ_MARK(4);
    const int ell_next = max(1, min(a.k_c + 3, m - 2));
    const int nwant = min(m, max(ell_next, a.k_c));
    // the eigenvalues split over the cluster's CTAs, each shared by DSMEM
    auto share_lam = [&](double* lam, int r, int nwn) {
      if (r < nwn && tid == 0)
        for (int dd = 0; dd < CS; ++dd) cluster.map_shared_rank(lam, dd)[r] = lam[r];
      cluster.sync();
    };
    rr_arrow(m, ell, nwant, a.H, M1, ts, thetaS, Ys, m, (a.prof && b == 0) ? a.prof + 8 : nullptr, b, CS,
             share_lam);
    LZ_MARK(5);
    const double beta_last = a.H[m * M1 + (m - 1)];
    if (tid == 0) {
      bool ok = true;
      const double tol_eff = a.tol * (1.0 + fabs(thetaS[0]));
      for (int u = 0; u < a.k_c; ++u) {
        const double r = fabs(beta_last * Ys[(m - 1) * m + u]);
        if (!(r <= tol_eff)) ok = false;
      }
      misc[2] = ok ? 1.0 : 0.0;
    }
    __syncthreads();
    if (b == 0) {
      for (int u = tid; u < nwant; u += nth) {
        a.theta[u] = thetaS[u];
        a.res[u] = fabs(beta_last * Ys[(m - 1) * m + u]);
      }
      if (tid == 0) a.hist[nhist] = thetaS[0];
    }
    ++nhist;
    if (misc[2] != 0.0) { converged = 1; break; }
    if (cycle == a.max_restarts) break;
    ell = ell_next;
    if (m == 32) {
      // Q[:, :ell] <- Q Y[:, :ell] on the FP64 tensor cores: a warp per block
      // of 8 rows, m8n8k4 over the 32 columns; the block's Q fragments are in
      // registers before any of its outputs is stored (row i of the product
      // depends on row i of Q only)
      const int g = lane >> 2, q4 = lane & 3, nrb = (nloc + 7) >> 3, ntl = (ell + 7) >> 3;
      for (int rbk = warp; rbk < nrb; rbk += nw) {
        const int i0 = rbk * 8, r = i0 + g;
        double af[8];
#pragma unroll
        for (int kc = 0; kc < 8; ++kc) af[kc] = Qs[(size_t)(kc * 4 + q4) * LDQ + r];
        for (int nt2 = 0; nt2 < ntl; ++nt2) {
          const int n0 = nt2 * 8;
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int kc = 0; kc < 8; ++kc) dmma_m8n8k4(d0, d1, af[kc], Ys[(kc * 4 + q4) * m + n0 + g], d0, d1);
          const int c0 = n0 + 2 * q4;
          if (r < nloc) {
            if (c0 < ell) Qs[(size_t)c0 * LDQ + r] = d0;
            if (c0 + 1 < ell) Qs[(size_t)(c0 + 1) * LDQ + r] = d1;
          }
        }
      }
      __syncthreads();  // column ell is an input of every row block above
      for (int il = tid; il < nloc; il += nth) Qs[(size_t)ell * LDQ + il] = Qs[(size_t)m * LDQ + il];
    } else {
      for (int il = tid; il < nloc; il += nth) {
        double qrow[32];
        load_qrow(il, qrow);
        for (int u = 0; u < ell; ++u) Qs[(size_t)u * LDQ + il] = qrow_dot(qrow, u);
        Qs[(size_t)ell * LDQ + il] = Qs[(size_t)m * LDQ + il];
      }
    }
    __syncthreads();  // Ys (the restart's Y) is read; the operand cache may return
    load_cache();
    ++restarts;
    jstart = ell;
    from_q = true;
    cluster.sync();
    if (b == 0) {
      for (int x = tid; x < M1 * M1; x += nth) a.H[x] = 0.0;
      __syncthreads();
      for (int u = tid; u < ell; u += nth) a.H[u * M1 + u] = thetaS[u];
      __syncthreads();
    }
    LZ_MARK(6);
  }
  if (a.prof && b == 0 && tid == 0)
    for (int s = 0; s < 8; ++s) a.prof[s] += lz_acc[s];
  for (int il = tid; il < nloc; il += nth) {
    double qrow[32];
    load_qrow(il, qrow);
    for (int u = 0; u < a.k_c; ++u) a.vecs_out[(int64_t)(r0 + il) * a.ldvecs + u] = qrow_dot(qrow, u);
  }
  if (b == 0 && tid == 0) {
    a.flags[F_EXIT] = EXIT_DONE;
    a.flags[F_CONV] = converged;
    a.flags[F_RESTARTS] = restarts;
    a.flags[F_NHIST] = nhist;
    a.flags[F_MATVECS] = matvecs;
  }
  cluster.sync();  // keep smem alive until every remote read is done
}

static size_t lz_cl_smem(int m, int R, int nth, int hmax) {
  const int M1 = m + 1, nw = nth / 32, LDQ = lz_ldq(R);
  return (size_t)((size_t)M1 * LDQ + 2 * LDQ + 16 * 32 * 2 + 16 * 16 + nw * 32 + hmax + 8 + 64 + 4 * m * m + 6 * 64) *
             sizeof(double) + (128 + R + 1) * sizeof(int) + ((2 * hmax + 7) & ~7) + 64;
}

// remote nonzeros of each CTA's row range (halo sizes of the cluster kernel)
__global__ void k_halo_count(int n, int R, const int* __restrict__ rowptr, const int* __restrict__ col, int* out) {
  __shared__ int tot;
  if (threadIdx.x == 0) tot = 0;
  __syncthreads();
  const int r0 = min(n, (int)blockIdx.x * R), r1 = min(n, r0 + R);
  int cnt = 0;
  for (int z = rowptr[r0] + threadIdx.x; z < rowptr[r1]; z += blockDim.x) {
    const int c = col[z];
    cnt += (c < r0 || c >= r1);
  }
  atomicAdd(&tot, cnt);
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = tot;
}

// ------------------------------------------------------------ small kernels
__global__ void k_copy(int64_t n, const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i];
}

// c[t] = Q[:, t] . v  for t < used  (one block per column, deterministic)
// reseed helpers on the row-blocked Q: c[t] = Q[:, t] . v (one block per t),
// v -= Q[:, :used] c, Q[:, t] = s * v (v == nullptr: zero)
__global__ void k_qcol_dot(int64_t n, const double* __restrict__ Q, int M1, const double* __restrict__ v,
                           double* __restrict__ c) {
  __shared__ double red[32];
  const int t = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(Q[qidx(i, t, M1)], v[i], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) c[t] = s;
}

__global__ void k_qcol_sub(int64_t n, const double* __restrict__ Q, int M1, int used, const double* __restrict__ c,
                           double* __restrict__ v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int t = 0; t < used; ++t) s = fma(Q[qidx(i, t, M1)], c[t], s);
    v[i] -= s;
  }
}

__global__ void k_qcol_set(int64_t n, const double* __restrict__ v, double sc, double* __restrict__ Q, int t,
                           int M1) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    Q[qidx(i, t, M1)] = v ? v[i] * sc : 0.0;
}

__global__ void k_norm2(int64_t n, const double* __restrict__ v, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(v[i], v[i], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[0] = s;
}

__global__ void k_scale_into(int64_t n, const double* __restrict__ v, double s, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = v[i] * s;
}

// ---- row-sharded Lanczos (dist.py): one step's epilogue on the device, so a
// cycle issues no host reads.  c1, c2: the allreduced CGS2 coefficients
// (j+1 each), nrm2 = ||w''||^2 allreduced.  Writes H[:j+1, j] = c1 + c2
// (symmetric), beta = ||w''|| into H[j+1, j] (0 on breakdown), the local
// rows of q_{j+1} = w'' / beta (0 on breakdown) and flags[0] = first breakdown
// step (eigsolve.py:136-147: beta <= 1e-13 max(1, max|c|)), flags[1] |= a
// non-finite matvec (eigsolve.py:128-129).
__global__ void k_lz_step_finish(int j, int m1, const double* __restrict__ c1, const double* __restrict__ c2,
                                 const double* __restrict__ nrm2, double* __restrict__ H, int* __restrict__ flags,
                                 const double* __restrict__ w, int64_t nl, int64_t ldw, double* __restrict__ q,
                                 int64_t ldq) {
  __shared__ double s_inv;
  if (threadIdx.x == 0) {
    double mx = 0.0;
    bool bad = false;
    for (int t = 0; t <= j; ++t) {
      const double c = c1[t] + c2[t];
      if (!isfinite(c)) bad = true;
      mx = fmax(mx, fabs(c));
    }
    const double beta = sqrt(fmax(nrm2[0], 0.0));
    if (!isfinite(beta)) bad = true;
    const bool brk = !(beta > 1e-13 * fmax(1.0, mx));
    s_inv = brk ? 0.0 : 1.0 / beta;
    if (blockIdx.x == 0) {
      for (int t = 0; t <= j; ++t) {
        const double c = c1[t] + c2[t];
        H[(int64_t)t * m1 + j] = c;
        H[(int64_t)j * m1 + t] = c;
      }
      H[(int64_t)(j + 1) * m1 + j] = brk ? 0.0 : beta;
      H[(int64_t)j * m1 + j + 1] = brk ? 0.0 : beta;
      if (brk && flags[0] < 0) flags[0] = j;
      if (bad) flags[1] = 1;
    }
  }
  __syncthreads();
  const double inv = s_inv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nl; i += (int64_t)gridDim.x * blockDim.x)
    q[i * ldq] = w[i * ldw] * inv;
}

// thick restart of the replicated H: H = diag(theta[:ell]) (eigsolve.py:175-176)
__global__ void k_lz_restart_h(int m1, int ell, const double* __restrict__ theta, double* __restrict__ H) {
  for (int x = threadIdx.x; x < m1 * m1; x += blockDim.x) {
    const int r = x / m1, c = x % m1;
    H[x] = (r == c && r < ell) ? theta[r] : 0.0;
  }
}

// dense fallback (eigsolve.py:66-80): Z = M I densely, symmetrise, eigh
__global__ void k_dense_eigh(int n, const int* __restrict__ rowptr, const int* __restrict__ col,
                             const double* __restrict__ val, int k, double* vals_out, double* vecs_out,
                             int64_t ldv, int* nonfinite) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* base = (double*)smem_raw;
  JacobiSmem js;
  js.A = base;
  js.A2 = js.A + n * n;
  js.V = js.A2 + n * n;
  js.V2 = js.V + n * n;
  double* vals = js.V2 + n * n;
  double* vecs = vals + 64;
  js.cself = vecs + n * n;
  js.cmate = js.cself + 64;
  js.red = js.cmate + 64;
  js.mate = (int*)(js.red + 32);
  js.flag = js.mate + 64;
  js.ptab = (unsigned char*)(js.flag + 4);
  for (int x = threadIdx.x; x < n * n; x += blockDim.x) js.A[x] = 0.0;
  __syncthreads();
  int bad = 0;
  for (int r = threadIdx.x; r < n; r += blockDim.x)
    for (int z = rowptr[r]; z < rowptr[r + 1]; ++z) {
      double v = val[z];
      if (!isfinite(v)) bad = 1;
      js.A[r * n + col[z]] += v;
    }
  bad = __syncthreads_or(bad);
  if (bad) {
    if (threadIdx.x == 0) *nonfinite = 1;
    return;
  }
  jacobi_eigh(n, js, vals, vecs, n);
  for (int u = threadIdx.x; u < k; u += blockDim.x) vals_out[u] = vals[u];
  for (int x = threadIdx.x; x < n * k; x += blockDim.x) {
    int r = x / k, u = x % k;
    vecs_out[(int64_t)r * ldv + u] = vecs[r * n + u];
  }
}

__global__ void k_small_eigh(int k, const double* __restrict__ a, double* vals_out, double* vecs_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* base = (double*)smem_raw;
  JacobiSmem js;
  js.A = base;
  js.A2 = js.A + k * k;
  js.V = js.A2 + k * k;
  js.V2 = js.V + k * k;
  double* vals = js.V2 + k * k;
  double* vecs = vals + 64;
  js.cself = vecs + k * k;
  js.cmate = js.cself + 64;
  js.red = js.cmate + 64;
  js.mate = (int*)(js.red + 32);
  js.flag = js.mate + 64;
  js.ptab = (unsigned char*)(js.flag + 4);
  for (int x = threadIdx.x; x < k * k; x += blockDim.x) js.A[x] = a[x];
  __syncthreads();
  jacobi_eigh(k, js, vals, vecs, k);
  for (int u = threadIdx.x; u < k; u += blockDim.x) vals_out[u] = vals[u];
  for (int x = threadIdx.x; x < k * k; x += blockDim.x) vecs_out[x] = vecs[x];
}

static size_t eigh_smem(int n) {
  return (size_t)(5 * n * n + 64 * 3 + 32) * sizeof(double) + 68 * sizeof(int) + JAC_PTAB_BYTES + 64;
}

void launch_small_eigh(usbs_ctx* ctx, int k, const double* a, double* vals, double* vecs) {
  size_t sm = eigh_smem(k);
  smem_optin(ctx, (const void*)k_small_eigh, 200 * 1024);
  k_small_eigh<<<1, 256, sm, ctx->stream>>>(k, a, vals, vecs);
  check_launch(ctx);
}

template <int LG, int NH>
static void lz_launch(usbs_ctx* ctx, LzArgs& a, int G, size_t smem) {
  auto fn = k_lanczos<LG, NH>;
  smem_optin(ctx, (const void*)fn, 200 * 1024);
  const int threads = NH == 1 ? 512 : 256;
  int per_sm = 0;
  USBS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem));
  if (per_sm * ctx->num_sms < G) fail(USBS_ERR_CUDA, "lanczos grid exceeds co-resident capacity");
  void* args[] = {&a};
  USBS_CUDA(cudaLaunchCooperativeKernel((const void*)fn, dim3(G), dim3(threads), args, smem, ctx->stream));
  check_launch(ctx);
}

// Cluster plan for the small-n variant: CS CTAs in one cluster, R rows each.
struct LzClusterPlan {
  int cs = 0, R = 0, lg = 32, hmax = 0;
  size_t smem = 0;
};

template <int LG>
static int lz_cl_max_clusters(int cs, size_t smem) {
  auto fn = k_lanczos_cl<LG>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nc = 0;
  if (cudaOccupancyMaxActiveClusters(&nc, (void*)fn, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return nc;
}

static int lz_cl_max_clusters_lg(int LG, int cs, size_t smem) {
  switch (LG) {
    case 1: return lz_cl_max_clusters<1>(cs, smem);
    case 4: return lz_cl_max_clusters<4>(cs, smem);
    case 8: return lz_cl_max_clusters<8>(cs, smem);
    case 16: return lz_cl_max_clusters<16>(cs, smem);
    default: return lz_cl_max_clusters<32>(cs, smem);
  }
}

// Picks the largest cluster (16, else 8) whose per-CTA Q slice fits in shared
// memory and that the device can schedule; cs = 0 means "use the grid kernel".
static LzClusterPlan lz_cluster_plan(usbs_ctx* ctx, usbs_problem* p, int m, int LG) {
  const int64_t n = p->n, nnz = p->nnz;
  LzClusterPlan pl;
  // short rows (<= 16 nnz on average): thread per row; else the grid
  // kernel's group size
  if (nnz <= 16 * n) LG = 1;
  const char* e = getenv("USBS_LZ_CLUSTER");
  if (e && e[0] == '0') return pl;
  if (m > 32) return pl;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  for (int cs : {16, 8}) {
    const int64_t R = ((n + cs - 1) / cs) | 1;  // odd: conflict-free column reads
    if (R < 32) continue;  // tiny operators: one warp-row per CTA at least
    if (n * R >= (int64_t(1) << 32)) continue;  // owner = c / R by multiply-high
    size_t sm = lz_cl_smem(m, (int)R, 512, 0);
    if (sm > (size_t)optin) continue;
    if (lz_cl_max_clusters_lg(LG, cs, sm) < 1) continue;
    pl.cs = cs;
    pl.R = (int)R;
    pl.smem = sm;
    pl.lg = LG;
    // halo SpMV when the largest per-CTA remote nonzero count fits
    const char* eh = getenv("USBS_LZ_HALO");
    if (LG == 1 && R < 2048 && n <= 65536 && !(eh && eh[0] == '0')) {
      int* dcnt = (int*)ctx->ws.get(WS_LZ_HALO, 16 * sizeof(int));
      k_halo_count<<<cs, 256, 0, ctx->stream>>>((int)n, (int)R, p->rowptr, p->col, dcnt);
      USBS_CUDA(cudaMemcpyAsync(ctx->pinned_i, dcnt, cs * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      USBS_CUDA(cudaStreamSynchronize(ctx->stream));
      int hmax = 0;
      for (int b = 0; b < cs; ++b) hmax = std::max(hmax, ctx->pinned_i[b]);
      const size_t smh = lz_cl_smem(m, (int)R, 512, std::max(hmax, 1));
      if (hmax > 0 && smh <= (size_t)optin && lz_cl_max_clusters_lg(LG, cs, smh) >= 1) {
        pl.hmax = hmax;
        pl.smem = smh;
      }
    }
    return pl;
  }
  return pl;
}

// plan cached per (problem, basis size)
static LzClusterPlan lz_cached_plan(usbs_ctx* ctx, usbs_problem* p, int m) {
  if (p->lz_cl_m != m) {
    const LzClusterPlan pl = lz_cluster_plan(ctx, p, m, p->spmv_group);
    p->lz_cl_m = m;
    p->lz_cl_cs = pl.cs;
    p->lz_cl_R = pl.R;
    p->lz_cl_lg = pl.lg;
    p->lz_cl_hmax = pl.hmax;
    p->lz_cl_smem = pl.smem;
  }
  LzClusterPlan pl;
  pl.cs = p->lz_cl_cs;
  pl.R = p->lz_cl_R;
  pl.lg = p->lz_cl_lg;
  pl.hmax = p->lz_cl_hmax;
  pl.smem = p->lz_cl_smem;
  return pl;
}

template <int LG>
static void lz_cl_launch_t(usbs_ctx* ctx, LzArgs& a, const LzClusterPlan& pl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.cs);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = pl.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  USBS_CUDA(cudaLaunchKernelEx(&cfg, k_lanczos_cl<LG>, a, pl.R, pl.hmax));
  check_launch(ctx);
}

static void lz_cl_launch(usbs_ctx* ctx, LzArgs& a, const LzClusterPlan& pl) {
  switch (pl.lg) {
    case 1: lz_cl_launch_t<1>(ctx, a, pl); break;
    case 4: lz_cl_launch_t<4>(ctx, a, pl); break;
    case 8: lz_cl_launch_t<8>(ctx, a, pl); break;
    case 16: lz_cl_launch_t<16>(ctx, a, pl); break;
    default: lz_cl_launch_t<32>(ctx, a, pl); break;
  }
}

template <int NH>
static void lz_dispatch(usbs_ctx* ctx, LzArgs& a, int G, int LG, size_t smem) {
  switch (LG) {
    case 4: lz_launch<4, NH>(ctx, a, G, smem); break;
    case 8: lz_launch<8, NH>(ctx, a, G, smem); break;
    case 16: lz_launch<16, NH>(ctx, a, G, smem); break;
    default: lz_launch<32, NH>(ctx, a, G, smem); break;
  }
}

}  // namespace usbs

using namespace usbs;

// Phase timers accumulated by k_lanczos when USBS_LZ_PROF is set (ns):
// [phase A, grid barriers, phase B, phase C, end of cycle, Rayleigh-Ritz, restart, -]
extern "C" usbs_status usbs_lanczos_profile(usbs_ctx* ctx, unsigned long long* out, int reset) {
  USBS_API_BEGIN
  auto* p = (unsigned long long*)ctx->ws.get(WS_LZ_PROF, 1024 * sizeof(unsigned long long));
  USBS_CUDA(cudaMemcpyAsync(out, p, 1024 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
  USBS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (reset) USBS_CUDA(cudaMemsetAsync(p, 0, 1024 * sizeof(unsigned long long), ctx->stream));
  USBS_API_END
}

extern "C" usbs_status usbs_lanczos_plan(usbs_ctx* ctx, usbs_problem* p, int m, int* cluster_size,
                                         int* rows_per_cta) {
  USBS_API_BEGIN
  if (m < 2 || m > 64) fail(USBS_ERR_CONFIG, "Lanczos basis size must be in [2, 64]");
  const LzClusterPlan pl = (p->n_cols == p->n) ? lz_cached_plan(ctx, p, m) : LzClusterPlan{};
  *cluster_size = pl.cs;
  *rows_per_cta = pl.R;
  USBS_API_END
}

extern "C" usbs_status usbs_lz_step_finish(usbs_ctx* ctx, int j, int m1, const double* c1, const double* c2,
                                           const double* nrm2, double* H, int* flags, const double* w, int64_t nl,
                                           int64_t ldw, double* q, int64_t ldq) {
  USBS_API_BEGIN
  if (j < 0 || j + 1 >= m1) fail(USBS_ERR_SHAPE, "lz_step_finish: 0 <= j < m");
  const int bl = (int)std::max<int64_t>(1, std::min<int64_t>((nl + 255) / 256, 4 * ctx->num_sms));
  k_lz_step_finish<<<bl, 256, 0, ctx->stream>>>(j, m1, c1, c2, nrm2, H, flags, w, nl, ldw, q, ldq);
  check_launch(ctx);
  USBS_API_END
}

extern "C" usbs_status usbs_lz_restart_h(usbs_ctx* ctx, int m1, int ell, const double* theta, double* H) {
  USBS_API_BEGIN
  k_lz_restart_h<<<1, 256, 0, ctx->stream>>>(m1, ell, theta, H);
  check_launch(ctx);
  USBS_API_END
}

extern "C" usbs_status usbs_small_eigh(usbs_ctx* ctx, int k, const double* a, double* vals, double* vecs) {
  USBS_API_BEGIN
  if (k < 1 || k > 64) fail(USBS_ERR_SHAPE, "small_eigh supports 1 <= k <= 64");
  launch_small_eigh(ctx, k, a, vals, vecs);
  USBS_API_END
}

extern "C" usbs_status usbs_lanczos_top(usbs_ctx* ctx, usbs_problem* p, int which, int k_c, int inner_iters,
                                        int max_restarts, double tol, const double* v0, usbs_rng_fill_fn reseed,
                                        void* user, double* vals, double* vecs_dev, int64_t ldvecs, double* res,
                                        int* converged, int* restarts, double* ritz_hist, int* n_hist,
                                        int* matvecs) {
  USBS_API_BEGIN
  const int64_t n = p->n;
  if (k_c < 1) fail(USBS_ERR_CONFIG, "k_c must be at least 1");
  if (p->n_cols != p->n) fail(USBS_ERR_SHAPE, "lanczos_top needs a square (unsharded) operator");
  if (max_restarts < 0 || inner_iters < 0) fail(USBS_ERR_CONFIG, "invalid Lanczos budget");
  if (ldvecs < k_c) fail(USBS_ERR_SHAPE, "ldvecs < k_c");
  const double* val = which ? p->zval : p->cval;
  cudaStream_t st = ctx->stream;
  const int m = std::max(std::max(inner_iters, k_c + 1), 2);
  if (k_c >= n || inner_iters >= n || m >= n) {
    // dense fallback
    if (n > 64) fail(USBS_ERR_CONFIG, "dense Lanczos fallback supports n <= 64");
    int* nf = (int*)ctx->ws.get(WS_LZ_FLAGS, 64 * sizeof(int));
    USBS_CUDA(cudaMemsetAsync(nf, 0, sizeof(int), st));
    double* dv = (double*)ctx->ws.get(WS_LZ_OUT, 64 * sizeof(double));
    const int k = (int)std::min<int64_t>(k_c, n);
    smem_optin(ctx, (const void*)k_dense_eigh, 200 * 1024);
    k_dense_eigh<<<1, 256, eigh_smem((int)n), st>>>((int)n, p->rowptr, p->col, val, k, dv, vecs_dev, ldvecs, nf);
    check_launch(ctx);
    USBS_CUDA(cudaMemcpyAsync(ctx->pinned, dv, k * sizeof(double), cudaMemcpyDeviceToHost, st));
    USBS_CUDA(cudaMemcpyAsync(ctx->pinned_i, nf, sizeof(int), cudaMemcpyDeviceToHost, st));
    USBS_CUDA(cudaStreamSynchronize(st));
    if (ctx->pinned_i[0]) fail(USBS_ERR_NONFINITE, "matvec returned non-finite values");
    for (int u = 0; u < k; ++u) {
      vals[u] = ctx->pinned[u];
      res[u] = 0.0;
    }
    *converged = 1;
    *restarts = 0;
    ritz_hist[0] = ctx->pinned[0];
    *n_hist = 1;
    *matvecs = (int)n;
    return USBS_OK;
  }
  if (m > 64) fail(USBS_ERR_CONFIG, "Lanczos basis size m > 64 is not supported");
  if (max_restarts > 3900) fail(USBS_ERR_CONFIG, "max_restarts > 3900 is not supported");
  const int NH = m <= 32 ? 1 : 2;
  const int G = p->lz_blocks;
  const int64_t ldq = (n + 31) / 32 * 32;
  double* Q = (double*)ctx->ws.get(WS_LZ_Q, (size_t)ldq * (m + 1) * sizeof(double));
  double* W = (double*)ctx->ws.get(WS_LZ_W, (size_t)2 * ldq * sizeof(double));
  double* H = (double*)ctx->ws.get(WS_LZ_H, (size_t)(m + 1) * (m + 1) * sizeof(double));
  double* P = (double*)ctx->ws.get(WS_LZ_P, (size_t)(G * 64 * 2 + G) * sizeof(double));
  int* flags = (int*)ctx->ws.get(WS_LZ_FLAGS, 64 * sizeof(int));
  double* out = (double*)ctx->ws.get(WS_LZ_OUT, (size_t)(m + m * m + m + max_restarts + 1 + 8) * sizeof(double));
  double* tmp = (double*)ctx->ws.get(WS_LZ_TMP, (size_t)(ldq + 128) * sizeof(double));
  // a (re)allocated basis / W workspace may hold the bytes of freed
  // allocations (NaN patterns): the kernels multiply not-yet-written columns
  // by zero coefficients, so zero them once per allocation
  if (ctx->lzq_ptr != (void*)Q || ctx->lzw_ptr != (void*)W) {
    USBS_CUDA(cudaMemsetAsync(Q, 0, (size_t)ldq * (m + 1) * sizeof(double), st));
    USBS_CUDA(cudaMemsetAsync(W, 0, (size_t)2 * ldq * sizeof(double), st));
    ctx->lzq_ptr = Q;
    ctx->lzw_ptr = W;
  }
  USBS_CUDA(cudaMemsetAsync(H, 0, (size_t)(m + 1) * (m + 1) * sizeof(double), st));
  USBS_CUDA(cudaMemsetAsync(flags, 0, 64 * sizeof(int), st));
  // padding rows of the last 32-row tile stay zero (the TMA variant streams
  // whole tiles), as do the padding rows of W
  if (n % 32) {
    USBS_CUDA(cudaMemsetAsync(Q + (n / 32) * (m + 1) * 32, 0, (size_t)(m + 1) * 32 * sizeof(double), st));
    USBS_CUDA(cudaMemsetAsync(W + n, 0, (size_t)(ldq - n) * sizeof(double), st));
    USBS_CUDA(cudaMemsetAsync(W + ldq + n, 0, (size_t)(ldq - n) * sizeof(double), st));
  }
  {
    int bl0 = (int)std::min<int64_t>((n + 255) / 256, 4 * ctx->num_sms);
    k_qcol_set<<<bl0, 256, 0, st>>>(n, v0, 1.0, Q, 0, m + 1);
    check_launch(ctx);
  }

  LzArgs a{};
  a.n = (int)n; a.m = m; a.k_c = k_c; a.max_restarts = max_restarts; a.ldq = ldq;
  a.tol = tol < 0 ? 1e-9 : tol;
  a.rowptr = p->rowptr; a.col = p->col; a.val = val;
  a.blk_row = p->blk_row; a.blk_seg = p->blk_seg; a.seg_r0 = p->seg_r0; a.seg_r1 = p->seg_r1;
  a.piece_z0 = p->lz_piece_z0; a.piece_z1 = p->lz_piece_z1;
  // small operators: one thread-block cluster with Q resident in smem; large
  // ones: the TMA-pipelined grid kernel (m <= 32) or the v1 grid kernel
  const LzClusterPlan clp = lz_cached_plan(ctx, p, m);
  const char* ev1 = getenv("USBS_LZ_V1");
  const bool use_tma = clp.cs == 0 && m <= 32 && !(ev1 && ev1[0] == '1');
  if (getenv("USBS_LZ_DEBUG"))
    fprintf(stderr, "[lanczos] n=%lld m=%d cluster=%d R=%d hmax=%d smem=%zu tma=%d\n", (long long)n, m, clp.cs, clp.R,
            clp.hmax, clp.smem, (int)use_tma);
  if (use_tma) lz_tma_plan(ctx, p);
  a.piece_sum = (double*)ctx->ws.get(
      WS_LZ_SPLIT, (size_t)std::max(1, std::max(p->lz_npieces, use_tma ? p->lzg_npieces : 0)) * sizeof(double));
  a.blk_split = p->lz_blk_split; a.split_row = p->lz_split_row; a.split_first = p->lz_split_first;
  a.split_cnt = p->lz_split_cnt;
  a.Q = Q; a.W0 = W; a.W1 = W + ldq; a.H = H;
  a.P1 = P; a.P2 = P + G * 64; a.P3 = P + 2 * G * 64;
  a.flags = flags;
  a.theta = out; a.Y = out + m; a.res = out + m + m * m; a.hist = out + 2 * m + m * m;
  a.vecs_out = vecs_dev; a.ldvecs = ldvecs;
  a.cycle0 = 0; a.ell0 = 0; a.j0 = 0; a.restarts0 = 0; a.nhist0 = 0; a.matvecs0 = 0; a.wbuf0 = 0;
  a.beta_prev = 1.0; a.first_from_q = 1;
  a.prof = nullptr;
  if (getenv("USBS_LZ_PROF")) {
    static bool zeroed = false;
    a.prof = (unsigned long long*)ctx->ws.get(WS_LZ_PROF, 1024 * sizeof(unsigned long long));
    if (!zeroed) {
      USBS_CUDA(cudaMemsetAsync(a.prof, 0, 1024 * sizeof(unsigned long long), st));
      zeroed = true;
    }
  }

  const int nw = (NH == 1 ? 512 : 256) / 32;
  size_t smem = (size_t)(nw * 32 * NH + 64 * 3 + 8 + 64 + m * m + 4 * m * m + 64 * 2 + 32) * sizeof(double) +
                68 * sizeof(int) + JAC_PTAB_BYTES + (6 * 64) * sizeof(double) + 128 * sizeof(int) + 64 +
                LZT_NNZ * sizeof(double) + (2 * LZT_ROWS + 2) * sizeof(int);
  if (use_tma) {
    // P partials are [32][G'] with the TMA plan's block count
    const int Gt = p->lzg_G;
    double* Pt = (double*)ctx->ws.get(WS_LZ_P, (size_t)(std::max(G, Gt) * 64 * 2 + std::max(G, Gt)) * sizeof(double));
    a.P1 = Pt; a.P2 = Pt + Gt * 64; a.P3 = Pt + 2 * Gt * 64;
  }
  int64_t ctr = 0;
  int* hf = ctx->pinned_i;
  for (;;) {
    if (clp.cs > 0) lz_cl_launch(ctx, a, clp);
    else if (use_tma) lz_tma_launch(ctx, p, a);
    else if (NH == 1) lz_dispatch<1>(ctx, a, G, p->spmv_group, smem);
    else lz_dispatch<2>(ctx, a, G, p->spmv_group, smem);
    // flags and (speculatively) the results in one round trip
    USBS_CUDA(cudaMemcpyAsync(hf, flags, 16 * sizeof(int), cudaMemcpyDeviceToHost, st));
    USBS_CUDA(cudaMemcpyAsync(ctx->pinned, a.theta, (size_t)k_c * sizeof(double), cudaMemcpyDeviceToHost, st));
    USBS_CUDA(cudaMemcpyAsync(ctx->pinned + 64, a.res, (size_t)k_c * sizeof(double), cudaMemcpyDeviceToHost, st));
    USBS_CUDA(cudaMemcpyAsync(ctx->pinned + 128, a.hist, (size_t)(max_restarts + 1) * sizeof(double),
                              cudaMemcpyDeviceToHost, st));
    USBS_CUDA(cudaStreamSynchronize(st));
    if (hf[F_EXIT] == EXIT_NONFINITE) fail(USBS_ERR_NONFINITE, "matvec returned non-finite values");
    if (hf[F_EXIT] == EXIT_DONE) break;
    // breakdown at step j: fresh direction for q_{j+1} (eigsolve.py:136-147, 55-63)
    const int j = hf[F_J], used = j + 1;
    ctr += 16;
    double* v = tmp;
    double* cbuf = tmp + ldq;
    bool got = false;
    for (int att = 0; att < 8 && !got; ++att) {
      if (!reseed) fail(USBS_ERR_CALLBACK, "Lanczos breakdown needs a reseed callback");
      if (reseed(user, ctr + att + 1, v, n) != 0) fail(USBS_ERR_CALLBACK, "reseed callback failed");
      // _seeded_unit normalises, then the projection, then the norm test
      k_norm2<<<1, 1024, 0, st>>>(n, v, cbuf + 64);
      check_launch(ctx);
      USBS_CUDA(cudaMemcpyAsync(ctx->pinned, cbuf + 64, sizeof(double), cudaMemcpyDeviceToHost, st));
      USBS_CUDA(cudaStreamSynchronize(st));
      double nv0 = std::sqrt(ctx->pinned[0]);
      int thr = 256, bl = (int)std::min<int64_t>((n + thr - 1) / thr, 4 * ctx->num_sms);
      k_scale_into<<<bl, thr, 0, st>>>(n, v, 1.0 / nv0, v);
      check_launch(ctx);
      k_qcol_dot<<<used, 512, 0, st>>>(n, Q, m + 1, v, cbuf);
      check_launch(ctx);
      k_qcol_sub<<<bl, thr, 0, st>>>(n, Q, m + 1, used, cbuf, v);
      check_launch(ctx);
      k_norm2<<<1, 1024, 0, st>>>(n, v, cbuf + 64);
      check_launch(ctx);
      USBS_CUDA(cudaMemcpyAsync(ctx->pinned, cbuf + 64, sizeof(double), cudaMemcpyDeviceToHost, st));
      USBS_CUDA(cudaStreamSynchronize(st));
      double nv = std::sqrt(ctx->pinned[0]);
      if (nv > 1e-8) {
        k_qcol_set<<<bl, thr, 0, st>>>(n, v, 1.0 / nv, Q, j + 1, m + 1);
        check_launch(ctx);
        got = true;
      }
    }
    if (!got) {
      int bl = (int)std::min<int64_t>((n + 255) / 256, 4 * ctx->num_sms);
      k_qcol_set<<<bl, 256, 0, st>>>(n, nullptr, 0.0, Q, j + 1, m + 1);
      check_launch(ctx);
    }
    const int M1 = m + 1;
    double zero = 0.0;
    USBS_CUDA(cudaMemcpyAsync(H + (j + 1) * M1 + j, &zero, sizeof(double), cudaMemcpyHostToDevice, st));
    USBS_CUDA(cudaMemcpyAsync(H + j * M1 + (j + 1), &zero, sizeof(double), cudaMemcpyHostToDevice, st));
    USBS_CUDA(cudaStreamSynchronize(st));
    a.cycle0 = hf[F_CYCLE]; a.ell0 = hf[F_ELL]; a.j0 = j + 1; a.restarts0 = hf[F_RESTARTS];
    a.nhist0 = hf[F_NHIST]; a.matvecs0 = hf[F_MATVECS]; a.wbuf0 = hf[F_PENDING];
    a.first_from_q = 1;
    USBS_CUDA(cudaMemsetAsync(flags, 0, 64 * sizeof(int), st));
  }
  const int nh = hf[F_NHIST];
  const double* ho = ctx->pinned;
  for (int u = 0; u < k_c; ++u) {
    vals[u] = ho[u];
    res[u] = ho[64 + u];
  }
  for (int h = 0; h < nh; ++h) ritz_hist[h] = ho[128 + h];
  *converged = hf[F_CONV];
  *restarts = hf[F_RESTARTS];
  *n_hist = nh;
  *matvecs = hf[F_MATVECS];
  USBS_API_END
}
