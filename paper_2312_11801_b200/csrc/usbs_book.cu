// Low-rank primal bookkeeping kernels (K4, K4w, K5, K8, K10, K13, K14 of
// SURVEY 2.2).  Reference behaviour (paths under pkg/src/specbundle/):
//   problem.py:151-155, 200-208  primal_image_lowrank / primal_image_factor
//   problem.py:169-173, 229-239  compressed_rows (never materialised here:
//                                rows are generated tile by tile in smem)
//   subqp.py:487-498, 509-510    quad_ss = a^2/rho C^T C, quad_s_eta, C^T w
//   bundle.py:307-316            F = V Q_c, trace / cost / image statistics
//   sketch.py:58-74              P <- eta P + (F L)(F^T Psi)
//   bundle.py:108-109            Xbar <- eta Xbar + F L F^T
//   problem.py:292-308, bundle.py:239-255, 344-372, subqp.py:595-598
//                                projections, candidate, residual norms
#include <algorithm>
#include <cmath>

#include "usbs_common.cuh"
#include "usbs_kernels.cuh"

namespace usbs {

// ------------------------------------------------------------- K5 images
// out[i] = beta*base[i] + A_i(V S V^T); S full k x k (sdiag=0) or diag (sdiag=1)
__global__ void __launch_bounds__(256) k_image_diag(int64_t n, const double* __restrict__ V, int64_t ldv, int k,
                                                    const double* __restrict__ S, int sdiag, double sscale,
                                                    const double* beta_dev, double beta,
                                                    const double* __restrict__ base, double* __restrict__ out) {
  // the block's 256 rows are staged with coalesced loads (odd row stride in
  // shared memory: conflict-free row reads), then a thread per row
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Ss = (double*)smem_raw;          // k * k
  double* rows = Ss + k * k;               // 256 * kp
  const int kp = k | 1;
  for (int x = threadIdx.x; x < (sdiag ? k : k * k); x += blockDim.x) Ss[x] = sscale * S[x];
  if (beta_dev) beta *= beta_dev[0];
  for (int64_t r0 = (int64_t)blockIdx.x * 256; r0 < n; r0 += (int64_t)gridDim.x * 256) {
    const int nr = (int)min((int64_t)256, n - r0);
    __syncthreads();
    for (int x = threadIdx.x; x < nr * k; x += blockDim.x) {
      const int r = x / k, c = x - r * k;
      rows[r * kp + c] = V[(r0 + r) * ldv + c];
    }
    __syncthreads();
    const int t = threadIdx.x;
    if (t < nr) {
      const double* v = rows + t * kp;
      double acc = 0.0;
      if (sdiag) {
        for (int j = 0; j < k; ++j) acc = fma(v[j] * v[j], Ss[j], acc);
      } else {
        for (int j = 0; j < k; ++j) {
          double tt = 0.0;
          for (int l = 0; l < k; ++l) tt = fma(Ss[j * k + l], v[l], tt);
          acc = fma(v[j], tt, acc);
        }
      }
      const int64_t i = r0 + t;
      out[i] = (base ? beta * base[i] : 0.0) + acc;
    }
  }
}

// A(V S V^T) for entry constraints: <A_i, V S V^T> = sum over the entries
// (r, c, val) of constraint i of (2 - [r == c]) val (V S V^T)[r, c], with
// (V S V^T)[r, c] = W[r, :] . V[c, :] and W = V S computed once by k_rowgemm
// (k FMAs per entry instead of k^2).  Eight lanes per constraint stride over
// its entries; a fixed shuffle tree sums them (deterministic).
__global__ void __launch_bounds__(256) k_image_entries(int64_t m, const int* __restrict__ cptr,
                                                       const int* __restrict__ cent, const int* __restrict__ erow,
                                                       const int* __restrict__ ecol, const double* __restrict__ eval,
                                                       const double* __restrict__ V, int64_t ldv,
                                                       const double* __restrict__ W, int64_t ldw, int k,
                                                       const double* __restrict__ S, int sdiag, double sscale,
                                                       const double* beta_dev, double beta,
                                                       const double* __restrict__ base, double* __restrict__ out) {
  __shared__ double Sd[64];
  if (sdiag)
    for (int x = threadIdx.x; x < k; x += blockDim.x) Sd[x] = sscale * S[x];
  if (beta_dev) beta *= beta_dev[0];
  __syncthreads();
  const int lane = threadIdx.x & 31, gw = lane >> 3, t = lane & 7;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t wb = wid * 4; wb < m; wb += nwarps * 4) {
    const int64_t i = wb + gw;
    double acc = 0.0;
    if (i < m) {
      for (int q = cptr[i] + t; q < cptr[i + 1]; q += 8) {
        const int e = cent[q];
        const int r = erow[e], c = ecol[e];
        const double* vc = V + (int64_t)c * ldv;
        double v = 0.0;
        if (sdiag) {
          const double* vr = V + (int64_t)r * ldv;
          for (int j = 0; j < k; ++j) v = fma(vr[j] * Sd[j], vc[j], v);
        } else {
          const double* wr = W + (int64_t)r * ldw;
          for (int j = 0; j < k; ++j) v = fma(wr[j], vc[j], v);
        }
        acc = fma(v, (r == c) ? eval[e] : 2.0 * eval[e], acc);
      }
    }
#pragma unroll
    for (int o = 4; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, 8);
    if (i < m && t == 0) out[i] = (base ? beta * base[i] : 0.0) + acc;
  }
}

// k_image_entries for problems whose constraints mostly have ONE entry
// (C3: 99%, C5: all): the entry comes from the flattened (row, col, value)
// arrays (one load level instead of cptr -> cent -> entry), and four lanes
// share a constraint's k-long dot product (lane t takes columns t, t + 4,
// ...; one row read by the four lanes is one contiguous range), two shuffle
// steps to combine, eight constraints per warp.  Constraints with a few
// entries (rc.x == -1) are summed by the group's lanes from the entry list;
// the ones with more than IMAGE_HEAVY entries (C3: one 400-entry row sum,
// which alone set the kernel's duration when four lanes walked it) are
// listed in heavy[1 .. heavy[0]] and each is summed by a whole block first:
// 64 lane groups over its entries, a fixed shuffle + shared-memory tree.
// Sum orders differ from k_image_entries (rounding level only).
constexpr int IMAGE_HEAVY = 32;

__global__ void __launch_bounds__(256) k_image_c1(int64_t m, const int2* __restrict__ c1rc,
                                                  const double* __restrict__ c1v, const int* __restrict__ heavy,
                                                  const int* __restrict__ cptr,
                                                  const int* __restrict__ cent, const int* __restrict__ erow,
                                                  const int* __restrict__ ecol, const double* __restrict__ eval,
                                                  const double* __restrict__ V, int64_t ldv,
                                                  const double* __restrict__ W, int64_t ldw, int k,
                                                  const double* __restrict__ S, int sdiag, double sscale,
                                                  const double* beta_dev, double beta,
                                                  const double* __restrict__ base, double* __restrict__ out) {
  __shared__ double Sd[64];
  __shared__ double red[8];
  if (sdiag)
    for (int x = threadIdx.x; x < k; x += blockDim.x) Sd[x] = sscale * S[x];
  if (beta_dev) beta *= beta_dev[0];
  __syncthreads();
  const int lane = threadIdx.x & 31, gq = lane >> 2, t = lane & 3;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // columns j0, j0 + js, ... of the entry's k-long dot
  auto pair = [&](int r, int c, int j0, int js) -> double {
    double v = 0.0;
    if (sdiag) {
      const double* vr = V + (int64_t)r * ldv;
      const double* vc = V + (int64_t)c * ldv;
      for (int j = j0; j < k; j += js) v = fma(vr[j] * Sd[j], vc[j], v);
    } else {
      const double* wr = W + (int64_t)r * ldw;
      const double* vc = V + (int64_t)c * ldv;
      for (int j = j0; j < k; j += js) v = fma(wr[j], vc[j], v);
    }
    return v;
  };
  const int nh = heavy ? heavy[0] : 0;
  for (int h = blockIdx.x; h < nh; h += gridDim.x) {
    const int i = heavy[1 + h];
    double acc = 0.0;
    for (int q = cptr[i] + (threadIdx.x >> 2); q < cptr[i + 1]; q += blockDim.x >> 2) {
      const int e = cent[q];
      const int r = erow[e], c = ecol[e];
      acc = fma(pair(r, c, t, 4), (r == c) ? eval[e] : 2.0 * eval[e], acc);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
      out[i] = (base ? beta * base[i] : 0.0) + s;
    }
    __syncthreads();
  }
  for (int64_t wb = wid * 8; wb < m; wb += nwarps * 8) {
    const int64_t i = wb + gq;
    double acc = 0.0;
    bool own = i < m;
    if (own) {
      const int2 rc = __ldg(c1rc + i);
      if (rc.x >= 0) {  // one entry: the four lanes split its dot
        const double val = __ldg(c1v + i);
        acc = pair(rc.x, rc.y, t, 4) * ((rc.x == rc.y) ? val : 2.0 * val);
      } else {  // several: the lanes split the entries, a whole dot each
        const int q0 = cptr[i], q1 = cptr[i + 1];
        if (heavy && q1 - q0 > IMAGE_HEAVY) {
          own = false;  // a block summed it
        } else {
          for (int q = q0 + t; q < q1; q += 4) {
            const int e = cent[q];
            const int r = erow[e], c = ecol[e];
            acc = fma(pair(r, c, 0, 1), (r == c) ? eval[e] : 2.0 * eval[e], acc);
          }
        }
      }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 2, 4);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1, 4);
    if (own && t == 0) out[i] = (base ? beta * base[i] : 0.0) + acc;
  }
}

// -------------------------------------------------- K4 / K4w compressed rows
// Row i of the (never stored) compressed matrix: c_i[p] = svec(V^T A_i V)[p].
// Tiles of TR constraints are generated into smem; each thread accumulates
// TPT 4x4 lower tiles of C^T C plus its share of C^T a and C^T w.
constexpr int CTR = 32;

__device__ __forceinline__ double crow_entry(int diag_only, int64_t i, int a, int b, double wp,
                                             const int* __restrict__ cptr, const int* __restrict__ cent,
                                             const int* __restrict__ erow, const int* __restrict__ ecol,
                                             const double* __restrict__ eval, const double* __restrict__ V,
                                             int64_t ldv) {
  if (diag_only) {
    const double* v = V + i * ldv;
    return v[a] * v[b] * wp;
  }
  double s = 0.0;
  for (int t = cptr[i]; t < cptr[i + 1]; ++t) {
    const int e = cent[t];
    const int r = erow[e], c = ecol[e];
    const double* vr = V + (int64_t)r * ldv;
    const double* vc = V + (int64_t)c * ldv;
    double g = vr[a] * vc[b] + vc[a] * vr[b];
    if (r == c) g *= 0.5;
    s += g * eval[e] * wp;
  }
  return s;
}

template <int TPT>
__global__ void __launch_bounds__(256) k_compressed(int64_t m, int diag_only, const int* __restrict__ cptr,
                                                    const int* __restrict__ cent, const int* __restrict__ erow,
                                                    const int* __restrict__ ecol, const double* __restrict__ eval,
                                                    const double* __restrict__ V, int64_t ldv, int k, int d,
                                                    const double* __restrict__ avec, const double* __restrict__ wvec,
                                                    int do_gram, double* __restrict__ gpart,
                                                    double* __restrict__ apart, double* __restrict__ wpart) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int dp = d + 1;  // padded row stride
  double* tile = (double*)smem_raw;         // CTR * dp
  double* aw = tile + CTR * dp;              // CTR
  double* ww = aw + CTR;                     // CTR
  unsigned char* pi = (unsigned char*)(ww + CTR);
  unsigned char* pj = pi + 600;
  if (threadIdx.x == 0) {
    int p = 0;
    for (int j = 0; j < k; ++j)
      for (int i = j; i < k; ++i) { pi[p] = (unsigned char)i; pj[p] = (unsigned char)j; ++p; }
  }
  const int64_t chunk = (m + gridDim.x - 1) / gridDim.x;
  const int64_t c0 = blockIdx.x * chunk, c1 = min(m, c0 + chunk);
  const int nt = (d + 3) / 4;
  const int ntiles = nt * (nt + 1) / 2;
  double acc[TPT][16];
  int tr_[TPT], tc_[TPT];
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
#pragma unroll
    for (int x = 0; x < 16; ++x) acc[u][x] = 0.0;
    int tix = threadIdx.x + u * 256;
    tr_[u] = -1;
    tc_[u] = 0;
    if (do_gram && tix < ntiles) {
      int r = (int)((sqrtf(8.0f * tix + 1.0f) - 1.0f) * 0.5f);
      while (r * (r + 1) / 2 > tix) --r;
      while ((r + 1) * (r + 2) / 2 <= tix) ++r;
      tr_[u] = r;
      tc_[u] = tix - r * (r + 1) / 2;
    }
  }
  double accA[3] = {0, 0, 0}, accW[3] = {0, 0, 0};  // d <= 768 with 256 threads
  __syncthreads();
  for (int64_t base = c0; base < c1; base += CTR) {
    const int rows = (int)min((int64_t)CTR, c1 - base);
    __syncthreads();
    for (int x = threadIdx.x; x < CTR * d; x += blockDim.x) {
      const int r = x / d, p = x % d;
      double v = 0.0;
      if (r < rows) {
        const int a = pi[p], b = pj[p];
        v = crow_entry(diag_only, base + r, a, b, a == b ? 1.0 : 1.4142135623730951, cptr, cent, erow, ecol,
                       eval, V, ldv);
      }
      tile[r * dp + p] = v;
    }
    for (int r = threadIdx.x; r < CTR; r += blockDim.x) {
      aw[r] = (avec && r < rows) ? avec[base + r] : 0.0;
      ww[r] = (wvec && r < rows) ? wvec[base + r] : 0.0;
    }
    __syncthreads();
    if (do_gram) {
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        if (tr_[u] < 0) continue;
        const int pa = tr_[u] * 4, pb = tc_[u] * 4;
        for (int r = 0; r < rows; ++r) {
          const double* row = tile + r * dp;
          double xa[4], xb[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            xa[q] = (pa + q < d) ? row[pa + q] : 0.0;
            xb[q] = (pb + q < d) ? row[pb + q] : 0.0;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int s = 0; s < 4; ++s) acc[u][q * 4 + s] = fma(xa[q], xb[s], acc[u][q * 4 + s]);
        }
      }
    }
    if (avec || wvec) {
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const int p = threadIdx.x + u * 256;
        if (p < d) {
          double sa = accA[u], sw = accW[u];
          for (int r = 0; r < rows; ++r) {
            const double c = tile[r * dp + p];
            sa = fma(aw[r], c, sa);
            sw = fma(ww[r], c, sw);
          }
          accA[u] = sa;
          accW[u] = sw;
        }
      }
    }
  }
  // partials: gram as full d x d (lower tiles mirrored later), vectors
  if (do_gram) {
#pragma unroll
    for (int u = 0; u < TPT; ++u) {
      if (tr_[u] < 0) continue;
      const int pa = tr_[u] * 4, pb = tc_[u] * 4;
      for (int q = 0; q < 4; ++q)
        for (int s = 0; s < 4; ++s) {
          const int P = pa + q, Qc = pb + s;
          if (P < d && Qc < d && Qc <= P) gpart[(int64_t)blockIdx.x * d * d + (int64_t)P * d + Qc] = acc[u][q * 4 + s];
        }
    }
  }
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    const int p = threadIdx.x + u * 256;
    if (p < d) {
      if (apart) apart[(int64_t)blockIdx.x * d + p] = accA[u];
      if (wpart) wpart[(int64_t)blockIdx.x * d + p] = accW[u];
    }
  }
}

// The same partial sums with the d x d Gram on the FP64 tensor cores: per
// 32-row tile of generated rows (smem, as above), G += T^T T as m8n8k4 MMAs
// over 8 x 8 output tiles of the lower triangle, TPW tiles per warp
// (16 warps), accumulators in registers for the whole row range; the
// tiles' (I, K) come from a smem table.
template <int TPW>
__global__ void __launch_bounds__(512, 1) k_compressed_mma(int64_t m, int diag_only, const int* __restrict__ cptr,
                                                        const int* __restrict__ cent, const int* __restrict__ erow,
                                                        const int* __restrict__ ecol, const double* __restrict__ eval,
                                                        const double* __restrict__ V, int64_t ldv, int k, int d,
                                                        const double* __restrict__ avec,
                                                        const double* __restrict__ wvec, double* __restrict__ gpart,
                                                        double* __restrict__ apart, double* __restrict__ wpart,
                                                        int runs) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // row stride = 8 (mod 16) doubles: the fragment loads (rows 4ks + q,
  // columns 8X + g) then hit every bank exactly twice
  const int dp = d + 1 + ((8 - (d + 1)) & 15);
  double* tile = (double*)smem_raw;  // CTR * dp
  double* aw = tile + CTR * dp;       // CTR
  double* ww = aw + CTR;              // CTR
  unsigned char* pi = (unsigned char*)(ww + CTR);
  unsigned char* pj = pi + 600;
  unsigned short* ttab = (unsigned short*)(pj + 600);  // (I << 8) | K of the 8 x 8 lower tiles
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nth = blockDim.x;
  const int g = lane >> 2, q = lane & 3;
  const int n8 = (d + 7) >> 3, nt8 = n8 * (n8 + 1) / 2;
  // tile u of this warp (-1: none): strided (t = y 16 + warp + 16 HY u) or a
  // contiguous run per warp of the CTA's share
  const int per_cta = (nt8 + (int)gridDim.y - 1) / (int)gridDim.y;
  const int per_warp = (per_cta + 15) / 16;
  const int cta_end = min(nt8, ((int)blockIdx.y + 1) * per_cta);
  auto tile_t = [&](int u) -> int {
    if (runs) {
      const int t = (int)blockIdx.y * per_cta + warp * per_warp + u;
      return (u < per_warp && t < cta_end) ? t : -1;
    }
    const int t = (int)blockIdx.y * 16 + warp + 16 * (int)gridDim.y * u;
    return t < nt8 ? t : -1;
  };
  if (tid == 0) {
    int p = 0;
    for (int j = 0; j < k; ++j)
      for (int i = j; i < k; ++i) { pi[p] = (unsigned char)i; pj[p] = (unsigned char)j; ++p; }
  }
  for (int t = tid; t < nt8; t += nth) {
    int I = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
    while (I * (I + 1) / 2 > t) --I;
    while ((I + 1) * (I + 2) / 2 <= t) ++I;
    ttab[t] = (unsigned short)((I << 8) | (t - I * (I + 1) / 2));
  }
  const int64_t chunk = (m + gridDim.x - 1) / gridDim.x;
  const int64_t c0 = blockIdx.x * chunk, c1 = min(m, c0 + chunk);
  double acc0[TPW], acc1[TPW];
#pragma unroll
  for (int u = 0; u < TPW; ++u) acc0[u] = acc1[u] = 0.0;
  double accA[2] = {0, 0}, accW[2] = {0, 0};
  __syncthreads();
  for (int64_t base = c0; base < c1; base += CTR) {
    const int rows = (int)min((int64_t)CTR, c1 - base);
    __syncthreads();
    // rows of the tile: a warp per constraint row (k <= 32), the V rows of
    // its entries loaded once per entry into the lanes and the d products
    // formed by shuffles, lane p handling entries p, p + 32, ...
    for (int r = warp; r < CTR; r += nth >> 5) {
      double accp[7];
#pragma unroll
      for (int jj = 0; jj < 7; ++jj) accp[jj] = 0.0;
      if (r < rows) {
        const int64_t i = base + r;
        const int t0 = diag_only ? 0 : cptr[i], t1 = diag_only ? 1 : cptr[i + 1];
        for (int t = t0; t < t1; ++t) {
          int rr, cc2;
          double val;
          if (diag_only) {
            rr = cc2 = (int)i;
            val = 1.0;
          } else {
            const int e = cent[t];
            rr = erow[e];
            cc2 = ecol[e];
            val = eval[e];
          }
          const double vr = lane < k ? V[(int64_t)rr * ldv + lane] : 0.0;
          const double vc = lane < k ? V[(int64_t)cc2 * ldv + lane] : 0.0;
          const double half = rr == cc2 ? 0.5 : 1.0;
#pragma unroll
          for (int jj = 0; jj < 7; ++jj) {
            const int pp = lane + 32 * jj;
            const int aa = pp < d ? pi[pp] : 0, bb = pp < d ? pj[pp] : 0;
            const double ra = __shfl_sync(0xffffffffu, vr, aa), cb = __shfl_sync(0xffffffffu, vc, bb);
            const double ca = __shfl_sync(0xffffffffu, vc, aa), rb = __shfl_sync(0xffffffffu, vr, bb);
            const double wpp = aa == bb ? 1.0 : 1.4142135623730951;
            double gg = ra * cb + ca * rb;
            gg *= half;
            accp[jj] += gg * val * wpp;
          }
        }
      }
#pragma unroll
      for (int jj = 0; jj < 7; ++jj) {
        const int pp = lane + 32 * jj;
        if (pp < d) tile[r * dp + pp] = accp[jj];
      }
    }
    for (int r = tid; r < CTR; r += nth) {
      aw[r] = (avec && r < rows) ? avec[base + r] : 0.0;
      ww[r] = (wvec && r < rows) ? wvec[base + r] : 0.0;
    }
    __syncthreads();
    if (runs) {
      // a contiguous run of lower-triangle tiles per warp: tiles of one tile
      // row share the A fragment, loaded once per k-step and row; k-steps
      // outer so the warp's tile chains interleave
#pragma unroll
      for (int ks = 0; ks < CTR / 4; ++ks) {
        const double* row = tile + (4 * ks + q) * dp;
        int iprev = -1;
        double av = 0.0;
#pragma unroll
        for (int u = 0; u < TPW; ++u) {
          const int t = tile_t(u);
          if (t >= 0) {
            const unsigned e = ttab[t];
            const int I = (int)(e >> 8);
            const int ca = 8 * I + g, cb = 8 * (int)(e & 255u) + g;
            if (I != iprev) {
              av = ca < d ? row[ca] : 0.0;
              iprev = I;
            }
            const double bv = cb < d ? row[cb] : 0.0;
            dmma_m8n8k4(acc0[u], acc1[u], av, bv, acc0[u], acc1[u]);
          }
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < TPW; ++u) {
        const int t = tile_t(u);
        if (t >= 0) {
          const unsigned e = ttab[t];
          const int ca = 8 * (int)(e >> 8) + g, cb = 8 * (int)(e & 255u) + g;
          const bool va = ca < d, vb = cb < d;
#pragma unroll
          for (int ks = 0; ks < CTR / 4; ++ks) {
            const double* row = tile + (4 * ks + q) * dp;
            const double av = va ? row[ca] : 0.0, bv = vb ? row[cb] : 0.0;
            dmma_m8n8k4(acc0[u], acc1[u], av, bv, acc0[u], acc1[u]);
          }
        }
      }
    }
    if ((avec || wvec) && blockIdx.y == 0) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int p = tid + u * 512;
        if (p < d) {
          double sa = accA[u], sw = accW[u];
          for (int r = 0; r < rows; ++r) {
            const double c = tile[r * dp + p];
            sa = fma(aw[r], c, sa);
            sw = fma(ww[r], c, sw);
          }
          accA[u] = sa;
          accW[u] = sw;
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < TPW; ++u) {
    const int t = tile_t(u);
    if (t >= 0) {
      const unsigned e = ttab[t];
      const int P = 8 * (int)(e >> 8) + g, Q0 = 8 * (int)(e & 255u) + 2 * q;
      double* out = gpart + (int64_t)blockIdx.x * d * d;
      if (P < d && Q0 < d && Q0 <= P) out[(int64_t)P * d + Q0] = acc0[u];
      if (P < d && Q0 + 1 < d && Q0 + 1 <= P) out[(int64_t)P * d + Q0 + 1] = acc1[u];
    }
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int p = tid + u * 512;
    if (p < d && blockIdx.y == 0) {
      if (apart) apart[(int64_t)blockIdx.x * d + p] = accA[u];
      if (wpart) wpart[(int64_t)blockIdx.x * d + p] = accW[u];
    }
  }
}

// Single-entry flattening for the pipelined K4: per constraint row the
// (row, col, value) of its entry when it has exactly one (C3: 99%, C5: all),
// else (-1, -1) and the row is generated from the entry list.
__global__ void k_c1_flatten(int64_t m, const int* __restrict__ cptr, const int* __restrict__ cent,
                             const int* __restrict__ erow, const int* __restrict__ ecol,
                             const double* __restrict__ eval, int2* __restrict__ rc, double* __restrict__ cv,
                             int* __restrict__ heavy) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const int t0 = cptr[i], t1 = cptr[i + 1];
    if (heavy && t1 - t0 > IMAGE_HEAVY) heavy[1 + atomicAdd(heavy, 1)] = (int)i;
    if (t1 - t0 == 1) {
      const int e = cent[t0];
      rc[i] = make_int2(erow[e], ecol[e]);
      cv[i] = eval[e];
    } else {
      rc[i] = make_int2(-1, -1);
      cv[i] = 0.0;
    }
  }
}

// K4 with the row generation pipelined behind the tensor-core Gram.  The
// 32-row tiles of generated rows are double buffered in smem and the
// generation of tile i+1 runs in the same barrier interval as the MMAs of
// tile i; its global loads are issued ahead: the constraints' single entries
// (row, col, value) three tiles ahead and their two V rows two tiles ahead,
// in flight while the warp runs its MMAs.  Warp w owns rows w and w + 16 of
// every tile.  Rows with several entries are generated from the entry list
// (synchronously).  The Gram is computed in 16 x 16 blocks of the lower
// triangle (2 x 2 tiles of 8, three on the diagonal), BPW blocks per warp
// strided over the warps of gridDim.y CTAs per row range: per k-step the
// warp loads two A and two B fragments for four m8n8k4 MMAs.
template <int BPW>
__global__ void __launch_bounds__(512, 1) k_compressed_mma_pipe(int64_t m, int diag_only,
    const int2* __restrict__ c1rc, const double* __restrict__ c1v, const int* __restrict__ cptr,
    const int* __restrict__ cent, const int* __restrict__ erow, const int* __restrict__ ecol,
    const double* __restrict__ eval, const double* __restrict__ V, int64_t ldv, int k, int d,
    double* __restrict__ gpart) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int dp = d + 1 + ((8 - (d + 1)) & 15);
  double* tbuf = (double*)smem_raw;  // 2 x CTR * dp
  unsigned char* pi = (unsigned char*)(tbuf + 2 * CTR * dp);
  unsigned char* pj = pi + 600;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int n16 = (d + 15) >> 4, nb16 = n16 * (n16 + 1) / 2;
  // block u of this warp: (BI, BK), BK <= BI, or BI = -1
  int bI[BPW], bK[BPW];
#pragma unroll
  for (int u = 0; u < BPW; ++u) {
    const int t = (int)blockIdx.y * 16 + warp + 16 * (int)gridDim.y * u;
    if (t < nb16) {
      int I = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
      while (I * (I + 1) / 2 > t) --I;
      while ((I + 1) * (I + 2) / 2 <= t) ++I;
      bI[u] = I;
      bK[u] = t - I * (I + 1) / 2;
    } else {
      bI[u] = -1;
      bK[u] = 0;
    }
  }
  if (tid == 0) {
    int p = 0;
    for (int j = 0; j < k; ++j)
      for (int i = j; i < k; ++i) { pi[p] = (unsigned char)i; pj[p] = (unsigned char)j; ++p; }
  }
  const int64_t chunk = (m + gridDim.x - 1) / gridDim.x;
  const int64_t c0 = blockIdx.x * chunk, c1 = min(m, c0 + chunk);
  const int ntile = (int)((max((int64_t)0, c1 - c0) + CTR - 1) / CTR);
  double acc[BPW][4][2];
#pragma unroll
  for (int u = 0; u < BPW; ++u)
#pragma unroll
    for (int x = 0; x < 4; ++x) acc[u][x][0] = acc[u][x][1] = 0.0;

  // prefetch state per owned row slot s (rows warp, warp + 16 of a tile):
  // A = entries of tile i+3, B = V rows of tile i+2, C = V rows of tile i+1
  int2 rcA[2], rcB[2], rcC[2];
  double vA[2], vB[2], vC[2], vrB[2], vcB[2], vrC[2], vcC[2];
  auto row_of = [&](int tl, int s) -> int64_t { return c0 + (int64_t)tl * CTR + warp + 16 * s; };
  auto load_info = [&](int tl) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int64_t i = row_of(tl, s);
      if (tl < ntile && i < c1) {
        if (diag_only) { rcA[s] = make_int2((int)i, (int)i); vA[s] = 1.0; }
        else { rcA[s] = __ldg(c1rc + i); vA[s] = __ldg(c1v + i); }
      } else {
        rcA[s] = make_int2(-2, -2);  // no row
        vA[s] = 0.0;
      }
    }
  };
  // B -> C, then A -> B with B's V rows issued
  auto advance = [&]() {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      rcC[s] = rcB[s]; vC[s] = vB[s]; vrC[s] = vrB[s]; vcC[s] = vcB[s];
      rcB[s] = rcA[s]; vB[s] = vA[s];
      const bool ok = rcA[s].x >= 0 && lane < k;
      vrB[s] = ok ? __ldg(V + (int64_t)rcA[s].x * ldv + lane) : 0.0;
      vcB[s] = ok ? __ldg(V + (int64_t)rcA[s].y * ldv + lane) : 0.0;
    }
  };
  // the lane's 7 svec slots (a, b) and weights, fixed for the kernel
  int pab[7];
#pragma unroll
  for (int jj = 0; jj < 7; ++jj) pab[jj] = 0;
  // products of one entry into the lane's 7 svec slots; a diagonal entry
  // (row == col) needs two shuffles per slot: (ra cb + ca rb) / 2 = ra rb
  // exactly when a_r == a_c
  auto entry = [&](double a_r, double a_c, bool same, double val, double (&accp)[7]) {
#pragma unroll
    for (int jj = 0; jj < 7; ++jj) {
      const int aa = pab[jj] & 255, bb = pab[jj] >> 8;
      const double wpp = aa == bb ? 1.0 : 1.4142135623730951;
      const double ra = __shfl_sync(0xffffffffu, a_r, aa), rb = __shfl_sync(0xffffffffu, a_r, bb);
      double gg;
      if (same) {
        gg = ra * rb;
      } else {
        const double cb = __shfl_sync(0xffffffffu, a_c, bb), ca = __shfl_sync(0xffffffffu, a_c, aa);
        gg = ra * cb + ca * rb;
      }
      accp[jj] += gg * val * wpp;
    }
  };
  // generate tile tl (stage C) into buf
  auto build = [&](int tl, double* buf) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int r = warp + 16 * s;
      double accp[7];
#pragma unroll
      for (int jj = 0; jj < 7; ++jj) accp[jj] = 0.0;
      if (rcC[s].x >= 0) {
        entry(vrC[s], vcC[s], rcC[s].x == rcC[s].y, vC[s], accp);
      } else if (rcC[s].x == -1) {  // several entries: from the list
        const int64_t i = row_of(tl, s);
        for (int t = cptr[i]; t < cptr[i + 1]; ++t) {
          const int e = cent[t];
          const int rr = erow[e], cc2 = ecol[e];
          const double a_r = lane < k ? V[(int64_t)rr * ldv + lane] : 0.0;
          const double a_c = lane < k ? V[(int64_t)cc2 * ldv + lane] : 0.0;
          entry(a_r, a_c, rr == cc2, eval[e], accp);
        }
      }
#pragma unroll
      for (int jj = 0; jj < 7; ++jj) {
        const int pp = lane + 32 * jj;
        if (pp < d) buf[r * dp + pp] = accp[jj];
      }
    }
  };

  __syncthreads();  // tables
#pragma unroll
  for (int jj = 0; jj < 7; ++jj) {
    const int pp = lane + 32 * jj;
    pab[jj] = pp < d ? (pi[pp] | (pj[pp] << 8)) : 0;
  }
  load_info(0);
  advance();          // B = tile 0
  load_info(1);
  advance();          // C = tile 0, B = tile 1
  load_info(2);
  if (ntile > 0) build(0, tbuf);
  advance();          // C = tile 1, B = tile 2
  load_info(3);
  __syncthreads();
  for (int tl = 0; tl < ntile; ++tl) {
    const double* cur = tbuf + (tl & 1) * CTR * dp;
    double* nxt = tbuf + ((tl + 1) & 1) * CTR * dp;
    // G += T^T T on the current tile (rows beyond the range are zero)
#pragma unroll
    for (int u = 0; u < BPW; ++u) {
      if (bI[u] >= 0) {
        const int ra0 = 16 * bI[u] + g, ra1 = ra0 + 8, rb0 = 16 * bK[u] + g, rb1 = rb0 + 8;
        const bool diagb = bI[u] == bK[u];
#pragma unroll
        for (int ks = 0; ks < CTR / 4; ++ks) {
          const double* row = cur + (4 * ks + q) * dp;
          const double a0 = ra0 < d ? row[ra0] : 0.0, a1 = ra1 < d ? row[ra1] : 0.0;
          const double b0 = rb0 < d ? row[rb0] : 0.0, b1 = rb1 < d ? row[rb1] : 0.0;
          dmma_m8n8k4(acc[u][0][0], acc[u][0][1], a0, b0, acc[u][0][0], acc[u][0][1]);
          dmma_m8n8k4(acc[u][2][0], acc[u][2][1], a1, b0, acc[u][2][0], acc[u][2][1]);
          dmma_m8n8k4(acc[u][3][0], acc[u][3][1], a1, b1, acc[u][3][0], acc[u][3][1]);
          if (!diagb) dmma_m8n8k4(acc[u][1][0], acc[u][1][1], a0, b1, acc[u][1][0], acc[u][1][1]);
        }
      }
    }
    if (tl + 1 < ntile) {
      build(tl + 1, nxt);  // stage C: V rows loaded two intervals ago
      advance();
      load_info(tl + 4);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < BPW; ++u) {
    if (bI[u] < 0) continue;
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int P = 16 * bI[u] + 8 * (x >> 1) + g, Q0 = 16 * bK[u] + 8 * (x & 1) + 2 * q;
      double* out = gpart + (int64_t)blockIdx.x * d * d;
      if (P < d && Q0 < d && Q0 <= P) out[(int64_t)P * d + Q0] = acc[u][x][0];
      if (P < d && Q0 + 1 < d && Q0 + 1 <= P) out[(int64_t)P * d + Q0 + 1] = acc[u][x][1];
    }
  }
}


// sum block partials in fixed order; gram output mirrored to full symmetric
__global__ void k_compressed_final(int nb, int d, const double* __restrict__ gpart, const double* __restrict__ apart,
                                   const double* __restrict__ wpart, double sg, double sa, double sw,
                                   double* __restrict__ G, double* __restrict__ A, double* __restrict__ W) {
  // a warp per output entry (lower triangle of G, then A, then W): the lanes
  // stride over the block partials with their loads in flight together
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t ntri = (int64_t)d * (d + 1) / 2, tot = (int64_t)d * d;
  if (wid < ntri) {
    if (!G) return;
    int P = (int)((sqrt(8.0 * (double)wid + 1.0) - 1.0) * 0.5);
    while ((int64_t)P * (P + 1) / 2 > wid) --P;
    while ((int64_t)(P + 1) * (P + 2) / 2 <= wid) ++P;
    const int Qc = (int)(wid - (int64_t)P * (P + 1) / 2);
    const int64_t x = (int64_t)P * d + Qc;
    double s = 0.0;
    for (int bb = lane; bb < nb; bb += 32) s += gpart[(int64_t)bb * tot + x];
    s = warp_sum(s);
    if (lane == 0) {
      G[(int64_t)P * d + Qc] = sg * s;
      G[(int64_t)Qc * d + P] = sg * s;
    }
  } else if (wid < ntri + 2 * d) {
    const bool isA = wid < ntri + d;
    const int p = (int)(wid - ntri - (isA ? 0 : d));
    const double* part = isA ? apart : wpart;
    double* out = isA ? A : W;
    if (!out) return;
    double s = 0.0;
    for (int bb = lane; bb < nb; bb += 32) s += part[(int64_t)bb * d + p];
    s = warp_sum(s);
    if (lane == 0) out[p] = (isA ? sa : sw) * s;
  }
}

// ------------------------------------------------------------- row GEMM
// Y[i,:] = alpha * X[i,:] B + beta * Y0[i,:]   (B ka x kb in smem)
__global__ void k_rowgemm(int64_t n, const double* __restrict__ X, int64_t ldx, int ka,
                          const double* __restrict__ B, int64_t ldb, int kb, const double* __restrict__ xs,
                          double alpha, double beta, const double* Y0, int64_t ldy0, double* Y, int64_t ldy) {
  // B' = diag(xs) B so that Y = alpha (X diag(xs)) B + beta Y0 (sketch.py:71)
  __shared__ double Bs[64 * 64];
  for (int x = threadIdx.x; x < ka * kb; x += blockDim.x) {
    const int u = x / kb, c = x % kb;
    Bs[x] = B[(int64_t)u * ldb + c];
  }
  __shared__ double xsv[64];
  for (int u = threadIdx.x; u < ka; u += blockDim.x) xsv[u] = xs ? xs[u] : 1.0;
  __syncthreads();
  if (xs) {
    const int64_t tot = n * kb;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = x / kb;
      const int c = (int)(x % kb);
      const double* xr = X + i * ldx;
      double s = 0.0;
      for (int u = 0; u < ka; ++u) s = fma(xr[u] * xsv[u], Bs[u * kb + c], s);
      double v = alpha * s;
      if (Y0) v += beta * Y0[i * ldy0 + c];
      Y[i * ldy + c] = v;
    }
    return;
  }
  const int64_t tot = n * kb;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = x / kb;
    const int c = (int)(x % kb);
    const double* xr = X + i * ldx;
    double s = 0.0;
    for (int u = 0; u < ka; ++u) s = fma(xr[u], Bs[u * kb + c], s);
    double v = alpha * s;
    if (Y0) v += beta * Y0[i * ldy0 + c];
    Y[i * ldy + c] = v;
  }
}

// Row-per-thread form of k_rowgemm for kb <= KBM: a thread keeps its output
// row in registers (every column of X read once per row instead of once per
// output entry); B (ka x kb, scaled by xs) in shared memory, read as
// broadcasts.  Same sums in the same order as k_rowgemm.
template <int KBM>
__global__ void __launch_bounds__(256) k_rowgemm_rt(int64_t n, const double* __restrict__ X, int64_t ldx, int ka,
                                                    const double* __restrict__ B, int64_t ldb, int kb,
                                                    const double* __restrict__ xs, double alpha, double beta,
                                                    const double* Y0, int64_t ldy0, double* Y, int64_t ldy) {
  __shared__ double Bs[64 * KBM];
  __shared__ double xsv[64];
  for (int x = threadIdx.x; x < ka * KBM; x += blockDim.x) {
    const int u = x / KBM, c = x % KBM;
    Bs[x] = c < kb ? B[(int64_t)u * ldb + c] : 0.0;
  }
  for (int u = threadIdx.x; u < ka; u += blockDim.x) xsv[u] = xs ? xs[u] : 1.0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double* xr = X + i * ldx;
    double o[KBM];
#pragma unroll
    for (int c = 0; c < KBM; ++c) o[c] = 0.0;
    for (int u = 0; u < ka; ++u) {
      const double xv = xs ? xr[u] * xsv[u] : xr[u];
      const double* br = Bs + u * KBM;
#pragma unroll
      for (int c = 0; c < KBM; ++c) o[c] = fma(xv, br[c], o[c]);
    }
    double* yr = Y + i * ldy;
    const double* y0r = Y0 ? Y0 + i * ldy0 : nullptr;
#pragma unroll
    for (int c = 0; c < KBM; ++c) {
      if (c < kb) {
        double v = alpha * o[c];
        if (y0r) v += beta * y0r[c];
        yr[c] = v;
      }
    }
  }
}

// sum_i sum_j F[i,j] G[i,j] w[j]  (deterministic two-pass)
__global__ void k_wcoldot_partial(int64_t n, const double* __restrict__ F, int64_t ldf,
                                  const double* __restrict__ G, int64_t ldg, int k,
                                  const double* __restrict__ w, double* __restrict__ part) {
  __shared__ double red[32];
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  double s = 0.0;
  for (int64_t x = r0 * k + threadIdx.x; x < r1 * k; x += blockDim.x) {
    const int64_t i = x / k;
    const int j = (int)(x % k);
    s = fma(F[i * ldf + j] * G[i * ldg + j], w[j], s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_sum_partials(int nb, const double* __restrict__ part, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[b];
    out[0] = s;
  }
}

// X = eta X + F diag(l) F^T  (n x n dense, explicit store)
__global__ void k_dense_update(int64_t n, double* __restrict__ X, double eta, const double* __restrict__ F,
                               int64_t ldf, int kc, const double* __restrict__ l) {
  const int64_t tot = n * n;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = x / n, c = x % n;
    double s = 0.0;
    for (int j = 0; j < kc; ++j) s = fma(F[r * ldf + j] * l[j], F[c * ldf + j], s);
    X[x] = eta * X[x] + s;
  }
}

// ------------------------------------------------------------- vector ops
enum VecOp {
  VOP_W = 0,         // out = y - (b + nu)/rho
  VOP_PROJN = 1,     // out = ineq ? min(z, 0) : 0
  VOP_AXPBY = 2,     // out = a*x + b*y
  VOP_NUNEXT = 3,    // out = projN(ax + rho*y - b); red0 += (out - nu)^2
  VOP_CAND = 4,      // out = y - (b - ax)/rho; ineq: nu<0 -> 0 else max(.,0)
  VOP_RESID = 5,     // diff = ax - projK(ax): red0 += diff^2, red1 = max|diff|
  VOP_DOT = 6,       // red0 += x*y
  VOP_MINI = 7,      // red1 = min over ineq of x  (stored as max of -x)
  VOP_RELU = 8,      // out = max(x, 0)
  VOP_DOTAFF = 9,    // red_out[0] = s0 * sum x*y + s1   (only one slot written)
  VOP_PSIWY = 10,    // red0 += (b + z - x) * y   (psi_value, subqp.py:546-549: w = b + nu - a_x)
  VOP_PSIWW = 11,    // red0 += (b + z - x)^2
};

// x, y, z are operand vectors; red: per-block partials [nb][2]
__global__ void k_vec(int op, int64_t m, const double* __restrict__ x, const double* __restrict__ y,
                      const double* __restrict__ z, const double* __restrict__ b, const double* __restrict__ ineq,
                      double s0, double s1, double* __restrict__ out, double* __restrict__ red) {
  __shared__ double sred[32];
  double r0 = 0.0, r1 = op == VOP_MINI ? -INFINITY : 0.0;
  const int64_t chunk = (m + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = blockIdx.x * chunk, i1 = min(m, i0 + chunk);
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const bool iq = ineq && ineq[i] != 0.0;
    switch (op) {
      case VOP_W: out[i] = x[i] - (b[i] + y[i]) / s0; break;
      case VOP_PROJN: out[i] = iq ? fmin(x[i], 0.0) : 0.0; break;
      case VOP_AXPBY: out[i] = s0 * x[i] + (y ? s1 * y[i] : 0.0); break;
      case VOP_NUNEXT: {
        double t = x[i] + s0 * y[i] - b[i];
        double v = iq ? fmin(t, 0.0) : 0.0;
        out[i] = v;
        double dlt = v - z[i];
        r0 = fma(dlt, dlt, r0);
        break;
      }
      case VOP_CAND: {
        double v = y[i] - (b[i] - x[i]) / s0;
        if (iq) v = (z[i] < 0.0) ? 0.0 : fmax(v, 0.0);
        out[i] = v;
        break;
      }
      case VOP_RESID: {
        double pk = iq ? fmin(x[i], b[i]) : b[i];
        double dlt = x[i] - pk;
        r0 = fma(dlt, dlt, r0);
        r1 = fmax(r1, fabs(dlt));
        break;
      }
      case VOP_DOT:
      case VOP_DOTAFF: r0 = fma(x[i], y[i], r0); break;
      case VOP_PSIWY: r0 = fma(b[i] + z[i] - x[i], y[i], r0); break;  // <b + nu - a_x, y>
      case VOP_PSIWW: {                                             // ||b + nu - a_x||^2
        const double w = b[i] + z[i] - x[i];
        r0 = fma(w, w, r0);
        break;
      }
      case VOP_RELU: out[i] = fmax(x[i], 0.0); break;
      case VOP_MINI:
        if (iq) r1 = fmax(r1, -x[i]);
        break;
    }
  }
  if (red) {
    double t0 = block_sum(r0, sred);
    double t1 = warp_max(r1);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = t1;
    __syncthreads();
    if (threadIdx.x == 0) {
      double mx = op == VOP_MINI ? -INFINITY : 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, sred[w]);
      red[2 * blockIdx.x] = t0;
      red[2 * blockIdx.x + 1] = mx;
    }
  }
}

__global__ void k_vec_final(int nb, const double* __restrict__ red, double* __restrict__ out, int is_min,
                            int affine, double s0, double s1) {
  if (threadIdx.x == 0) {
    double s = 0.0, mx = is_min ? -INFINITY : 0.0;
    for (int b = 0; b < nb; ++b) {
      s += red[2 * b];
      mx = fmax(mx, red[2 * b + 1]);
    }
    if (affine) {
      out[0] = s0 * s + s1;
    } else {
      out[0] = s;
      out[1] = mx;
    }
  }
}

// pivoted Cholesky of a small Gram (c <= 64) with the column-pivoted
// Gram-Schmidt drop rule of symlin.orthonormalize (symlin.py:148-190):
// pick max remaining norm; stop when <= drop_tol * max input column norm.
// Outputs: perm[r] (chosen columns), rank, Rinv (r x r upper, row-major, ld c),
// cond flag = min(selected residual / max norm) for the exact-path guard.
// Block-parallel; every matrix element sees the same operation sequence as
// a serial left-to-right sweep (bit-reproducible, no atomics).
__global__ void __launch_bounds__(256) k_pivchol(int c, const double* __restrict__ G, double drop_tol,
                                                 int* __restrict__ perm, double* __restrict__ Rinv,
                                                 double* __restrict__ info) {
  __shared__ double A[40 * 40];
  __shared__ double R[40 * 40];
  __shared__ double X[40 * 40];
  __shared__ int alive[40];
  __shared__ int sel_s, ok_s;
  __shared__ double bn_s, maxn_s, rjj_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nth = blockDim.x;
  for (int x = tid; x < c * c; x += nth) A[x] = G[x];
  for (int x = tid; x < 40 * 40; x += nth) R[x] = 0.0;
  for (int x = tid; x < c; x += nth) alive[x] = 1;
  __syncthreads();
  if (warp == 0) {
    double mx = 0.0;
    for (int jj = lane; jj < c; jj += 32) mx = fmax(mx, sqrt(fmax(A[jj * c + jj], 0.0)));
    mx = warp_max(mx);
    if (lane == 0) maxn_s = mx;
  }
  __syncthreads();
  const double mx = maxn_s;
  const double thresh = drop_tol < 0.0 ? 0.0 : drop_tol * mx;
  int r = 0;
  double minratio = 1.0;
  if (mx > 0.0) {
    for (int step = 0; step < c; ++step) {
      if (warp == 0) {
        // pivot: largest remaining column norm, first index on ties; natural
        // order (first alive column) without pivoting
        double bn = -1.0;
        int best = 1 << 30;
        for (int jj = lane; jj < c; jj += 32)
          if (alive[jj]) {
            const double nj = sqrt(fmax(A[jj * c + jj], 0.0));
            const bool take = drop_tol < 0.0 ? (jj < best) : (nj > bn || (nj == bn && jj < best));
            if (take) { bn = nj; best = jj; }
          }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, bn, o);
          const int oj = __shfl_xor_sync(0xffffffffu, best, o);
          const bool take = drop_tol < 0.0 ? (oj < best) : (ob > bn || (ob == bn && oj < best));
          if (take) { bn = ob; best = oj; }
        }
        if (lane == 0) {
          sel_s = best < (1 << 30) ? best : -1;
          bn_s = bn;
          if (best < (1 << 30) && !(bn <= thresh)) alive[best] = 0;
        }
      }
      __syncthreads();
      const int best = sel_s;
      const double bn = bn_s;
      if (best < 0 || bn <= thresh) break;
      minratio = fmin(minratio, bn / mx);
      if (tid == 0) perm[r] = best;
      const double rb = sqrt(A[best * c + best]);
      for (int x = tid; x < c * c; x += nth) {
        const int i2 = x / c, jj = x % c;
        if (alive[i2] && alive[jj]) A[i2 * c + jj] -= (A[best * c + i2] / rb) * (A[best * c + jj] / rb);
      }
      ++r;
      __syncthreads();
    }
  }
  __syncthreads();
  // R = chol(G_pp) in pivot order (row-oriented: R[j][b] = (G_pp[j][b] -
  // sum_{q<j} R[q][j] R[q][b]) / R[j][j], q ascending)
  double mr = minratio;
  if (r > 0) {
    for (int x = tid; x < r * r; x += nth) {
      const int a2 = x / r, b2 = x % r;
      A[a2 * 40 + b2] = G[perm[a2] * c + perm[b2]];
    }
    if (tid == 0) ok_s = 1;
    __syncthreads();
    for (int j = 0; j < r; ++j) {
      if (tid == 0) {
        double s = A[j * 40 + j];
        for (int q = 0; q < j; ++q) s -= R[q * 40 + j] * R[q * 40 + j];
        if (!(s > 0.0)) ok_s = 0;
        rjj_s = sqrt(s);
        if (s > 0.0) R[j * 40 + j] = rjj_s;
      }
      __syncthreads();
      if (!ok_s) break;
      const double rjj = rjj_s;
      for (int b2 = j + 1 + tid; b2 < r; b2 += nth) {
        double t = A[j * 40 + b2];
        for (int q = 0; q < j; ++q) t -= R[q * 40 + j] * R[q * 40 + b2];
        R[j * 40 + b2] = t / rjj;
      }
      __syncthreads();
    }
    if (!ok_s) mr = 0.0;
    // Rinv (upper) by back substitution, one thread per column
    for (int col = tid; col < r; col += nth)
      for (int row = r - 1; row >= 0; --row) {
        double s = (row == col) ? 1.0 : 0.0;
        for (int q = row + 1; q < r; ++q) s -= R[row * 40 + q] * X[q * 40 + col];
        X[row * 40 + col] = (row <= col) ? s / R[row * 40 + row] : 0.0;
      }
    __syncthreads();
    // r x r upper inverse, zero elsewhere (callers may reuse the buffer)
    for (int x = tid; x < c * c; x += nth) {
      const int i = x / c, j = x % c;
      Rinv[x] = (i < r && j < r) ? X[i * 40 + j] : 0.0;
    }
  }
  if (tid == 0) {
    info[0] = r;
    info[1] = mr;
    info[2] = mx;
  }
}

// ---------------------------------------------------------- cut rounding
// maxcut_round (rounding.py:34-51): x = sign(U[:, j]) (zero -> +1) and
// 0.25 x^T L x = sum_e w_e [x_u != x_v] (each undirected edge counted once:
// x^T L x = sum_e w_e (x_u - x_v)^2).  Exact for integer weights, so the
// value equals the reference's bit for bit in that case.
__global__ void k_cut_partial(int64_t ne, const int* __restrict__ eu, const int* __restrict__ ev,
                              const double* __restrict__ ew, const double* __restrict__ U, int64_t ldu,
                              double* __restrict__ part) {
  __shared__ double red[32];
  const int j = blockIdx.y;
  double acc = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    const bool su = U[(int64_t)eu[e] * ldu + j] >= 0.0, sv = U[(int64_t)ev[e] * ldu + j] >= 0.0;
    if (su != sv) acc += ew[e];
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) part[(int64_t)j * gridDim.x + blockIdx.x] = acc;
}

__global__ void k_cut_final(int nb, int r, const double* __restrict__ part, double* __restrict__ vals,
                            int* __restrict__ best) {
  __shared__ double v[64];
  for (int j = threadIdx.x; j < r; j += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[(int64_t)j * nb + b];
    v[j] = s;
    vals[j] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int bj = 0;
    for (int j = 1; j < r; ++j)
      if (v[j] > v[bj]) bj = j;  // first maximum, as the reference's strict '>'
    best[0] = bj;
  }
}

__global__ void k_cut_assign(int64_t n, const double* __restrict__ U, int64_t ldu, const int* __restrict__ best,
                             int* __restrict__ x) {
  const int j = best[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = U[i * ldu + j] >= 0.0 ? 1 : -1;
}

__global__ void k_gather(int64_t n, const int64_t* __restrict__ idx, const double* __restrict__ src,
                         double* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

// dst[i, :k] = src[idx[i], :k] (row-major), a zero row where idx[i] < 0:
// the embedding scatter of warm_start_pad (bundle.py:781-792) as a gather
// through the inverse map
__global__ void k_gather_rows(int64_t n, int k, const int64_t* __restrict__ idx, const double* __restrict__ src,
                              int64_t lds, double* __restrict__ dst, int64_t ldd) {
  const int64_t tot = n * k;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = x / k;
    const int j = (int)(x - i * k);
    const int64_t s = idx[i];
    dst[i * ldd + j] = s >= 0 ? src[s * lds + j] : 0.0;
  }
}

// orthonormalize's first CholQR factor: B[perm[i], j] = Rinv[i, j] for
// i, j < r (r = info[0], the pivoted Cholesky rank), zero elsewhere
__global__ void k_perm_rows(int c, const int* __restrict__ perm, const double* __restrict__ rinv,
                            const double* __restrict__ info, double* __restrict__ out) {
  const int r = (int)info[0];
  for (int x = threadIdx.x; x < c * c; x += blockDim.x) out[x] = 0.0;
  __syncthreads();
  for (int x = threadIdx.x; x < c * c; x += blockDim.x) {
    const int i = x / c, j = x % c;
    if (i < r && j < r) out[perm[i] * c + j] = rinv[i * c + j];
  }
}

// --------------------------------------------- constraint-bundle surface
// primal_image_dense (problem.py:157-158, 210-212): sum over constraint i's
// entries of (2 - [r == c]) val X[r, c]; diagonal family: X[i, i]
__global__ void __launch_bounds__(256) k_image_dense(int64_t m, int diag_only, const int* __restrict__ cptr,
                                                     const int* __restrict__ cent, const int* __restrict__ erow,
                                                     const int* __restrict__ ecol, const double* __restrict__ eval,
                                                     const double* __restrict__ X, int64_t ldx,
                                                     double* __restrict__ out) {
  const int lane = threadIdx.x & 31, gw = lane >> 3, t = lane & 7;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t wb = wid * 4; wb < m; wb += nwarps * 4) {
    const int64_t i = wb + gw;
    double acc = 0.0;
    if (i < m) {
      if (diag_only) {
        if (t == 0) acc = X[i * ldx + i];
      } else {
        for (int q = cptr[i] + t; q < cptr[i + 1]; q += 8) {
          const int e = cent[q];
          const int r = erow[e], c = ecol[e];
          acc = fma(X[(int64_t)r * ldx + c], (r == c) ? eval[e] : 2.0 * eval[e], acc);
        }
      }
    }
#pragma unroll
    for (int o = 4; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, 8);
    if (i < m && t == 0) out[i] = acc;
  }
}

// compressed_rows (problem.py:169-173, 229-239): row i = svec(V^T A_i V),
// column-major lower-triangle order with sqrt(2) off the diagonal
__global__ void k_compressed_rows(int64_t m, int diag_only, const int* __restrict__ cptr,
                                  const int* __restrict__ cent, const int* __restrict__ erow,
                                  const int* __restrict__ ecol, const double* __restrict__ eval,
                                  const double* __restrict__ V, int64_t ldv, int k, double* __restrict__ out,
                                  int64_t ldo) {
  const int d = k * (k + 1) / 2;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < m * d; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = x / d;
    int rem = (int)(x % d), j = 0;
    while (rem >= k - j) { rem -= k - j; ++j; }
    const int a = j + rem, bcol = j;  // svec position -> (row a, column b), a >= b
    out[i * ldo + (x % d)] = crow_entry(diag_only, i, a, bcol, a == bcol ? 1.0 : 1.4142135623730951, cptr, cent,
                                        erow, ecol, eval, V, ldv);
  }
}

}  // namespace usbs

using namespace usbs;

static int nblocks(usbs_ctx* ctx, int64_t work, int per = 256, int mult = 8) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((work + per - 1) / per, (int64_t)mult * ctx->num_sms));
}

// the flattened single-entry view of the constraint list (lazy, once)
static void ensure_c1(usbs_ctx* ctx, usbs_problem* p) {
  if (p->c1_rc) return;
  p->c1_rc = dev_alloc<int2>(p, (size_t)p->m);
  p->c1_val = dev_alloc<double>(p, (size_t)p->m);
  if (p->max_entries_per_cons > IMAGE_HEAVY) {
    p->c1_heavy = dev_alloc<int>(p, (size_t)p->m + 1);
    USBS_CUDA(cudaMemsetAsync(p->c1_heavy, 0, sizeof(int), ctx->stream));
  }
  k_c1_flatten<<<nblocks(ctx, p->m), 256, 0, ctx->stream>>>(p->m, p->cptr, p->cent, p->e_row, p->e_col, p->e_val,
                                                            p->c1_rc, p->c1_val, p->c1_heavy);
  check_launch(ctx);
}

extern "C" {

usbs_status usbs_cons_image(usbs_ctx* ctx, usbs_problem* p, const double* V, int64_t ldv, int k, const double* S,
                            int s_is_diag, double s_scale, const double* beta_dev, double beta, const double* base,
                            double* out) {
  USBS_API_BEGIN
  if (k < 1 || k > 64) fail(USBS_ERR_SHAPE, "cons_image: 1 <= k <= 64");
  if (p->diag_only) {
    const size_t smi = (size_t)(k * k + 256 * (k | 1)) * sizeof(double);
    smem_optin(ctx, (const void*)k_image_diag, (int)smi);
    const int bl = (int)std::max<int64_t>(1, std::min<int64_t>((p->n + 255) / 256, 8 * ctx->num_sms));
    k_image_diag<<<bl, 256, smi, ctx->stream>>>(p->n, V, ldv, k, S, s_is_diag, s_scale, beta_dev, beta, base, out);
  } else {
    const double* W = nullptr;
    if (!s_is_diag) {
      if (k * k > 4096) fail(USBS_ERR_SHAPE, "cons_image: k too large for a dense S");
      const int64_t nv = std::max<int64_t>(p->n, p->n_cols);
      double* Wb = (double*)ctx->ws.get(WS_BOOK_W, (size_t)nv * k * sizeof(double));
      k_rowgemm<<<nblocks(ctx, nv * k), 256, 0, ctx->stream>>>(nv, V, ldv, k, S, k, k, nullptr, s_scale, 0.0,
                                                               nullptr, 0, Wb, k);
      check_launch(ctx);
      W = Wb;
    }
    const char* ev1 = getenv("USBS_IMAGE_V1");
    if (!(ev1 && ev1[0] == '1')) {  // A/B: USBS_IMAGE_V1=1 -> eight lanes over each constraint's entry list
      ensure_c1(ctx, p);
      k_image_c1<<<nblocks(ctx, (p->m + 7) / 8 * 32), 256, 0, ctx->stream>>>(
          p->m, p->c1_rc, p->c1_val, p->c1_heavy, p->cptr, p->cent, p->e_row, p->e_col, p->e_val, V, ldv, W, k, k, S, s_is_diag,
          s_scale, beta_dev, beta, base, out);
    } else {
      k_image_entries<<<nblocks(ctx, (p->m + 3) / 4 * 32), 256, 0, ctx->stream>>>(
          p->m, p->cptr, p->cent, p->e_row, p->e_col, p->e_val, V, ldv, W, k, k, S, s_is_diag, s_scale, beta_dev,
          beta, base, out);
    }
  }
  check_launch(ctx);
  USBS_API_END
}


__global__ void k_svec(int k, const double* __restrict__ A, double scale, double* __restrict__ out);

usbs_status usbs_cons_compressed(usbs_ctx* ctx, usbs_problem* p, const double* V, int64_t ldv, int k,
                                 double scale_gram, double* gram_out, const double* a_vec, double scale_a,
                                 double* a_out, const double* w_vec, double scale_w, double* w_out) {
  USBS_API_BEGIN
  if (k < 1 || k > 32) fail(USBS_ERR_SHAPE, "cons_compressed: 1 <= k <= 32");
  if (!p->diag_only && p->n_cols == p->n && (a_vec || w_vec)) {
    // sum_i v_i c_i = svec(V^T A*(v) V): assemble A*(v) on the merged
    // pattern, one SpMM and one Gram (O(E + nnz k + n k^2) instead of the
    // O(E d) row-by-row generation); the d x d Gram below needs the rows
    double* tval = (double*)ctx->ws.get(WS_BOOK_T, (size_t)p->nnz * sizeof(double));
    double* Y = (double*)ctx->ws.get(WS_BOOK_W, (size_t)p->n * k * sizeof(double));
    double* G = (double*)ctx->ws.get(WS_BOOK_G, (size_t)k * k * sizeof(double));
    for (int u = 0; u < 2; ++u) {
      const double* vec = u ? w_vec : a_vec;
      if (!vec) continue;
      launch_adjoint_values(ctx, p, vec, tval);
      launch_spmm_vals(ctx, p, tval, V, ldv, k, Y, k);
      launch_gram_tn(ctx, p->n, V, ldv, k, Y, k, k, G, true);
      k_svec<<<1, 256, 0, ctx->stream>>>(k, G, u ? scale_w : scale_a, u ? w_out : a_out);
      check_launch(ctx);
    }
    a_vec = nullptr;
    w_vec = nullptr;
    if (!gram_out) return USBS_OK;
  }
  if (p->diag_only && p->n >= 1024 && (a_vec || w_vec) && ((uintptr_t)V & 15) == 0 && ldv <= 128) {
    // diagonal constraints: sum_i v_i svec(v_i v_i^T) = svec(V^T diag(v) V),
    // a row-weighted Gram on the TMA Gram kernel (O(n k^2), memory-bound)
    double* G = (double*)ctx->ws.get(WS_BOOK_G, (size_t)k * k * sizeof(double));
    for (int u = 0; u < 2; ++u) {
      const double* vec = u ? w_vec : a_vec;
      if (!vec) continue;
      launch_gram_tn(ctx, p->n, V, ldv, k, V, ldv, k, G, true, vec);
      k_svec<<<1, 256, 0, ctx->stream>>>(k, G, u ? scale_w : scale_a, u ? w_out : a_out);
      check_launch(ctx);
    }
    a_vec = nullptr;
    w_vec = nullptr;
    if (!gram_out) return USBS_OK;
  }
  const int d = k * (k + 1) / 2;
  const int nt = (d + 3) / 4, ntiles = nt * (nt + 1) / 2;
  const int tpt = gram_out ? (ntiles + 255) / 256 : 1;
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms, (p->m + 63) / 64));
  const size_t gbytes = gram_out ? (size_t)nb * d * d * sizeof(double) : 0;
  double* ws = (double*)ctx->ws.get(WS_BOOK, gbytes + (size_t)2 * nb * d * sizeof(double) + 64);
  double* gpart = gram_out ? ws : nullptr;
  double* apart = a_vec ? ws + (gram_out ? (size_t)nb * d * d : 0) : nullptr;
  double* wpart = w_vec ? ws + (gram_out ? (size_t)nb * d * d : 0) + (size_t)nb * d : nullptr;
  const size_t sm = (size_t)(CTR * (d + 1) + 2 * CTR) * sizeof(double) + 1200;
  const int dg = gram_out ? 1 : 0;
#define USBS_COMP(T)                                                                                      \
  {                                                                                                       \
    smem_optin(ctx, (const void*)k_compressed<T>, 200 * 1024);                                            \
    k_compressed<T><<<nb, 256, sm, ctx->stream>>>(p->m, p->diag_only ? 1 : 0, p->cptr, p->cent, p->e_row,  \
                                                  p->e_col, p->e_val, V, ldv, k, d, a_vec, w_vec, dg, gpart, \
                                                  apart, wpart);                                          \
  }
  const int n8 = (d + 7) / 8, nt8 = n8 * (n8 + 1) / 2;
  const char* emma = getenv("USBS_COMPRESSED_MMA");
  const char* eruns = getenv("USBS_K4_RUNS");
  const int runs = (eruns && eruns[0] == '1') ? 1 : 0;  // contiguous runs measured slower (profiles/k4_time.py)
  if (gram_out && nt8 <= 16 * 24 && !(emma && emma[0] == '0')) {
    // tensor-core Gram (d <= 216)
    const size_t smm = (size_t)(CTR * (d + 1 + ((8 - (d + 1)) & 15)) + 2 * CTR) * sizeof(double) + 1200 + 2 * nt8 + 16;
#define USBS_COMP_MMA(T, HY)                                                                               \
  {                                                                                                        \
    smem_optin(ctx, (const void*)k_compressed_mma<T>, 200 * 1024);                                         \
    k_compressed_mma<T><<<dim3(nb, HY), 512, smm, ctx->stream>>>(p->m, p->diag_only ? 1 : 0, p->cptr, p->cent, p->e_row, \
                                                       p->e_col, p->e_val, V, ldv, k, d, a_vec, w_vec, gpart, \
                                                       apart, wpart, runs);                                \
  }
    const char* ev1 = getenv("USBS_K4_V1");
    if (!a_vec && !w_vec && !(ev1 && ev1[0] == '1')) {
      // pipelined row generation (A/B: USBS_K4_V1=1)
      if (!p->diag_only) ensure_c1(ctx, p);
      const size_t smp = (size_t)(2 * CTR * (d + 1 + ((8 - (d + 1)) & 15))) * sizeof(double) + 1200 + 16;
      const int n16 = (d + 15) / 16, nb16 = n16 * (n16 + 1) / 2;
#define USBS_COMP_PIPE(T, HY)                                                                              \
  {                                                                                                        \
    smem_optin(ctx, (const void*)k_compressed_mma_pipe<T>, 200 * 1024);                                    \
    k_compressed_mma_pipe<T><<<dim3(nb, HY), 512, smp, ctx->stream>>>(                                     \
        p->m, p->diag_only ? 1 : 0, p->c1_rc, p->c1_val, p->cptr, p->cent, p->e_row, p->e_col, p->e_val, V, \
        ldv, k, d, gpart);                                                                                 \
  }
      if (nb16 <= 16) USBS_COMP_PIPE(1, 1)
      else if (nb16 <= 32) USBS_COMP_PIPE(2, 1)
      else if (nb16 <= 64) USBS_COMP_PIPE(2, 2)
      else USBS_COMP_PIPE(4, 2)  // d = 210: 105 blocks over two CTAs per row range (four: 7% slower)
#undef USBS_COMP_PIPE
    } else {
    if (nt8 <= 16 * 3) USBS_COMP_MMA(3, 1)
    else if (nt8 <= 16 * 8) USBS_COMP_MMA(8, 1)
    else USBS_COMP_MMA(12, 2)  // the tiles split over two CTAs per row range: 24 accumulators a lane, no spill
    }
#undef USBS_COMP_MMA
  } else if (tpt <= 1) USBS_COMP(1)
  else if (tpt <= 2) USBS_COMP(2)
  else if (tpt <= 4) USBS_COMP(4)
  else if (tpt <= 6) USBS_COMP(6)
  else if (tpt <= 8) USBS_COMP(8)
  else fail(USBS_ERR_SHAPE, "cons_compressed: d too large");
#undef USBS_COMP
  check_launch(ctx);
  k_compressed_final<<<(int)(((int64_t)d * (d + 1) / 2 + 2 * d + 7) / 8), 256, 0, ctx->stream>>>(
      nb, d, gpart, apart, wpart, scale_gram, scale_a, scale_w, gram_out, a_vec ? a_out : nullptr,
      w_vec ? w_out : nullptr);
  check_launch(ctx);
  USBS_API_END
}

usbs_status usbs_rowgemm(usbs_ctx* ctx, int64_t n, const double* X, int64_t ldx, int ka, const double* B,
                         int64_t ldb, int kb, const double* xs, double alpha, double beta, const double* Y0,
                         int64_t ldy0, double* Y, int64_t ldy) {
  USBS_API_BEGIN
  if (ka < 1 || kb < 1 || ka > 64 || ka * kb > 4096) fail(USBS_ERR_SHAPE, "rowgemm: ka <= 64, ka*kb <= 4096");
  const char* ev = getenv("USBS_ROWGEMM_V1");
  if (kb <= 32 && !(ev && ev[0] == '1')) {
    // a thread per output row (A/B: USBS_ROWGEMM_V1=1 -> a thread per entry)
    const int bl = nblocks(ctx, n);
    if (kb <= 4) k_rowgemm_rt<4><<<bl, 256, 0, ctx->stream>>>(n, X, ldx, ka, B, ldb, kb, xs, alpha, beta, Y0, ldy0, Y, ldy);
    else if (kb <= 8) k_rowgemm_rt<8><<<bl, 256, 0, ctx->stream>>>(n, X, ldx, ka, B, ldb, kb, xs, alpha, beta, Y0, ldy0, Y, ldy);
    else if (kb <= 12) k_rowgemm_rt<12><<<bl, 256, 0, ctx->stream>>>(n, X, ldx, ka, B, ldb, kb, xs, alpha, beta, Y0, ldy0, Y, ldy);
    else if (kb <= 16) k_rowgemm_rt<16><<<bl, 256, 0, ctx->stream>>>(n, X, ldx, ka, B, ldb, kb, xs, alpha, beta, Y0, ldy0, Y, ldy);
    else if (kb <= 24) k_rowgemm_rt<24><<<bl, 256, 0, ctx->stream>>>(n, X, ldx, ka, B, ldb, kb, xs, alpha, beta, Y0, ldy0, Y, ldy);
    else k_rowgemm_rt<32><<<bl, 256, 0, ctx->stream>>>(n, X, ldx, ka, B, ldb, kb, xs, alpha, beta, Y0, ldy0, Y, ldy);
  } else {
    k_rowgemm<<<nblocks(ctx, n * kb), 256, 0, ctx->stream>>>(n, X, ldx, ka, B, ldb, kb, xs, alpha, beta, Y0, ldy0, Y,
                                                             ldy);
  }
  check_launch(ctx);
  USBS_API_END
}

usbs_status usbs_gram(usbs_ctx* ctx, int64_t n, const double* A, int64_t lda, int ka, const double* B, int64_t ldb,
                      int kb, double* out, int sym) {
  USBS_API_BEGIN
  launch_gram_tn(ctx, n, A, lda, ka, B, ldb, kb, out, sym != 0);
  USBS_API_END
}

usbs_status usbs_wcoldot(usbs_ctx* ctx, int64_t n, const double* F, int64_t ldf, const double* G, int64_t ldg, int k,
                         const double* w, double* out) {
  USBS_API_BEGIN
  int nb = (int)std::min<int64_t>(2 * ctx->num_sms, std::max<int64_t>(1, (n * k + 2047) / 2048));
  double* part = (double*)ctx->ws.get(WS_RED, (size_t)nb * sizeof(double));
  k_wcoldot_partial<<<nb, 256, 0, ctx->stream>>>(n, F, ldf, G, ldg, k, w, part);
  check_launch(ctx);
  k_sum_partials<<<1, 32, 0, ctx->stream>>>(nb, part, out);
  check_launch(ctx);
  USBS_API_END
}

usbs_status usbs_dense_update(usbs_ctx* ctx, int64_t n, double* X, double eta, const double* F, int64_t ldf, int kc,
                              const double* lams) {
  USBS_API_BEGIN
  k_dense_update<<<nblocks(ctx, n * n), 256, 0, ctx->stream>>>(n, X, eta, F, ldf, kc, lams);
  check_launch(ctx);
  USBS_API_END
}

usbs_status usbs_vec(usbs_ctx* ctx, int op, int64_t m, const double* x, const double* y, const double* z,
                     const double* b, const double* ineq, double s0, double s1, double* out, double* red_out) {
  USBS_API_BEGIN
  int nb = (int)std::min<int64_t>(2 * ctx->num_sms, std::max<int64_t>(1, (m + 2047) / 2048));
  double* red = red_out ? (double*)ctx->ws.get(WS_RED + 1, (size_t)2 * nb * sizeof(double)) : nullptr;
  k_vec<<<nb, 256, 0, ctx->stream>>>(op, m, x, y, z, b, ineq, s0, s1, out, red);
  check_launch(ctx);
  if (red_out) {
    k_vec_final<<<1, 32, 0, ctx->stream>>>(nb, red, red_out, op == VOP_MINI ? 1 : 0, op == VOP_DOTAFF ? 1 : 0, s0,
                                           s1);
    check_launch(ctx);
  }
  USBS_API_END
}

__global__ void k_svec(int k, const double* __restrict__ A, double scale, double* __restrict__ out) {
  // column-major lower triangle, sqrt(2) off the diagonal (symlin.py:57-79)
  const int d = k * (k + 1) / 2;
  for (int p = threadIdx.x; p < d; p += blockDim.x) {
    int j = 0, rem = p;
    while (rem >= k - j) { rem -= k - j; ++j; }
    const int i = j + rem;
    out[p] = scale * (A[i * k + j] * (i == j ? 1.0 : 1.4142135623730951));
  }
}

usbs_status usbs_svec(usbs_ctx* ctx, int k, const double* A, double scale, double* out) {
  USBS_API_BEGIN
  if (k < 1 || k > 64) fail(USBS_ERR_SHAPE, "svec: 1 <= k <= 64");
  k_svec<<<1, 256, 0, ctx->stream>>>(k, A, scale, out);
  check_launch(ctx);
  USBS_API_END
}

usbs_status usbs_pivchol(usbs_ctx* ctx, int c, const double* G, double drop_tol, int* perm, double* Rinv,
                         double* info) {
  USBS_API_BEGIN
  if (c < 1 || c > 40) fail(USBS_ERR_SHAPE, "pivchol: 1 <= c <= 40");
  k_pivchol<<<1, 256, 0, ctx->stream>>>(c, G, drop_tol, perm, Rinv, info);
  check_launch(ctx);
  USBS_API_END
}

usbs_status usbs_maxcut_round(usbs_ctx* ctx, int64_t n, int64_t ne, const int32_t* eu, const int32_t* ev,
                              const double* ew, const double* U, int64_t ldu, int r, double* vals, int* best,
                              int32_t* x) {
  USBS_API_BEGIN
  if (n < 1 || r < 1 || r > 64 || ldu < r) fail(USBS_ERR_SHAPE, "factor must be a nonempty n x r matrix, r <= 64");
  const int nbx = (int)std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms, (ne + 255) / 256));
  double* part = (double*)ctx->ws.get(WS_RED + 50, (size_t)nbx * r * sizeof(double) + 64 * sizeof(double) + 64);
  double* dv = part + (size_t)nbx * r;
  int* db = (int*)(dv + 64);
  k_cut_partial<<<dim3(nbx, r), 256, 0, ctx->stream>>>(ne, eu, ev, ew, U, ldu, part);
  check_launch(ctx);
  k_cut_final<<<1, 64, 0, ctx->stream>>>(nbx, r, part, dv, db);
  check_launch(ctx);
  k_cut_assign<<<nblocks(ctx, n), 256, 0, ctx->stream>>>(n, U, ldu, db, x);
  check_launch(ctx);
  USBS_CUDA(cudaMemcpyAsync(ctx->pinned, dv, r * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  USBS_CUDA(cudaMemcpyAsync(ctx->pinned_i, db, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  USBS_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int j = 0; j < r; ++j) vals[j] = ctx->pinned[j];
  *best = ctx->pinned_i[0];
  USBS_API_END
}

usbs_status usbs_gather(usbs_ctx* ctx, int64_t n, const int64_t* idx, const double* src, double* dst) {
  USBS_API_BEGIN
  if (n < 0) fail(USBS_ERR_SHAPE, "gather: n < 0");
  if (n > 0) {
    k_gather<<<nblocks(ctx, n), 256, 0, ctx->stream>>>(n, idx, src, dst);
    check_launch(ctx);
  }
  USBS_API_END
}

usbs_status usbs_gather_rows(usbs_ctx* ctx, int64_t n, int k, const int64_t* idx, const double* src, int64_t lds,
                             double* dst, int64_t ldd) {
  USBS_API_BEGIN
  if (n < 0 || k < 1 || lds < k || ldd < k) fail(USBS_ERR_SHAPE, "gather_rows: n >= 0, k >= 1, ld >= k");
  if (n > 0) {
    k_gather_rows<<<nblocks(ctx, n * k), 256, 0, ctx->stream>>>(n, k, idx, src, lds, dst, ldd);
    check_launch(ctx);
  }
  USBS_API_END
}

usbs_status usbs_perm_rows(usbs_ctx* ctx, int c, const int32_t* perm, const double* rinv, const double* info,
                           double* out) {
  USBS_API_BEGIN
  if (c < 1 || c > 64) fail(USBS_ERR_SHAPE, "perm_rows: 1 <= c <= 64");
  k_perm_rows<<<1, 256, 0, ctx->stream>>>(c, perm, rinv, info, out);
  check_launch(ctx);
  USBS_API_END
}

usbs_status usbs_cons_adjoint_apply(usbs_ctx* ctx, usbs_problem* p, const double* y, const double* V, int64_t ldv,
                                    int k, double* Y, int64_t ldy, double* gram) {
  USBS_API_BEGIN
  if (p->n_cols != p->n) fail(USBS_ERR_SHAPE, "cons_adjoint_apply needs an unsharded problem");
  if (k < 1 || ldv < k || ldy < k) fail(USBS_ERR_SHAPE, "cons_adjoint_apply: bad k / leading dimension");
  double* tval = (double*)ctx->ws.get(WS_BOOK_T, (size_t)p->nnz * sizeof(double));
  launch_adjoint_values(ctx, p, y, tval);
  launch_spmm_vals(ctx, p, tval, V, ldv, k, Y, ldy);
  if (gram) launch_gram_tn(ctx, p->n, V, ldv, k, Y, ldy, k, gram, true);
  USBS_API_END
}

usbs_status usbs_cons_adjoint_values(usbs_ctx* ctx, usbs_problem* p, const double* y, double* vals) {
  USBS_API_BEGIN
  launch_adjoint_values(ctx, p, y, vals);
  USBS_API_END
}

usbs_status usbs_problem_pattern(usbs_problem* p, int64_t* rowptr, int32_t* col, int32_t* nent) {
  USBS_API_BEGIN
  ensure_slot_lists(p->ctx, p);
  USBS_CUDA(cudaStreamSynchronize(p->ctx->stream));
  std::vector<int32_t> rp(p->n + 1), ap(p->nnz + 1);
  USBS_CUDA(cudaMemcpy(rp.data(), p->rowptr, (p->n + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost));
  USBS_CUDA(cudaMemcpy(col, p->col, p->nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
  USBS_CUDA(cudaMemcpy(ap.data(), p->aptr, (p->nnz + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i <= p->n; ++i) rowptr[i] = rp[i];
  for (int64_t s = 0; s < p->nnz; ++s) nent[s] = ap[s + 1] - ap[s];
  USBS_API_END
}

usbs_status usbs_cons_image_dense(usbs_ctx* ctx, usbs_problem* p, const double* X, int64_t ldx, double* out) {
  USBS_API_BEGIN
  if (p->n_cols != p->n) fail(USBS_ERR_SHAPE, "cons_image_dense needs an unsharded problem");
  k_image_dense<<<nblocks(ctx, (p->m + 3) / 4 * 32), 256, 0, ctx->stream>>>(
      p->m, p->diag_only ? 1 : 0, p->cptr, p->cent, p->e_row, p->e_col, p->e_val, X, ldx, out);
  check_launch(ctx);
  USBS_API_END
}

usbs_status usbs_cons_compressed_rows(usbs_ctx* ctx, usbs_problem* p, const double* V, int64_t ldv, int k,
                                      double* out, int64_t ldo) {
  USBS_API_BEGIN
  if (k < 1 || k > 64 || ldo < k * (k + 1) / 2) fail(USBS_ERR_SHAPE, "cons_compressed_rows: bad k / ldo");
  const int64_t tot = p->m * (int64_t)(k * (k + 1) / 2);
  k_compressed_rows<<<nblocks(ctx, tot), 256, 0, ctx->stream>>>(p->m, p->diag_only ? 1 : 0, p->cptr, p->cent,
                                                                p->e_row, p->e_col, p->e_val, V, ldv, k, out, ldo);
  check_launch(ctx);
  USBS_API_END
}

}  // extern "C"
