// Tall-skinny dense kernels on row-major n x k blocks (k <= 64):
//   gram_tn: out = A^T B (optionally symmetrised 0.5 (G + G^T)), two-pass
//            deterministic reduction (per-block partials, fixed-order sum).
//   dot:     deterministic x . y.
// Used for V^T (M V) Grams (problem.py:284-286, 166-167/225-227,
// subqp.py:459), F^T Psi of the sketch update (sketch.py:71) and the
// orthonormalisation Grams.
#include <algorithm>

#include "usbs_common.cuh"
#include "usbs_kernels.cuh"
#include "usbs_tma.cuh"

namespace usbs {

constexpr int GRAM_TR = 32;  // rows per smem tile

// grid: nb blocks, each over a contiguous chunk of rows; 256 threads; each
// thread owns output pairs p = tid, tid + 256, ... < ka * kb
__global__ void __launch_bounds__(256) k_gram_partial(int64_t n, const double* __restrict__ A, int64_t lda, int ka,
                                                      const double* __restrict__ B, int64_t ldb, int kb,
                                                      double* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sa = (double*)smem_raw;  // GRAM_TR * ka
  double* sb = sa + GRAM_TR * ka;  // GRAM_TR * kb
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  const int npair = ka * kb;
  constexpr int MAXP = 16;  // 64*64/256
  double acc[MAXP];
#pragma unroll
  for (int u = 0; u < MAXP; ++u) acc[u] = 0.0;
  for (int64_t base = r0; base < r1; base += GRAM_TR) {
    const int rows = (int)((r1 - base) < GRAM_TR ? (r1 - base) : GRAM_TR);
    __syncthreads();
    for (int x = threadIdx.x; x < rows * ka; x += blockDim.x) {
      int r = x / ka, c = x % ka;
      sa[r * ka + c] = A[(base + r) * lda + c];
    }
    for (int x = threadIdx.x; x < rows * kb; x += blockDim.x) {
      int r = x / kb, c = x % kb;
      sb[r * kb + c] = B[(base + r) * ldb + c];
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < MAXP; ++u) {
      const int p = threadIdx.x + u * 256;
      if (p < npair) {
        const int ia = p / kb, ib = p % kb;
        double s = acc[u];
        for (int r = 0; r < rows; ++r) s = fma(sa[r * ka + ia], sb[r * kb + ib], s);
        acc[u] = s;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < MAXP; ++u) {
    const int p = threadIdx.x + u * 256;
    if (p < npair) part[(int64_t)blockIdx.x * npair + p] = acc[u];
  }
}

// a warp per output entry: lanes stride over the block partials (fixed
// order), then a warp reduction; the symmetric variant averages the entry
// with its transpose
__global__ void k_gram_final(int nb, int ka, int kb, const double* __restrict__ part, double* __restrict__ out,
                             int sym) {
  const int npair = ka * kb;
  const int lane = threadIdx.x & 31;
  const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= npair) return;
  const int ia = p / kb, ib = p % kb;
  const int pt = ib * kb + ia;
  double s = 0.0, st = 0.0;
  for (int b = lane; b < nb; b += 32) {
    s += part[(int64_t)b * npair + p];
    if (sym) st += part[(int64_t)b * npair + pt];
  }
  s = warp_sum(s);
  if (sym) st = warp_sum(st);
  if (lane == 0) out[p] = sym ? 0.5 * (s + st) : s;
}

// TMA-fed Gram for 16-byte-aligned row-major operands: a block streams its
// row chunk in tiles of R rows through GB_S shared-memory stages (one
// cp.async.bulk per operand per tile -- rows of a row-major block are one
// contiguous range whatever the column count used -- completing on the
// stage's mbarrier); 256 threads own 4 x 4 output blocks of A^T B for a
// subset of rows each (register blocking: 16 FMAs per 8 shared loads); the
// row groups are summed in fixed order at the end, then the blocks
// (k_gram_final).  Memory-bound: (ka + kb) 8 bytes per row.
constexpr int GB_S = 3;
constexpr int GB_THREADS = 256;

__global__ void __launch_bounds__(GB_THREADS, 2) k_gram_bulk(int64_t n, const double* __restrict__ A, int64_t lda,
                                                          int ka, const double* __restrict__ B, int64_t ldb, int kb,
                                                          int R, int64_t rows_per_block, double* __restrict__ part,
                                                          const double* __restrict__ rw) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block, r1 = min(n, r0 + rows_per_block);
  const int stA = R * (int)lda, stB = R * (int)ldb;
  const int stride = (stA + stB + 1) & ~1;
  double* st = (double*)smem_raw;
  uint64_t* bar = (uint64_t*)(st + GB_S * stride);
  const int tid = threadIdx.x;
  const int nt = r1 > r0 ? (int)((r1 - r0 + R - 1) / R) : 0;
  if (tid == 0) {
    for (int s = 0; s < GB_S; ++s) mbar_init(bar + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int t) {
    const int s = t % GB_S;
    const int64_t row = r0 + (int64_t)t * R;
    const int rows = (int)min((int64_t)R, r1 - row);
    const uint32_t na = (uint32_t)rows * (uint32_t)lda, nb = (uint32_t)rows * (uint32_t)ldb;
    const uint32_t ba = (na * 8u) & ~15u, bb = (nb * 8u) & ~15u;
    double* sa = st + s * stride;
    double* sb = sa + stA;
    fence_proxy_smem();  // this thread's earlier plain stores into the stage
    mbar_expect_tx(bar + s, ba + bb);
    if (ba) bulk_g2s(sa, A + row * lda, ba, bar + s);
    if (bb) bulk_g2s(sb, B + row * ldb, bb, bar + s);
    // an odd element count leaves the last element to a plain load
    if (na & 1u) sa[na - 1] = A[row * lda + na - 1];
    if (nb & 1u) sb[nb - 1] = B[row * ldb + nb - 1];
  };
  if (tid == 0)
    for (int t = 0; t < GB_S && t < nt; ++t) issue(t);
  const int cbA = (ka + 3) >> 2, cbB = (kb + 3) >> 2, nob = cbA * cbB;
  const int nrg = GB_THREADS / nob;
  const int ob = tid % nob, rg = tid / nob;
  const bool act = rg < nrg;
  const int ia = (ob / cbB) * 4, ib = (ob % cbB) * 4;
  double acc[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) acc[u] = 0.0;
  for (int t = 0; t < nt; ++t) {
    const int s = t % GB_S;
    mbar_wait(bar + s, (uint32_t)(t / GB_S) & 1u);
    __syncthreads();  // the odd-element plain loads of this stage (thread 0)
    const double* sa = st + s * stride;
    const double* sb = sa + stA;
    const int rows = (int)min((int64_t)R, r1 - (r0 + (int64_t)t * R));
    if (act) {
      const int64_t row0 = r0 + (int64_t)t * R;
      for (int r = rg; r < rows; r += nrg) {
        double av[4], bv[4];
        const double wr = rw ? rw[row0 + r] : 1.0;  // optional row weights: A^T diag(rw) B
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          av[u] = ia + u < ka ? sa[r * lda + ia + u] * wr : 0.0;
          bv[u] = ib + u < kb ? sb[r * ldb + ib + u] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u * 4 + v] = fma(av[u], bv[v], acc[u * 4 + v]);
      }
    }
    __syncthreads();  // stage s free
    if (tid == 0 && t + GB_S < nt) issue(t + GB_S);
  }
  // fixed-order sum over the row groups (stage memory reused)
  double* red = st;
  const int np = ka * kb;
  if (act)
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (ia + u < ka && ib + v < kb) red[rg * np + (ia + u) * kb + ib + v] = acc[u * 4 + v];
  __syncthreads();
  for (int p = tid; p < np; p += GB_THREADS) {
    double sm = 0.0;
    for (int g = 0; g < nrg; ++g) sm += red[g * np + p];
    part[(int64_t)blockIdx.x * np + p] = sm;
  }
}

void launch_gram_tn(usbs_ctx* ctx, int64_t n, const double* A, int64_t lda, int ka, const double* B, int64_t ldb,
                    int kb, double* out, bool sym, const double* rw) {
  if (ka < 1 || kb < 1 || ka > 64 || kb > 64) fail(USBS_ERR_SHAPE, "gram: 1 <= k <= 64");
  if (sym && ka != kb) fail(USBS_ERR_SHAPE, "gram: symmetric output needs ka == kb");
  const char* eg = getenv("USBS_GRAM_V1");
  if (rw && !(n >= 1024 && lda <= 128 && ldb <= 128 && ((uintptr_t)A & 15) == 0 && ((uintptr_t)B & 15) == 0))
    fail(USBS_ERR_SHAPE, "weighted gram needs the TMA path (aligned operands, n >= 1024)");
  if (n >= 1024 && lda <= 128 && ldb <= 128 && ((uintptr_t)A & 15) == 0 && ((uintptr_t)B & 15) == 0 &&
      !(eg && eg[0] == '1')) {
    int R = (int)std::min<int64_t>(128, std::max<int64_t>(16, 4096 / (lda + ldb)));
    R &= ~15;
    int nb = (int)std::min<int64_t>(2 * ctx->num_sms, (n + R - 1) / R);
    int64_t rpb = ((n + nb - 1) / nb + R - 1) / R * R;
    nb = (int)((n + rpb - 1) / rpb);
    const int stride = (int)((R * (lda + ldb) + 1) & ~1);
    const size_t sm = (size_t)GB_S * stride * sizeof(double) + GB_S * sizeof(uint64_t);
    const int nob = ((ka + 3) / 4) * ((kb + 3) / 4);
    if ((size_t)(GB_THREADS / nob) * ka * kb <= (size_t)GB_S * stride) {
      smem_optin(ctx, (const void*)k_gram_bulk, (int)sm);
      double* part = (double*)ctx->ws.get(WS_GRAM_PARTIAL, (size_t)nb * ka * kb * sizeof(double));
      k_gram_bulk<<<nb, GB_THREADS, sm, ctx->stream>>>(n, A, lda, ka, B, ldb, kb, R, rpb, part, rw);
      check_launch(ctx);
      k_gram_final<<<(ka * kb + 7) / 8, 256, 0, ctx->stream>>>(nb, ka, kb, part, out, sym ? 1 : 0);
      check_launch(ctx);
      return;
    }
  }
  if (rw) fail(USBS_ERR_SHAPE, "weighted gram: shape outside the TMA path");
  // one block per SM for n >= 148 * 64 rows, else a 64-row chunk per block:
  // the partial pass is latency-bound per tile, so short chunks win
  int nb = (int)std::min<int64_t>(ctx->num_sms, std::max<int64_t>(1, (n + 63) / 64));
  double* part = (double*)ctx->ws.get(WS_GRAM_PARTIAL, (size_t)nb * ka * kb * sizeof(double));
  size_t sm = (size_t)GRAM_TR * (ka + kb) * sizeof(double);
  k_gram_partial<<<nb, 256, sm, ctx->stream>>>(n, A, lda, ka, B, ldb, kb, part);
  check_launch(ctx);
  k_gram_final<<<(ka * kb + 7) / 8, 256, 0, ctx->stream>>>(nb, ka, kb, part, out, sym ? 1 : 0);
  check_launch(ctx);
}

__global__ void k_dot_partial(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                              double* __restrict__ part) {
  __shared__ double red[32];
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  double s = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) s = fma(x[i], y[i], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_sum_final(int nb, const double* __restrict__ part, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[b];
    out[0] = s;
  }
}

void launch_dot(usbs_ctx* ctx, int64_t n, const double* x, const double* y, double* out) {
  int nb = (int)std::min<int64_t>(2 * ctx->num_sms, std::max<int64_t>(1, (n + 1023) / 1024));
  double* part = (double*)ctx->ws.get(WS_RED, (size_t)nb * sizeof(double));
  k_dot_partial<<<nb, 256, 0, ctx->stream>>>(n, x, y, part);
  check_launch(ctx);
  k_sum_final<<<1, 32, 0, ctx->stream>>>(nb, part, out);
  check_launch(ctx);
}

}  // namespace usbs
