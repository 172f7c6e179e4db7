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

void launch_gram_tn(usbs_ctx* ctx, int64_t n, const double* A, int64_t lda, int ka, const double* B, int64_t ldb,
                    int kb, double* out, bool sym) {
  if (ka < 1 || kb < 1 || ka > 64 || kb > 64) fail(USBS_ERR_SHAPE, "gram: 1 <= k <= 64");
  if (sym && ka != kb) fail(USBS_ERR_SHAPE, "gram: symmetric output needs ka == kb");
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
