// K1q: the quadratic-assignment cost as a dense contraction on the FP64
// tensor cores.  build_qap (problem.py:462-477) sets C = -(D (x) W) / scale_c
// on the lifted block, with composite index a = i*l + k (problem.py:364-371:
// i the distance factor, k the weight factor) and an empty row/column 0, so
// for a column v:
//
//     (C v)[1 + i*l + k] = coef * (D X W^T)[i, k],   X[j, m] = v[1 + j*l + m]
//
// (coef = -1/scale_c).  k_kron_apply computes T = X W^T, then D T, for one
// column per CTA with mma.sync.m8n8k4 f64 on l padded to a multiple of 8
// (the padding is zero), operands in shared memory: 2 (L/8)^2 (L/4) DMMAs per
// column (l = 20: 108) against the l^2 (~0.9 l^2) nonzeros of the sparse cost
// row block per output row.  The slack operator Z = C - A*(y) is applied as
// this contraction plus a sparse pass over the adjoint values A*(y) on the
// merged pattern (usbs_sparse.cu, launch_adjoint_values), so
// Z V = C V - A*(y) V (problem.py:311-314).
#include <algorithm>

#include "usbs_common.cuh"
#include "usbs_kernels.cuh"

namespace usbs {

// D = A B + C, A 8x4 row-major, B 4x8 col-major (usbs_common.cuh dmma_m8n8k4)
template <int L>
__global__ void __launch_bounds__(128) k_kron_apply(int l, const double* __restrict__ D,
                                                     const double* __restrict__ W, double coef,
                                                     const double* __restrict__ V, int64_t ldv,
                                                     double* __restrict__ Y, int64_t ldy, double beta) {
  __shared__ double Xs[L * L], Ws[L * L], Ds[L * L], Ts[L * L];
  const int c = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int x = tid; x < L * L; x += blockDim.x) {
    const int r = x / L, q = x % L;
    const bool in = r < l && q < l;
    Xs[x] = in ? V[(int64_t)(1 + r * l + q) * ldv + c] : 0.0;
    Ws[x] = in ? W[r * l + q] : 0.0;
    Ds[x] = in ? D[r * l + q] : 0.0;
  }
  __syncthreads();
  constexpr int NT = L / 8, NK = L / 4;
  const int ar = lane >> 2, ac = lane & 3;
  // T = X W^T: T[j][k] = sum_m X[j][m] W[k][m]
  for (int t = warp; t < NT * NT; t += 4) {
    const int jt = t / NT, kt = t % NT;
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int ks = 0; ks < NK; ++ks) {
      const double a = Xs[(jt * 8 + ar) * L + ks * 4 + ac];   // A[row][q] = X[j][m]
      const double b = Ws[(kt * 8 + ar) * L + ks * 4 + ac];   // B[q][col] = W[k][m]
      dmma_m8n8k4(d0, d1, a, b, d0, d1);
    }
    Ts[(jt * 8 + ar) * L + kt * 8 + 2 * ac] = d0;
    Ts[(jt * 8 + ar) * L + kt * 8 + 2 * ac + 1] = d1;
  }
  __syncthreads();
  // Y = D T: Y[i][k] = sum_j D[i][j] T[j][k]
  for (int t = warp; t < NT * NT; t += 4) {
    const int it = t / NT, kt = t % NT;
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int ks = 0; ks < NK; ++ks) {
      const double a = Ds[(it * 8 + ar) * L + ks * 4 + ac];   // A[row][q] = D[i][j]
      const double b = Ts[(ks * 4 + ac) * L + kt * 8 + ar];   // B[q][col] = T[j][k]
      dmma_m8n8k4(d0, d1, a, b, d0, d1);
    }
    const int i = it * 8 + ar;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = kt * 8 + 2 * ac + h;
      if (i < l && k < l) {
        double* yp = Y + (int64_t)(1 + i * l + k) * ldy + c;
        const double v = coef * (h ? d1 : d0);
        *yp = beta != 0.0 ? fma(beta, *yp, v) : v;
      }
    }
  }
  if (tid == 0) Y[c] = beta != 0.0 ? beta * Y[c] : 0.0;  // row 0 of C is empty
}

void launch_kron_apply(usbs_ctx* ctx, usbs_problem* p, const double* V, int64_t ldv, int k, double* Y, int64_t ldy,
                       double beta) {
  const int l = p->kron_l;
  if (l <= 8) k_kron_apply<8><<<k, 128, 0, ctx->stream>>>(l, p->kron_D, p->kron_W, p->kron_coef, V, ldv, Y, ldy, beta);
  else if (l <= 16) k_kron_apply<16><<<k, 128, 0, ctx->stream>>>(l, p->kron_D, p->kron_W, p->kron_coef, V, ldv, Y, ldy, beta);
  else if (l <= 24) k_kron_apply<24><<<k, 128, 0, ctx->stream>>>(l, p->kron_D, p->kron_W, p->kron_coef, V, ldv, Y, ldy, beta);
  else if (l <= 32) k_kron_apply<32><<<k, 128, 0, ctx->stream>>>(l, p->kron_D, p->kron_W, p->kron_coef, V, ldv, Y, ldy, beta);
  else fail(USBS_ERR_SHAPE, "kron apply: l <= 32");
  check_launch(ctx);
}

bool kron_enabled(const usbs_problem* p) {
  if (!p->kron_l) return false;
  const char* e = getenv("USBS_KRON");
  return !(e && e[0] == '0');
}

}  // namespace usbs

using namespace usbs;

extern "C" usbs_status usbs_problem_set_kron(usbs_ctx* ctx, usbs_problem* p, int l, const double* D, const double* W,
                                             double coef) {
  USBS_API_BEGIN
  if (!ctx || !p) fail(USBS_ERR_CONFIG, "null context/problem");
  if (l < 1 || l > 32) fail(USBS_ERR_SHAPE, "kron factors: 1 <= l <= 32");
  if (p->n != (int64_t)l * l + 1 || p->n_cols != p->n) fail(USBS_ERR_SHAPE, "kron factors: n must be l^2 + 1");
  p->kron_D = dev_upload(p, D, (size_t)l * l);
  p->kron_W = dev_upload(p, W, (size_t)l * l);
  p->kron_coef = coef;
  p->aval = dev_alloc<double>(p, p->nnz);
  USBS_CUDA(cudaMemset(p->aval, 0, (size_t)p->nnz * sizeof(double)));  // Z = C until the first assembly
  p->kron_l = l;
  USBS_API_END
}
