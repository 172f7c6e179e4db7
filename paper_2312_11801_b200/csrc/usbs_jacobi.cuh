// Block-cooperative cyclic Jacobi eigensolver for small symmetric matrices
// (N <= 64), FP64, in shared memory.  Replaces symlin.small_eigh
// (symlin.py:193-198, LAPACK syevd through numpy) inside the device kernels:
// Lanczos Rayleigh-Ritz (eigsolve.py:152), model_update (bundle.py:302).
//
// Parallel round-robin ordering: P = N rounded up to even, P/2 disjoint
// rotations per round, P-1 rounds per sweep.  Each round applies all
// rotations at once: A <- J^T A J computed element-wise from the previous
// buffer (4-term formula), V <- V J.  Rotation parameters follow Golub & Van
// Loan's sym.schur2; the annihilated pair entry is set to exactly zero.
// Termination (as in the classical threshold Jacobi): from the fourth sweep
// on, an off-diagonal entry that is negligible next to both diagonal entries
// (|a_pp| + 100|a_pq| == |a_pp| and likewise for a_qq) is set to zero
// without rotating; the solver stops after a sweep without rotations.
// Output: eigenvalues descending, eigenvector columns in matching order.
#pragma once
#include "usbs_common.cuh"

namespace usbs {

struct JacobiSmem {
  double* A;      // N*N
  double* A2;     // N*N
  double* V;      // N*N
  double* V2;     // N*N
  double* cself;  // 64
  double* cmate;  // 64
  int* mate;      // 64
  double* red;    // 32
  int* flag;      // 1
};

constexpr int JAC_MAXE = 16;  // elements per thread: N*N <= 4096, blockDim >= 256

// On entry: js.A holds the symmetric input (row-major, ld = N).  All threads
// of the block must call (blockDim >= 256 when N > 32).  On exit: vals[0..N)
// descending, vecs (row-major N x N, column c = eigenvector c).
__device__ inline int jacobi_eigh(int N, JacobiSmem js, double* vals, double* vecs, int ldvec) {
  int sweeps_done = 0;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int NN = N * N;
  double* A = js.A;
  double* A2 = js.A2;
  double* V = js.V;
  double* V2 = js.V2;
  // element ownership, computed once (no integer division inside the rounds)
  short er[JAC_MAXE], ec[JAC_MAXE];
  int ne = 0;
#pragma unroll
  for (int u = 0; u < JAC_MAXE; ++u) {
    const int x = tid + u * nth;
    er[u] = (short)(x < NN ? x / N : 0);
    ec[u] = (short)(x < NN ? x % N : 0);
    if (x < NN) ne = u + 1;
  }
  // symmetrise (small_eigh does 0.5 (s + s^T)) and V = I
#pragma unroll
  for (int u = 0; u < JAC_MAXE; ++u) {
    if (u >= ne) break;
    const int r = er[u], c = ec[u], x = r * N + c;
    A2[x] = (r == c) ? A[x] : 0.5 * (A[r * N + c] + A[c * N + r]);
    V[x] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  { double* t = A; A = A2; A2 = t; }
  const int P = N + (N & 1);
  if (N > 1) {
    for (int sweep = 0; sweep < 50; ++sweep) {
      if (tid == 0) *js.flag = 0;
      __syncthreads();
      for (int r = 0; r < P - 1; ++r) {
        for (int i = tid; i < P / 2; i += nth) {
          int a, b;
          if (i == 0) { a = r; b = P - 1; }
          else { a = (r + i) % (P - 1); b = (r - i + (P - 1)) % (P - 1); }
          const int p = a < b ? a : b, q = a < b ? b : a;
          if (q < N) {
            const double apq = A[p * N + q];
            const double app = A[p * N + p], aqq = A[q * N + q];
            double c = 1.0, s = 0.0;
            int zero = 0;
            if (apq != 0.0) {
              const double g = 100.0 * fabs(apq);
              if (sweep >= 3 && fabs(app) + g == fabs(app) && fabs(aqq) + g == fabs(aqq)) {
                zero = 1;  // negligible: annihilate without rotating
              } else {
                const double tau = (aqq - app) / (2.0 * apq);
                const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                c = 1.0 / sqrt(1.0 + t * t);
                s = t * c;
                zero = 1;
                *js.flag = 1;
              }
            }
            // mate < 0 encodes "no coupling"; the pair entry is zeroed when zero = 1
            js.mate[p] = zero ? q : (q | 0x100);
            js.cself[p] = c; js.cmate[p] = -s;
            js.mate[q] = zero ? p : (p | 0x100);
            js.cself[q] = c; js.cmate[q] = s;
          } else if (p < N) {
            js.mate[p] = p | 0x100; js.cself[p] = 1.0; js.cmate[p] = 0.0;
          }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < JAC_MAXE; ++u) {
          if (u >= ne) break;
          const int rr = er[u], cc = ec[u];
          const int mrr = js.mate[rr], mcc = js.mate[cc];
          const int mr = mrr & 0xff, mc = mcc & 0xff;
          const double sr = js.cself[rr], tr = js.cmate[rr], sc = js.cself[cc], tc = js.cmate[cc];
          if (rr >= cc) {
            double v;
            if (mr == cc && rr != cc && !(mrr & 0x100)) {
              v = 0.0;
            } else {
              const double x0 = sc * A[rr * N + cc] + (mc != cc ? tc * A[rr * N + mc] : 0.0);
              const double x1 = (mr != rr) ? (sc * A[mr * N + cc] + (mc != cc ? tc * A[mr * N + mc] : 0.0)) : 0.0;
              v = sr * x0 + (mr != rr ? tr * x1 : 0.0);
            }
            A2[rr * N + cc] = v;
            A2[cc * N + rr] = v;
          }
          V2[rr * N + cc] = sc * V[rr * N + cc] + (mc != cc ? tc * V[rr * N + mc] : 0.0);
        }
        __syncthreads();
        { double* t = A; A = A2; A2 = t; }
        { double* t = V; V = V2; V2 = t; }
      }
      const int rotated = *js.flag;
      __syncthreads();
      ++sweeps_done;
      if (!rotated) break;
    }
  }
  // sort descending by rank (ties by index)
  for (int i = tid; i < N; i += nth) {
    const double li = A[i * N + i];
    int rank = 0;
    for (int j = 0; j < N; ++j) {
      const double lj = A[j * N + j];
      if (lj > li || (lj == li && j < i)) ++rank;
    }
    js.mate[i] = rank;
  }
  __syncthreads();
  for (int i = tid; i < N; i += nth) vals[js.mate[i]] = A[i * N + i];
#pragma unroll
  for (int u = 0; u < JAC_MAXE; ++u) {
    if (u >= ne) break;
    const int rr = er[u], cc = ec[u];
    vecs[rr * ldvec + js.mate[cc]] = V[rr * N + cc];
  }
  __syncthreads();
  return sweeps_done;
}

}  // namespace usbs
