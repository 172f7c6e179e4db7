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

__device__ inline size_t jacobi_smem_bytes(int N) {
  return (size_t)4 * N * N * sizeof(double) + 64 * 2 * sizeof(double) + 64 * sizeof(int) +
         32 * sizeof(double) + 16;
}

// On entry: js.A holds the symmetric input (row-major, ld = N).  All threads
// of the block must call.  On exit: vals[0..N) descending, vecs (row-major
// N x N, column c = eigenvector c) written to the given pointers (may be
// shared or global).
__device__ inline void jacobi_eigh(int N, JacobiSmem js, double* vals, double* vecs, int ldvec) {
  const int tid = threadIdx.x, nth = blockDim.x;
  double* A = js.A;
  double* A2 = js.A2;
  double* V = js.V;
  double* V2 = js.V2;
  // symmetrise (small_eigh does 0.5 (s + s^T)) and V = I
  for (int x = tid; x < N * N; x += nth) {
    int r = x / N, c = x % N;
    if (r > c) {
      double s = 0.5 * (A[r * N + c] + A[c * N + r]);
      A2[r * N + c] = s;
      A2[c * N + r] = s;
    } else if (r == c) {
      A2[x] = A[x];
    }
    V[x] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  { double* t = A; A = A2; A2 = t; }
  // Frobenius norm for thresholds
  double fro2 = 0.0;
  for (int x = tid; x < N * N; x += nth) fro2 += A[x] * A[x];
  fro2 = block_sum(fro2, js.red);
  const double fro = sqrt(fro2);
  const double skip = 1e-300 + 1e-18 * fro;
  const int P = N + (N & 1);
  if (N > 1 && fro > 0.0) {
    for (int sweep = 0; sweep < 40; ++sweep) {
      if (tid == 0) *js.flag = 0;
      __syncthreads();
      for (int r = 0; r < P - 1; ++r) {
        // rotation parameters
        for (int i = tid; i < P / 2; i += nth) {
          int a, b;
          if (i == 0) { a = r; b = P - 1; }
          else { a = (r + i) % (P - 1); b = (r - i + (P - 1)) % (P - 1); }
          int p = a < b ? a : b, q = a < b ? b : a;
          if (q < N) {
            double apq = A[p * N + q];
            double c = 1.0, s = 0.0;
            if (fabs(apq) > skip) {
              double tau = (A[q * N + q] - A[p * N + p]) / (2.0 * apq);
              double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
              c = 1.0 / sqrt(1.0 + t * t);
              s = t * c;
              *js.flag = 1;
            }
            js.mate[p] = q; js.cself[p] = c; js.cmate[p] = -s;
            js.mate[q] = p; js.cself[q] = c; js.cmate[q] = s;
          } else if (p < N) {
            js.mate[p] = p; js.cself[p] = 1.0; js.cmate[p] = 0.0;
          }
        }
        __syncthreads();
        for (int x = tid; x < N * N; x += nth) {
          int rr = x / N, cc = x % N;
          int mr = js.mate[rr], mc = js.mate[cc];
          double sr = js.cself[rr], tr = js.cmate[rr], sc = js.cself[cc], tc = js.cmate[cc];
          if (rr >= cc) {
            double v;
            if (mr == cc && rr != cc) {
              v = 0.0;
            } else {
              double x0 = sc * A[rr * N + cc] + (mc != cc ? tc * A[rr * N + mc] : 0.0);
              double x1 = (mr != rr) ? (sc * A[mr * N + cc] + (mc != cc ? tc * A[mr * N + mc] : 0.0)) : 0.0;
              v = sr * x0 + (mr != rr ? tr * x1 : 0.0);
            }
            A2[rr * N + cc] = v;
            A2[cc * N + rr] = v;
          }
          V2[x] = sc * V[rr * N + cc] + (mc != cc ? tc * V[rr * N + mc] : 0.0);
        }
        __syncthreads();
        { double* t = A; A = A2; A2 = t; }
        { double* t = V; V = V2; V2 = t; }
      }
      // convergence: off-diagonal mass
      double off = 0.0;
      for (int x = tid; x < N * N; x += nth) {
        int rr = x / N, cc = x % N;
        if (rr != cc) off += A[x] * A[x];
      }
      off = block_sum(off, js.red);
      int rotated = *js.flag;
      __syncthreads();
      if (!rotated || off <= 1e-32 * fro2) break;
    }
  }
  // sort descending by rank (ties by index)
  for (int i = tid; i < N; i += nth) {
    double li = A[i * N + i];
    int rank = 0;
    for (int j = 0; j < N; ++j) {
      double lj = A[j * N + j];
      if (lj > li || (lj == li && j < i)) ++rank;
    }
    js.mate[i] = rank;
  }
  __syncthreads();
  for (int i = tid; i < N; i += nth) vals[js.mate[i]] = A[i * N + i];
  for (int x = tid; x < N * N; x += nth) {
    int rr = x / N, cc = x % N;
    vecs[rr * ldvec + js.mate[cc]] = V[x];
  }
  __syncthreads();
}

}  // namespace usbs
