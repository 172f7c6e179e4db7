// Block-cooperative cyclic Jacobi eigensolver for small symmetric matrices
// (N <= 64), FP64, in shared memory.  Replaces symlin.small_eigh
// (symlin.py:193-198, LAPACK syevd through numpy) inside the device kernels:
// Lanczos Rayleigh-Ritz (eigsolve.py:152), model_update (bundle.py:302).
//
// Parallel round-robin ordering (circle method): P = N rounded up to even,
// P/2 disjoint rotations per round, P-1 rounds per sweep; the pair table is
// built once per call.  Each round: P/2 threads compute the rotations
// (Golub & Van Loan sym.schur2 written with one division:
//   x = a_qq - a_pp, y = 2 a_pq, t = sign(x y) |y| / (|x| + hypot(x, y)),
//   c = rsqrt(1 + t^2), s = t c), then the block applies all of them at once,
// A <- J^T A J element-wise from the previous buffer and V <- V J; the pair
// entry becomes exactly zero.  Entries with |a_pq| <= 1e-16 ||A||_F are
// annihilated without rotating (backward error at LAPACK level); the solver
// stops after a sweep without rotations.
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
  unsigned char* ptab;  // 64*64 pair table (round, slot) -> (p, q) packed
};

constexpr int JAC_MAXE = 16;  // elements per thread: N*N <= 4096, blockDim >= 256
constexpr size_t JAC_PTAB_BYTES = 64 * 64;

// On entry: js.A holds the symmetric input (row-major, ld = N).  All threads
// of the block must call (blockDim * 16 >= N * N).  On exit: vals[0..N)
// descending, vecs (row-major N x N, column c = eigenvector c).  Returns the
// number of sweeps.
__device__ inline int jacobi_eigh(int N, JacobiSmem js, double* vals, double* vecs, int ldvec) {
  int sweeps_done = 0;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int NN = N * N;
  const int P = N + (N & 1);
  double* A = js.A;
  double* A2 = js.A2;
  double* V = js.V;
  double* V2 = js.V2;
  short er[JAC_MAXE], ec[JAC_MAXE];
  int ne = 0;
#pragma unroll
  for (int u = 0; u < JAC_MAXE; ++u) {
    const int x = tid + u * nth;
    er[u] = (short)(x < NN ? x / N : 0);
    ec[u] = (short)(x < NN ? x % N : 0);
    if (x < NN) ne = u + 1;
  }
  // pair table: round r, slot i -> (min, max) packed as two bytes
  for (int x = tid; x < (P - 1) * (P / 2); x += nth) {
    const int r = x / (P / 2), i = x % (P / 2);
    int a, b;
    if (i == 0) { a = r; b = P - 1; }
    else { a = (r + i) % (P - 1); b = (r - i + (P - 1)) % (P - 1); }
    js.ptab[2 * x] = (unsigned char)(a < b ? a : b);
    js.ptab[2 * x + 1] = (unsigned char)(a < b ? b : a);
  }
  // symmetrise (small_eigh does 0.5 (s + s^T)), V = I, ||A||_F
  double f2 = 0.0;
#pragma unroll
  for (int u = 0; u < JAC_MAXE; ++u) {
    if (u >= ne) break;
    const int r = er[u], c = ec[u], x = r * N + c;
    const double v = (r == c) ? A[x] : 0.5 * (A[r * N + c] + A[c * N + r]);
    A2[x] = v;
    V[x] = (r == c) ? 1.0 : 0.0;
    f2 = fma(v, v, f2);
  }
  f2 = block_sum(f2, js.red);  // includes barriers
  { double* t = A; A = A2; A2 = t; }
  const double thr = 1e-16 * sqrt(f2);
  if (N > 1 && f2 > 0.0) {
    for (int sweep = 0; sweep < 40; ++sweep) {
      int any = 0;
      for (int r = 0; r < P - 1; ++r) {
        if (tid < P / 2) {
          const int x = r * (P / 2) + tid;
          const int p = js.ptab[2 * x], q = js.ptab[2 * x + 1];
          if (q < N) {
            const double apq = A[p * N + q];
            double c = 1.0, s = 0.0;
            int flag = 0;  // bit0: pair entry annihilated
            if (apq != 0.0) {
              flag = 1;
              if (fabs(apq) > thr) {
                const double xx = A[q * N + q] - A[p * N + p], yy = 2.0 * apq;
                double t = fabs(yy) / (fabs(xx) + sqrt(fma(xx, xx, yy * yy)));
                if ((xx < 0.0) != (yy < 0.0) && xx != 0.0) t = -t;
                c = rsqrt(fma(t, t, 1.0));
                s = t * c;
                any = 1;
              }
            }
            js.mate[p] = q | (flag << 8);
            js.cself[p] = c;
            js.cmate[p] = -s;
            js.mate[q] = p | (flag << 8);
            js.cself[q] = c;
            js.cmate[q] = s;
          } else if (p < N) {
            js.mate[p] = p;
            js.cself[p] = 1.0;
            js.cmate[p] = 0.0;
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
            if (mr == cc && rr != cc && (mrr >> 8)) {
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
      ++sweeps_done;
      if (!__syncthreads_or(any)) break;
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
