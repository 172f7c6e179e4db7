// Microbenchmark (diagnostic): rr_arrow (Lanczos Rayleigh-Ritz on the
// arrowhead + tridiagonal projection) on one CTA of 512 threads, N = 32,
// ell = 13, nw = 13, phase times in cycles via clock64.
#include <cstdio>
#include <cmath>
#include "../../paper_2312_11801_b200/csrc/usbs_tridiag.cuh"
using namespace usbs;

__global__ void __launch_bounds__(512, 1) k(const double* H, int N, int ell, int nw, double* vals, double* Yout,
                                            unsigned long long* prof, int reps) {
  extern __shared__ __align__(16) double sm[];
  double* Ys = sm;
  TriSmem ts;
  ts.A = Ys + N * N; ts.Q = ts.A + N * N; ts.Z = ts.Q + N * N; ts.v = ts.Z + N * N;
  ts.p = ts.v + 64; ts.dd = ts.p + 64; ts.ee = ts.dd + 64; ts.lam = ts.ee + 64; ts.red = ts.lam + 64;
  ts.iw = (int*)(ts.red + 64);
  __shared__ double th[64];
  for (int r = 0; r < reps; ++r) rr_arrow(N, ell, nw, H, N + 1, ts, th, Ys, N, prof);
  for (int x = threadIdx.x; x < N * nw; x += blockDim.x) Yout[x] = Ys[(x / nw) * N + (x % nw)];
  for (int x = threadIdx.x; x < nw; x += blockDim.x) vals[x] = th[x];
}

int main() {
  const int N = 32, M1 = N + 1, ell = 13, nw = 13;
  double h[M1 * M1] = {0};
  // arrowhead: theta_k descending, b_k; then tridiagonal
  for (int k2 = 0; k2 < ell; ++k2) { h[k2 * M1 + k2] = 1.0 - 0.05 * k2 - 0.001 * k2 * k2; h[k2 * M1 + ell] = h[ell * M1 + k2] = 1e-3 * (k2 + 1); }
  for (int i = ell; i < N; ++i) { h[i * M1 + i] = 0.3 * std::sin(1.7 * i); if (i + 1 < N) h[(i + 1) * M1 + i] = h[i * M1 + i + 1] = 0.2 + 0.01 * i; }
  double *dH, *dv, *dY; unsigned long long* dp;
  cudaMalloc(&dH, sizeof(h)); cudaMalloc(&dv, 64 * 8); cudaMalloc(&dY, 64 * 64 * 8); cudaMalloc(&dp, 16 * 8);
  cudaMemcpy(dH, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemset(dp, 0, 16 * 8);
  const size_t smem = (4 * N * N + 6 * 64) * 8 + 128 * 4 + 64;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int reps = 20;
  k<<<1, 512, smem>>>(dH, N, ell, nw, dv, dY, dp, reps);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long p[16]; double vals[64];
  cudaMemcpy(p, dp, 16 * 8, cudaMemcpyDeviceToHost); cudaMemcpy(vals, dv, 64 * 8, cudaMemcpyDeviceToHost);
  printf("%s  setup %.2f  bisect %.2f  inv-it %.2f  out %.2f | factor+start %.2f (factor alone %.2f) us\n", cudaGetErrorString(e),
         p[0] / 1e3 / reps, p[1] / 1e3 / reps, p[2] / 1e3 / reps, p[3] / 1e3 / reps, p[4] / 1e3 / reps, p[7] / 1e3 / reps);
  printf("theta: %.15f %.15f %.15f\n", vals[0], vals[1], vals[12]);
  return 0;
}
