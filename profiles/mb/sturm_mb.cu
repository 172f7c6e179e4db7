// Microbenchmark (diagnostic): cycles per Sturm count / per multisection
// iteration of rr_arrow on a synthetic arrow+tridiagonal H (N = 33, ell = 13).
#include <cstdio>
#include "../../paper_2312_11801_b200/csrc/usbs_tridiag.cuh"
using namespace usbs;

__global__ void k_mb(int N, int ell, const double* dd_g, const double* sq_g, long long* out, int* cnt_out) {
  __shared__ double d[64], sq[64];
  for (int i = threadIdx.x; i < N; i += blockDim.x) { d[i] = dd_g[i]; sq[i] = sq_g[i]; }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  long long t0 = clock64();
  int acc = 0;
  for (int rep = 0; rep < 100; ++rep) {
    const double sig = -1.0 + 2.0 * (lane + rep * 32) / 3200.0;
    acc += sturm_arrow(N, ell, d, sq, sig, 1e-300);
  }
  long long t1 = clock64();
  // one division-based multisection step
  double lo = -1.0, hi = 1.0;
  long long t2 = clock64();
  for (int rep = 0; rep < 100; ++rep) {
    const double s2 = lo + (hi - lo) * (double)(lane + 1) / 33.0;
    acc += s2 > 0.0;
    lo += 1e-3 * s2;
  }
  long long t3 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / 100; out[1] = (t3 - t2) / 100; }
  cnt_out[threadIdx.x] = acc;
}

int main() {
  const int N = 33, ell = 13;
  double hd[64], hs[64];
  for (int i = 0; i < N; ++i) { hd[i] = 0.5 * __builtin_sin(i * 1.3); hs[i] = 0.01 + 0.1 * (i % 5); }
  double *dd, *ds; long long* o; int* c;
  cudaMalloc(&dd, 64 * 8); cudaMalloc(&ds, 64 * 8); cudaMalloc(&o, 16); cudaMalloc(&c, 4096);
  cudaMemcpy(dd, hd, 64 * 8, cudaMemcpyHostToDevice); cudaMemcpy(ds, hs, 64 * 8, cudaMemcpyHostToDevice);
  for (int w = 1; w <= 16; w *= 4) {
    k_mb<<<1, 32 * w>>>(N, ell, dd, ds, o, c);
    long long h[2];
    cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    printf("warps %2d: sturm count %lld cycles (%.1f / row), division step %lld cycles\n", w, h[0], h[0] / (double)N, h[1]);
  }
  return 0;
}
