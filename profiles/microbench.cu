// Latency microbenchmarks on B200 (sm_100a) for the latency-bound small
// dense kernels (IPM, Rayleigh-Ritz): cycles per dependent op.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb profiles/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double* out, long long* cyc, double seed, int iters) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = seed + i;
  __syncthreads();
  double x = seed + threadIdx.x * 1e-3;
  long long t0, t1;
  // 0: dependent DFMA
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
  // 1: dependent double division
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 + 1e-3 / x;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0);
  // 2: dependent rsqrt
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = rsqrt(x) + 0.5;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0);
  // 3: dependent sqrt
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = sqrt(x) + 0.5;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0);
  // 4: dependent smem load (pointer chase through indices)
  int idx = threadIdx.x & 511;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) idx = ((int)sm[idx] + 1) & 511;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0);
  // 5: __syncthreads
  t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0);
  // 6: shuffle chain
  double y = x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) y = __shfl_xor_sync(0xffffffffu, y, 1) + 1e-9;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0);
  // 7: DMUL chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = x * 1.0000001;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[7] = (t1 - t0);
  out[threadIdx.x] = x + y + idx;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  const char* names[] = {"dfma", "ddiv", "drsqrt", "dsqrt", "lds-chase", "syncthreads(512)", "shfl.f64", "dmul"};
  for (int threads : {32, 512}) {
    k_lat<<<1, threads>>>(out, cyc, 1.5, 1000);
    cudaDeviceSynchronize();
    k_lat<<<1, threads>>>(out, cyc, 1.5, 1000);
    cudaDeviceSynchronize();
    printf("threads=%d\n", threads);
    for (int i = 0; i < 8; ++i) printf("  %-18s %8.1f cycles/op\n", names[i], cyc[i] / 1000.0);
  }
  return 0;
}
