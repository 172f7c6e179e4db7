// Microbenchmark (diagnostic): dependent-chain latencies on this GPU.
#include <cstdio>
__global__ void k(double* out, long long* cyc, int nwarps_busy) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1e-3 * (i % 13);
  __syncthreads();
  double a = out[0], b = out[1];
  long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) a = fma(a, b, 1e-9);
  long long t1 = clock64();
  float fa = (float)a, fb = (float)b;
  for (int i = 0; i < 1000; ++i) fa = fmaf(fa, fb, 1e-9f);
  long long t2 = clock64();
  int idx = 0;
  for (int i = 0; i < 1000; ++i) idx = (int)(sm[idx & 1023] * 0.0) + (i & 7);  // LDS chain
  long long t3 = clock64();
  double c = a;
  for (int i = 0; i < 1000; ++i) c = c + b;
  long long t4 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
  out[2 + threadIdx.x] = a + fa + idx + c;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1100); cudaMalloc(&c, 64);
  double h[2] = {0.999, 1.0001}; cudaMemcpy(o, h, 16, cudaMemcpyHostToDevice);
  for (int th : {32, 128, 512}) {
    k<<<1, th>>>(o, c, 0); cudaDeviceSynchronize();
    long long r[4]; cudaMemcpy(r, c, 32, cudaMemcpyDeviceToHost);
    printf("threads %3d: DFMA %.1f  FFMA %.1f  LDS-chain %.1f  DADD %.1f cycles/op\n", th, r[0] / 1000.0, r[1] / 1000.0, r[2] / 1000.0, r[3] / 1000.0);
  }
  return 0;
}
