// Microbenchmark (diagnostic): mma.sync m8n8k4 f64 latency / throughput on
// this GPU versus plain DFMA.
#include <cstdio>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}
__global__ void k(double* io, long long* cyc) {
  const int lane = threadIdx.x & 31;
  double a = io[lane], b = io[32 + lane], c0 = 0, c1 = 0;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) dmma(c0, c1, a, b, c0, c1);  // dependent chain
  long long t1 = clock64();
  double e0 = 0, e1 = 0, f0 = 0, f1 = 0, g0 = 0, g1 = 0, h0 = 0, h1 = 0;
  for (int i = 0; i < 64; ++i) {  // 4 independent chains
    dmma(e0, e1, a, b, e0, e1); dmma(f0, f1, a, b, f0, f1); dmma(g0, g1, a, b, g0, g1); dmma(h0, h1, a, b, h0, h1);
  }
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[blockIdx.x * 2] = t1 - t0; cyc[blockIdx.x * 2 + 1] = t2 - t1; }
  io[64 + threadIdx.x] = c0 + c1 + e0 + e1 + f0 + f1 + g0 + g1 + h0 + h1;
}
int main() {
  double* io; long long* c; cudaMalloc(&io, 8 * 2048); cudaMalloc(&c, 64);
  cudaMemset(io, 0, 8 * 2048);
  for (int th : {32, 128, 512}) {
    k<<<1, th>>>(io, c); cudaDeviceSynchronize();
    long long r[2]; cudaMemcpy(r, c, 16, cudaMemcpyDeviceToHost);
    printf("threads %3d: dependent DMMA %.1f cycles each; 4 chains %.1f cycles per DMMA (per warp)\n", th, r[0] / 256.0, r[1] / 256.0);
  }
  return 0;
}
