// Microbenchmark (diagnostic): one panel's trailing tile update of the IPM
// Cholesky (d = 210, J = 0: 351 tile pairs over 15 warps), cycles per panel.
//   mode 0: full (decode + load + 2 DMMA + store, next tile prefetched)
//   mode 1: loads + store only (no DMMA)
//   mode 2: DMMA on register operands only (no smem)
//   mode 3: decode only
#include <cstdio>
constexpr int D = 210;
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}
__device__ __forceinline__ int t_sw(int r) { return ((r >> 1) & 3) << 1; }
__device__ __forceinline__ int t_base(int d, int I, int K) { return 32 * I * (I + 1) + K * min(8, d - 8 * I) * 8; }
__device__ __forceinline__ void pair_decode(int pq, int& I, int& K) {
  int i = (int)((sqrtf(8.0f * (float)pq + 1.0f) - 1.0f) * 0.5f);
  while ((i + 1) * (i + 2) / 2 <= pq) ++i;
  while (i * (i + 1) / 2 > pq) --i;
  I = i; K = pq - i * (i + 1) / 2;
}
struct TileFrag { double a0, a1, b0, b1; double2 c; int cpos; bool st; };
__device__ __forceinline__ void tile_load(const double* __restrict__ M, int d, int J, int I, int K, TileFrag& f) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3, sg = t_sw(g);
  const int rbI = min(8, d - 8 * I), rbK = min(8, d - 8 * K);
  const double* A = M + t_base(d, I, J) + g * 8;
  const double* B = M + t_base(d, K, J) + g * 8;
  const bool vi = g < rbI, vk = g < rbK;
  f.a0 = vi ? -A[q ^ sg] : 0.0; f.a1 = vi ? -A[(q + 4) ^ sg] : 0.0;
  f.b0 = vk ? B[q ^ sg] : 0.0; f.b1 = vk ? B[(q + 4) ^ sg] : 0.0;
  f.cpos = t_base(d, I, K) + g * 8 + ((2 * q) ^ sg);
  f.st = vi;
  f.c = vi ? *reinterpret_cast<const double2*>(M + f.cpos) : make_double2(0.0, 0.0);
}
__device__ __forceinline__ void tile_apply(double* __restrict__ M, const TileFrag& f) {
  double d0, d1;
  dmma(d0, d1, f.a0, f.b0, f.c.x, f.c.y);
  dmma(d0, d1, f.a1, f.b1, d0, d1);
  if (f.st) *reinterpret_cast<double2*>(M + f.cpos) = make_double2(d0, d1);
}
__device__ __forceinline__ int pidx(int i, int j) { return i * (i + 1) / 2 + j; }
__global__ void __launch_bounds__(512, 1) k(int mode, long long* out, double* sink) {
  extern __shared__ __align__(16) double M[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3, sg = t_sw(g);
  for (int x = tid; x < 24000; x += 512) M[x] = 1e-3 * (x % 17);
  __shared__ unsigned short ptab[400];
  for (int pq = tid; pq < 351; pq += 512) {
    int I = 0; while ((I + 1) * (I + 2) / 2 <= pq) ++I;
    ptab[pq] = (unsigned short)((I << 8) | (pq - I * (I + 1) / 2));
  }
  __syncthreads();
  const int J = 0, R = 26, npairs = R * (R + 1) / 2, nw1 = 15;
  double acc = 0.0;
  long long t0 = clock64();
  for (int rep = 0; rep < 10; ++rep) {
    if (mode == 7 || mode == 8) {
      // packed lower storage; panel J = 0 (jb = 8), tile rows I = 1..26
      // mode 7: pair round robin (the kernel's two-tile jobs are similar)
      // mode 8: a warp per tile row, the row's A fragments loaded once
      const int d = D, j0 = 0, jb = 8;
      if (mode == 8) {
        if (warp >= 1) {
          for (int Ir = warp - 1; Ir < 26; Ir += 15) {
            const int I = 26 - Ir;  // longest rows first
            const int ra = I * 8 + g;
            const bool va = ra < d;
            const int oa = va ? pidx(ra, 0) : 0;
            const double a0 = va ? -M[oa + j0 + q] : 0.0, a1 = va ? -M[oa + j0 + 4 + q] : 0.0;
            for (int K = 1; K <= I; ++K) {
              const int rb = K * 8 + g;
              const int ob = rb < d ? pidx(rb, 0) : 0;
              const double b0 = rb < d ? M[ob + j0 + q] : 0.0, b1 = rb < d ? M[ob + j0 + 4 + q] : 0.0;
              const int cc = K * 8 + 2 * q;
              const bool v0 = va && cc <= ra, v1 = va && cc + 1 <= ra;
              double c0 = v0 ? M[oa + cc] : 0.0, c1 = v1 ? M[oa + cc + 1] : 0.0;
              double d0, d1;
              dmma(d0, d1, a0, b0, c0, c1);
              dmma(d0, d1, a1, b1, d0, d1);
              if (v0) M[oa + cc] = d0;
              if (v1) M[oa + cc + 1] = d1;
            }
          }
        }
      } else if (warp >= 1) {
        int I = 0, K = warp - 1;
        while (K > I) { K -= I + 1; ++I; }
        for (int pq = warp - 1; pq < npairs; pq += 15) {
          const int Ia = I + 1, Ka = K + 1;
          const int ra = Ia * 8 + g, rb = Ka * 8 + g;
          const int oa = ra < d ? pidx(ra, 0) : 0, ob = rb < d ? pidx(rb, 0) : 0;
          const double a0 = (ra < d && q < jb) ? -M[oa + j0 + q] : 0.0, a1 = (ra < d && q + 4 < jb) ? -M[oa + j0 + 4 + q] : 0.0;
          const double b0 = (rb < d && q < jb) ? M[ob + j0 + q] : 0.0, b1 = (rb < d && q + 4 < jb) ? M[ob + j0 + 4 + q] : 0.0;
          const int cc = Ka * 8 + 2 * q;
          const bool v0 = ra < d && cc <= ra, v1 = ra < d && cc + 1 <= ra;
          double c0 = v0 ? M[oa + cc] : 0.0, c1 = v1 ? M[oa + cc + 1] : 0.0;
          double d0, d1;
          dmma(d0, d1, a0, b0, c0, c1);
          dmma(d0, d1, a1, b1, d0, d1);
          if (v0) M[oa + cc] = d0;
          if (v1) M[oa + cc + 1] = d1;
          K += 15;
          while (K > I) { K -= I + 1; ++I; }
        }
      }
    } else if (mode >= 4) {
      if (warp & 3) {
        const int nup = 12, w = warp - 1 - (warp >> 2);
        for (int pq = w; pq < npairs; pq += nup) {
          const unsigned e = ptab[pq];
          if (mode == 5) { acc += (double)e; continue; }
          TileFrag f;
          tile_load(M, D, J, J + 1 + (int)(e >> 8), J + 1 + (int)(e & 255u), f);
          if (mode == 6) { *reinterpret_cast<double2*>(M + f.cpos) = f.c; acc += f.a0 + f.a1 + f.b0 + f.b1; continue; }
          tile_apply(M, f);
        }
      }
    } else if (warp >= 1) {
      for (int pq = warp - 1; pq < npairs; pq += nw1) {
        int I, K;
        pair_decode(pq, I, K);
        I += J + 1; K += J + 1;
        if (mode == 3) { acc += I + K; continue; }
        if (mode == 2) {
          double d0, d1;
          dmma(d0, d1, acc, 1.0 + pq, acc, 0.5);
          dmma(d0, d1, acc, 2.0, d0, d1);
          acc += d0 + d1;
          continue;
        }
        const double* A = M + t_base(D, I, J) + g * 8;
        const double* B = M + t_base(D, K, J) + g * 8;
        const double a0 = -A[q ^ sg], a1 = -A[(q + 4) ^ sg], b0 = B[q ^ sg], b1 = B[(q + 4) ^ sg];
        const int cpos = t_base(D, I, K) + g * 8 + ((2 * q) ^ sg);
        double2 c = *reinterpret_cast<const double2*>(M + cpos);
        double d0 = c.x + a0 * b0 + a1 * b1, d1 = c.y;
        if (mode == 0) {
          dmma(d0, d1, a0, b0, c.x, c.y);
          dmma(d0, d1, a1, b1, d0, d1);
        }
        *reinterpret_cast<double2*>(M + cpos) = make_double2(d0, d1);
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 32) out[0] = (t1 - t0) / 10;
  if (acc == 1.2345) sink[0] = acc;
}
int main() {
  long long* o; double* s; cudaMalloc(&o, 64); cudaMalloc(&s, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* nm[] = {"full", "loads+store", "dmma only", "decode only", "kernel path", "ptab only", "kernel no dmma", "packed pairs", "packed rows"};
  for (int mode = 0; mode < 9; ++mode) {
    k<<<1, 512, 24000 * 8>>>(mode, o, s);
    cudaError_t e = cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("%-12s %6lld cycles per panel (351 pairs, 15 warps) %s\n", nm[mode], h, cudaGetErrorString(e));
  }
  return 0;
}
