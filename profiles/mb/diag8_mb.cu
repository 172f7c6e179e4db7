// Microbenchmark (diagnostic): the IPM Cholesky's 8 x 8 diagonal-block
// factorisation by one warp (packed lower storage), cycles per call:
//   v0 two entries per lane (the round's first version; shuffle chain)
//   v1 rows in lanes 0..7 (row r in lane r, all 8 entries in registers)
//   v2 v1 with an FP32-seeded rsqrt
//   v3 the whole block in every lane, factored redundantly (no shuffles)
// B200, d = 64 block: v0 2321, v1 1638 (the kernel's), v2 2173, v3 2678
// cycles; v1 = v3 bit for bit (single-lane issue makes v3 slower)
#include <cstdio>
__device__ __forceinline__ int pidx(int i, int j) { return i * (i + 1) / 2 + j; }
__device__ __forceinline__ void chol_diag8(double* Mp, int d, int J, double* rdiag, int* flag) {
  const int lane = threadIdx.x & 31;
  const int j0 = J * 8, jb = min(8, d - j0);
  const int t = lane & 7, ia = lane >> 3, ib = 4 + (lane >> 3);
  double ea = (ia < jb && t <= ia) ? Mp[pidx(j0 + ia, j0 + t)] : 0.0;
  double eb = (ib < jb && t <= ib) ? Mp[pidx(j0 + ib, j0 + t)] : 0.0;
  int ok = 1;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (c < jb) {
      const double pv = __shfl_sync(0xffffffffu, c < 4 ? ea : eb, (c & 3) * 8 + c);
      if (!(pv > 0.0)) ok = 0;
      const double r = ok ? rsqrt(pv) : 0.0;
      if (t == c) {
        if (ia > c) ea *= r; else if (ia == c) ea = pv * r;
        if (ib > c) eb *= r; else if (ib == c) eb = pv * r;
      }
      if (lane == 0) rdiag[j0 + c] = r;
      const double lia = __shfl_sync(0xffffffffu, ea, (ia & 3) * 8 + c);
      const double lib = __shfl_sync(0xffffffffu, eb, (ib & 3) * 8 + c);
      const double lta_a = __shfl_sync(0xffffffffu, ea, (t & 3) * 8 + c);
      const double lta_b = __shfl_sync(0xffffffffu, eb, (t & 3) * 8 + c);
      const double lta = t < 4 ? lta_a : lta_b;
      if (t > c) {
        if (t <= ia) ea -= lia * lta;
        if (t <= ib) eb -= lib * lta;
      }
    }
  }
  if (ia < jb && t <= ia) Mp[pidx(j0 + ia, j0 + t)] = ea;
  if (ib < jb && t <= ib) Mp[pidx(j0 + ib, j0 + t)] = eb;
  if (lane == 0) *flag = ok;
}
// v1: lane r (< 8) holds row r of the block; per column c the pivot row's
// entries come by shuffle from lane c (row c, columns <= c are final)
__device__ __forceinline__ void chol_diag8_v1(double* Mp, int d, int J, double* rdiag, int* flag) {
  const int lane = threadIdx.x & 31;
  const int j0 = J * 8, jb = min(8, d - j0);
  const int r = lane & 7;
  double a[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) a[t] = (r < jb && t <= r) ? Mp[pidx(j0 + r, j0 + t)] : 0.0;
  int ok = 1;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (c < jb) {
      const double pv = __shfl_sync(0xffffffffu, a[c], c);   // A(c, c) after the updates so far
      if (!(pv > 0.0)) ok = 0;
      const double rs = ok ? rsqrt(pv) : 0.0;
      if (lane == 0) rdiag[j0 + c] = rs;
      // column c: L(r, c) = A(r, c) / L(c, c); the diagonal L(c, c) = pv rs
      a[c] = (r == c) ? pv * rs : a[c] * rs;
      // trailing update of row r: A(r, t) -= L(r, c) L(t, c), c < t <= r
#pragma unroll
      for (int t = c + 1; t < 8; ++t) {
        const double ltc = __shfl_sync(0xffffffffu, a[c], t);  // L(t, c) from lane t
        if (t <= r) a[t] -= a[c] * ltc;
      }
    }
  }
  if (lane < 8 && r < jb) {
#pragma unroll
    for (int t = 0; t < 8; ++t) if (t <= r) Mp[pidx(j0 + r, j0 + t)] = a[t];
  }
  if (lane == 0) *flag = ok;
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  double r = (double)rsqrtf((float)x);
  r = r * fma(-0.5 * x * r, r, 1.5);
  r = r * fma(-0.5 * x * r, r, 1.5);
  return r;
}
__device__ __forceinline__ void chol_diag8_v2(double* Mp, int d, int J, double* rdiag, int* flag) {
  const int lane = threadIdx.x & 31;
  const int j0 = J * 8, jb = min(8, d - j0);
  const int r = lane & 7;
  double a[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) a[t] = (r < jb && t <= r) ? Mp[pidx(j0 + r, j0 + t)] : 0.0;
  int ok = 1;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (c < jb) {
      const double pv = __shfl_sync(0xffffffffu, a[c], c);
      if (!(pv > 0.0)) ok = 0;
      const double rs = ok ? rsqrt_nr(pv) : 0.0;
      if (lane == 0) rdiag[j0 + c] = rs;
      a[c] = (r == c) ? pv * rs : a[c] * rs;
#pragma unroll
      for (int t = c + 1; t < 8; ++t) {
        const double ltc = __shfl_sync(0xffffffffu, a[c], t);
        if (t <= r) a[t] -= a[c] * ltc;
      }
    }
  }
  if (lane < 8 && r < jb) {
#pragma unroll
    for (int t = 0; t < 8; ++t) if (t <= r) Mp[pidx(j0 + r, j0 + t)] = a[t];
  }
  if (lane == 0) *flag = ok;
}

// v3: every lane holds the whole 8 x 8 lower block and factors it
// redundantly (no shuffles; same per-entry operation sequence as v1);
// lane r (< 8) stores row r
__device__ __forceinline__ void chol_diag8_v3(double* Mp, int d, int J, double* rdiag, int* flag) {
  const int lane = threadIdx.x & 31;
  const int j0 = J * 8, jb = min(8, d - j0);
  double a[36];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int t = 0; t <= r; ++t) a[r * (r + 1) / 2 + t] = (r < jb) ? Mp[pidx(j0 + r, j0 + t)] : 0.0;
  int ok = 1;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (c < jb) {
      const double pv = a[c * (c + 1) / 2 + c];
      if (!(pv > 0.0)) ok = 0;
      const double rs = ok ? rsqrt(pv) : 0.0;
      if (lane == 0) rdiag[j0 + c] = rs;
      a[c * (c + 1) / 2 + c] = pv * rs;
#pragma unroll
      for (int r = c + 1; r < 8; ++r) a[r * (r + 1) / 2 + c] *= rs;
#pragma unroll
      for (int r = c + 1; r < 8; ++r)
#pragma unroll
        for (int t = c + 1; t <= r; ++t) a[r * (r + 1) / 2 + t] -= a[r * (r + 1) / 2 + c] * a[t * (t + 1) / 2 + c];
    }
  }
  const int r = lane & 7;
  if (lane < 8 && r < jb) {
#pragma unroll
    for (int rr = 0; rr < 8; ++rr)
      if (rr == r)
#pragma unroll
        for (int t = 0; t <= rr; ++t) Mp[pidx(j0 + rr, j0 + t)] = a[rr * (rr + 1) / 2 + t];
  }
  if (lane == 0) *flag = ok;
}
__global__ void k(int v, double* g, long long* out) {
  __shared__ double Mp[64 * 65 / 2];
  __shared__ double rd[64];
  __shared__ int flag;
  const int d = 64;
  for (int x = threadIdx.x; x < d * (d + 1) / 2; x += blockDim.x) Mp[x] = g[x];
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 50; ++rep) {
    if (v == 0) chol_diag8(Mp, d, rep & 7, rd, &flag); else if (v == 1) chol_diag8_v1(Mp, d, rep & 7, rd, &flag); else if (v == 2) chol_diag8_v2(Mp, d, rep & 7, rd, &flag); else chol_diag8_v3(Mp, d, rep & 7, rd, &flag);
    __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[v] = (t1 - t0) / 50;
  for (int x = threadIdx.x; x < 64; x += blockDim.x) g[4096 + x] = rd[x];
}
int main() {
  const int d = 64;
  static double h[8192];
  for (int i = 0; i < d; ++i) for (int j = 0; j <= i; ++j) h[i * (i + 1) / 2 + j] = (i == j) ? 100.0 + i : 1.0 / (1 + i + j);
  double* g; long long* o; cudaMalloc(&g, 8192 * 8); cudaMalloc(&o, 64);
  double rd0[64], rd1[64], rd2[64], rd3[64];
  for (int v = 0; v < 4; ++v) {
    cudaMemcpy(g, h, 8192 * 8, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(v, g, o);
    cudaDeviceSynchronize();
    cudaMemcpy(v == 3 ? rd3 : v == 2 ? rd2 : (v ? rd1 : rd0), g + 4096, 64 * 8, cudaMemcpyDeviceToHost);
  }
  long long c[4]; cudaMemcpy(c, o, 32, cudaMemcpyDeviceToHost);
  double mx = 0, mx2 = 0, mx3 = 0; for (int i = 0; i < 64; ++i) { mx3 = fmax(mx3, fabs(rd3[i] - rd1[i])); mx = fmax(mx, fabs(rd0[i] - rd1[i])); mx2 = fmax(mx2, fabs(rd0[i] - rd2[i]) / fabs(rd0[i])); }
  printf("diag8 v0 %lld cycles, v1 %lld cycles, v2 %lld cycles, v3 %lld cycles, v1 diff %.3e, v2 rel diff %.3e, v3-v1 diff %.3e\n", c[0], c[1], c[2], c[3], mx, mx2, mx3);
  return 0;
}
