// Microbenchmark (diagnostic): a 16-CTA cluster exchanging 32-double
// partials every repetition, (0) DSMEM push + cluster.sync versus (1) DSMEM
// push + remote mbarrier arrive (release.cluster) + local try_wait.parity.
// Checks the exchanged sums and reports cycles per exchange.
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t ca) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ca) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t a, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
               : "=r"(ok) : "r"(a), "r"(parity) : "memory");
  return ok != 0;
}

__global__ void __launch_bounds__(512, 1) k(int mode, int reps, long long* out, int* err) {
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ __align__(16) double XA[2][16 * 32];
  __shared__ __align__(8) unsigned long long bar[2];
  __shared__ __align__(16) double mine[3][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = (int)cluster.block_rank(), CS = 16;
  if (tid == 0) {
    mbar_init(smem_u32(&bar[0]), CS);
    mbar_init(smem_u32(&bar[1]), CS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster.sync();
  uint32_t ph[2] = {0, 0};
  long long t0 = clock64();
  int bad = 0;
  for (int r = 0; r < reps; ++r) {
    const int s = r & 1;  // alternate buffers / barriers (as two exchange kinds in a step)
    double* X = XA[s];
    if (mode == 2) {
      // pull: publish the own partials locally, barrier, warp w fetches CTA w's
      double* M = mine[r % 3];
      if (warp == 0) M[lane] = 1000.0 * r + 10.0 * b + lane;
      cluster.sync();
      if (warp < CS) X[warp * 32 + lane] = cluster.map_shared_rank(M, warp)[lane];
      __syncthreads();
      double sum = 0.0;
      for (int src = 0; src < CS; ++src) sum += X[src * 32 + lane];
      const double want = 16.0 * (1000.0 * r + lane) + 10.0 * 120.0;
      if (sum != want) bad = 2;
      continue;
    }
    if (warp == 0) {
      const double v = 1000.0 * r + 10.0 * b + lane;
      for (int d = 0; d < CS; ++d) cluster.map_shared_rank(X, d)[b * 32 + lane] = v;
      if (mode == 1) {
        __syncwarp();
        if (lane < CS) mbar_arrive_remote(mapa_u32(smem_u32(&bar[s]), lane));
      }
    }
    if (mode == 0) {
      cluster.sync();
    } else {
      const uint32_t a = smem_u32(&bar[s]);
      int spins = 0;
      while (!mbar_try(a, ph[s])) {
        if (++spins > (1 << 24)) { bad = 1; break; }
      }
      ph[s] ^= 1;
    }
    // every warp checks the sums (the data must be visible)
    double sum = 0.0;
    for (int src = 0; src < CS; ++src) sum += X[src * 32 + lane];
    const double want = 16.0 * (1000.0 * r + lane) + 10.0 * 120.0;
    if (sum != want) bad = 2;
    if (mode == 1) __syncthreads();  // reads of X[s] done before it is rewritten two reps later
  }
  long long t1 = clock64();
  if (tid == 0) out[b] = (t1 - t0) / reps;
  if (bad) atomicExch(err, bad);
  cluster.sync();
}

int main() {
  long long* o; int* e;
  cudaMalloc(&o, 64 * 8); cudaMalloc(&e, 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(e, 0, 4);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16); cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaError_t le = cudaLaunchKernelEx(&cfg, k, mode, 400, o, e);
    cudaError_t se = cudaDeviceSynchronize();
    long long h[16]; int he;
    cudaMemcpy(h, o, 16 * 8, cudaMemcpyDeviceToHost); cudaMemcpy(&he, e, 4, cudaMemcpyDeviceToHost);
    long long mx = 0; for (int i = 0; i < 16; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("mode %d (%s): %lld cycles per exchange, err %d, %s %s\n", mode, mode == 2 ? "pull" : (mode ? "mbarrier" : "cluster.sync"), mx, he,
           cudaGetErrorString(le), cudaGetErrorString(se));
  }
  return 0;
}
