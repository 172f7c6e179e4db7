// K1 for 2 <= k <= 32 columns: Y = M V on the merged CSR (problem.py:311-314
// matmat, :284-289 cost_quad / cost_factor_ip, subqp.py:459), CSR-stream by
// blocks.  A tile is a run of consecutive rows with at most T nonzeros
// (T = 6144 / k, so the products of a tile fit 48 KB of shared memory):
//   1. its column indices and values are staged in shared memory (coalesced);
//   2. the products val[z] * V[col[z], c] are gathered with lane = column c
//      (consecutive lanes read one nonzero's contiguous V row, ~3 nonzeros per
//      warp instruction, every thread keeping 8 gathers in flight) into
//      shared memory;
//   3. each (row, column) pair is summed serially in CSR order (the order of
//      scipy's csr_matvec) and written once.
// Rows above T nonzeros are cut into T-nonzero chunks whose per-column sums
// (a fixed-order tree within the chunk) are added up chunk by chunk, in order,
// by a combine kernel: deterministic, no atomics.
#include <algorithm>
#include <vector>

#include "usbs_common.cuh"
#include "usbs_kernels.cuh"

namespace usbs {

constexpr int SPT_THREADS = 256;
constexpr int SPT_ROWS = 1024;  // rows per tile

static int spmm_tile_nnz(int k) { return std::max(64, std::min(1024, 6144 / k)); }

__global__ void __launch_bounds__(SPT_THREADS) k_spmm_tiles(int ntiles, const int* __restrict__ t_r0,
                                                            const int* __restrict__ t_r1, int nch,
                                                            const int* __restrict__ ch_z0,
                                                            const int* __restrict__ ch_z1,
                                                            const int* __restrict__ rowptr,
                                                            const int* __restrict__ col,
                                                            const double* __restrict__ val,
                                                            const double* __restrict__ V, int64_t ldv, int k,
                                                            double* __restrict__ Y, int64_t ldy,
                                                            double* __restrict__ partial, int T) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* prod = (double*)smem_raw;        // T * k
  double* sval = prod + (size_t)T * k;     // T
  int* scol = (int*)(sval + T);            // T
  const int tid = threadIdx.x;
  const int nzl = SPT_THREADS / k;
  const int zl = tid / k, c = tid - zl * k;
  const bool act = zl < nzl;
  const int b = blockIdx.x;
  int z0, cnt, r0 = 0, r1 = 0;
  if (b < ntiles) {
    r0 = t_r0[b];
    r1 = t_r1[b];
    z0 = rowptr[r0];
    cnt = rowptr[r1] - z0;
  } else {
    z0 = ch_z0[b - ntiles];
    cnt = ch_z1[b - ntiles] - z0;
  }
  for (int z = tid; z < cnt; z += SPT_THREADS) {
    scol[z] = __ldcs(col + z0 + z);
    sval[z] = __ldcs(val + z0 + z);
  }
  __syncthreads();
  if (act) {
    int z = zl;
    for (; z + 7 * nzl < cnt; z += 8 * nzl) {
      double g[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) g[u] = V[(int64_t)scol[z + u * nzl] * ldv + c];
#pragma unroll
      for (int u = 0; u < 8; ++u) prod[(z + u * nzl) * k + c] = sval[z + u * nzl] * g[u];
    }
    for (; z < cnt; z += nzl) prod[z * k + c] = sval[z] * V[(int64_t)scol[z] * ldv + c];
  }
  __syncthreads();
  if (b < ntiles) {
    if (act)
      for (int r = zl; r < r1 - r0; r += nzl) {
        const int a = rowptr[r0 + r] - z0, e = rowptr[r0 + r + 1] - z0;
        double s = 0.0;
        for (int z = a; z < e; ++z) s += prod[z * k + c];
        Y[(int64_t)(r0 + r) * ldy + c] = s;
      }
  } else {
    // chunk of a long row: per-column sums, then the lanes' sums in fixed order
    double s = 0.0;
    if (act)
      for (int z = zl; z < cnt; z += nzl) s += prod[z * k + c];
    __syncthreads();
    if (act) prod[zl * k + c] = s;
    __syncthreads();
    if (tid < k) {
      double t = 0.0;
      for (int q = 0; q < nzl; ++q) t += prod[q * k + tid];
      partial[(int64_t)(b - ntiles) * k + tid] = t;
    }
  }
}

__global__ void k_spmm_chunks_combine(int nh, const int* __restrict__ h_row, const int* __restrict__ h_first,
                                      const int* __restrict__ h_cnt, const double* __restrict__ partial, int k,
                                      double* __restrict__ Y, int64_t ldy) {
  const int64_t tot = (int64_t)nh * k;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(x / k), c = (int)(x % k);
    const int f = h_first[r], n = h_cnt[r];
    double s = 0.0;
    for (int q = 0; q < n; ++q) s += partial[(int64_t)(f + q) * k + c];
    Y[(int64_t)h_row[r] * ldy + c] = s;
  }
}

// tile / chunk lists for a given T, built once per (problem, T) on the host
static void spmm_plan(usbs_problem* p, int T) {
  if (p->spt_T == T) return;
  const std::vector<int32_t>& rp = p->h_rowptr;
  const int64_t n = p->n;
  std::vector<int32_t> r0, r1, cz0, cz1, hrow, hfirst, hcnt;
  int64_t i = 0;
  while (i < n) {
    if (rp[i + 1] - rp[i] > T) {
      hrow.push_back((int32_t)i);
      hfirst.push_back((int32_t)cz0.size());
      int c = 0;
      for (int32_t z = rp[i]; z < rp[i + 1]; z += T, ++c) {
        cz0.push_back(z);
        cz1.push_back(std::min<int32_t>(rp[i + 1], z + T));
      }
      hcnt.push_back(c);
      ++i;
      continue;
    }
    const int64_t s0 = i;
    while (i < n && i - s0 < SPT_ROWS && rp[i + 1] - rp[i] <= T && rp[i + 1] - rp[s0] <= T) ++i;
    r0.push_back((int32_t)s0);
    r1.push_back((int32_t)i);
  }
  p->spt_ntiles = (int)r0.size();
  p->spt_nch = (int)cz0.size();
  p->spt_nhuge = (int)hrow.size();
  p->spt_r0 = dev_upload(p, r0.data(), r0.size());
  p->spt_r1 = dev_upload(p, r1.data(), r1.size());
  p->spt_z0 = dev_upload(p, cz0.data(), cz0.size());
  p->spt_z1 = dev_upload(p, cz1.data(), cz1.size());
  p->spt_hrow = dev_upload(p, hrow.data(), hrow.size());
  p->spt_hfirst = dev_upload(p, hfirst.data(), hfirst.size());
  p->spt_hcnt = dev_upload(p, hcnt.data(), hcnt.size());
  p->spt_T = T;
}

bool spmm_tiles_ok(const usbs_problem* p, int k) {
  const char* e = getenv("USBS_SPMM_V1");
  if (!e) return false;  // A/B only: the v1 warp-per-row kernel is faster at C4 / C5 (profiles/spmm_ab.py)
  return k >= 2 && k <= 32 && (int64_t)p->h_rowptr.size() == p->n + 1 && e[0] == '0';
}

void launch_spmm_tiles(usbs_ctx* ctx, usbs_problem* p, const double* val, const double* V, int64_t ldv, int k,
                       double* Y, int64_t ldy) {
  const int T = spmm_tile_nnz(k);
  spmm_plan(p, T);
  const size_t sm = (size_t)T * k * sizeof(double) + (size_t)T * (sizeof(double) + sizeof(int));
  smem_optin(ctx, (const void*)k_spmm_tiles, (int)sm);
  double* part = p->spt_nch ? (double*)ctx->ws.get(WS_SPMM_PARTIAL + 100, (size_t)p->spt_nch * k * sizeof(double))
                            : nullptr;
  const int nb = p->spt_ntiles + p->spt_nch;
  if (nb > 0) {
    k_spmm_tiles<<<nb, SPT_THREADS, sm, ctx->stream>>>(p->spt_ntiles, p->spt_r0, p->spt_r1, p->spt_nch, p->spt_z0,
                                                       p->spt_z1, p->rowptr, p->col, val, V, ldv, k, Y, ldy, part, T);
    check_launch(ctx);
  }
  if (p->spt_nhuge) {
    const int64_t tot = (int64_t)p->spt_nhuge * k;
    const int bl = (int)std::min<int64_t>((tot + 255) / 256, 4 * ctx->num_sms);
    k_spmm_chunks_combine<<<std::max(bl, 1), 256, 0, ctx->stream>>>(p->spt_nhuge, p->spt_hrow, p->spt_hfirst,
                                                                     p->spt_hcnt, part, k, Y, ldy);
    check_launch(ctx);
  }
}

}  // namespace usbs
