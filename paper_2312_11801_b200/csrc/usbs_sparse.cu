// Context, problem upload, slack assembly (Z = C - A*(y)) and the
// operator apply Y = M V (K1) with an optional V^T Y Gram epilogue.
//
// Reference behaviour replaced (paths under /root/reference/pkg/src/specbundle):
//   problem.py:311-314  dual_slack_operator: CSR of C - A*(y) rebuilt per call,
//                       matvec/matmat through scipy _sparsetools csr_matvec(s)
//   problem.py:160-161, 214-220  adjoint_matrix (diag / entry families)
//   problem.py:284-286  cost_quad = sym(V^T C V)
//   subqp.py:459        V^T A*(y) V - V^T C V  (= -sym(V^T Z V))
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>

#include "usbs_common.cuh"
#include "usbs_kernels.cuh"

// std::allocator whose value construction default-initialises (no zero fill
// for arithmetic types): for host arrays that are written completely anyway
template <typename T>
struct DefaultInitAlloc : std::allocator<T> {
  template <typename U>
  struct rebind {
    using other = DefaultInitAlloc<U>;
  };
  DefaultInitAlloc() = default;
  template <typename U>
  DefaultInitAlloc(const DefaultInitAlloc<U>&) {}
  template <typename U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <typename U, typename... Args>
  void construct(U* p, Args&&... args) {
    ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
  }
};

namespace usbs {
void staged_h2d(usbs_ctx* ctx, void* dst, const void* src, size_t bytes) {
  constexpr size_t CH = 8u << 20;
  if (bytes <= (1u << 20)) {
    USBS_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
    return;
  }
  for (int k = 0; k < 2; ++k)
    if (!ctx->stage[k]) {
      USBS_CUDA(cudaMallocHost(&ctx->stage[k], CH));
      USBS_CUDA(cudaEventCreateWithFlags(&ctx->stage_ev[k], cudaEventDisableTiming));
    }
  size_t off = 0;
  int k = 0;
  while (off < bytes) {
    const size_t len = std::min(CH, bytes - off);
    USBS_CUDA(cudaEventSynchronize(ctx->stage_ev[k]));  // the chunk's previous copy has drained
    std::memcpy(ctx->stage[k], (const unsigned char*)src + off, len);
    USBS_CUDA(cudaMemcpyAsync((unsigned char*)dst + off, ctx->stage[k], len, cudaMemcpyHostToDevice, ctx->stream));
    USBS_CUDA(cudaEventRecord(ctx->stage_ev[k], ctx->stream));
    off += len;
    k ^= 1;
  }
  USBS_CUDA(cudaStreamSynchronize(ctx->stream));
}
}  // namespace usbs

namespace usbs {

static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }

// ----------------------------------------------------------------- assembly
// zval[s] = cval[s] - sum_{e in slot s} y[idx[e]] * val[e]   (problem.py:313)
__global__ void k_slack_assemble(int64_t nnz, const double* __restrict__ cval,
                                 const int* __restrict__ aptr, const int* __restrict__ aent,
                                 const int* __restrict__ eidx, const double* __restrict__ eval,
                                 const double* __restrict__ y, double* __restrict__ zval) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nnz;
       s += (int64_t)gridDim.x * blockDim.x) {
    int a = aptr[s], b = aptr[s + 1];
    double acc = 0.0;
    for (int t = a; t < b; ++t) {
      int e = aent[t];
      acc += y[eidx[e]] * eval[e];
    }
    zval[s] = (a == b) ? cval[s] : cval[s] - acc;
  }
}

// diag_only fast path: copy C values, then overwrite the n diagonal slots
__global__ void k_slack_diag(int64_t n, const int* __restrict__ dslot, const double* __restrict__ cval,
                             const double* __restrict__ y, double* __restrict__ zval) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int s = dslot[i];
    zval[s] = cval[s] - y[i];
  }
}

// ----------------------------------------------------------------- SpMM
// Y[row, :] = sum_nz M[row, col] * V[col, :], one LG-lane group per item,
// lane t owns output column t (column chunks of LG for k > LG).
template <int LG>
__global__ void __launch_bounds__(256) k_spmm(int n_items, const int* __restrict__ it_row,
                                              const int* __restrict__ it_beg,
                                              const int* __restrict__ it_end,
                                              const int* __restrict__ it_slot,
                                              const int* __restrict__ col,
                                              const double* __restrict__ val,
                                              const double* __restrict__ V, int64_t ldv, int k,
                                              double* __restrict__ Y, int64_t ldy,
                                              double* __restrict__ partial) {
  const int groups_per_block = blockDim.x / LG;
  const int g = threadIdx.x / LG, t = threadIdx.x % LG;
  for (int it = blockIdx.x * groups_per_block + g; it < n_items; it += gridDim.x * groups_per_block) {
    const int row = it_row[it], b = it_beg[it], e = it_end[it], slot = it_slot[it];
    for (int c0 = 0; c0 < k; c0 += LG) {
      const int c = c0 + t;
      const bool on = c < k;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int z = b;
      for (; z + 4 <= e; z += 4) {
        int j0 = col[z], j1 = col[z + 1], j2 = col[z + 2], j3 = col[z + 3];
        double v0 = val[z], v1 = val[z + 1], v2 = val[z + 2], v3 = val[z + 3];
        if (on) {
          a0 = fma(v0, V[(int64_t)j0 * ldv + c], a0);
          a1 = fma(v1, V[(int64_t)j1 * ldv + c], a1);
          a2 = fma(v2, V[(int64_t)j2 * ldv + c], a2);
          a3 = fma(v3, V[(int64_t)j3 * ldv + c], a3);
        }
      }
      for (; z < e; ++z) {
        int j0 = col[z];
        double v0 = val[z];
        if (on) a0 = fma(v0, V[(int64_t)j0 * ldv + c], a0);
      }
      double acc = (a0 + a1) + (a2 + a3);
      if (on) {
        if (slot < 0) Y[(int64_t)row * ldy + c] = acc;
        else partial[(int64_t)slot * k + c] = acc;
      }
    }
  }
}

// k = 1: rows longer than SHORT_ROW nonzeros get a warp (<= 256) or a block
// (> 256); the short ones go through CSR-stream tiles.
constexpr int SHORT_ROW = 32;

// CSR-stream tiles: the tile's nonzeros are read fully coalesced (one per
// thread, 8 in flight), their products staged in shared memory, then one
// thread per row sums its products in column order (a sequential CSR loop's
// order).
constexpr int ST_ROWS = 1024;  // rows per tile (empty rows add no nonzeros)

// All of a k = 1 apply in ONE launch, block roles by blockIdx (huge rows
// first so they never form the tail): [0, H) one block per row with more
// than ST_NNZ nonzeros (thread-strided partial sums, fixed-order block
// tree); then the CSR-stream tiles, each a run of consecutive rows with at
// most ST_NNZ nonzeros in total; inside a tile a thread sums each short row
// (<= SHORT_ROW) and a warp each longer one.  Deterministic, no atomics.
template <int ST_NNZ, int ST_THREADS, int MINB>
__global__ void __launch_bounds__(ST_THREADS, MINB) k_spmv_fused(int nhuge, const int* __restrict__ huge_rows, int ntiles,
                                                    const int* __restrict__ tile_r0, const int* __restrict__ tile_r1,
                                                    const int* __restrict__ rowptr, const int* __restrict__ col,
                                                    const double* __restrict__ val, const double* __restrict__ x,
                                                    int64_t ldx, double* __restrict__ y, int64_t ldy) {
  __shared__ double prod[ST_NNZ];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int b = blockIdx.x;
  if (b < nhuge) {
    const int r = __ldg(huge_rows + b);
    const int zb = __ldg(rowptr + r), ze = __ldg(rowptr + r + 1);
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    for (int z0 = zb; z0 < ze; z0 += ST_THREADS * 4) {
      int cc[4];
      double vv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int z = z0 + tid + ST_THREADS * u;
        cc[u] = z < ze ? __ldcg(col + z) : -1;
        vv[u] = z < ze ? __ldcg(val + z) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (cc[u] >= 0) a[u & 3] = fma(vv[u], __ldg(x + (int64_t)cc[u] * ldx), a[u & 3]);
    }
    double s = warp_sum((a[0] + a[1]) + (a[2] + a[3]));
    if (lane == 0) prod[warp] = s;
    __syncthreads();
    if (warp == 0) {
      s = lane < ST_THREADS / 32 ? prod[lane] : 0.0;
      s = warp_sum(s);
      if (lane == 0) y[(int64_t)r * ldy] = s;
    }
    return;
  }
  b -= nhuge;
  if (b >= ntiles) return;
  __shared__ int rps[ST_ROWS + 1];  // tile row pointers relative to base
  __shared__ int longl[ST_ROWS];    // tile rows longer than SHORT_ROW
  __shared__ int nlong;
  const int r0 = __ldg(tile_r0 + b), r1 = __ldg(tile_r1 + b);
  const int base = __ldg(rowptr + r0), cnt = __ldg(rowptr + r1) - base;
  int cc[ST_NNZ / ST_THREADS];
  double vv[ST_NNZ / ST_THREADS];
#pragma unroll
  for (int u = 0; u < ST_NNZ / ST_THREADS; ++u) {
    const int z = tid + u * ST_THREADS;
    cc[u] = z < cnt ? __ldcg(col + base + z) : 0;
    vv[u] = z < cnt ? __ldcg(val + base + z) : 0.0;
  }
  for (int i = tid; i <= r1 - r0; i += ST_THREADS) rps[i] = __ldg(rowptr + r0 + i) - base;
  if (tid == 0) nlong = 0;
#pragma unroll
  for (int u = 0; u < ST_NNZ / ST_THREADS; ++u) {
    const int z = tid + u * ST_THREADS;
    if (z < cnt) prod[z] = vv[u] * __ldg(x + (int64_t)cc[u] * ldx);
  }
  __syncthreads();
  for (int il = tid; il < r1 - r0; il += ST_THREADS) {
    const int bb = rps[il], e = rps[il + 1];
    if (e - bb > SHORT_ROW) {
      longl[atomicAdd(&nlong, 1)] = il;  // list order is irrelevant: one row, one sum
      continue;
    }
    double s = 0.0;
    for (int z = bb; z < e; ++z) s += prod[z];
    y[(int64_t)(r0 + il) * ldy] = s;
  }
  __syncthreads();
  for (int t = warp; t < nlong; t += ST_THREADS / 32) {
    const int il = longl[t];
    const int bb = rps[il], e = rps[il + 1];
    double s = 0.0;
    for (int z = bb + lane; z < e; z += 32) s += prod[z];
    s = warp_sum(s);
    if (lane == 0) y[(int64_t)(r0 + il) * ldy] = s;
  }
}

// SpMM for 2 <= k <= 16: a warp per row segment, two 16-lane slots each
// taking every other nonzero (lane c of a slot owns column c), 4 nonzeros
// per slot in flight; slots are combined with one shuffle.
__global__ void __launch_bounds__(256) k_spmm16x2(int n_items, const int* __restrict__ it_row,
                                                  const int* __restrict__ it_beg, const int* __restrict__ it_end,
                                                  const int* __restrict__ it_slot, const int* __restrict__ col,
                                                  const double* __restrict__ val, const double* __restrict__ V,
                                                  int64_t ldv, int k, double* __restrict__ Y, int64_t ldy,
                                                  double* __restrict__ partial) {
  const int lane = threadIdx.x & 31, s = lane >> 4, c = lane & 15;
  const bool on = c < k;
  const int warps_total = (gridDim.x * blockDim.x) >> 5;
  for (int it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < n_items; it += warps_total) {
    const int b = __ldg(it_beg + it), e = __ldg(it_end + it);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int z = b + s;
    for (; z + 6 < e; z += 8) {
      const int j0 = __ldg(col + z), j1 = __ldg(col + z + 2), j2 = __ldg(col + z + 4), j3 = __ldg(col + z + 6);
      const double v0 = __ldg(val + z), v1 = __ldg(val + z + 2), v2 = __ldg(val + z + 4), v3 = __ldg(val + z + 6);
      if (on) {
        a0 = fma(v0, __ldg(V + (int64_t)j0 * ldv + c), a0);
        a1 = fma(v1, __ldg(V + (int64_t)j1 * ldv + c), a1);
        a2 = fma(v2, __ldg(V + (int64_t)j2 * ldv + c), a2);
        a3 = fma(v3, __ldg(V + (int64_t)j3 * ldv + c), a3);
      }
    }
    for (; z < e; z += 2) {
      const int j0 = __ldg(col + z);
      const double v0 = __ldg(val + z);
      if (on) a0 = fma(v0, __ldg(V + (int64_t)j0 * ldv + c), a0);
    }
    double acc = (a0 + a1) + (a2 + a3);
    acc += __shfl_xor_sync(0xffffffffu, acc, 16);
    if (s == 0 && on) {
      const int sl = __ldg(it_slot + it);
      if (sl < 0) Y[(int64_t)__ldg(it_row + it) * ldy + c] = acc;
      else partial[(int64_t)sl * k + c] = acc;
    }
  }
}

// combine the partials of split rows in a fixed order (deterministic)

// 2 <= k <= 15: G-lane groups (G = 3, 4, 6, 8 for k <= 5, 7, 11, 15), 32/G
// items per warp at once (the per-item index, col/val and V round trips of
// several rows overlap).  A group gathers a row of V with 16-byte loads: the
// k (+1) doubles from the row start rounded down to 16 bytes, lane c of the
// group holding window elements 2c, 2c+1 -- columns 2c - s, 2c + 1 - s,
// where s is the row start's 8-byte parity.  Products accumulate per parity
// (even: ae0/ae1, odd: ao0/ao1); column 2c = ae0 + ao1 of lane c and column
// 2c+1 = ae1 of lane c + ao0 of lane c+1, each parity summed in CSR order.
// Any ldv; V's base 16-byte aligned (the launcher checks), so no window
// starts before V's first entry; vend = elements of V that may be read.
template <int G>
__global__ void __launch_bounds__(256) k_spmm_g(int n_items, const int* __restrict__ it_row,
                                                const int* __restrict__ it_beg, const int* __restrict__ it_end,
                                                const int* __restrict__ it_slot, const int* __restrict__ col,
                                                const double* __restrict__ val, const double* __restrict__ V,
                                                int64_t ldv, int64_t vend, int k, double* __restrict__ Y,
                                                int64_t ldy, double* __restrict__ partial) {
  constexpr int NG = 32 / G;
  const int lane = threadIdx.x & 31, g = lane / G, c = lane % G;
  const bool live = g < NG;
  const int warps_total = (gridDim.x * blockDim.x) >> 5;
  const uintptr_t vb = (uintptr_t)V;
  for (int it0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * NG; it0 < n_items; it0 += warps_total * NG) {
    const int it = it0 + g;
    const bool on = live && it < n_items;
    int b = 0, e = 0;
    if (on) { b = __ldg(it_beg + it); e = __ldg(it_end + it); }
    double ae0 = 0.0, ae1 = 0.0, ao0 = 0.0, ao1 = 0.0;
    int len = e - b;
    // warp-uniform trip count: the longest item of the warp
    int mx = len;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    for (int u = 0; u < mx; u += 2) {
      const bool h0 = u < len, h1 = u + 1 < len;
      const int j0 = h0 ? __ldg(col + b + u) : 0, j1 = h1 ? __ldg(col + b + u + 1) : 0;
      const double v0 = h0 ? __ldg(val + b + u) : 0.0, v1 = h1 ? __ldg(val + b + u + 1) : 0.0;
      const int64_t r0 = (int64_t)j0 * ldv, r1 = (int64_t)j1 * ldv;
      const int s0 = (int)(((vb >> 3) + r0) & 1), s1 = (int)(((vb >> 3) + r1) & 1);
      const int64_t w0 = r0 - s0 + 2 * c, w1 = r1 - s1 + 2 * c;  // window element of this lane
      double2 x0 = make_double2(0.0, 0.0), x1 = make_double2(0.0, 0.0);
      if (h0 && 2 * c - s0 < k) {
        if (w0 + 1 < vend) x0 = __ldg(reinterpret_cast<const double2*>(V + w0));
        else if (w0 >= 0 && w0 < vend) x0.x = __ldg(V + w0);
      }
      if (h1 && 2 * c - s1 < k) {
        if (w1 + 1 < vend) x1 = __ldg(reinterpret_cast<const double2*>(V + w1));
        else if (w1 >= 0 && w1 < vend) x1.x = __ldg(V + w1);
      }
      if (h0) {
        if (s0) { ao0 = fma(v0, x0.x, ao0); ao1 = fma(v0, x0.y, ao1); }
        else { ae0 = fma(v0, x0.x, ae0); ae1 = fma(v0, x0.y, ae1); }
      }
      if (h1) {
        if (s1) { ao0 = fma(v1, x1.x, ao0); ao1 = fma(v1, x1.y, ao1); }
        else { ae0 = fma(v1, x1.x, ae0); ae1 = fma(v1, x1.y, ae1); }
      }
    }
    const double nxt = __shfl_down_sync(0xffffffffu, ao0, 1);  // lane c+1's odd-parity column 2c+1
    if (on) {
      const int c0 = 2 * c, c1 = 2 * c + 1;
      const double y0 = ae0 + ao1;
      const double y1 = ae1 + (c + 1 < G ? nxt : 0.0);
      const int sl = __ldg(it_slot + it);
      double* out = sl < 0 ? Y + (int64_t)__ldg(it_row + it) * ldy : partial + (int64_t)sl * k;
      if (c0 < k) out[c0] = y0;
      if (c1 < k) out[c1] = y1;
    }
  }
}

__global__ void k_spmm_combine(int n_sr, const int* __restrict__ sr_row, const int* __restrict__ sr_first,
                               const int* __restrict__ sr_count, const double* __restrict__ partial,
                               int k, double* __restrict__ Y, int64_t ldy) {
  int64_t total = (int64_t)n_sr * k;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    int r = (int)(x / k), c = (int)(x % k);
    int f = sr_first[r], cnt = sr_count[r];
    double acc = 0.0;
    for (int s = 0; s < cnt; ++s) acc += partial[(int64_t)(f + s) * k + c];
    Y[(int64_t)sr_row[r] * ldy + c] = acc;
  }
}

// ---------------------------------------------------------------- host helpers
static int pick_group(double avg) {
  int g = 4;
  while (g < 32 && g < avg) g <<= 1;
  return g;
}

}  // namespace usbs

using namespace usbs;

extern "C" {

int usbs_abi_version(void) { return USBS_ABI_VERSION; }

const char* usbs_last_error(void) { return g_err.c_str(); }

usbs_status usbs_ctx_create(int device, void* stream, usbs_ctx** out) {
  USBS_API_BEGIN
  if (!out) fail(USBS_ERR_CONFIG, "null output pointer");
  USBS_CUDA(cudaSetDevice(device));
  auto* c = new usbs_ctx();
  c->device = device;
  // NULL is the legacy default stream (what torch reports for its default
  // stream), so work stays ordered with the caller's tensor operations
  c->stream = (cudaStream_t)stream;
  cudaDeviceProp prop;
  USBS_CUDA(cudaGetDeviceProperties(&prop, device));
  c->num_sms = prop.multiProcessorCount;
  USBS_CUDA(cudaMallocHost(&c->pinned, 4096 * sizeof(double)));
  USBS_CUDA(cudaMallocHost(&c->pinned_i, 256 * sizeof(int)));
  *out = c;
  USBS_API_END
}

usbs_status usbs_ctx_destroy(usbs_ctx* c) {
  USBS_API_BEGIN
  if (!c) return USBS_OK;
  cudaStreamSynchronize(c->stream);
  c->ws.release();
  for (int k = 0; k < 2; ++k) {
    if (c->stage[k]) cudaFreeHost(c->stage[k]);
    if (c->stage_ev[k]) cudaEventDestroy(c->stage_ev[k]);
  }
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->pinned_i) cudaFreeHost(c->pinned_i);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
  USBS_API_END
}

usbs_status usbs_ctx_sync(usbs_ctx* c) {
  USBS_API_BEGIN
  USBS_CUDA(cudaStreamSynchronize(c->stream));
  USBS_API_END
}

int64_t usbs_ctx_launches(usbs_ctx* c) { return c ? c->launches : -1; }

usbs_status usbs_memcpy_h2d(usbs_ctx* c, void* dst, const void* src, int64_t bytes) {
  USBS_API_BEGIN
  if (bytes > 0) {
    USBS_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, c->stream));
    USBS_CUDA(cudaStreamSynchronize(c->stream));
  }
  USBS_API_END
}

usbs_status usbs_memcpy_d2h(usbs_ctx* c, void* dst, const void* src, int64_t bytes) {
  USBS_API_BEGIN
  if (bytes > 0) {
    USBS_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost, c->stream));
    USBS_CUDA(cudaStreamSynchronize(c->stream));
  }
  USBS_API_END
}


static void create_problem(usbs_ctx* ctx, int64_t n, int64_t n_cols, int64_t m, const int64_t* c_indptr,
                           const int32_t* c_indices, const double* c_data, int64_t ne, const int64_t* e_idx,
                           const int64_t* e_rows, const int64_t* e_cols, const double* e_vals, int diag_only,
                           int directed, usbs_problem** out);

usbs_status usbs_problem_create(usbs_ctx* ctx, int64_t n, int64_t m, const int64_t* c_indptr,
                                const int32_t* c_indices, const double* c_data, int64_t ne,
                                const int64_t* e_idx, const int64_t* e_rows, const int64_t* e_cols,
                                const double* e_vals, int diag_only, usbs_problem** out) {
  USBS_API_BEGIN
  create_problem(ctx, n, n, m, c_indptr, c_indices, c_data, ne, e_idx, e_rows, e_cols, e_vals, diag_only, 0, out);
  USBS_API_END
}

usbs_status usbs_problem_create_shard(usbs_ctx* ctx, int64_t n_rows, int64_t n_cols, int64_t m,
                                      const int64_t* c_indptr, const int32_t* c_indices, const double* c_data,
                                      int64_t ne, const int64_t* e_idx, const int64_t* e_rows,
                                      const int64_t* e_cols, const double* e_vals, int diag_only,
                                      usbs_problem** out) {
  USBS_API_BEGIN
  create_problem(ctx, n_rows, n_cols, m, c_indptr, c_indices, c_data, ne, e_idx, e_rows, e_cols, e_vals, diag_only, 1,
                 out);
  USBS_API_END
}

static void create_problem(usbs_ctx* ctx, int64_t n, int64_t n_cols, int64_t m, const int64_t* c_indptr,
                           const int32_t* c_indices, const double* c_data, int64_t ne, const int64_t* e_idx,
                           const int64_t* e_rows, const int64_t* e_cols, const double* e_vals, int diag_only,
                           int directed, usbs_problem** out) {
  if (!ctx || !out) fail(USBS_ERR_CONFIG, "null context/output");
  if (n < 1 || n_cols < 1 || m < 0 || ne < 0) fail(USBS_ERR_SHAPE, "invalid problem dimensions");
  if (n >= (1LL << 31) - 1 || n_cols >= (1LL << 31) - 1) fail(USBS_ERR_SHAPE, "n exceeds int32 indexing");
  USBS_CUDA(cudaSetDevice(ctx->device));
  // USBS_PLAN_PROF=1: host planning phase times on stderr
  const bool tprof = getenv("USBS_PLAN_PROF") != nullptr;
  auto tlast = std::chrono::steady_clock::now();
  auto PT = [&](const char* what) {
    if (!tprof) return;
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[plan] %-28s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - tlast).count());
    tlast = now;
  };
  auto* p = new usbs_problem();
  p->ctx = ctx;
  p->n = n;
  p->n_cols = n_cols;
  p->m = m;
  p->ne = ne;
  p->diag_only = diag_only != 0;
  p->nnz_c = c_indptr[n];

  // --- extra (row, col, entry, role) pairs from the constraint entries
  // (square problems mirror off-diagonal entries; shard problems receive the
  // directed entries of their own rows, with global columns)
  std::vector<int64_t> xcnt(n + 1, 0);
  for (int64_t e = 0; e < ne; ++e) {
    int64_t r = e_rows[e], c = e_cols[e], ci = e_idx[e];
    if (r < 0 || c < 0 || r >= n || c >= n_cols || (!directed && r > c))
      fail(USBS_ERR_SHAPE, "constraint entry out of range or rows > cols");
    if (ci < 0 || ci >= m) fail(USBS_ERR_SHAPE, "constraint index out of range");
    xcnt[r + 1]++;
    if (!directed && r != c) xcnt[c + 1]++;
  }
  for (int64_t i = 0; i < n; ++i) xcnt[i + 1] += xcnt[i];
  std::vector<int32_t> xcol(xcnt[n]);
  std::vector<int64_t> xent(xcnt[n]);
  std::vector<int64_t> xpos_r(ne), xpos_c(ne, -1);  // x-positions of each entry (slot -> entries below)
  {
    std::vector<int64_t> pos(xcnt.begin(), xcnt.end() - 1);
    for (int64_t e = 0; e < ne; ++e) {
      int64_t r = e_rows[e], c = e_cols[e];
      xpos_r[e] = pos[r];
      xcol[pos[r]] = (int32_t)c;
      xent[pos[r]++] = e;
      if (!directed && r != c) {
        xpos_c[e] = pos[c];
        xcol[pos[c]] = (int32_t)r;
        xent[pos[c]++] = e;
      }
    }
  }
  PT("constraint entries -> rows");
  // --- merge per row: C columns (sorted, duplicates summed) with the extra
  // columns.  Two passes over row ranges on host threads: merged lengths,
  // then the merged pattern written in place (same result as a serial merge).
  std::vector<int64_t> rowptr(n + 1, 0);
  std::vector<int64_t> slot_of_x(xcnt[n]);
  const int nthr = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(16u, std::max(1u, std::thread::hardware_concurrency())),
                                                              n / 4096 + 1));
  // merged columns / values: filled completely below, so not zero-initialised
  std::vector<int32_t, DefaultInitAlloc<int32_t>> col;
  std::vector<double, DefaultInitAlloc<double>> cval;
  {
    std::vector<std::string> errs(nthr);
    auto merge_rows = [&](int th, int64_t i0, int64_t i1, bool write) {
      std::vector<std::pair<int32_t, double>> crow;
      std::vector<std::pair<int32_t, int64_t>> xrow;
      for (int64_t i = i0; i < i1; ++i) {
        crow.clear();
        for (int64_t z = c_indptr[i]; z < c_indptr[i + 1]; ++z) {
          if (c_indices[z] < 0 || c_indices[z] >= n_cols) {
            errs[th] = "cost column index out of range";
            return;
          }
          crow.emplace_back(c_indices[z], c_data[z]);
        }
        if (!std::is_sorted(crow.begin(), crow.end(), [](auto& a, auto& b) { return a.first < b.first; }))
          std::stable_sort(crow.begin(), crow.end(), [](auto& a, auto& b) { return a.first < b.first; });
        xrow.clear();
        for (int64_t t = xcnt[i]; t < xcnt[i + 1]; ++t) xrow.emplace_back(xcol[t], t);
        if (xrow.size() > 1)
          std::stable_sort(xrow.begin(), xrow.end(), [](auto& a, auto& b) { return a.first < b.first; });
        size_t a = 0, b = 0;
        int64_t o = write ? rowptr[i] : 0;
        while (a < crow.size() || b < xrow.size()) {
          int32_t cc = INT32_MAX;
          if (a < crow.size()) cc = crow[a].first;
          if (b < xrow.size()) cc = std::min(cc, xrow[b].first);
          double v = 0.0;
          while (a < crow.size() && crow[a].first == cc) v += crow[a++].second;  // duplicate C entries summed
          while (b < xrow.size() && xrow[b].first == cc) {
            if (write) slot_of_x[xrow[b].second] = o;
            ++b;
          }
          if (write) {
            col[o] = cc;
            cval[o] = v;
          }
          ++o;
        }
        if (!write) rowptr[i + 1] = o;  // row length (prefix-summed below)
      }
    };
    auto run = [&](bool write) {
      std::vector<std::thread> ts;
      for (int th = 0; th < nthr; ++th) {
        const int64_t i0 = n * th / nthr, i1 = n * (th + 1) / nthr;
        ts.emplace_back(merge_rows, th, i0, i1, write);
      }
      for (auto& t : ts) t.join();
      for (auto& e : errs)
        if (!e.empty()) fail(USBS_ERR_SHAPE, e);
    };
    // diagonal constraints (one x-entry per row, column i) with sorted cost
    // rows without duplicates: the merged row is the cost row with the
    // diagonal inserted -- no per-row sort
    bool fast = diag_only && !directed;
    if (fast) {
      // one threaded pass: rows strictly increasing (sorted, no duplicates),
      // columns in range, merged row lengths (the diagonal added if absent)
      std::vector<char> ok(nthr, 1), inrange(nthr, 1);
      auto scan = [&](int th, int64_t i0, int64_t i1) {
        for (int64_t i = i0; i < i1; ++i) {
          bool has = false;
          for (int64_t z = c_indptr[i]; z < c_indptr[i + 1]; ++z) {
            const int32_t c = c_indices[z];
            if (c < 0 || c >= n_cols) inrange[th] = 0;
            if (z > c_indptr[i] && c <= c_indices[z - 1]) ok[th] = 0;
            has |= (c == i);
          }
          rowptr[i + 1] = (c_indptr[i + 1] - c_indptr[i]) + (has ? 0 : 1);
        }
      };
      std::vector<std::thread> ts;
      for (int th = 0; th < nthr; ++th) ts.emplace_back(scan, th, n * th / nthr, n * (th + 1) / nthr);
      for (auto& t : ts) t.join();
      for (int th = 0; th < nthr; ++th) {
        if (!inrange[th]) fail(USBS_ERR_SHAPE, "cost column index out of range");
        fast = fast && ok[th];
      }
    }
    if (fast) {
      for (int64_t i = 0; i < n; ++i) rowptr[i + 1] += rowptr[i];
      col.resize(rowptr[n]);
      cval.resize(rowptr[n]);
      auto fill = [&](int64_t i0, int64_t i1) {
        for (int64_t i = i0; i < i1; ++i) {
          int64_t o = rowptr[i];
          bool put = false;
          for (int64_t z = c_indptr[i]; z < c_indptr[i + 1]; ++z) {
            const int32_t c = c_indices[z];
            if (c < 0 || c >= n_cols) continue;  // reported below
            if (!put && c >= i) {
              if (c != i) { col[o] = (int32_t)i; cval[o] = 0.0; ++o; }
              slot_of_x[xcnt[i]] = c == i ? o : o - 1;
              put = true;
            }
            col[o] = c;
            cval[o] = c_data[z];
            ++o;
          }
          if (!put) {
            slot_of_x[xcnt[i]] = o;
            col[o] = (int32_t)i;
            cval[o] = 0.0;
          }
        }
      };
      std::vector<std::thread> ts;
      for (int th = 0; th < nthr; ++th) ts.emplace_back(fill, n * th / nthr, n * (th + 1) / nthr);
      for (auto& t : ts) t.join();
    } else {
      std::fill(rowptr.begin(), rowptr.end(), 0);
      run(false);
      for (int64_t i = 0; i < n; ++i) rowptr[i + 1] += rowptr[i];
      col.resize(rowptr[n]);
      cval.resize(rowptr[n]);
      run(true);
    }
  }
  PT("merge C with the entries");
  p->nnz = (int64_t)col.size();
  if (p->nnz >= (1LL << 31) - 1) fail(USBS_ERR_SHAPE, "nnz exceeds int32 indexing");
  // --- slot -> entries (ascending entry id within a slot): counting pass
  // over the entries in order
  // (diagonal problems: built lazily on the device, ensure_slot_lists --
  // only the constraint duck type's adjoint evaluations read them)
  const bool lazy_slots = diag_only && !directed;
  std::vector<int32_t> aptr(lazy_slots ? 1 : p->nnz + 1, 0);
  if (!lazy_slots) {
    for (int64_t t = 0; t < (int64_t)slot_of_x.size(); ++t) aptr[slot_of_x[t] + 1]++;
    for (int64_t s = 0; s < p->nnz; ++s) aptr[s + 1] += aptr[s];
  }
  std::vector<int32_t> aent(lazy_slots ? 0 : aptr[p->nnz]);
  if (!lazy_slots) {
    std::vector<int32_t> cur(aptr.begin(), aptr.end() - 1);
    for (int64_t e = 0; e < ne; ++e) {
      aent[cur[slot_of_x[xpos_r[e]]]++] = (int32_t)e;
      if (xpos_c[e] >= 0) aent[cur[slot_of_x[xpos_c[e]]]++] = (int32_t)e;
    }
  }
  PT("slot -> entries");
  std::vector<int32_t> rp32(n + 1);
  for (int64_t i = 0; i <= n; ++i) rp32[i] = (int32_t)rowptr[i];

  // --- work items (row segments)
  double avg = (double)p->nnz / (double)n;
  p->spmv_group = pick_group(avg);
  const int SEG = 16 * p->spmv_group;
  std::vector<int32_t> irow, ibeg, iend, islot, srow, sfirst, scount;
  {
    const size_t cap = (size_t)n + (size_t)(p->nnz / SEG) + 16;  // one item per row plus the extra pieces of split rows
    irow.reserve(cap); ibeg.reserve(cap); iend.reserve(cap); islot.reserve(cap);
  }
  int nsplit = 0;
  for (int64_t i = 0; i < n; ++i) {
    int32_t b = rp32[i], e = rp32[i + 1];
    if (e - b <= SEG) {
      irow.push_back((int32_t)i); ibeg.push_back(b); iend.push_back(e); islot.push_back(-1);
    } else {
      srow.push_back((int32_t)i); sfirst.push_back(nsplit);
      int cnt = 0;
      for (int32_t z = b; z < e; z += SEG) {
        irow.push_back((int32_t)i); ibeg.push_back(z); iend.push_back(std::min(e, z + SEG));
        islot.push_back(nsplit++); cnt++;
      }
      scount.push_back(cnt);
    }
  }
  p->n_items = (int)irow.size();
  p->n_split_items = nsplit;
  p->n_split_rows = (int)srow.size();

  PT("SpMM work items");
  // --- Lanczos grid partition: rows for the Q passes, SpMV segments apart
  // leave 4 SMs free for kernels that overlap the Lanczos kernel (the
  // model-evaluation IPM on the auxiliary stream)
  int G = (int)std::min<int64_t>(std::max(1, ctx->num_sms - 4),
                                 std::max<int64_t>(1, std::max<int64_t>((n + 63) / 64, (p->nnz + n + 4095) / 4096)));
  if (const char* env = getenv("USBS_LZ_BLOCKS")) G = std::max(1, std::min(ctx->num_sms, atoi(env)));
  p->lz_blocks = G;
  std::vector<int32_t> blk_row(G + 1, (int32_t)n), blk_seg(G + 1, 0), seg_r0, seg_r1;
  {
    // rows (the CGS2 passes over Q): balanced on rows; the SpMV runs in its
    // own phase, so its segments are balanced separately on nonzeros
    const double NNZCOST = 0.0;  // the Q passes cost per row only (measured, C4)
    double total = (double)n + NNZCOST * (double)p->nnz;
    double acc = 0.0;
    int b = 0;
    blk_row[0] = 0;
    for (int64_t i = 0; i < n && b + 1 < G; ++i) {
      acc += 1.0 + NNZCOST * (rp32[i + 1] - rp32[i]);
      if (acc >= total * (b + 1) / G) blk_row[++b] = (int32_t)(i + 1);
    }
    for (int bb = b + 1; bb < G; ++bb) blk_row[bb] = (int32_t)n;
    blk_row[G] = (int32_t)n;
    // align the boundaries to the 32-row tiles of the Lanczos basis layout
    for (int bb = 1; bb < G; ++bb) blk_row[bb] = (int32_t)std::min<int64_t>(n, (blk_row[bb] + 31) / 32 * 32);
    for (int bb = 1; bb <= G; ++bb) blk_row[bb] = std::max(blk_row[bb], blk_row[bb - 1]);
    // SpMV segments over the whole matrix: <= LZT_NNZ nonzeros and
    // <= LZT_ROWS rows; a row with more is cut into LZT_NNZ-nonzero pieces
    // (segment r1 = -(piece + 1)) whose partial sums its row owner adds up
    std::vector<int32_t> pz0, pz1, srow, sfirst, scnt;
    int64_t i = 0;
    while (i < n) {
      const int64_t s0 = i;
      if (rp32[i + 1] - rp32[i] > LZT_NNZ) {
        srow.push_back((int32_t)i);
        sfirst.push_back((int32_t)pz0.size());
        int c = 0;
        for (int32_t z = rp32[i]; z < rp32[i + 1]; z += LZT_NNZ, ++c) {
          seg_r0.push_back((int32_t)i);
          seg_r1.push_back(-(int32_t)pz0.size() - 1);
          pz0.push_back(z);
          pz1.push_back(std::min(rp32[i + 1], z + LZT_NNZ));
        }
        scnt.push_back(c);
        ++i;
        continue;
      }
      while (i < n && i - s0 < LZT_ROWS && rp32[i + 1] - rp32[i] <= LZT_NNZ && rp32[i + 1] - rp32[s0] <= LZT_NNZ)
        ++i;
      seg_r0.push_back((int32_t)s0);
      seg_r1.push_back((int32_t)i);
    }
    p->lz_npieces = (int)pz0.size();
    p->lz_piece_z0 = dev_upload(p, pz0.data(), pz0.size());
    p->lz_piece_z1 = dev_upload(p, pz1.data(), pz1.size());
    // split rows per row block (both lists ascend in row order)
    std::vector<int32_t> blk_sp(G + 1, 0);
    for (int bb = 0; bb <= G; ++bb)
      blk_sp[bb] = (int32_t)(std::lower_bound(srow.begin(), srow.end(), blk_row[bb]) - srow.begin());
    p->lz_blk_split = dev_upload(p, blk_sp.data(), blk_sp.size());
    p->lz_split_row = dev_upload(p, srow.data(), srow.size());
    p->lz_split_first = dev_upload(p, sfirst.data(), sfirst.size());
    p->lz_split_cnt = dev_upload(p, scnt.data(), scnt.size());
    // contiguous segment ranges per block, balanced on the measured cost of
    // each row kind (least-squares fit of the C4 per-block timers, in units
    // of a short-row nonzero): short rows (a thread per row) 1.0 per nonzero
    // + 0.36 per row; rows of 33..128 nonzeros (a warp per row, lanes half
    // idle) 1.5; longer rows 1.15; pieces of rows above LZT_NNZ (a block per
    // piece) 0.74
    const int64_t ns = (int64_t)seg_r0.size();
    auto seg_cost = [&](int64_t e) -> double {
      if (seg_r1[e] < 0) {
        const int pc = -seg_r1[e] - 1;
        return 0.74 * (double)(pz1[pc] - pz0[pc]);
      }
      double c = 0.0;
      for (int32_t r = seg_r0[e]; r < seg_r1[e]; ++r) {
        const int32_t len = rp32[r + 1] - rp32[r];
        c += len <= 32 ? len + 0.36 : (len <= 128 ? 1.5 * len : 1.15 * len);
      }
      return c;
    };
    double stot = 0.0;
    for (int64_t e = 0; e < ns; ++e) stot += seg_cost(e);
    double sacc = 0.0;
    int sb = 0;
    blk_seg[0] = 0;
    for (int64_t e = 0; e < ns && sb + 1 < G; ++e) {
      sacc += seg_cost(e);
      if (sacc >= stot * (sb + 1) / G) blk_seg[++sb] = (int32_t)(e + 1);
    }
    for (int bb = sb + 1; bb <= G; ++bb) blk_seg[bb] = (int32_t)ns;
  }
  PT("v1 Lanczos partition");
  std::vector<int32_t> diag_slot;
  if (p->diag_only) {
    if (m != n || ne != n) fail(USBS_ERR_SHAPE, "diag_only requires m == n == entries");
    diag_slot.resize(n);
    for (int64_t e = 0; e < ne; ++e) {
      if ((!directed && e_rows[e] != e_cols[e]) || e_idx[e] != e_rows[e] || e_rows[e] != e || e_vals[e] != 1.0)
        fail(USBS_ERR_SHAPE, "diag_only entries must be (i, i, col_i, 1.0) in row order");
    }
    // each row holds exactly one entry, at x-position xcnt[i]
    for (int64_t i = 0; i < n; ++i) diag_slot[i] = (int32_t)slot_of_x[xcnt[i]];
  }

  PT("diag slots");
  // --- upload
  p->rowptr = dev_upload(p, rp32.data(), rp32.size());
  p->h_rowptr = rp32;
  p->col = dev_upload(p, col.data(), col.size());
  p->cval = dev_upload(p, cval.data(), cval.size());
  p->zval = dev_alloc<double>(p, p->nnz);
  USBS_CUDA(cudaMemcpy(p->zval, p->cval, p->nnz * sizeof(double), cudaMemcpyDeviceToDevice));
  PT("  upload C pattern + values");
  if (!lazy_slots) {
    p->aptr = dev_upload(p, aptr.data(), aptr.size());
    p->aent = dev_upload(p, aent.data(), aent.size());
  }
  {
    std::vector<int32_t> ei(ne), er(ne), ec(ne);
    for (int64_t e = 0; e < ne; ++e) {
      ei[e] = (int32_t)e_idx[e]; er[e] = (int32_t)e_rows[e]; ec[e] = (int32_t)e_cols[e];
    }
    p->e_idx = dev_upload(p, ei.data(), ne);
    p->e_row = dev_upload(p, er.data(), ne);
    p->e_col = dev_upload(p, ec.data(), ne);
    p->e_val = dev_upload(p, e_vals, ne);
  }
  PT("  upload entries");
  if (p->diag_only) p->diag_slot = dev_upload(p, diag_slot.data(), n);
  {
    std::vector<int32_t> cptr(m + 1, 0), cent(ne);
    for (int64_t e = 0; e < ne; ++e) cptr[e_idx[e] + 1]++;
    int mx = 0;
    for (int64_t i = 0; i < m; ++i) { mx = std::max(mx, cptr[i + 1]); cptr[i + 1] += cptr[i]; }
    std::vector<int32_t> pos(cptr.begin(), cptr.end() - 1);
    for (int64_t e = 0; e < ne; ++e) cent[pos[e_idx[e]]++] = (int32_t)e;
    p->cptr = dev_upload(p, cptr.data(), cptr.size());
    p->cent = dev_upload(p, cent.data(), cent.size());
    p->max_entries_per_cons = mx;
  }
  PT("  constraint lists");
  {
    std::vector<int32_t> lr, lb, le, ls;
    for (size_t t = 0; t < irow.size(); ++t) {
      const int32_t r = irow[t];
      if (rp32[r + 1] - rp32[r] > SHORT_ROW) {
        lr.push_back(r); lb.push_back(ibeg[t]); le.push_back(iend[t]); ls.push_back(islot[t]);
      }
    }
    // CSR-stream tiles: maximal runs of at most ST_ROWS consecutive rows with
    // at most ST_NNZ nonzeros in total; longer rows get a block of their own
    {
      const int ST_NNZ = 1024;  // the tile size k_spmv_fused is instantiated for
      p->st_nnz = ST_NNZ;
      std::vector<int32_t> t0, t1, hr;
      int64_t i = 0;
      while (i < n) {
        if (rp32[i + 1] - rp32[i] > ST_NNZ) { hr.push_back((int32_t)i); ++i; continue; }
        const int64_t s0 = i;
        while (i < n && i - s0 < ST_ROWS && rp32[i + 1] - rp32[i] <= ST_NNZ && rp32[i + 1] - rp32[s0] <= ST_NNZ) ++i;
        t0.push_back((int32_t)s0);
        t1.push_back((int32_t)i);
      }
      p->n_stiles = (int)t0.size();
      p->stile_r0 = dev_upload(p, t0.data(), t0.size());
      p->stile_r1 = dev_upload(p, t1.data(), t1.size());
      p->n_huge_rows = (int)hr.size();
      p->huge_rows = dev_upload(p, hr.data(), hr.size());
    }
    p->n_long_items = (int)lr.size();
    p->lit_row = dev_upload(p, lr.data(), lr.size());
    p->lit_beg = dev_upload(p, lb.data(), lb.size());
    p->lit_end = dev_upload(p, le.data(), le.size());
    p->lit_slot = dev_upload(p, ls.data(), ls.size());
  }
  p->it_row = dev_upload(p, irow.data(), irow.size());
  p->it_beg = dev_upload(p, ibeg.data(), ibeg.size());
  p->it_end = dev_upload(p, iend.data(), iend.size());
  p->it_slot = dev_upload(p, islot.data(), islot.size());
  p->sr_row = dev_upload(p, srow.data(), srow.size());
  p->sr_first = dev_upload(p, sfirst.data(), sfirst.size());
  p->sr_count = dev_upload(p, scount.data(), scount.size());
  p->blk_row = dev_upload(p, blk_row.data(), blk_row.size());
  p->blk_seg = dev_upload(p, blk_seg.data(), blk_seg.size());
  p->seg_r0 = dev_upload(p, seg_r0.data(), seg_r0.size());
  p->seg_r1 = dev_upload(p, seg_r1.data(), seg_r1.size());
  PT("uploads + tiles + lists");
  *out = p;
}

usbs_status usbs_problem_destroy(usbs_problem* p) {
  USBS_API_BEGIN
  if (!p) return USBS_OK;
  cudaStreamSynchronize(p->ctx->stream);
  for (void* d : p->owned) cudaFree(d);
  delete p;
  USBS_API_END
}

usbs_status usbs_problem_info(usbs_problem* p, int64_t* nnz_z, int64_t* nnz_c, int* lz_blocks,
                              int* group) {
  USBS_API_BEGIN
  if (nnz_z) *nnz_z = p->nnz;
  if (nnz_c) *nnz_c = p->nnz_c;
  if (lz_blocks) *lz_blocks = p->lz_blocks;
  if (group) *group = p->spmv_group;
  USBS_API_END
}

usbs_status usbs_slack_assemble(usbs_ctx* ctx, usbs_problem* p, const double* y) {
  USBS_API_BEGIN
  launch_slack_assemble(ctx, p, y);
  USBS_API_END
}

usbs_status usbs_op_apply(usbs_ctx* ctx, usbs_problem* p, int which, const double* V, int64_t ldv, int k,
                          double* Y, int64_t ldy, double* gram) {
  USBS_API_BEGIN
  if (k < 1 || ldv < k || ldy < k) fail(USBS_ERR_SHAPE, "op_apply: bad k / leading dimension");
  if (kron_enabled(p)) {
    // QAP cost on the FP64 tensor cores; Z V = C V - A*(y) V
    if (which) {
      launch_spmm_vals(ctx, p, p->aval, V, ldv, k, Y, ldy);
      launch_kron_apply(ctx, p, V, ldv, k, Y, ldy, -1.0);
    } else {
      launch_kron_apply(ctx, p, V, ldv, k, Y, ldy, 0.0);
    }
  } else {
    launch_spmm(ctx, p, which, V, ldv, k, Y, ldy);
  }
  if (gram) launch_gram_tn(ctx, p->n, V, ldv, k, Y, ldy, k, gram, true);
  USBS_API_END
}

}  // extern "C"

namespace usbs {

void launch_slack_assemble(usbs_ctx* ctx, usbs_problem* p, const double* y) {
  if (p->diag_only) {
    // zval already equals cval off the diagonal (it is only ever written here)
    int th = 256, bl = (int)std::min<int64_t>((p->n + th - 1) / th, 4 * ctx->num_sms);
    k_slack_diag<<<bl, th, 0, ctx->stream>>>(p->n, p->diag_slot, p->cval, y, p->zval);
    check_launch(ctx);
  } else {
    int th = 256, bl = (int)std::min<int64_t>((p->nnz + th - 1) / th, 8 * ctx->num_sms);
    k_slack_assemble<<<std::max(bl, 1), th, 0, ctx->stream>>>(p->nnz, p->cval, p->aptr, p->aent, p->e_idx,
                                                              p->e_val, y, p->zval);
    check_launch(ctx);
  }
  if (p->kron_l) launch_adjoint_values(ctx, p, y, p->aval);  // the sparse part of Z V on the Kronecker path
}

void launch_spmm(usbs_ctx* ctx, usbs_problem* p, int which, const double* V, int64_t ldv, int k,
                 double* Y, int64_t ldy) {
  launch_spmm_vals(ctx, p, which ? p->zval : p->cval, V, ldv, k, Y, ldy);
}

// T = A*(w) on the merged pattern: tval[s] = sum_{e in slot s} w[idx[e]] val[e]
__global__ void k_adjoint_values(int64_t nnz, const int* __restrict__ aptr, const int* __restrict__ aent,
                                 const int* __restrict__ eidx, const double* __restrict__ eval,
                                 const double* __restrict__ w, double* __restrict__ tval) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nnz;
       s += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int t = aptr[s]; t < aptr[s + 1]; ++t) {
      const int e = aent[t];
      acc += w[eidx[e]] * eval[e];
    }
    tval[s] = acc;
  }
}

// slot -> entries lists of a diagonal problem, built on first use: row i's
// single entry (id i) sits at diag_slot[i] (increasing in i), so
// aptr[s] = #{i : diag_slot[i] < s} and aent[i] = i
__global__ void k_diag_slot_lists(int64_t n, int64_t nnz, const int* __restrict__ dslot, int* __restrict__ aptr,
                                  int* __restrict__ aent) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s <= nnz; s += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (dslot[mid] < s) lo = mid + 1;
      else hi = mid;
    }
    aptr[s] = (int)lo;
    if (s < n) aent[s] = (int)s;
  }
}

void ensure_slot_lists(usbs_ctx* ctx, usbs_problem* p) {
  if (p->aptr) return;
  if (!p->diag_only || !p->diag_slot) fail(USBS_ERR_CONFIG, "slot lists missing");
  p->aptr = dev_alloc<int>(p, p->nnz + 1);
  p->aent = dev_alloc<int>(p, p->n);
  const int bl = (int)std::min<int64_t>((p->nnz + 256) / 256, 8 * ctx->num_sms);
  k_diag_slot_lists<<<std::max(bl, 1), 256, 0, ctx->stream>>>(p->n, p->nnz, p->diag_slot, p->aptr, p->aent);
  check_launch(ctx);
}

void launch_adjoint_values(usbs_ctx* ctx, usbs_problem* p, const double* w, double* tval) {
  ensure_slot_lists(ctx, p);
  int th = 256, bl = (int)std::min<int64_t>((p->nnz + th - 1) / th, 8 * ctx->num_sms);
  k_adjoint_values<<<std::max(bl, 1), th, 0, ctx->stream>>>(p->nnz, p->aptr, p->aent, p->e_idx, p->e_val, w, tval);
  check_launch(ctx);
}

void launch_spmm_vals(usbs_ctx* ctx, usbs_problem* p, const double* val, const double* V, int64_t ldv, int k,
                      double* Y, int64_t ldy) {
  if (spmm_tiles_ok(p, k)) {  // block CSR-stream SpMM (usbs_spmm.cu; A/B via USBS_SPMM_V1=0)
    launch_spmm_tiles(ctx, p, val, V, ldv, k, Y, ldy);
    return;
  }
  double* partial = nullptr;
  if (p->n_split_items) partial = (double*)ctx->ws.get(WS_SPMM_PARTIAL, (size_t)p->n_split_items * k * sizeof(double));
  const int th = 256;
  if (k == 1) {
    const int64_t nb = (int64_t)p->n_huge_rows + p->n_stiles;
    if (nb > 0) {
k_spmv_fused<1024, 256, 6><<<(unsigned)nb, 256, 0, ctx->stream>>>(
          p->n_huge_rows, p->huge_rows, p->n_stiles, p->stile_r0, p->stile_r1, p->rowptr, p->col, val, V, ldv, Y,
          ldy);
      check_launch(ctx);
    }
    return;
  } else if (k <= 15 && p->nnz <= 16 * p->n && ((uintptr_t)V & 15) == 0 && !getenv("USBS_SPMM_16X2")) {
    // (a 16-byte-aligned base: no row's window starts before V's first entry)
    // short rows (C4: 9 per row): grouped 16-byte-gather kernel, several rows
    // per warp; long rows (C5: 41) keep the half-warp kernel, which is faster
    // there (profiles/spmm_ab.py; A/B: USBS_SPMM_16X2=1)
    const int G = k <= 5 ? 3 : k <= 7 ? 4 : k <= 11 ? 6 : 8;
    const int per = (th / 32) * (32 / G);
    int bl = (int)std::min<int64_t>((p->n_items + per - 1) / per, 16 * ctx->num_sms);
    const int64_t vend = (int64_t)(p->n_cols - 1) * ldv + k;  // V has n_cols rows (local + ghost for shards)
    auto args = [&](auto kern) {
      kern<<<std::max(bl, 1), th, 0, ctx->stream>>>(p->n_items, p->it_row, p->it_beg, p->it_end, p->it_slot,
                                                    p->col, val, V, ldv, vend, k, Y, ldy, partial);
    };
    if (G == 3) args(k_spmm_g<3>);
    else if (G == 4) args(k_spmm_g<4>);
    else if (G == 6) args(k_spmm_g<6>);
    else args(k_spmm_g<8>);
  } else if (k <= 16) {
    int bl = (int)std::min<int64_t>((p->n_items + 7) / 8, 16 * ctx->num_sms);
    k_spmm16x2<<<std::max(bl, 1), th, 0, ctx->stream>>>(p->n_items, p->it_row, p->it_beg, p->it_end, p->it_slot,
                                                        p->col, val, V, ldv, k, Y, ldy, partial);
  } else {
    int per = th / 32;
    int bl = (int)std::min<int64_t>((p->n_items + per - 1) / per, 16 * ctx->num_sms);
    k_spmm<32><<<std::max(bl, 1), th, 0, ctx->stream>>>(p->n_items, p->it_row, p->it_beg, p->it_end, p->it_slot,
                                                        p->col, val, V, ldv, k, Y, ldy, partial);
  }
  check_launch(ctx);
  if (p->n_split_rows) {
    int64_t tot = (int64_t)p->n_split_rows * k;
    int bl = (int)std::min<int64_t>((tot + 255) / 256, 4 * ctx->num_sms);
    k_spmm_combine<<<std::max(bl, 1), 256, 0, ctx->stream>>>(p->n_split_rows, p->sr_row, p->sr_first,
                                                             p->sr_count, partial, k, Y, ldy);
    check_launch(ctx);
  }
}

}  // namespace usbs
