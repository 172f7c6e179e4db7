// Shared internals of libusbs_b200 (sm_100a).  Not part of the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>
#include <unordered_map>
#include <mutex>
#include <map>
#include <utility>

#include "../../include/usbs_b200.h"

namespace usbs {

void set_error(const std::string& msg);

struct CudaError {
  cudaError_t e;
  const char* what;
};

#define USBS_CUDA(call)                                                        \
  do {                                                                         \
    cudaError_t _e = (call);                                                   \
    if (_e != cudaSuccess) throw ::usbs::CudaError{_e, #call};                 \
  } while (0)

struct StatusError {
  usbs_status s;
  std::string msg;
};

[[noreturn]] inline void fail(usbs_status s, const std::string& m) { throw StatusError{s, m}; }

// Scratch buffer cache keyed by slot id; grows on demand, never shrinks.
struct Workspace {
  std::unordered_map<int, std::pair<void*, size_t>> bufs;
  void* get(int slot, size_t bytes) {
    auto& b = bufs[slot];
    if (b.second < bytes) {
      if (b.first) cudaFree(b.first);
      size_t nb = bytes < 256 ? 256 : bytes;
      USBS_CUDA(cudaMalloc(&b.first, nb));
      b.second = nb;
    }
    return b.first;
  }
  void release() {
    for (auto& kv : bufs)
      if (kv.second.first) cudaFree(kv.second.first);
    bufs.clear();
  }
};

}  // namespace usbs

struct usbs_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  int64_t launches = 0;
  usbs::Workspace ws;
  double* pinned = nullptr;  // 4096 doubles of pinned host scratch
  int* pinned_i = nullptr;   // 256 ints
  unsigned char* stage[2] = {nullptr, nullptr};  // pinned upload staging (lazy)
  void* lzq_ptr = nullptr;  // Lanczos basis / W workspaces last zeroed (usbs_lanczos_top)
  void* lzw_ptr = nullptr;
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
};

struct usbs_problem {
  usbs_ctx* ctx = nullptr;
  int64_t n = 0, n_cols = 0, m = 0, nnz = 0, nnz_c = 0, ne = 0;  // n = rows (local for shards)
  bool diag_only = false;
  // merged CSR pattern of C - A*(y)
  int* rowptr = nullptr;
  int* col = nullptr;
  double* cval = nullptr;  // C values in the merged pattern (0 where only A* lives)
  double* zval = nullptr;  // assembled Z = C - A*(y)
  int* diag_slot = nullptr;  // slot of (i,i) (diag_only)
  // slack assembly: slot -> contributing entries
  int* aptr = nullptr;   // nnz + 1
  int* aent = nullptr;   // entry ids
  // constraint -> entries (ascending entry id), for row-wise constraint kernels
  int* cptr = nullptr;  // m + 1
  int2* c1_rc = nullptr;      // per constraint: (row, col) of its single entry, (-1, -1) if it has several
  double* c1_val = nullptr;   // that entry's value (lazy, first compressed-Gram call)
  int* c1_heavy = nullptr;    // [0] = count h, [1 .. h] = constraints with > IMAGE_HEAVY entries (any order)
  int* cent = nullptr;  // ne
  int max_entries_per_cons = 0;
  // flat constraint entries (device copies)
  int* e_idx = nullptr;
  int* e_row = nullptr;
  int* e_col = nullptr;
  double* e_val = nullptr;
  // SpMM work items: row segments (rows longer than SEG are split)
  int n_items = 0;
  int* it_row = nullptr;
  int* it_beg = nullptr;
  int* it_end = nullptr;
  int* it_slot = nullptr;  // -1: whole row, else index into the split-partial scratch
  // k = 1 SpMV: rows with more than 2048 nonzeros get a block each
  int n_huge_rows = 0;
  int* huge_rows = nullptr;
  int n_stiles = 0;  // CSR-stream tiles of consecutive rows (k = 1 SpMV)
  int st_nnz = 1024;  // nonzeros per tile (rows above it get a block)
  int* stile_r0 = nullptr;
  int* stile_r1 = nullptr;
  // the subset of items that belong to rows longer than 32
  int n_long_items = 0;
  int* lit_row = nullptr;
  int* lit_beg = nullptr;
  int* lit_end = nullptr;
  int* lit_slot = nullptr;
  int n_split_items = 0;
  int n_split_rows = 0;
  int* sr_row = nullptr;    // split rows
  int* sr_first = nullptr;  // first split slot
  int* sr_count = nullptr;
  int* sr_block = nullptr;  // owning Lanczos block of each split row (ascending)
  // Lanczos partition: block b owns rows [blk_row[b], blk_row[b+1])
  int lz_blocks = 0;
  int spmv_group = 32;
  // cached cluster-Lanczos plan (usbs_lanczos.cu): basis size it was made
  // for, cluster size (0 = grid kernel), rows per CTA, dynamic smem bytes
  int lz_cl_m = -1, lz_cl_cs = 0, lz_cl_R = 0, lz_cl_lg = 32;  // lg: SpMV lanes per row
  int lz_cl_hmax = 0;  // halo slots per CTA (0: DSMEM gathers inside the SpMV)
  size_t lz_cl_smem = 0;
  int* blk_row = nullptr;
  int* blk_seg = nullptr;  // Lanczos block b's SpMV segments [blk_seg[b], blk_seg[b+1])
  int* seg_r0 = nullptr;   // segment rows [seg_r0, seg_r1): <= LZT_NNZ nonzeros or one row
  int* seg_r1 = nullptr;
  int lz_npieces = 0;             // pieces of rows above LZT_NNZ nonzeros
  int* lz_piece_z0 = nullptr;     //   nonzero range of each piece
  int* lz_piece_z1 = nullptr;
  int* lz_blk_split = nullptr;    // row block b's split rows [lz_blk_split[b], [b+1])
  int* lz_split_row = nullptr;    //   row, first piece, piece count
  int* lz_split_first = nullptr;
  int* lz_split_cnt = nullptr;
  // tiled SpMM plan (usbs_spmm.cu), built per tile size on first use
  int spt_T = 0, spt_ntiles = 0, spt_nch = 0, spt_nhuge = 0;
  int *spt_r0 = nullptr, *spt_r1 = nullptr, *spt_z0 = nullptr, *spt_z1 = nullptr;
  int *spt_hrow = nullptr, *spt_hfirst = nullptr, *spt_hcnt = nullptr;
  // Kronecker-structured cost (QAP, usbs_kron.cu): C = coef (0 (+) D (x) W)
  int kron_l = 0;
  double* kron_D = nullptr;
  double* kron_W = nullptr;
  double kron_coef = 0.0;
  double* aval = nullptr;  // A*(y) on the merged pattern (set by slack assembly)
  // TMA-pipelined grid Lanczos plan (usbs_lanczos_grid.cu), built on first use
  std::vector<int32_t> h_rowptr;  // host copy of rowptr (the plan's input)
  int lzg_ready = 0, lzg_G = 0, lzg_npieces = 0, lzg_nsplit = 0, lzg_tail0 = 0, lzg_tail1 = 0;
  int* lzg_blk_row = nullptr;
  int* lzg_blk_item = nullptr;
  int4* lzg_items = nullptr;
  int* lzg_split_row = nullptr;
  int* lzg_split_first = nullptr;
  int* lzg_split_cnt = nullptr;
  int* lzg_blk_split = nullptr;
  std::vector<void*> owned;
};

namespace usbs {

// grid-Lanczos SpMV segments: at most LZT_NNZ nonzeros and LZT_ROWS rows
constexpr int LZT_NNZ = 4096;
constexpr int LZT_ROWS = 2048;

// Host -> device copy through two pinned staging chunks (host memcpy of one
// chunk overlaps the DMA of the other); small arrays go directly.
void staged_h2d(usbs_ctx* ctx, void* dst, const void* src, size_t bytes);

template <typename T>
T* dev_upload(usbs_problem* p, const T* host, size_t count) {
  T* d = nullptr;
  size_t bytes = count * sizeof(T);
  USBS_CUDA(cudaMalloc(&d, bytes < 16 ? 16 : bytes));
  if (count) staged_h2d(p->ctx, d, host, bytes);
  p->owned.push_back(d);
  return d;
}

template <typename T>
T* dev_alloc(usbs_problem* p, size_t count) {
  T* d = nullptr;
  size_t bytes = count * sizeof(T);
  USBS_CUDA(cudaMalloc(&d, bytes < 16 ? 16 : bytes));
  p->owned.push_back(d);
  return d;
}

inline void note_launch(usbs_ctx* c, int n = 1) { c->launches += n; }

// Large dynamic shared memory opt-in for kernel `fn` on the context's device.
// cudaFuncSetAttribute acts on the current device only, so the opt-in is
// recorded per (kernel, device) as the largest size requested so far (the
// attribute is an upper bound: raising it never breaks smaller launches);
// thread-safe.
inline void smem_optin(const usbs_ctx* c, const void* fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  std::lock_guard<std::mutex> g(mu);
  int& cur = done[std::make_pair(fn, c->device)];
  if (bytes <= cur) return;
  USBS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  cur = bytes;
}

inline void check_launch(usbs_ctx* c) {
  note_launch(c);
  USBS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------- device utils
// D = A B + C on the FP64 tensor cores (mma.sync m8n8k4, row.col): lane l
// holds a = A[l >> 2][l & 3], b = B[l & 3][l >> 2], c/d = C[l >> 2][2 (l & 3) + {0, 1}]
__device__ __forceinline__ void dmma_m8n8k4(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// block-wide sum, result broadcast to all threads; red must hold >= 32 doubles
__device__ inline double block_sum(double v, double* red) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = lane < nw ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

__device__ __forceinline__ double ldg_nc(const double* p) { return __ldg(p); }

}  // namespace usbs

// Every C-ABI entry point is wrapped in this to map exceptions to statuses.
#define USBS_API_BEGIN try {
#define USBS_API_END                                                              \
  }                                                                               \
  catch (const ::usbs::StatusError& e) {                                          \
    ::usbs::set_error(e.msg);                                                     \
    return e.s;                                                                   \
  }                                                                               \
  catch (const ::usbs::CudaError& e) {                                            \
    ::usbs::set_error(std::string(e.what) + ": " + cudaGetErrorString(e.e));      \
    return USBS_ERR_CUDA;                                                         \
  }                                                                               \
  catch (const std::exception& e) {                                               \
    ::usbs::set_error(e.what());                                                  \
    return USBS_ERR_CUDA;                                                         \
  }                                                                               \
  return USBS_OK;
