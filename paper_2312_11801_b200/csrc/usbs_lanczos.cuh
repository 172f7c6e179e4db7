// Shared definitions of the persistent Lanczos kernels (usbs_lanczos.cu:
// cluster and v1 grid variants; usbs_lanczos_grid.cu: the TMA-pipelined grid
// variant).  Internal, not part of the C ABI.
#pragma once
#include "usbs_common.cuh"

namespace usbs {

enum LzFlag { F_EXIT = 0, F_J = 1, F_CYCLE = 2, F_ELL = 3, F_RESTARTS = 4, F_CONV = 5, F_NHIST = 6,
              F_MATVECS = 7, F_NONFINITE = 8, F_PENDING = 9 };
enum LzExit { EXIT_DONE = 0, EXIT_BREAKDOWN = 1, EXIT_NONFINITE = 2 };

struct LzArgs {
  int n, m, k_c, max_restarts;
  int64_t ldq;  // row stride of W0/W1 (>= n)
  double tol;
  const int* rowptr;
  const int* col;
  const double* val;
  const int* blk_row;  // block b owns rows [blk_row[b], blk_row[b+1]) (Q passes)
  const int* blk_seg;  // ... and SpMV segments [blk_seg[b], blk_seg[b+1]) (nnz-balanced)
  const int* seg_r0;   // segment: rows [seg_r0, seg_r1), <= LZT_NNZ nonzeros,
  const int* seg_r1;   //   or (seg_r1 < 0) piece -seg_r1-1 of a longer row
  const int* piece_z0;  // nonzero range of each piece
  const int* piece_z1;
  double* piece_sum;    // partial sum of each piece
  const int* blk_split;  // row block b's split rows [blk_split[b], blk_split[b+1])
  const int* split_row;
  const int* split_first;
  const int* split_cnt;
  double* Q;
  double* W0;
  double* W1;
  double* H;
  double* P1;  // [64][G] column partials, P1[t * G + b]
  double* P2;  // [64][G]
  double* P3;  // [G]
  int* flags;
  double* theta;  // [m]   output (after the last Rayleigh-Ritz)
  double* Y;      // [m*m] output
  double* res;    // [m]
  double* hist;   // [max_restarts + 1]
  // resume state
  int cycle0, ell0, j0, restarts0, nhist0, matvecs0, wbuf0;
  double beta_prev;  // beta of the step before j0 (only used if first step gathers from W)
  int first_from_q;  // 1: q_{j0} is materialised in Q (start/restart/reseed)
  double* vecs_out;  // n x k_c row-major (written when done)
  int64_t ldvecs;
  unsigned long long* prof;  // optional phase timer accumulators (ns), block 0
  // TMA-pipelined grid variant (usbs_lanczos_grid.cu)
  const int4* items;       // SpMV work items of every block (see LzGridPlan)
  const int* blk_item;     // block b's items [blk_item[b], blk_item[b+1])
  int nsplit;              // rows whose SpMV is cut into pieces spread over blocks
  const int* gsplit_row;   //   ascending row ids
  const int* gsplit_first; //   first piece of each split row
  const int* gsplit_cnt;   //   its piece count
  const int* blk_gsplit;   // block b owns split rows [blk_gsplit[b], blk_gsplit[b+1])
  int tail0, tail1;        // the shared SpMV item pool [tail0, tail1)
  int* steal;              // its two claim counters (step parity)
  int lz_opt;              // A/B switches of the TMA variant (bit 0: column sums from shared memory)
};

// Q element (row i, column t) in the row-blocked layout
__host__ __device__ __forceinline__ int64_t qidx(int64_t i, int t, int M1) {
  return ((i >> 5) * M1 + t) * 32 + (i & 31);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}


// TMA-pipelined grid variant (usbs_lanczos_grid.cu)
void lz_tma_plan(usbs_ctx* ctx, usbs_problem* p);
void lz_tma_launch(usbs_ctx* ctx, usbs_problem* p, LzArgs& a);

}  // namespace usbs
