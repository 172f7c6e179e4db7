// Internal launch helpers shared between translation units.
#pragma once
#include "usbs_common.cuh"

namespace usbs {

// workspace slot ids
enum WsSlot {
  WS_SPMM_PARTIAL = 1,
  WS_GRAM_PARTIAL = 2,
  WS_LZ_Q = 10,
  WS_LZ_W = 11,
  WS_LZ_H = 12,
  WS_LZ_P = 13,
  WS_LZ_SPLIT = 14,
  WS_LZ_FLAGS = 15,
  WS_LZ_OUT = 16,
  WS_LZ_TMP = 17,
  WS_LZ_PROF = 18,
  WS_LZ_HALO = 19,
  WS_SMALL = 20,
  WS_RED = 21,
  WS_IPM = 30,
  WS_BOOK = 40,
  WS_BOOK_T = 41,
  WS_BOOK_W = 42,
  WS_BOOK_G = 43,
};

void launch_slack_assemble(usbs_ctx* ctx, usbs_problem* p, const double* y);
void launch_spmm(usbs_ctx* ctx, usbs_problem* p, int which, const double* V, int64_t ldv, int k,
                 double* Y, int64_t ldy);
void launch_spmm_vals(usbs_ctx* ctx, usbs_problem* p, const double* val, const double* V, int64_t ldv, int k,
                      double* Y, int64_t ldy);
void launch_adjoint_values(usbs_ctx* ctx, usbs_problem* p, const double* w, double* tval);
void ensure_slot_lists(usbs_ctx* ctx, usbs_problem* p);
bool kron_enabled(const usbs_problem* p);
bool spmm_tiles_ok(const usbs_problem* p, int k);
void launch_spmm_tiles(usbs_ctx* ctx, usbs_problem* p, const double* val, const double* V, int64_t ldv, int k,
                       double* Y, int64_t ldy);
void launch_kron_apply(usbs_ctx* ctx, usbs_problem* p, const double* V, int64_t ldv, int k, double* Y, int64_t ldy,
                       double beta);
// out (ka x kb, row-major, dev) = A^T B for row-major n x ka A and n x kb B;
// sym: out = 0.5 (G + G^T) (requires ka == kb)
void launch_gram_tn(usbs_ctx* ctx, int64_t n, const double* A, int64_t lda, int ka, const double* B, int64_t ldb,
                    int kb, double* out, bool sym, const double* rw = nullptr);
// deterministic sum-of-squares / dot over n (result in dev scalar)
void launch_dot(usbs_ctx* ctx, int64_t n, const double* x, const double* y, double* out);

}  // namespace usbs
