/*
 * usbs_b200.h -- C ABI of the B200-native USBS hot path (sm_100a).
 *
 * Drop-in boundary for the per-iteration hot path of the reference package
 * specbundle 0.1.0 (arXiv 2312.11801).  The reference is pure Python, so
 * there is no FFI today; each entry point below names the Python interface
 * it replaces (paths relative to /root/reference/pkg/src/specbundle/).  The
 * Python host layer (paper_2312_11801_b200/) binds this header with ctypes
 * and mirrors the reference operator/solver interfaces on top of it.
 *
 * Conventions
 *   - plain C types only: pointers, int32/int64, double.  No torch types.
 *   - "host" pointers are read synchronously; "dev" pointers are device
 *     addresses (caller-owned buffers, e.g. torch CUDA tensors) consumed on
 *     the context's stream.  Calls returning host scalars synchronise.
 *   - dense n x k blocks are ROW-MAJOR with leading dimension ld >= k (the
 *     reference's C-order numpy layout); small k x k / d x d matrices are
 *     dense row-major with ld = k (symmetric ones are stored in full).
 *   - all arithmetic is FP64.
 *   - status codes map 1:1 onto the reference exceptions (see usbs_status).
 */
#ifndef USBS_B200_H
#define USBS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define USBS_ABI_VERSION 1

typedef enum {
  USBS_OK = 0,
  USBS_ERR_SHAPE = 1,       /* ValueError (shapes / dimensions)                 */
  USBS_ERR_CONFIG = 2,      /* ValueError (invalid configuration)               */
  USBS_ERR_NONFINITE = 3,   /* eigsolve.NumericError       eigsolve.py:21-22    */
  USBS_ERR_NOT_PD = 4,      /* symlin.ConditioningError    symlin.py:34-35      */
  USBS_ERR_STEP_FAIL = 5,   /* subqp.StepFailureError      subqp.py:56-57       */
  USBS_ERR_EMPTY_BASIS = 6, /* symlin.EmptyBasisError      symlin.py:38-39      */
  USBS_ERR_CUDA = 7,        /* CUDA runtime failure (RuntimeError)              */
  USBS_ERR_CALLBACK = 8     /* a host callback reported failure                 */
} usbs_status;

typedef struct usbs_ctx usbs_ctx;
typedef struct usbs_problem usbs_problem;

/* ---- context ------------------------------------------------------------ */
int usbs_abi_version(void);
/* Message for the last non-OK status returned on this thread. */
const char* usbs_last_error(void);
/* stream: a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream);
 * NULL is the legacy default stream.  All work of the context is ordered on
 * it, so caller-side copies on the same stream need no extra sync. */
usbs_status usbs_ctx_create(int device, void* stream, usbs_ctx** out);
usbs_status usbs_ctx_destroy(usbs_ctx* ctx);
usbs_status usbs_ctx_sync(usbs_ctx* ctx);
/* number of kernel launches issued by this context so far (bench evidence) */
int64_t usbs_ctx_launches(usbs_ctx* ctx);
/* stream-ordered host <-> device copies of plain buffers (synchronising) */
usbs_status usbs_memcpy_h2d(usbs_ctx* ctx, void* dst_dev, const void* src_host, int64_t bytes);
usbs_status usbs_memcpy_d2h(usbs_ctx* ctx, void* dst_host, const void* src_dev, int64_t bytes);

/* ---- problem upload: SdpProblem.cost + constraint bundle ----------------
 * Replaces the scipy CSR + constraint objects consumed by
 * problem.py:311-314 (dual_slack_operator), 284-289 (cost_quad,
 * cost_factor_ip), 144-243 (DiagonalConstraints / SparseConstraintFamilies).
 * C: CSR (host, int64 indptr, int32 indices, sorted or not, no duplicates).
 * Constraints as flat entries (host): constraint e_idx[e] has
 * A[e_rows[e], e_cols[e]] = A[e_cols[e], e_rows[e]] = e_vals[e], rows <= cols.
 * Diagonal constraints (MaxCut) are passed as entries (i, i, i, 1.0) and
 * flagged diag_only = 1, which enables the row-wise fast paths.
 * The library builds the merged pattern of C - A*(y) once (the reference
 * rebuilds that CSR on every evaluation, problem.py:313). */
usbs_status usbs_problem_create(usbs_ctx* ctx, int64_t n, int64_t m,
                                const int64_t* c_indptr, const int32_t* c_indices,
                                const double* c_data, int64_t n_entries,
                                const int64_t* e_idx, const int64_t* e_rows,
                                const int64_t* e_cols, const double* e_vals,
                                int diag_only, usbs_problem** out);
/* Row shard of a problem for multi-GPU runs: the rank's n_rows rows of C
 * (CSR with global column indices < n_cols) and the DIRECTED constraint
 * entries of those rows (local row, global column, local constraint index;
 * no mirroring).  diag_only: entry i is (i, i, row_offset + i, 1.0). */
usbs_status usbs_problem_create_shard(usbs_ctx* ctx, int64_t n_rows, int64_t n_cols, int64_t m,
                                      const int64_t* c_indptr, const int32_t* c_indices,
                                      const double* c_data, int64_t n_entries, const int64_t* e_idx,
                                      const int64_t* e_rows, const int64_t* e_cols,
                                      const double* e_vals, int diag_only, usbs_problem** out);
usbs_status usbs_problem_destroy(usbs_problem* p);
/* nnz of the merged slack pattern and the lanczos grid size (for reporting) */
usbs_status usbs_problem_info(usbs_problem* p, int64_t* nnz_z, int64_t* nnz_c,
                              int* lanczos_blocks, int* spmv_group);

/* ---- K1: operator apply ------------------------------------------------- */
/* Z = C - A*(y) assembled in place (problem.py:313 "(cost - adjoint_matrix(y))"). */
usbs_status usbs_slack_assemble(usbs_ctx* ctx, usbs_problem* p, const double* y_dev);
/* Y = M V with M = C (which = 0) or the assembled Z (which = 1), V n x k;
 * optionally gram = sym(V^T Y) (k x k, dev).  Replaces LinOp.matmat
 * (eigsolve.py:25-36 via problem.py:314), cost_quad (problem.py:284-286) and
 * the Z-Gram of assemble_eval_coeffs (subqp.py:459). */
usbs_status usbs_op_apply(usbs_ctx* ctx, usbs_problem* p, int which, const double* v_dev,
                          int64_t ldv, int k, double* y_dev, int64_t ldy, double* gram_dev);

/* Kronecker-structured cost (build_qap, problem.py:462-477): C = coef *
 * (0 (+) D (x) W) with composite index a = i*l + k (problem.py:364-371),
 * D, W host l x l row-major, n = l^2 + 1.  op_apply then runs C V as the
 * contraction coef * D X W^T on the FP64 tensor cores (mma.sync m8n8k4) and
 * Z V as that minus a sparse pass over A*(y) (USBS_KRON=0 disables it). */
usbs_status usbs_problem_set_kron(usbs_ctx* ctx, usbs_problem* p, int l, const double* d_host,
                                  const double* w_host, double coef);

/* ---- K2/K3: thick-restart Lanczos --------------------------------------- */
/* Row-sharded Lanczos (dist.lanczos_sharded; eigsolve.py:125-176 per rank):
 * the epilogue of step j on the device -- H[:j+1, j] = c1 + c2, beta =
 * sqrt(nrm2) into H[j+1, j], q_{j+1} = w / beta on the local rows (zero on
 * breakdown), flags[0] = first breakdown step (beta <= 1e-13 max(1, max|c|),
 * eigsolve.py:136-147), flags[1] |= non-finite -- and the thick-restart reset
 * H = diag(theta[:ell]).  c1, c2, nrm2 are the allreduced (replicated) CGS2
 * coefficients and norm; no host reads inside a cycle. */
usbs_status usbs_lz_step_finish(usbs_ctx* ctx, int j, int m1, const double* c1_dev, const double* c2_dev,
                                const double* nrm2_dev, double* h_dev, int* flags_dev, const double* w_dev,
                                int64_t nl, int64_t ldw, double* q_dev, int64_t ldq);
usbs_status usbs_lz_restart_h(usbs_ctx* ctx, int m1, int ell, const double* theta_dev, double* h_dev);
/* Host callback producing the PCG64 stream of eigsolve._seeded_unit for a
 * counter (eigsolve.py:49-52) into a device n-vector (unnormalised normals).
 * Returns 0 on success. */
typedef int (*usbs_rng_fill_fn)(void* user, int64_t counter, double* out_dev, int64_t n);
/* lanczos_top (eigsolve.py:83-181) on M = C (which = 0) or Z (which = 1).
 * v0_dev: the normalised start vector _seeded_unit(n, seed, 0).
 * Outputs: vals (host, k_c, descending), vecs_dev (n x k_c row-major, ld),
 * res (host, k_c), *converged, *restarts, ritz_hist (host, >= max_restarts+1
 * entries, *n_hist written), *matvecs.  tol < 0 means the default 1e-9. */
usbs_status usbs_lanczos_top(usbs_ctx* ctx, usbs_problem* p, int which, int k_c,
                             int inner_iters, int max_restarts, double tol,
                             const double* v0_dev, usbs_rng_fill_fn reseed, void* user,
                             double* vals, double* vecs_dev, int64_t ldvecs, double* res,
                             int* converged, int* restarts, double* ritz_hist, int* n_hist,
                             int* matvecs);

/* Phase timers of the Lanczos kernel (ns, accumulated while the environment
 * variable USBS_LZ_PROF is set); out_host holds 1024 entries: [0..7] phase A,
 * barriers, phase B, phase C, end of cycle, Rayleigh-Ritz, restart, SpMV
 * (cluster kernel), all measured on block 0; [8..11] Rayleigh-Ritz setup,
 * bisection, inverse iteration, output; [32 + 4b + s] block b's work in the
 * SpMV, the Q^T w sums, phase B and phase C with barrier waits excluded
 * (grid kernel).  reset != 0
 * zeroes them. */
usbs_status usbs_lanczos_profile(usbs_ctx* ctx, unsigned long long* out_host, int reset);

/* Execution plan usbs_lanczos_top uses for basis size m on p: *cluster_size
 * CTAs in one thread-block cluster holding *rows_per_cta rows of Q each in
 * shared memory, or *cluster_size = 0 for the grid-wide cooperative kernel
 * (*rows_per_cta = 0).  The environment variable USBS_LZ_CLUSTER=0, read when
 * the plan is first made for p, forces the grid kernel. */
usbs_status usbs_lanczos_plan(usbs_ctx* ctx, usbs_problem* p, int m, int* cluster_size,
                              int* rows_per_cta);

/* ---- K3: small symmetric eigendecomposition ----------------------------- */
/* small_eigh (symlin.py:193-198): symmetrise, eigendecompose, descending.
 * k <= 64; a_dev, vals_dev (k), vecs_dev (k x k, columns = eigenvectors). */
usbs_status usbs_small_eigh(usbs_ctx* ctx, int k, const double* a_dev, double* vals_dev,
                            double* vecs_dev);

/* ---- K12: interior-point bundle subproblem (single CTA) ------------------
 * _ipm_solve (subqp.py:353-435) behind ipm_quad / ipm_eval (438-448).
 * Coefficients (dev): Q11 = quad_ss (d x d, NULL = 0 for ipm_eval),
 * q12 = quad_s_eta (d, NULL = 0), lin_s (d), scal = [quad_eta, lin_eta].
 * State (dev, usbs_ipm_state_len(k) doubles): S, T (k x k), eta, zeta, omega,
 * mu, has_eta, k, valid -- IpmState (subqp.py:111-147).  warm_state may be
 * NULL (cold start) and may alias state_out.
 * result (dev, 5): value, newton_iters, exact, eta_opt, trailing failures.
 * opts (host, 8 or NULL = IpmOptions defaults): mu_tol, kkt_tol, max_newton,
 * step_frac, backtrack, min_step, max_step_failures, warm_blend. */
usbs_status usbs_ipm_solve(usbs_ctx* ctx, int k, int has_eta, const double* Q11_dev,
                           const double* q12_dev, const double* lin_s_dev, const double* scal_dev,
                           const double* warm_state_dev, double* state_out_dev, double* result_dev,
                           const double* opts);
int usbs_ipm_state_len(int k);
/* Phase timers of the IPM kernel (ns, 10 slots, accumulated while the
 * environment variable USBS_IPM_PROF is set); reset != 0 zeroes them. */
usbs_status usbs_ipm_profile(usbs_ctx* ctx, unsigned long long* out_host, int reset);

/* ---- K5: constraint image A(V S V^T) ------------------------------------
 * out = beta * base + A(V S V^T); S k x k (s_is_diag = 0) or its diagonal
 * (s_is_diag = 1: A(U diag(l) U^T)).  primal_image_lowrank / _factor
 * (problem.py:151-155, 200-208).  base may be NULL. */
usbs_status usbs_cons_image(usbs_ctx* ctx, usbs_problem* p, const double* v_dev, int64_t ldv,
                            int k, const double* s_dev, int s_is_diag, double s_scale,
                            const double* beta_dev, double beta, const double* base_dev,
                            double* out_dev);
/* (S is scaled by s_scale; beta is multiplied by *beta_dev when non-NULL) */

/* ---- K4/K4w: compressed constraint rows c_i = svec(V^T A_i V) -----------
 * gram_out = scale_gram * C^T C (d x d), a_out = scale_a * C^T a,
 * w_out = scale_w * C^T w; any output may be NULL.  compressed_rows
 * (problem.py:169-173, 229-239) and its uses in assemble_quad_coeffs
 * (subqp.py:487-498, 510).  C is never materialised. */
usbs_status usbs_cons_compressed(usbs_ctx* ctx, usbs_problem* p, const double* v_dev,
                                 int64_t ldv, int k, double scale_gram, double* gram_out_dev,
                                 const double* a_dev, double scale_a, double* a_out_dev,
                                 const double* w_dev, double scale_w, double* w_out_dev);

/* ---- tall-skinny dense helpers (row-major blocks, k <= 64) -------------- */
/* Y = alpha (X diag(xs)) B + beta Y0 (X n x ka, B ka x kb with ld ldb, dev;
 * xs (ka) and Y0 may be NULL; Y0 may alias Y) */
usbs_status usbs_rowgemm(usbs_ctx* ctx, int64_t n, const double* x_dev, int64_t ldx, int ka,
                         const double* b_dev, int64_t ldb, int kb, const double* xs_dev,
                         double alpha, double beta, const double* y0_dev, int64_t ldy0,
                         double* y_dev, int64_t ldy);
/* out = A^T B (ka x kb); sym: 0.5 (G + G^T) */
usbs_status usbs_gram(usbs_ctx* ctx, int64_t n, const double* a_dev, int64_t lda, int ka,
                      const double* b_dev, int64_t ldb, int kb, double* out_dev, int sym);
/* out[0] = sum_ij F_ij G_ij w_j  (cost_factor_ip, problem.py:288-289) */
usbs_status usbs_wcoldot(usbs_ctx* ctx, int64_t n, const double* f_dev, int64_t ldf,
                         const double* g_dev, int64_t ldg, int k, const double* w_dev,
                         double* out_dev);
/* X = eta X + F diag(l) F^T (ExplicitStore.update, bundle.py:108-109) */
usbs_status usbs_dense_update(usbs_ctx* ctx, int64_t n, double* x_dev, double eta,
                              const double* f_dev, int64_t ldf, int kc, const double* l_dev);
/* m-vector operations (op codes in csrc/usbs_book.cu VecOp); red_out (dev, 2)
 * receives [sum, max] reductions where the op defines them.  Ops 10/11 are the
 * two reductions of psi_value (subqp.py:546-549): <b + nu - a_x, y> and
 * ||b + nu - a_x||^2 with x = a_x, z = nu. */
usbs_status usbs_vec(usbs_ctx* ctx, int op, int64_t m, const double* x, const double* y,
                     const double* z, const double* b, const double* ineq, double s0, double s1,
                     double* out, double* red_out);
/* out (d) = scale * svec(A), A k x k symmetric (symlin.svec, symlin.py:72-79) */
usbs_status usbs_svec(usbs_ctx* ctx, int k, const double* a_dev, double scale, double* out_dev);
/* pivoted Cholesky of a c x c Gram with orthonormalize's drop rule
 * (symlin.py:148-190): perm (dev int, c), Rinv (dev, c x c upper, ld c),
 * info (dev, 3) = [rank, min selected residual ratio, max column norm]. */
usbs_status usbs_pivchol(usbs_ctx* ctx, int c, const double* g_dev, double drop_tol,
                         int* perm_dev, double* rinv_dev, double* info_dev);
/* B (c x c, dev) with B[perm[i], j] = Rinv[i, j] for i, j < r = info[0] and
 * zero elsewhere: orthonormalize's first CholQR factor built on the device
 * from usbs_pivchol's outputs, so the host reads the rank only once. */
usbs_status usbs_perm_rows(usbs_ctx* ctx, int c, const int32_t* perm_dev, const double* rinv_dev,
                           const double* info_dev, double* out_dev);

/* ---- the constraint-bundle duck type (problem.py:144-243) ------------------
 * Device halves of DiagonalConstraints / SparseConstraintFamilies for an
 * unsharded problem (the Python shim constraints.DeviceConstraints returns
 * numpy on demand). */
/* Y = A*(y) V (n x k, dev), optionally gram = sym(V^T Y): adjoint_matvec /
 * adjoint_inner_lowrank (problem.py:163-167, 222-227). */
usbs_status usbs_cons_adjoint_apply(usbs_ctx* ctx, usbs_problem* p, const double* y_dev,
                                    const double* v_dev, int64_t ldv, int k, double* y_out_dev,
                                    int64_t ldy, double* gram_dev);
/* A*(y) on the problem's merged pattern (nnz values, dev) and that pattern
 * (host: rowptr int64 n+1, col int32 nnz, nent int32 nnz = constraint
 * entries per slot, zero for slots that only hold cost entries):
 * adjoint_matrix (problem.py:160-161, 214-220). */
usbs_status usbs_cons_adjoint_values(usbs_ctx* ctx, usbs_problem* p, const double* y_dev,
                                     double* vals_dev);
usbs_status usbs_problem_pattern(usbs_problem* p, int64_t* rowptr, int32_t* col, int32_t* nent);
/* out (m, dev) = A(X) for a dense n x n X (dev, ld): primal_image_dense
 * (problem.py:157-158, 210-212). */
usbs_status usbs_cons_image_dense(usbs_ctx* ctx, usbs_problem* p, const double* x_dev, int64_t ldx,
                                  double* out_dev);
/* out (m x d, dev, ld >= d) = rows svec(V^T A_i V): compressed_rows
 * (problem.py:169-173, 229-239); the solver itself never materialises it. */
usbs_status usbs_cons_compressed_rows(usbs_ctx* ctx, usbs_problem* p, const double* v_dev,
                                      int64_t ldv, int k, double* out_dev, int64_t ldo);

/* dst[i] = src[idx[i]] for i < n (dev): the ghost-dual refresh of an
 * entry-family row shard (the mirrored Z slots of constraints owned by
 * another rank read these copies; dist.EntryShardPlan). */
usbs_status usbs_gather(usbs_ctx* ctx, int64_t n, const int64_t* idx_dev, const double* src_dev,
                        double* dst_dev);

/* dst[i, :k] = src[idx[i], :k] for i < n (dev, row-major, leading dimensions
 * lds, ldd >= k); a zero row where idx[i] < 0.  warm_start_pad's embedding of
 * the dual vectors, basis and primal factor into a larger problem
 * (bundle.py:781-792: y[cmap] = prev.y, basis[vmap] = model.basis, ...),
 * evaluated through the inverse map. */
usbs_status usbs_gather_rows(usbs_ctx* ctx, int64_t n, int k, const int64_t* idx_dev, const double* src_dev,
                             int64_t lds, double* dst_dev, int64_t ldd);

/* ---- device-controlled loop (alternating_max, subqp.py:552-614) -------------
 * Everything the context launches between usbs_loop_begin and usbs_loop_end is
 * captured as the body of a CUDA-graph WHILE node instead of being run; a
 * one-thread kernel closing the body does counter[0] += 1 and continues while
 * sqrt(max(red[0], 0)) > thresh and counter[0] < max_iters -- the reference's
 * "until ||nu' - nu|| <= tol (1 + ||b||) or max_passes" evaluated on the device,
 * so the passes run back to back with no host read.  usbs_loop_end launches the
 * loop on the context's stream (the body runs at least once); the caller zeroes
 * counter_dev first and reads it afterwards.  usbs_loop_abort drops a capture
 * after a failed call inside the body. */
usbs_status usbs_loop_begin(usbs_ctx* ctx);
usbs_status usbs_loop_end(usbs_ctx* ctx, const double* red_dev, double thresh, int max_iters,
                          int* counter_dev);
usbs_status usbs_loop_abort(usbs_ctx* ctx);

/* ---- rounding -------------------------------------- */
/* make_test_matrix (sketch.py:25-27): rows [row0, row1) of
 * np.random.RandomState(seed & 0x7FFFFFFF).standard_normal((n, r)) into
 * host memory out (C order), bit-identical to numpy's legacy MT19937 +
 * polar Gaussian.  Host-only (no device, no context): native so the fill
 * runs outside the Python GIL while the problem is planned; pipelined over
 * host threads (USBS_PSI_THREADS overrides the count; 0 = the caller only). */
usbs_status usbs_make_test_matrix(int64_t seed, int64_t n, int r, int64_t row0, int64_t row1, double* out);

/* maxcut_round (rounding.py:34-51): for every column j of the factor U
 * (n x r, dev, row-major, ld >= r, r <= 64) the cut value of
 * x = sign(U[:, j]) (zero signs to +1), 0.25 x^T L x = sum_e w_e [x_u != x_v]
 * over the graph's edges (dev: eu < ev int32, ew double, ne of them) --
 * exact, hence equal to the reference bit for bit, for integer weights.
 * Outputs: vals (host, r), *best (host, first maximum, the reference's
 * strict '>'), x_dev (dev int32, n) = the assignment of the best column. */
usbs_status usbs_maxcut_round(usbs_ctx* ctx, int64_t n, int64_t ne, const int32_t* eu_dev,
                              const int32_t* ev_dev, const double* ew_dev, const double* u_dev,
                              int64_t ldu, int r, double* vals, int* best, int32_t* x_dev);

#ifdef __cplusplus
}
#endif
#endif /* USBS_B200_H */
