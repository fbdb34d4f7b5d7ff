/*
 * otn_b200.h — C-ABI of the B200-native truncated-Newton EOT solver.
 *
 * This is the drop-in boundary for the reference's hot path (otnewton 0.1.0,
 * arXiv 2504.02067).  Each entry point replaces one operator of the
 * reference's internal operator seam; the reference interface
 * it replaces is cited as  file:line  relative to /root/reference/pkg/src/otnewton.
 *
 * Conventions
 *  - All array arguments are DEVICE pointers to float64 data owned by the
 *    caller (e.g. torch CUDA tensors).  No torch types cross this boundary.
 *  - n x n matrices (cost C, plan P) are row-major with leading dimension
 *    `ld` (fixed at otn_create; a multiple of 32, padding columns ignored on
 *    read and written as 0 on write).  Vectors have n entries.
 *  - Calls are stream-ordered on the context's stream.  Only calls that return
 *    host scalars (pointer arguments named host_*) synchronize the stream.
 *  - Return value: OTN_OK, an OTN_ERR_* failure, or an OTN_ST_* solver status
 *    that the host maps onto the reference's exception taxonomy
 *    (errors.py:11-65) with the same diagnostics.
 *  - A context is single-owner and not thread-safe, like the reference's
 *    DualState (dual.py:22-28).
 *  - Reductions are fixed-order trees without floating-point atomics: results
 *    are bit-reproducible run to run.
 */
#ifndef OTN_B200_H
#define OTN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OTN_ABI_VERSION 2

enum otn_status {
  OTN_OK = 0,
  OTN_ERR_CUDA = 1,              /* CUDA runtime failure; see otn_last_error()            */
  OTN_ERR_ARG = 2,               /* bad argument                                          */
  OTN_ST_PLAN_OVERFLOW = 10,     /* PlanOverflowError   (_kernels.py:55-58)               */
  OTN_ST_NONPOSITIVE_SUMS = 11,  /* ConditioningError   (newton.py:76-77)                 */
  OTN_ST_BREAKDOWN = 12,         /* ConditioningError   (newton.py:155-156)               */
  OTN_ST_PRECOND = 13,           /* ConditioningError   (newton.py:137-139)               */
  OTN_ST_NONCONVERGENCE = 14,    /* NonconvergenceError (newton.py:168-172), best = x     */
  OTN_ST_STAGNATION = 15,        /* StagnationError     (newton.py:202-205)               */
  OTN_ST_DOMAIN = 16             /* DomainError         (core.py:47-50)                   */
};

/* Vector ops for otn_vec (element-wise, operand order as in the reference). */
enum otn_vec_op {
  OTN_VEC_ADD_SUB = 0,  /* out = (a + b) - c        projector.py:146, dual.py:189          */
  OTN_VEC_AXPY = 1,     /* out = a + s*b            projector.py:234                        */
  OTN_VEC_STEP_V = 2,   /* out = (a + s*b) + (c - d) projector.py:235                       */
  OTN_VEC_EXTRAP = 3,   /* out = a + s*(a - b)      driver.py:170-175                       */
  OTN_VEC_EXP = 4,      /* out = exp(a)             dual.py:134-138                         */
  OTN_VEC_GRAD = 5,     /* out = exp(a) - b         projector.py:176                        */
  OTN_VEC_MUL_SUB = 6,  /* out = a*b - s*c          newton.py:102-105 (rP*d - rho*P(..))    */
  OTN_VEC_DIV = 7,      /* out = a / b              newton.py:98,112,158                    */
  OTN_VEC_SUB = 8,      /* out = a - b              newton.py:146,164                       */
  OTN_VEC_ADD = 9,      /* out = a + b              newton.py:199                           */
  OTN_VEC_PRECOND = 10, /* out = a * (1 - s*b)      newton.py:137                           */
  OTN_VEC_NEG_DIV = 11, /* out = (-a) / b           newton.py:192, projector.py:201         */
  OTN_VEC_RESCALE = 12, /* out = a * exp(b - c)     (sharded column-LSE combine)            */
  OTN_VEC_LSE_FIN = 13, /* out = a + (b finite ? b + log(c) : -inf)   _kernels.py:36-42     */
  OTN_VEC_LSE_FIN_SUB = 14, /* out = a - (b finite ? b + log(c) : -inf)  dual.py:182        */
  OTN_VEC_ROUND_SCALE = 15, /* out = b > 0 ? min(1, a / b) : 1          driver.py:193,198     */
  OTN_VEC_SUB_MUL = 16, /* out = a - b*c              driver.py:201-202                     */
  OTN_VEC_MUL = 17,     /* out = a * b                newton.py:102                         */
  OTN_VEC_COPY = 18     /* out = a                    dual.py:183 (log c(P) := log c)       */
};

/* Reductions for otn_reduce; results go to host_out[0..1]. */
enum otn_reduce_op {
  OTN_RED_ROW_STATS = 0, /* [sum|exp(a)-b|, sum b*b/exp(a)]; flags: exp(a)<=0 -> 1, b<0 -> 2
                            (projector.py:176-177, core.py:42-52)                         */
  OTN_RED_GRAD_L1 = 1,   /* [sum|exp(a)-b|, sum|exp(c)-d|]   dual.py:142-148              */
  OTN_RED_SUM_EXP = 2,   /* [sum exp(a)]                      projector.py:122-126         */
  OTN_RED_DOT = 3,       /* [sum a*b]                         dual.py:150-153              */
  OTN_RED_L1 = 4,        /* [sum |a|]                                                      */
  OTN_RED_L1_ADD = 5,    /* [sum |a + b|]                     newton.py:199-200            */
  OTN_RED_NONPOS = 6,    /* [count(a <= 0)]                   newton.py:138                */
  OTN_RED_MAX = 7,       /* [max a]                                                        */
  OTN_RED_L1_DOT = 8,    /* [sum |a|, sum a*b]                newton.py:162-165            */
  OTN_RED_OUTSIDE = 9    /* [count(!(2^-700 <= a <= 2^700))]  shifted column-LSE check     */
};

/* Point-cloud pass operations for otn_pc_pass. */
enum otn_pc_op {
  OTN_PC_LSE = 0,   /* out_i = outer_i +/- LSE_j(e_ij)                                     */
  OTN_PC_DOT = 1,   /* out_i = sum_j exp(e_ij) vec_j                                       */
  OTN_PC_DIAG = 2,  /* out_i = sum_j exp(e_ij)^2 vec_j; out2_i = max_j e_ij                */
  OTN_PC_MAXD = 3,  /* out_i = max_j D_ij (raw squared distance; pass cmax = 0)             */
  OTN_PC_LSE_PART = 4, /* out_i = max_j e_ij, out2_i = sum_j exp(e_ij - out_i) (shard partial) */
  OTN_PC_DOTC = 5,  /* out_i = sum_j exp(e_ij) C_ij vec_j   (primal cost <P, C>)            */
  OTN_PC_CDOT = 6,  /* out_i = sum_j C_ij vec_j             (rank-one term of <P, C>)       */
  OTN_PC_LSE_SHIFT = 7 /* out_i = sum_j exp(e_ij - outer_i)  (shard partial against a known
                          shift: ONE sum-allreduce per sharded column LSE)                 */
};

typedef struct otn_ctx otn_ctx;

/* Outcome of otn_newton / otn_pcg (host copy of the device record). */
typedef struct {
  int32_t status;      /* OTN_OK or OTN_ST_*                                         */
  int32_t pcg_calls;   /* pcg_solve calls made (op tally: diag_prc on the first)   */
  int64_t cg_iters;    /* newton: total CG iterations; pcg: iterations             */
  int64_t hvps;        /* F(rho)x products with rho != 0 (2 matvec passes each)    */
  double rho_final;    /* newton: discount of the last PCG call (newton.py:209)    */
  double resid_l1;     /* newton: undiscounted residual L1 (newton.py:199-201)     */
  double slope;        /* newton: -(grad_u . d_u)  (projector.py:205)              */
  double diag_rho;     /* NonconvergenceError diagnostics: rho                     */
  double diag_resid;   /* NonconvergenceError diagnostics: residual_l1             */
  int32_t plan_mode;   /* plan access of the launch: 0 streamed ring, 2 / 3 compressed
                          rows in shared / global memory (k_partition)             */
  int32_t plan_rows_max; /* most rows owned by one CTA                               */
  int64_t plan_nnz;    /* nonzero plan entries (materialize's per-row counts)      */
  int64_t plan_span;   /* entries inside the rows' nonzero 64-column segments: what
                          the ring streams per pass (roofline bytes = 8 x this)     */
} otn_solve_result;

/* ---- context ---------------------------------------------------------- */
int otn_abi_version(void);
const char* otn_last_error(void);
/* Allocate the device workspace for problems of size n (leading dim ld). */
int otn_create(otn_ctx** out, int device, int64_t n, int64_t ld, void* stream);
int otn_destroy(otn_ctx* ctx);
int otn_set_stream(otn_ctx* ctx, void* stream);
/* out4 = {n, ld, persistent-solver CTAs, workspace bytes} */
int otn_info(const otn_ctx* ctx, int64_t* out4);
/* out4 = {SMs, row-LSE path (0 register streaming, >0 CTAs of the bulk-copy
 * row LSE), column-reduction slabs, last configuration error code}          */
int otn_config(const otn_ctx* ctx, int64_t* out4);
/* Synchronize and copy the row partition and plan mode of the last
 * persistent-solver launch: host[0..G] = row boundaries of the G CTAs,
 * host[G+1] = plan mode (0 streamed ring, 2 sparse shared-memory rows, 3
 * sparse global-memory rows; 1 is retired); G = otn_info()[2].  Diagnostic (bench / tests).     */
int otn_coop_layout(otn_ctx* ctx, int* host);
/* Stream-ordered copies of n doubles (no host synchronization): device to
 * device, and host (page-locked for asynchrony) to device.  The solver's
 * vector bookkeeping (log-marginal caches, targets) on the ctx stream.     */
int otn_copy(otn_ctx* ctx, double* dst, const double* src, int64_t n);
int otn_upload(otn_ctx* ctx, double* dst, const double* host_src, int64_t n);
/* Zero `bytes` bytes of device memory, stream-ordered (buffer setup without
 * a framework fill kernel).                                                 */
int otn_zero(otn_ctx* ctx, void* dst, int64_t bytes);
/* Cost preparation, once per problem (dual.py:77-89): host_sym = (C == C^T)
 * over the n x n block of the ld-strided C (synchronizes); otn_transpose
 * writes C^T (padding columns 0) for the column passes of an asymmetric C.  */
int otn_is_symmetric(otn_ctx* ctx, const double* C, int* host_sym);
int otn_transpose(otn_ctx* ctx, double* out, const double* C);
/* Squared-Euclidean cost of 8-bit point sets on the tensor cores (K10, the
 * setup GEMM of problems.py:87-111 for 784-d pixel sets): X, Y are n x d
 * row-major float64 DEVICE arrays whose entries are integers in [0, 255];
 * C (n x ld) := max(|x_i|^2 + |y_j|^2 - 2 x_i.y_j, 0) / (its maximum),
 * padding columns 0.  The dot products run as exact u8 x u8 -> s32 MMAs, so
 * C equals the host's float64 evaluation bit for bit.  host_max receives the
 * maximum before normalization.  OTN_ERR_ARG when an entry is not an
 * integer in [0, 255].  Synchronizes.                                        */
int otn_pixel_cost(otn_ctx* ctx, const double* X, const double* Y, int64_t d, double* C,
                   double* host_max);
/* Synchronize and copy the four device status flags to the host:
 * [0] plan overflow, [1] nonpositive sums, [2] reduce domain, [3] rounding. */
int otn_read_flags(otn_ctx* ctx, int* host4);

/* ---- log-domain reductions (K1, K2, K3) --------------------------------- */
/* out_i = outer_i + LSE_j(neg_gamma*C_ij + inner_j); outer may be NULL (0.0).
 * Replaces _kernels.py:22-42 log_plan_row_sums(K, u, v) with K = -gamma*C
 * formed in registers (same single rounding as dual.py:74).               */
int otn_lse_rows(otn_ctx* ctx, const double* C, double neg_gamma, const double* outer,
                 const double* inner, double* out);
/* out_j = outer_j + LSE_i(neg_gamma*C_ij + inner_i) — the column reduction
 * log_plan_row_sums(K^T, v, u) of dual.py:91-102 / dual.py:186-194.  With
 * symmetric != 0 the rows of C are read instead (K^T aliases K, dual.py:80-88);
 * a caller holding a materialized transpose (as the reference holds K^T,
 * dual.py:77-89) passes it with symmetric = 1: a coalesced row pass.        */
int otn_lse_cols(otn_ctx* ctx, const double* C, int symmetric, double neg_gamma,
                 const double* outer, const double* inner, double* out);
/* v_j = log_c_j - LSE_i(neg_gamma*C_ij + u_i)   (rebalance_columns, dual.py:179-184) */
int otn_rebalance_cols(otn_ctx* ctx, const double* C, int symmetric, double neg_gamma,
                       const double* log_c, const double* u, double* v_out);
/* Line-search objective: out_j = (v + alpha*dv)_j + LSE_i(neg_gamma*C_ij + (u + alpha*du)_i)
 * and *host_mass = sum_j exp(out_j) (overflow -> inf).
 * Replaces dual.py:171-175 trial_log_col_sums + projector.py:122-126 _mass. */
int otn_trial_cols(otn_ctx* ctx, const double* C, int symmetric, double neg_gamma,
                   const double* u, const double* du, const double* v, const double* dv,
                   double alpha, double* out, double* host_mass);

/* ---- plan (K4 + K5) ------------------------------------------------------ */
/* A plan is the pair (P, seg_mask).  seg_mask (nullable = dense) holds one bit
 * per 64-column (512-byte) row segment, set iff the segment has a nonzero, and
 * the row's nonzero count: n rows x OTN_MASK_WORDS(ld) uint64 words, bit s%64
 * of word s/64 for segment s, then one count word.  The Hessian-vector
 * kernels skip all-zero segments (exp underflow makes most of the plan
 * exactly 0 at weak regularization) and, when the plan is sparse enough,
 * compress each CTA's rows into shared memory; skipped terms are exact zeros.*/
#define OTN_MASK_WORDS(ld) (((ld) + 4095) / 4096 + 1)
/* P_ij = exp((neg_gamma*C_ij + v_j) + u_i), and seg_mask if non-NULL.  If
 * icP != NULL also mu_i = (sum_j P_ij^2 icP_j) / rP_i (the Jacobi diagonal,
 * K5 fused).  Overflow (an exponent > 700) sets a device flag that the next
 * otn_newton reports as OTN_ST_PLAN_OVERFLOW; when host_overflow != NULL the
 * call synchronizes and returns the flag.  Replaces _kernels.py:45-61
 * materialize_plan and newton.py:107-112 diag_prc / _kernels.py:64-74.     */
int otn_materialize(otn_ctx* ctx, const double* C, double neg_gamma, const double* u,
                    const double* v, double* P, const double* icP, const double* rP,
                    double* mu, int* host_overflow, uint64_t* seg_mask);
/* seg_mask of an externally supplied plan. */
int otn_plan_mask(otn_ctx* ctx, const double* P, uint64_t* seg_mask);
/* rP = exp(log_rP), cP = exp(log_cP), icP = 1/cP; nonpositive sums set the
 * OTN_ST_NONPOSITIVE_SUMS flag (DiscountedSystem.__init__, newton.py:72-90). */
int otn_system_prep(otn_ctx* ctx, const double* log_rP, const double* log_cP, double* rP,
                    double* cP, double* icP, int* host_bad);
/* (P*P) @ w   (_kernels.py:64-74) */
int otn_square_matvec(otn_ctx* ctx, const double* P, const double* w, double* out);

/* ---- Hessian-vector products (K6, K7) ------------------------------------ */
int otn_matvec(otn_ctx* ctx, const double* P, const uint64_t* seg_mask, const double* x,
               double* out);                                      /* newton.py:43-48  */
int otn_rmatvec(otn_ctx* ctx, const double* P, const uint64_t* seg_mask, const double* x,
                double* out);                                     /* newton.py:51-56  */
/* out = rP*d - rho*P((P^T d)/cP)   (newton.py:100-105) */
int otn_apply_F(otn_ctx* ctx, const double* P, const uint64_t* seg_mask, const double* rP,
                const double* cP, double rho, const double* d, double* out);
/* out = (P^T d)/cP   (newton.py:96-98) */
int otn_apply_pc(otn_ctx* ctx, const double* P, const uint64_t* seg_mask, const double* cP,
                 const double* d, double* out);

/* ---- device-resident solvers (K8 + the CG / Newton loops) ----------------- */
/* Jacobi-PCG on F(rho) x = b to L1 recurrence residual <= tol, x in/out
 * (has_x0 = 0: start from zero).  One persistent cooperative launch, no host
 * round trip per iteration.  Replaces newton.py:123-172 pcg_solve.          */
int otn_pcg(otn_ctx* ctx, const double* P, const uint64_t* seg_mask, const double* rP,
            const double* cP, const double* mu, double rho, const double* b, double tol,
            double* x, int has_x0, int64_t max_iters, otn_solve_result* host_res);
/* Annealed truncated-Newton direction (newton.py:175-210) for gradient g,
 * forcing eta, starting discount rho0; writes d_u and, if d_v != NULL, the
 * back-substitution d_v = -(P^T d_u)/cP plus the slope -(g.d_u)
 * (projector.py:196-205).  One persistent cooperative launch.               */
int otn_newton(otn_ctx* ctx, const double* P, const uint64_t* seg_mask, const double* rP,
               const double* cP, const double* mu, const double* g, double eta, double rho0,
               int zero_init, int64_t max_iters, double* d_u, double* d_v,
               otn_solve_result* host_res);

/* One projector Newton step with its first line-search trial and, when that
 * trial is accepted, the accept path — all enqueued back to back, one host
 * synchronization (projector.py:196-238 for alpha = 1).  Runs otn_newton;
 * then, if the status is OK and the slope positive, the trial column sums at
 * alpha = 1 into `trial` (as otn_trial_cols on (C_cols, symmetric),
 * projector.py:122-126; the row LSE below reads C) and their
 * mass; then, only if the full step passes the mass-form Armijo test with
 * (armijo_c1, slope_floor) (projector.py:215-217: no backtracking), the
 * accept path: u += d_u; v = (v + d_v) + (log_c - trial); lc := log_c;
 * lr = row LSE (u, v) (dual.py:203-208); grad = exp(lr) - r; row statistics
 * as OTN_RED_ROW_STATS on (lr, r).  Device-side flags gate the launches, so
 * a step that must backtrack (or falls back) leaves u, v, lc, lr untouched
 * and the host continues exactly as after otn_newton + otn_trial_cols.
 * host_out = {mass, row-stats[0], row-stats[1], trial ran (0/1),
 * accepted (0/1)}; host_flags[0] = row-stats flags.  Returns the Newton
 * status like otn_newton.                                                    */
int otn_newton_step(otn_ctx* ctx, const double* P, const uint64_t* seg_mask, const double* rP,
                    const double* cP, const double* mu, const double* g, double eta, double rho0,
                    int zero_init, int64_t max_iters, double* d_u, double* d_v, const double* C,
                    const double* C_cols, int symmetric, double neg_gamma, double* u, double* v,
                    const double* r,
                    const double* log_c, double* trial, double* lc, double* lr, double* grad,
                    double armijo_c1, double slope_floor, otn_solve_result* host_res,
                    double* host_out, int* host_flags);
/* host_out == NULL: otn_newton_step only enqueues (the host is free until
 * the results are needed); otn_newton_step_wait synchronizes and fills
 * host_res / host_out / host_flags as otn_newton_step would have.           */
int otn_newton_step_wait(otn_ctx* ctx, otn_solve_result* host_res, double* host_out,
                         int* host_flags);

/* Telemetry: with timing on, every persistent-solver launch (the partition
 * kernel + k_coop) is bracketed by CUDA events; otn_coop_ms waits for the
 * last one and returns its device time in milliseconds.                      */
int otn_set_timing(otn_ctx* ctx, int on);
int otn_coop_ms(otn_ctx* ctx, float* ms);

/* Diagnostic: run building block `what` of the persistent solver `reps` times
 * in one launch (0 grid barrier, 1 grid reduction, 2 column-partial pass,
 * 3 row pass, 4 P^T x with its reductions, 5 full HVP).  Tooling only.     */
int otn_probe(otn_ctx* ctx, const double* P, const uint64_t* seg_mask, const double* cP,
              const double* rP, const double* x, double* out, int what, int64_t reps);

/* ---- on-the-fly point-cloud cost (D4/D5; no n x n array anywhere) ----------
 * One pass over all (row point a_i, column point b_j) pairs of the two SoA
 * point sets A (na points, lda stride between coordinates) and B:
 *   C_ij = (sum_k (a_ik - b_jk)^2) / cmax  (left-to-right sum, IEEE division:
 *          bit-identical to PointCloudProblem.materialize_cost),
 *   e_ij = order 0: (neg_gamma*C_ij + colpot_j) + rowpot_i
 *          order 1: (neg_gamma*C_ij + rowpot_i) + colpot_j
 *   with colpot_j += alpha*colpot_d_j when colpot_d != NULL and absent
 *   potentials treated as "not added".
 * Row passes of the reference's operators use A = X, B = Y; column passes
 * (P^T x, column LSE: log_plan_row_sums(K^T, ...), dual.py:97-175) swap the
 * point sets and use order 1 so the exponent keeps the reference's rounding
 * ((K + v) + u, _kernels.py:52-53).  For a row-sharded solve A holds this
 * rank's rows; column passes then produce per-rank partials the caller
 * combines with an allreduce.                                                */
int otn_pc_pass(otn_ctx* ctx, int op, const double* A, int64_t na, int64_t lda, const double* B,
                int64_t nb, int64_t ldb, int d, double cmax, double neg_gamma, int order,
                const double* colpot, const double* colpot_d, double alpha, const double* rowpot,
                const double* vec, const double* outer, const double* outer_d, int mode,
                double* out, double* out2);
/* Element-wise op / reduction on explicit lengths (sharded vectors). */
int otn_vec_n(otn_ctx* ctx, int64_t n, int op, double s, const double* a, const double* b,
              const double* c, const double* d, double* out);
int otn_reduce_n(otn_ctx* ctx, int64_t n, int op, const double* a, const double* b,
                 const double* c, const double* d, double* host_out, int* host_flags);
/* As otn_reduce_n, the two results written stream-ordered to DEVICE memory
 * dev_out[0..1] (no host synchronization): a row-sharded solve reduces its
 * shard into a device buffer, allreduces the buffer (NCCL, same stream order)
 * and reads all of a step's scalars back once.                              */
int otn_reduce_dev(otn_ctx* ctx, int64_t n, int op, const double* a, const double* b,
                   const double* c, const double* d, double* dev_out);

/* ---- projector / driver vector work ------------------------------------- */
int otn_vec(otn_ctx* ctx, int op, double s, const double* a, const double* b, const double* c,
            const double* d, double* out);
int otn_reduce(otn_ctx* ctx, int op, const double* a, const double* b, const double* c,
               const double* d, double* host_out, int* host_flags);
/* Row statistics of the projector (projector.py:176, core.py:42-52) in one
 * pass: g = exp(lr) - r (as OTN_VEC_GRAD) and host_out = OTN_RED_ROW_STATS of
 * (lr, r), host_flags its domain flags.  Synchronizes.                      */
int otn_row_stats(otn_ctx* ctx, const double* lr, const double* r, double* g, double* host_out,
                  int* host_flags);
/* The accept step's vector updates (projector.py:234-236) in one launch:
 * u += alpha*d_u; v = (v + alpha*d_v) + (log_c - trial); lc := log_c.       */
int otn_accept(otn_ctx* ctx, double alpha, double* u, const double* d_u, double* v,
               const double* d_v, const double* log_c, const double* trial, double* lc);
/* As otn_reduce without the host synchronization: the two results are copied
 * stream-ordered into host_out, which must be page-locked; they are valid
 * once the stream has passed this point (record an event after the call).
 * For read-backs the control flow does not wait on (per-stage telemetry). */
int otn_reduce_async(otn_ctx* ctx, int op, const double* a, const double* b, const double* c,
                     const double* d, double* host_out_pinned);
/* Round P onto U(r, c) in place and return host_out = {<P, C>, deficit}
 * (driver.py:178-208 round_plan + driver.py:306-310 vdot).  C may be NULL
 * (primal cost skipped).  host_flags: 1 = negative entry (DomainError),
 * 2 = zero total mass (DegenerateInputError).                               */
int otn_round_plan(otn_ctx* ctx, double* P, const double* C, const double* r, const double* c,
                   double* host_out, int* host_flags);

#ifdef __cplusplus
}
#endif

#endif /* OTN_B200_H */
