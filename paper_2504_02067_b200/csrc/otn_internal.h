// Internal declarations shared by the kernel translation units and the C-ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/otn_b200.h"

namespace otn {

constexpr int kCoopThreads = 512;       // one CTA per SM for the persistent solver
constexpr int kLseThreads = 256;        // 8 warps: one row per warp
constexpr int kColTile = 64;            // columns per CTA in column reductions
constexpr int kRedSlots = 2;            // rotating grid-reduction slots
constexpr int kRedWidth = 4;            // values per grid reduction (at most)
constexpr int kRedStride = 256;         // CTA partials per value (>= persistent-solver CTAs)
constexpr int kSegCols = 64;            // plan segment (zero-skip granularity): 64 cols = 512 B
constexpr int kSegWordCols = 64 * kSegCols;  // columns covered by one 64-bit mask word

// Device-side solver record (mirrored by otn_solve_result on the host).
struct DevResult {
  int32_t status;
  int32_t pcg_calls;    // pcg_solve invocations (diag_prc is tallied on the first)
  int64_t cg_iters;     // newton: total CG iterations; pcg: iterations
  int64_t hvps;         // Hessian-vector products with rho != 0 (2 matvec passes each)
  double rho_final;     // rho of the last PCG call (newton.py:209)
  double resid_l1;      // undiscounted residual (newton) / recurrence residual (pcg)
  double slope;         // -(grad_u . d_u)  (projector.py:205)
  double diag_rho;      // NonconvergenceError diagnostics (newton.py:168-172)
  double diag_resid;
  int32_t plan_mode;    // k_partition's choice for this launch
  int32_t plan_rows_max;
  int64_t plan_nnz;     // nonzeros of the plan
  int64_t plan_span;    // entries in nonzero 64-column segments
};

}  // namespace otn

struct otn_ctx {
  int device;
  int64_t n, ld;
  cudaStream_t stream;
  int num_sms;
  int coop_blocks;        // grid size of the persistent solver (all co-resident)
  int lse_slabs;          // row slabs of the column reductions
  // device workspace (one allocation)
  void* ws;
  size_t ws_bytes;
  double *r, *z, *p, *q, *M, *wc, *sv, *vtmp0, *vtmp1;   // length ld each
  double* wpart;          // coop_blocks x ld column partials
  double* red;            // grid-exchange slots: kRedSlots x kRedWidth x kRedStride x 16 B
  uint32_t* gs_epoch;     // last grid-exchange epoch (k_coop reads it at start, writes at exit)
  double* lse_part;       // lse_slabs x ld x 2 (m, s) column-LSE partials
  int lse_bulk_ctas;      // persistent CTAs of the bulk-copy row LSE (0: register streaming)
  int cfg_err;            // first error while configuring optional kernels (diagnostic)
  void* pix_scratch;      // otn_pixel_cost: packed u8 point sets + norms (grown on demand)
  size_t pix_scratch_bytes;
  int pc_exact;           // on-the-fly passes: exact-cost exponent everywhere (OTN_PC_EXACT=1)
  double* scal;           // 64 device scalars
  int* flags;             // 16 device flag words
  int* part;              // coop_blocks + 2 ints: row partition + plan mode (k_partition)
  void* sg;               // coop_blocks x kSparseGBytes (ld <= 4096 only; else nullptr)
  otn::DevResult* dres;
  // pinned host mirrors
  double* h_scal;
  int* h_flags;
  otn::DevResult* h_res;
  int time_coop;          // record ev_coop around every persistent-solver launch
  cudaEvent_t ev_coop[2];
};

// Launchers (all stream-ordered on ctx->stream; return cudaError_t).
namespace otn {
// gate (nullable): a device flag; the launch does nothing when *gate == 0
// (otn_newton_step enqueues the accept path before the host sees the result).
int lse_bulk_grid(int num_sms, int64_t n, int64_t ld, int* err);
cudaError_t launch_lse_rows(otn_ctx* x, const double* C, double ng, const double* outer,
                            const double* outer_d, const double* inner, const double* inner_d,
                            double alpha, int mode, double* out, const int* gate = nullptr);
cudaError_t launch_lse_cols(otn_ctx* x, const double* C, double ng, const double* outer,
                            const double* outer_d, const double* inner, const double* inner_d,
                            double alpha, int mode, double* out, const int* gate = nullptr);
cudaError_t launch_materialize(otn_ctx* x, const double* C, double ng, const double* u,
                               const double* v, double* P, const double* icP, const double* rP,
                               double* mu, int* flag, uint64_t* mask);
cudaError_t launch_plan_mask(otn_ctx* x, const double* P, uint64_t* mask);
cudaError_t launch_sys_prep(otn_ctx* x, const double* log_rP, const double* log_cP, double* rP,
                            double* cP, double* icP, int* flag);
cudaError_t launch_square_matvec(otn_ctx* x, const double* P, const double* w, double* out);

// Persistent cooperative solver.
enum CoopMode { kModeNewton = 0, kModePcg = 1, kModeHvp = 2, kModePc = 3, kModeMatvec = 4,
                kModeRmatvec = 5, kModeProbe = 6 };
struct CoopArgs {
  const double* P;
  int64_t n, ld;
  const double* rP;
  const double* cP;
  const double* mu;
  const double* g;        // newton: grad_u
  const double* b;        // pcg: right-hand side
  const double* xin;      // hvp / pc / matvec: input vector
  double* d;              // newton: d_u out; pcg: x in/out; others: output vector
  double* dv;             // newton: optional d_v out
  double eta, rho0, rho, tol;
  int zero_init, has_x0, mode, pad;
  int64_t max_iters;
  const int* pre_flags;   // materialize / prep flags checked first (nullable)
  const uint64_t* mask;   // plan segment occupancy (nullable = dense); mw words per row
  int64_t mw;
  int stages;             // shared-memory ring stages (set by launch_coop)
  int pad2;
  const int* part;        // row partition + plan mode (k_partition, set by launch_coop)
  void* sg;               // compressed-rows buffer of kPlanSparseG (nullable; set by launch_coop)
  // workspace
  double *r, *z, *p, *q, *M, *wc, *sv, *wpart;
  double* red;            // grid exchange slots (k_coop gs_exchange: 2 x kRedWidth x kRedStride x 16 B)
  uint32_t* gs_epoch;     // last grid-exchange epoch of the context
  DevResult* res;
  int* step_flags;        // nullable: otn_newton_step's gate words (see k_step_gate stage 0)
};
cudaError_t launch_coop(otn_ctx* x, const CoopArgs& a);
// K10 for 8-bit point sets (otn_pix.cu): C := squared distances / max, exact.
cudaError_t launch_pixel_cost(otn_ctx* x, const double* X, const double* Y, int64_t d, double* C,
                              unsigned long long* cmax_bits, int* err);
size_t sparse_g_bytes_per_cta();        // kPlanSparseG buffer slice (allocated when ld <= 4096)

// Vector kernels and single-CTA reductions.
cudaError_t launch_vec(otn_ctx* x, int op, int64_t n, double s0, const double* a, const double* b,
                       const double* c, const double* d, double* out, const int* gate = nullptr);
cudaError_t launch_reduce(otn_ctx* x, int op, int64_t n, const double* a, const double* b,
                          const double* c, const double* d, double* dst, int* flag,
                          const int* gate = nullptr);
// Newton-step gates (otn_newton_step): stage 0 -> flags[0] = (status OK and
// slope > 0), flags[2] = 0; stage 1 -> flags[1] = flags[0] and the Armijo test
// passes at alpha = 1 (mass = *mass).
// The accept path's vector updates in one launch (projector.py:234-236):
// u += s*du; v = (v + s*dv) + (logc - trial); lc = logc over ld entries.
cudaError_t launch_accept(otn_ctx* x, double s, double* u, const double* du, double* v,
                          const double* dv, const double* logc, const double* trial, double* lc,
                          const int* gate);
// OTN_RED_ROW_STATS that also writes g = exp(a) - b (OTN_VEC_GRAD) to `g`.
constexpr int kRedRowStatsGrad = 100;
cudaError_t launch_step_gate(otn_ctx* x, int stage, const DevResult* res, const double* mass,
                             double slope_floor, double armijo_c1, int* flags);
cudaError_t launch_symmetric(otn_ctx* x, const double* C, int* flag);
cudaError_t launch_transpose(otn_ctx* x, double* out, const double* C);
cudaError_t launch_round(otn_ctx* x, double* P, const double* C, const double* r, const double* c,
                         double* scratch_scalars, int* flag);

// On-the-fly point-cloud passes (otn_pc.cu).
struct PairArgs {
  const double* A;       // row points, SoA: A[k * lda + i]
  int64_t na, lda;
  const double* B;       // column points, SoA: B[k * ldb + j]
  int64_t nb, ldb;
  int d, op, order, mode;
  double cmax, ng;
  const double* colpot;    // added first (nullable)
  const double* colpot_d;  // colpot_eff = colpot + alpha * colpot_d (nullable)
  const double* rowpot;    // added second (nullable)
  double alpha;
  const double* vec;       // per-column vector (DOT / DIAG)
  const double* outer;     // LSE: out = outer +/- lse (nullable -> 0)
  const double* outer_d;
  double* out;             // per-row result
  double* out2;            // per-row aux (DIAG: max exponent; MAXD unused)
};
cudaError_t launch_pair(otn_ctx* x, const PairArgs& p);
}  // namespace otn
