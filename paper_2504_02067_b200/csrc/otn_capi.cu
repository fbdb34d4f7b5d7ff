// extern "C" boundary: context management and the entry points declared in
// include/otn_b200.h.  Every function validates its arguments, launches on the
// context's stream, and returns an otn_status code.
#include <sched.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>

#include "otn_internal.h"

namespace otn {
int coop_occupancy(int* blocks_per_sm);
}

namespace {

thread_local std::string g_err;

int fail(int code, const char* what, cudaError_t e = cudaSuccess) {
  char buf[512];
  if (e != cudaSuccess)
    snprintf(buf, sizeof(buf), "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  else
    snprintf(buf, sizeof(buf), "%s", what);
  g_err = buf;
  return code;
}

#define OTN_CUDA(call, what)                               \
  do {                                                     \
    cudaError_t e_ = (call);                               \
    if (e_ != cudaSuccess) return fail(OTN_ERR_CUDA, what, e_); \
  } while (0)

#define OTN_REQUIRE(cond, what) \
  do {                          \
    if (!(cond)) return fail(OTN_ERR_ARG, what); \
  } while (0)

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Wait for the stream by polling: the solver's host decisions wait on one
// scalar after every short kernel sequence, and a blocking synchronize adds
// the driver's wake-up latency to each of those round trips.  The busy poll
// is bounded: after 2 ms the thread yields between polls, after 20 ms it
// sleeps 100 us between polls (on-the-fly passes run for seconds; one core
// per rank must not spin for all of it).
cudaError_t stream_wait(cudaStream_t s) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  cudaError_t e;
  while ((e = cudaStreamQuery(s)) == cudaErrorNotReady) {
    const auto waited = clk::now() - t0;
    if (waited > std::chrono::milliseconds(20))
      std::this_thread::sleep_for(std::chrono::microseconds(100));
    else if (waited > std::chrono::milliseconds(2))
      sched_yield();
  }
  return e;
}

// The library links the static CUDA runtime, whose current device is per
// host thread and separate from torch's: every entry point that launches
// makes its context's device current for the call and restores the caller's.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const otn_ctx* x) {
    int cur = -1;
    if (x && cudaGetDevice(&cur) == cudaSuccess && cur != x->device) {
      if (cudaSetDevice(x->device) == cudaSuccess) prev = cur;
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int sync_copy(otn_ctx* x, void* host, const void* dev, size_t bytes, const char* what) {
  OTN_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, x->stream), what);
  OTN_CUDA(stream_wait(x->stream), what);
  return OTN_OK;
}

otn::CoopArgs base_args(otn_ctx* x, const double* P) {
  otn::CoopArgs a{};
  a.P = P;
  a.n = x->n;
  a.ld = x->ld;
  a.r = x->r;
  a.z = x->z;
  a.p = x->p;
  a.q = x->q;
  a.M = x->M;
  a.wc = x->wc;
  a.sv = x->sv;
  a.wpart = x->wpart;
  a.red = x->red;
  a.gs_epoch = x->gs_epoch;
  a.res = x->dres;
  return a;
}

int finish_solve(otn_ctx* x, otn_solve_result* host_res, const char* what) {
  int rc = sync_copy(x, x->h_res, x->dres, sizeof(otn::DevResult), what);
  if (rc) return rc;
  if (host_res) std::memcpy(host_res, x->h_res, sizeof(otn_solve_result));
  return x->h_res->status;
}

}  // namespace

static_assert(sizeof(otn_solve_result) == sizeof(otn::DevResult), "result layout");

extern "C" {

int otn_abi_version(void) { return OTN_ABI_VERSION; }

const char* otn_last_error(void) { return g_err.c_str(); }

int otn_create(otn_ctx** out, int device, int64_t n, int64_t ld, void* stream) {
  OTN_REQUIRE(out != nullptr, "otn_create: out is NULL");
  OTN_REQUIRE(n >= 1, "otn_create: n must be >= 1");
  OTN_REQUIRE(ld >= n && ld % 32 == 0, "otn_create: ld must be >= n and a multiple of 32");
  *out = nullptr;
  OTN_CUDA(cudaSetDevice(device), "otn_create: cudaSetDevice");
  otn_ctx* x = new otn_ctx();
  std::memset(x, 0, sizeof(otn_ctx));
  x->device = device;
  x->n = n;
  x->ld = ld;
  x->stream = static_cast<cudaStream_t>(stream);
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) { delete x; return fail(OTN_ERR_CUDA, "otn_create: properties", e); }
  if (!prop.cooperativeLaunch) { delete x; return fail(OTN_ERR_CUDA, "otn_create: no cooperative launch"); }
  x->num_sms = prop.multiProcessorCount;
  int per_sm = 0;
  e = (cudaError_t)otn::coop_occupancy(&per_sm);
  if (e != cudaSuccess || per_sm < 1) {
    delete x;
    return fail(OTN_ERR_CUDA, "otn_create: persistent solver does not fit on an SM", e);
  }
  x->coop_blocks = x->num_sms < otn::kRedStride ? x->num_sms : otn::kRedStride;   // one CTA per SM
  {
    // the persistent solver stages each CTA's (row, tile) spans in shared memory
    const int64_t rows = (n + x->coop_blocks - 1) / x->coop_blocks;
    const int64_t tiles = (ld + 4095) / 4096;
    if (rows * tiles > 8192 || tiles > 64) {
      delete x;
      return fail(OTN_ERR_ARG, "otn_create: n too large for the stored-plan solver "
                               "(rows per SM x 4096-column tiles must be <= 8192)");
    }
  }
  // column-reduction slabs: ~4 CTAs per SM over ld/64 column tiles
  {
    const int64_t tiles = (ld + otn::kColTile - 1) / otn::kColTile;
    int64_t want = (4LL * x->num_sms + tiles - 1) / tiles;
    if (want < 1) want = 1;
    if (want > 64) want = 64;
    if (want > n) want = n;
    x->lse_slabs = int(want);
  }
  const size_t vec = align_up(size_t(ld) * sizeof(double), 256);
  size_t off = 0;
  size_t o_r = off; off += vec;
  size_t o_z = off; off += vec;
  size_t o_p = off; off += vec;
  size_t o_q = off; off += vec;
  size_t o_M = off; off += vec;
  size_t o_wc = off; off += vec;
  size_t o_sv = off; off += vec;
  size_t o_t0 = off; off += vec;
  size_t o_t1 = off; off += vec;
  size_t o_wp = off; off += align_up(size_t(x->coop_blocks) * ld * sizeof(double), 256);
  size_t o_red = off; off += align_up(size_t(otn::kRedSlots) * otn::kRedStride * otn::kRedWidth * 16, 256);
  size_t o_gse = off; off += 256;
  size_t o_lse = off; off += align_up(size_t(x->lse_slabs) * ld * 2 * sizeof(double), 256);
  {
    // the bulk-copy row LSE is opt-in (OTN_LSE_BULK=1): measured slower than
    // the register-streaming kernel on B200 (tools/lse_bench.py)
    const char* exact = std::getenv("OTN_PC_EXACT");  // separable exponent off (A/B)
    x->pc_exact = exact && exact[0] == '1';
    const char* bulk = std::getenv("OTN_LSE_BULK");
    x->lse_bulk_ctas = (bulk && bulk[0] == '1') ? otn::lse_bulk_grid(x->num_sms, n, ld, &x->cfg_err)
                                                : 0;
  }
  size_t o_sc = off; off += align_up(64 * sizeof(double), 256);
  size_t o_fl = off; off += align_up(16 * sizeof(int), 256);
  size_t o_res = off; off += align_up(sizeof(otn::DevResult), 256);
  // part: G + 1 row boundaries, the plan mode, then 4 ints of plan statistics
  // (nnz and span as int64 pairs, k_partition)
  size_t o_part = off; off += align_up(size_t(x->coop_blocks + 8) * sizeof(int), 256);
  x->ws_bytes = off;
  e = cudaMalloc(&x->ws, off);
  if (e != cudaSuccess) { delete x; return fail(OTN_ERR_CUDA, "otn_create: cudaMalloc", e); }
  // compressed-rows buffer of the global sparse plan mode (one tile, and large
  // enough that a CTA's nonzeros can outgrow shared memory)
  x->sg = nullptr;
  if (ld <= 4096 && n >= 1024) {
    e = cudaMalloc(&x->sg, size_t(x->coop_blocks) * otn::sparse_g_bytes_per_cta());
    if (e != cudaSuccess) { cudaFree(x->ws); delete x; return fail(OTN_ERR_CUDA, "otn_create: sparse buffer", e); }
  }
  cudaMemset(x->ws, 0, off);
  char* base = static_cast<char*>(x->ws);
  x->r = (double*)(base + o_r);
  x->z = (double*)(base + o_z);
  x->p = (double*)(base + o_p);
  x->q = (double*)(base + o_q);
  x->M = (double*)(base + o_M);
  x->wc = (double*)(base + o_wc);
  x->sv = (double*)(base + o_sv);
  x->vtmp0 = (double*)(base + o_t0);
  x->vtmp1 = (double*)(base + o_t1);
  x->wpart = (double*)(base + o_wp);
  x->red = (double*)(base + o_red);
  x->gs_epoch = (uint32_t*)(base + o_gse);
  x->lse_part = (double*)(base + o_lse);

  x->scal = (double*)(base + o_sc);
  x->flags = (int*)(base + o_fl);
  x->dres = (otn::DevResult*)(base + o_res);
  x->part = (int*)(base + o_part);
  e = cudaMallocHost((void**)&x->h_scal, 64 * sizeof(double));
  if (e == cudaSuccess) e = cudaMallocHost((void**)&x->h_flags, 16 * sizeof(int));
  if (e == cudaSuccess) e = cudaMallocHost((void**)&x->h_res, sizeof(otn::DevResult));
  if (e == cudaSuccess) e = cudaEventCreate(&x->ev_coop[0]);
  if (e == cudaSuccess) e = cudaEventCreate(&x->ev_coop[1]);
  if (e != cudaSuccess) { otn_destroy(x); return fail(OTN_ERR_CUDA, "otn_create: pinned host", e); }
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { otn_destroy(x); return fail(OTN_ERR_CUDA, "otn_create: sync", e); }
  *out = x;
  return OTN_OK;
}

int otn_destroy(otn_ctx* x) {
  DeviceGuard dg_(x);
  if (!x) return OTN_OK;
  if (x->ws) cudaFree(x->ws);
  if (x->sg) cudaFree(x->sg);
  if (x->pix_scratch) cudaFree(x->pix_scratch);
  if (x->h_scal) cudaFreeHost(x->h_scal);
  if (x->h_flags) cudaFreeHost(x->h_flags);
  if (x->h_res) cudaFreeHost(x->h_res);
  if (x->ev_coop[0]) cudaEventDestroy(x->ev_coop[0]);
  if (x->ev_coop[1]) cudaEventDestroy(x->ev_coop[1]);
  delete x;
  return OTN_OK;
}

int otn_set_stream(otn_ctx* x, void* stream) {
  OTN_REQUIRE(x, "otn_set_stream: NULL ctx");
  x->stream = static_cast<cudaStream_t>(stream);
  return OTN_OK;
}

int otn_info(const otn_ctx* x, int64_t* out4) {
  OTN_REQUIRE(x && out4, "otn_info: NULL argument");
  out4[0] = x->n;
  out4[1] = x->ld;
  out4[2] = x->coop_blocks;
  out4[3] = int64_t(x->ws_bytes);
  return OTN_OK;
}

int otn_config(const otn_ctx* x, int64_t* out4) {
  OTN_REQUIRE(x && out4, "otn_config: NULL argument");
  out4[0] = x->num_sms;
  out4[1] = x->lse_bulk_ctas;
  out4[2] = x->lse_slabs;
  out4[3] = x->cfg_err;
  return OTN_OK;
}

int otn_copy(otn_ctx* x, double* dst, const double* src, int64_t n) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && dst && src && n >= 0, "otn_copy: bad argument");
  OTN_CUDA(cudaMemcpyAsync(dst, src, size_t(n) * sizeof(double), cudaMemcpyDeviceToDevice,
                           x->stream), "otn_copy");
  return OTN_OK;
}

int otn_upload(otn_ctx* x, double* dst, const double* host_src, int64_t n) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && dst && host_src && n >= 0, "otn_upload: bad argument");
  OTN_CUDA(cudaMemcpyAsync(dst, host_src, size_t(n) * sizeof(double), cudaMemcpyHostToDevice,
                           x->stream), "otn_upload");
  return OTN_OK;
}

int otn_zero(otn_ctx* x, void* dst, int64_t bytes) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && dst && bytes >= 0, "otn_zero: bad argument");
  OTN_CUDA(cudaMemsetAsync(dst, 0, size_t(bytes), x->stream), "otn_zero");
  return OTN_OK;
}

int otn_is_symmetric(otn_ctx* x, const double* C, int* host_sym) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && C && host_sym, "otn_is_symmetric: NULL argument");
  OTN_CUDA(cudaMemsetAsync(x->flags + 10, 0, sizeof(int), x->stream), "otn_is_symmetric: flag");
  OTN_CUDA(otn::launch_symmetric(x, C, x->flags + 10), "otn_is_symmetric");
  int rc = sync_copy(x, x->h_flags + 10, x->flags + 10, sizeof(int), "otn_is_symmetric: copy");
  if (rc) return rc;
  *host_sym = x->h_flags[10] == 0;
  return OTN_OK;
}

int otn_transpose(otn_ctx* x, double* out, const double* C) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && out && C && out != C, "otn_transpose: bad argument");
  OTN_CUDA(otn::launch_transpose(x, out, C), "otn_transpose");
  return OTN_OK;
}

int otn_pixel_cost(otn_ctx* x, const double* X, const double* Y, int64_t d, double* C,
                   double* host_max) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && X && Y && C && host_max, "otn_pixel_cost: NULL argument");
  OTN_REQUIRE(d >= 1 && d <= (int64_t(1) << 15), "otn_pixel_cost: d must be in [1, 32768]");
  // scratch words: the maximum's bits in scal[40], the range flag in flags[12]
  unsigned long long* cmax_bits = reinterpret_cast<unsigned long long*>(x->scal + 40);
  int* err = x->flags + 12;
  OTN_CUDA(otn::launch_pixel_cost(x, X, Y, d, C, cmax_bits, err), "otn_pixel_cost");
  int rc = sync_copy(x, x->h_scal + 40, x->scal + 40, sizeof(double), "otn_pixel_cost: max");
  if (rc) return rc;
  rc = sync_copy(x, x->h_flags + 12, x->flags + 12, sizeof(int), "otn_pixel_cost: flags");
  if (rc) return rc;
  OTN_REQUIRE(x->h_flags[12] == 0, "otn_pixel_cost: an entry is not an integer in [0, 255]");
  *host_max = x->h_scal[40];
  return OTN_OK;
}

int otn_coop_layout(otn_ctx* x, int* host) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && host, "otn_coop_layout: NULL argument");
  return sync_copy(x, host, x->part, size_t(x->coop_blocks + 2) * sizeof(int), "otn_coop_layout");
}

int otn_set_timing(otn_ctx* x, int on) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x, "otn_set_timing: NULL context");
  x->time_coop = on != 0;
  return OTN_OK;
}

int otn_coop_ms(otn_ctx* x, float* ms) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && ms, "otn_coop_ms: NULL argument");
  OTN_REQUIRE(x->time_coop, "otn_coop_ms: timing is off (otn_set_timing)");
  OTN_CUDA(cudaEventSynchronize(x->ev_coop[1]), "otn_coop_ms: sync");
  OTN_CUDA(cudaEventElapsedTime(ms, x->ev_coop[0], x->ev_coop[1]), "otn_coop_ms");
  return OTN_OK;
}

int otn_read_flags(otn_ctx* x, int* host4) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && host4, "otn_read_flags: NULL argument");
  int rc = sync_copy(x, x->h_flags, x->flags, 4 * sizeof(int), "otn_read_flags");
  if (rc) return rc;
  std::memcpy(host4, x->h_flags, 4 * sizeof(int));
  return OTN_OK;
}

// ---- log-domain reductions -----------------------------------------------
int otn_lse_rows(otn_ctx* x, const double* C, double ng, const double* outer, const double* inner,
                 double* out) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && C && inner && out, "otn_lse_rows: NULL argument");
  OTN_CUDA(otn::launch_lse_rows(x, C, ng, outer, nullptr, inner, nullptr, 0.0, 0, out),
           "otn_lse_rows");
  return OTN_OK;
}

static int lse_cols_any(otn_ctx* x, const double* C, int sym, double ng, const double* outer,
                        const double* outer_d, const double* inner, const double* inner_d,
                        double alpha, int mode, double* out, const char* what) {
  DeviceGuard dg_(x);
  cudaError_t e = sym ? otn::launch_lse_rows(x, C, ng, outer, outer_d, inner, inner_d, alpha, mode, out)
                      : otn::launch_lse_cols(x, C, ng, outer, outer_d, inner, inner_d, alpha, mode, out);
  OTN_CUDA(e, what);
  return OTN_OK;
}

int otn_lse_cols(otn_ctx* x, const double* C, int sym, double ng, const double* outer,
                 const double* inner, double* out) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && C && inner && out, "otn_lse_cols: NULL argument");
  return lse_cols_any(x, C, sym, ng, outer, nullptr, inner, nullptr, 0.0, 0, out, "otn_lse_cols");
}

int otn_rebalance_cols(otn_ctx* x, const double* C, int sym, double ng, const double* log_c,
                       const double* u, double* v_out) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && C && log_c && u && v_out, "otn_rebalance_cols: NULL argument");
  return lse_cols_any(x, C, sym, ng, log_c, nullptr, u, nullptr, 0.0, 1, v_out,
                      "otn_rebalance_cols");
}

int otn_trial_cols(otn_ctx* x, const double* C, int sym, double ng, const double* u,
                   const double* du, const double* v, const double* dv, double alpha, double* out,
                   double* host_mass) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && C && u && du && v && dv && out, "otn_trial_cols: NULL argument");
  int rc = lse_cols_any(x, C, sym, ng, v, dv, u, du, alpha, 0, out, "otn_trial_cols");
  if (rc) return rc;
  if (host_mass) {
    OTN_CUDA(otn::launch_reduce(x, OTN_RED_SUM_EXP, x->n, out, nullptr, nullptr, nullptr, x->scal,
                                x->flags + 4),
             "otn_trial_cols: mass");
    rc = sync_copy(x, x->h_scal, x->scal, sizeof(double), "otn_trial_cols: mass copy");
    if (rc) return rc;
    *host_mass = x->h_scal[0];
  }
  return OTN_OK;
}

// ---- plan ----------------------------------------------------------------
int otn_materialize(otn_ctx* x, const double* C, double ng, const double* u, const double* v,
                    double* P, const double* icP, const double* rP, double* mu, int* host_overflow,
                    uint64_t* seg_mask) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && C && u && v && P, "otn_materialize: NULL argument");
  OTN_REQUIRE(!icP || (rP && mu), "otn_materialize: icP needs rP and mu");
  OTN_CUDA(cudaMemsetAsync(x->flags + 0, 0, sizeof(int), x->stream), "otn_materialize: flag");
  OTN_CUDA(otn::launch_materialize(x, C, ng, u, v, P, icP, rP, mu, x->flags + 0, seg_mask),
           "otn_materialize");
  if (host_overflow) {
    int rc = sync_copy(x, x->h_flags, x->flags, sizeof(int), "otn_materialize: flag copy");
    if (rc) return rc;
    *host_overflow = x->h_flags[0];
    if (x->h_flags[0]) return OTN_ST_PLAN_OVERFLOW;
  }
  return OTN_OK;
}

int otn_plan_mask(otn_ctx* x, const double* P, uint64_t* seg_mask) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && P && seg_mask, "otn_plan_mask: NULL argument");
  // a system built from caller arrays (not from a materialized state) must not
  // inherit the overflow / nonpositive-sum flags of an earlier solve on this
  // context: the persistent solver checks flags[0..1] first
  OTN_CUDA(cudaMemsetAsync(x->flags, 0, 2 * sizeof(int), x->stream), "otn_plan_mask: flags");
  OTN_CUDA(otn::launch_plan_mask(x, P, seg_mask), "otn_plan_mask");
  return OTN_OK;
}

int otn_system_prep(otn_ctx* x, const double* lr, const double* lc, double* rP, double* cP,
                    double* icP, int* host_bad) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && lr && lc && rP && cP && icP, "otn_system_prep: NULL argument");
  OTN_CUDA(cudaMemsetAsync(x->flags + 1, 0, sizeof(int), x->stream), "otn_system_prep: flag");
  OTN_CUDA(otn::launch_sys_prep(x, lr, lc, rP, cP, icP, x->flags + 1), "otn_system_prep");
  if (host_bad) {
    int rc = sync_copy(x, x->h_flags, x->flags + 1, sizeof(int), "otn_system_prep: flag copy");
    if (rc) return rc;
    *host_bad = x->h_flags[0];
    if (x->h_flags[0]) return OTN_ST_NONPOSITIVE_SUMS;
  }
  return OTN_OK;
}

int otn_square_matvec(otn_ctx* x, const double* P, const double* w, double* out) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && P && w && out, "otn_square_matvec: NULL argument");
  OTN_CUDA(otn::launch_square_matvec(x, P, w, out), "otn_square_matvec");
  return OTN_OK;
}

// ---- HVP seam operators (single cooperative launch each) -------------------
static otn::CoopArgs plan_args(otn_ctx* x, const double* P, const uint64_t* seg_mask) {
  otn::CoopArgs a = base_args(x, P);
  a.mask = seg_mask;
  a.mw = OTN_MASK_WORDS(x->ld);
  return a;
}

static int coop_op(otn_ctx* x, int mode, const double* P, const uint64_t* seg_mask,
                   const double* rP, const double* cP, double rho, const double* xin, double* out,
                   const char* what) {
  DeviceGuard dg_(x);
  otn::CoopArgs a = plan_args(x, P, seg_mask);
  a.mode = mode;
  a.rP = rP;
  a.cP = cP;
  a.rho = rho;
  a.xin = xin;
  a.d = out;
  OTN_CUDA(otn::launch_coop(x, a), what);
  return OTN_OK;
}

int otn_matvec(otn_ctx* x, const double* P, const uint64_t* m, const double* v, double* out) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && P && v && out, "otn_matvec: NULL argument");
  return coop_op(x, otn::kModeMatvec, P, m, nullptr, nullptr, 0.0, v, out, "otn_matvec");
}

int otn_rmatvec(otn_ctx* x, const double* P, const uint64_t* m, const double* v, double* out) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && P && v && out, "otn_rmatvec: NULL argument");
  return coop_op(x, otn::kModeRmatvec, P, m, nullptr, nullptr, 0.0, v, out, "otn_rmatvec");
}

int otn_apply_F(otn_ctx* x, const double* P, const uint64_t* m, const double* rP,
                const double* cP, double rho, const double* d, double* out) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && P && rP && cP && d && out, "otn_apply_F: NULL argument");
  return coop_op(x, otn::kModeHvp, P, m, rP, cP, rho, d, out, "otn_apply_F");
}

int otn_apply_pc(otn_ctx* x, const double* P, const uint64_t* m, const double* cP,
                 const double* d, double* out) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && P && cP && d && out, "otn_apply_pc: NULL argument");
  return coop_op(x, otn::kModePc, P, m, nullptr, cP, 0.0, d, out, "otn_apply_pc");
}

// ---- solvers ---------------------------------------------------------------
int otn_pcg(otn_ctx* x, const double* P, const uint64_t* m, const double* rP, const double* cP,
            const double* mu, double rho, const double* b, double tol, double* xv, int has_x0,
            int64_t max_iters, otn_solve_result* host_res) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && P && rP && cP && mu && b && xv, "otn_pcg: NULL argument");
  OTN_REQUIRE(max_iters >= 0, "otn_pcg: max_iters < 0");
  otn::CoopArgs a = plan_args(x, P, m);
  a.mode = otn::kModePcg;
  a.rP = rP;
  a.cP = cP;
  a.mu = mu;
  a.rho = rho;
  a.b = b;
  a.tol = tol;
  a.d = xv;
  a.has_x0 = has_x0;
  a.max_iters = max_iters;
  OTN_CUDA(otn::launch_coop(x, a), "otn_pcg");
  return finish_solve(x, host_res, "otn_pcg: result");
}

int otn_newton(otn_ctx* x, const double* P, const uint64_t* m, const double* rP, const double* cP,
               const double* mu, const double* g, double eta, double rho0, int zero_init,
               int64_t max_iters, double* d_u, double* d_v, otn_solve_result* host_res) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && P && rP && cP && mu && g && d_u, "otn_newton: NULL argument");
  OTN_REQUIRE(max_iters >= 0, "otn_newton: max_iters < 0");
  otn::CoopArgs a = plan_args(x, P, m);
  a.mode = otn::kModeNewton;
  a.rP = rP;
  a.cP = cP;
  a.mu = mu;
  a.g = g;
  a.eta = eta;
  a.rho0 = rho0;
  a.zero_init = zero_init;
  a.max_iters = max_iters;
  a.d = d_u;
  a.dv = d_v;
  a.pre_flags = x->flags;
  OTN_CUDA(otn::launch_coop(x, a), "otn_newton");
  return finish_solve(x, host_res, "otn_newton: result");
}

int otn_newton_step(otn_ctx* x, const double* P, const uint64_t* m, const double* rP,
                    const double* cP, const double* mu, const double* g, double eta, double rho0,
                    int zero_init, int64_t max_iters, double* d_u, double* d_v, const double* C,
                    const double* Ccols, int sym, double ng, double* u, double* v, const double* r,
                    const double* log_c,
                    double* trial, double* lc, double* lr, double* grad, double armijo_c1,
                    double slope_floor, otn_solve_result* host_res, double* host_out,
                    int* host_flags) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && P && rP && cP && mu && g && d_u && d_v && C && Ccols && u && v && r && log_c &&
                  trial && lc && lr && grad,
              "otn_newton_step: NULL argument");
  OTN_REQUIRE(max_iters >= 0, "otn_newton_step: max_iters < 0");
  otn::CoopArgs a = plan_args(x, P, m);
  a.mode = otn::kModeNewton;
  a.rP = rP;
  a.cP = cP;
  a.mu = mu;
  a.g = g;
  a.eta = eta;
  a.rho0 = rho0;
  a.zero_init = zero_init;
  a.max_iters = max_iters;
  a.d = d_u;
  a.dv = d_v;
  a.pre_flags = x->flags;
  a.step_flags = x->flags + 6;                      // the first gate is set by k_coop itself
  OTN_CUDA(otn::launch_coop(x, a), "otn_newton_step");
  // scalars: scal[32] trial mass, scal[33..34] row statistics;
  // flags[6] trial gate, flags[7] accept gate, flags[8] row-statistics flags
  int* gates = x->flags + 6;
  const int n = int(x->n);
  cudaError_t e = sym ? otn::launch_lse_rows(x, Ccols, ng, v, d_v, u, d_u, 1.0, 0, trial, gates)
                      : otn::launch_lse_cols(x, Ccols, ng, v, d_v, u, d_u, 1.0, 0, trial, gates);
  OTN_CUDA(e, "otn_newton_step: trial");
  OTN_CUDA(otn::launch_reduce(x, OTN_RED_SUM_EXP, n, trial, nullptr, nullptr, nullptr,
                              x->scal + 32, x->flags + 4, gates),
           "otn_newton_step: mass");
  OTN_CUDA(otn::launch_step_gate(x, 1, x->dres, x->scal + 32, slope_floor, armijo_c1, gates),
           "otn_newton_step: armijo");
  const int* acc = gates + 1;
  OTN_CUDA(otn::launch_accept(x, 1.0, u, d_u, v, d_v, log_c, trial, lc, acc),
           "otn_newton_step: accept");
  OTN_CUDA(otn::launch_lse_rows(x, C, ng, u, nullptr, v, nullptr, 0.0, 0, lr, acc),
           "otn_newton_step: rows");
  OTN_CUDA(otn::launch_reduce(x, otn::kRedRowStatsGrad, n, lr, r, grad, nullptr, x->scal + 33,
                              x->flags + 8, acc),
           "otn_newton_step: row stats + gradient");
  OTN_CUDA(cudaMemcpyAsync(x->h_scal + 32, x->scal + 32, 3 * sizeof(double),
                           cudaMemcpyDeviceToHost, x->stream), "otn_newton_step: copy");
  OTN_CUDA(cudaMemcpyAsync(x->h_flags + 6, x->flags + 6, 3 * sizeof(int), cudaMemcpyDeviceToHost,
                           x->stream), "otn_newton_step: copy");
  if (!host_out) return OTN_OK;                     // collected by otn_newton_step_wait
  return otn_newton_step_wait(x, host_res, host_out, host_flags);
}

int otn_newton_step_wait(otn_ctx* x, otn_solve_result* host_res, double* host_out,
                         int* host_flags) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && host_out, "otn_newton_step_wait: NULL argument");
  int rc = finish_solve(x, host_res, "otn_newton_step: result");
  const bool ran = x->h_flags[6] != 0, ok = x->h_flags[7] != 0;
  host_out[0] = ran ? x->h_scal[32] : 0.0;
  host_out[1] = ok ? x->h_scal[33] : 0.0;
  host_out[2] = ok ? x->h_scal[34] : 0.0;
  host_out[3] = ran ? 1.0 : 0.0;
  host_out[4] = ok ? 1.0 : 0.0;
  if (host_flags) host_flags[0] = ok ? x->h_flags[8] : 0;
  return rc;
}

int otn_probe(otn_ctx* x, const double* P, const uint64_t* m, const double* cP, const double* rP,
              const double* xin, double* out, int what, int64_t reps) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && P && cP && rP && xin && out, "otn_probe: NULL argument");
  otn::CoopArgs a = plan_args(x, P, m);
  a.mode = otn::kModeProbe;
  a.cP = cP;
  a.rP = rP;
  a.xin = xin;
  a.d = out;
  a.has_x0 = what;
  a.max_iters = reps;
  OTN_CUDA(otn::launch_coop(x, a), "otn_probe");
  return OTN_OK;
}

// ---- point clouds ------------------------------------------------------------
int otn_pc_pass(otn_ctx* x, int op, const double* A, int64_t na, int64_t lda, const double* B,
                int64_t nb, int64_t ldb, int d, double cmax, double ng, int order,
                const double* colpot, const double* colpot_d, double alpha, const double* rowpot,
                const double* vec, const double* outer, const double* outer_d, int mode,
                double* out, double* out2) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && A && B && out, "otn_pc_pass: NULL argument");
  OTN_REQUIRE(d >= 1 && d <= 4, "otn_pc_pass: point dimension must be 1..4");
  OTN_REQUIRE(na >= 1 && nb >= 1 && lda >= na && ldb >= nb, "otn_pc_pass: bad sizes");
  OTN_REQUIRE(op >= OTN_PC_LSE && op <= OTN_PC_LSE_SHIFT, "otn_pc_pass: bad op");
  OTN_REQUIRE(op != OTN_PC_LSE_SHIFT || outer != nullptr, "otn_pc_pass: LSE_SHIFT needs outer");
  OTN_REQUIRE((op != OTN_PC_DOT && op != OTN_PC_DIAG && op != OTN_PC_DOTC && op != OTN_PC_CDOT) ||
                  vec != nullptr, "otn_pc_pass: DOT/DIAG/DOTC/CDOT need vec");
  OTN_REQUIRE(op != OTN_PC_LSE_PART || out2 != nullptr, "otn_pc_pass: LSE_PART needs out2");
  otn::PairArgs p{A, na, lda, B, nb, ldb, d, op, order, mode, cmax, ng, colpot, colpot_d, rowpot,
                  alpha, vec, outer, outer_d, out, out2};
  OTN_CUDA(otn::launch_pair(x, p), "otn_pc_pass");
  return OTN_OK;
}

int otn_vec_n(otn_ctx* x, int64_t n, int op, double s, const double* a, const double* b,
              const double* c, const double* d, double* out) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && a && out && n >= 0, "otn_vec_n: bad argument");
  OTN_REQUIRE(op >= OTN_VEC_ADD_SUB && op <= OTN_VEC_COPY, "otn_vec_n: bad op");
  if (n == 0) return OTN_OK;
  OTN_CUDA(otn::launch_vec(x, op, n, s, a, b, c, d, out), "otn_vec_n");
  return OTN_OK;
}

int otn_reduce_n(otn_ctx* x, int64_t n, int op, const double* a, const double* b, const double* c,
                 const double* d, double* host_out, int* host_flags) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && a && host_out && n >= 0, "otn_reduce_n: bad argument");
  OTN_REQUIRE(op >= OTN_RED_ROW_STATS && op <= OTN_RED_OUTSIDE, "otn_reduce_n: bad op");
  OTN_CUDA(cudaMemsetAsync(x->flags + 2, 0, sizeof(int), x->stream), "otn_reduce_n: flag");
  OTN_CUDA(otn::launch_reduce(x, op, n, a, b, c, d, x->scal + 8, x->flags + 2), "otn_reduce_n");
  OTN_CUDA(cudaMemcpyAsync(x->h_scal + 8, x->scal + 8, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                           x->stream), "otn_reduce_n: copy");
  OTN_CUDA(cudaMemcpyAsync(x->h_flags + 2, x->flags + 2, sizeof(int), cudaMemcpyDeviceToHost,
                           x->stream), "otn_reduce_n: copy");
  OTN_CUDA(stream_wait(x->stream), "otn_reduce_n: sync");
  host_out[0] = x->h_scal[8];
  host_out[1] = x->h_scal[9];
  if (host_flags) *host_flags = x->h_flags[2];
  return OTN_OK;
}

int otn_reduce_dev(otn_ctx* x, int64_t n, int op, const double* a, const double* b,
                   const double* c, const double* d, double* dev_out) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && a && dev_out && n >= 0, "otn_reduce_dev: bad argument");
  OTN_REQUIRE(op >= OTN_RED_GRAD_L1 && op <= OTN_RED_OUTSIDE && op != OTN_RED_MAX,
              "otn_reduce_dev: bad op (sums only)");
  OTN_CUDA(otn::launch_reduce(x, op, n, a, b, c, d, dev_out, x->flags + 2), "otn_reduce_dev");
  return OTN_OK;
}

// ---- vector work -----------------------------------------------------------
int otn_vec(otn_ctx* x, int op, double s, const double* a, const double* b, const double* c,
            const double* d, double* out) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && a && out, "otn_vec: NULL argument");
  OTN_REQUIRE(op >= OTN_VEC_ADD_SUB && op <= OTN_VEC_COPY, "otn_vec: bad op");
  OTN_CUDA(otn::launch_vec(x, op, x->n, s, a, b, c, d, out), "otn_vec");
  return OTN_OK;
}

int otn_reduce_async(otn_ctx* x, int op, const double* a, const double* b, const double* c,
                     const double* d, double* host_out) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && a && host_out, "otn_reduce_async: NULL argument");
  OTN_REQUIRE(op >= OTN_RED_ROW_STATS && op <= OTN_RED_L1_DOT, "otn_reduce_async: bad op");
  // own scalar slot (40..41) and flag word (9): later reductions cannot
  // overwrite the result before the copy runs (stream order), nor race it
  OTN_CUDA(otn::launch_reduce(x, op, x->n, a, b, c, d, x->scal + 40, x->flags + 9),
           "otn_reduce_async");
  OTN_CUDA(cudaMemcpyAsync(host_out, x->scal + 40, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                           x->stream), "otn_reduce_async: copy");
  return OTN_OK;
}

int otn_row_stats(otn_ctx* x, const double* lr, const double* r, double* g, double* host_out,
                  int* host_flags) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && lr && r && g && host_out, "otn_row_stats: NULL argument");
  OTN_CUDA(cudaMemsetAsync(x->flags + 2, 0, sizeof(int), x->stream), "otn_row_stats: flag");
  OTN_CUDA(otn::launch_reduce(x, otn::kRedRowStatsGrad, x->n, lr, r, g, nullptr, x->scal + 8,
                              x->flags + 2),
           "otn_row_stats");
  OTN_CUDA(cudaMemcpyAsync(x->h_scal + 8, x->scal + 8, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                           x->stream), "otn_row_stats: copy");
  OTN_CUDA(cudaMemcpyAsync(x->h_flags + 2, x->flags + 2, sizeof(int), cudaMemcpyDeviceToHost,
                           x->stream), "otn_row_stats: copy");
  OTN_CUDA(stream_wait(x->stream), "otn_row_stats: sync");
  host_out[0] = x->h_scal[8];
  host_out[1] = x->h_scal[9];
  if (host_flags) *host_flags = x->h_flags[2];
  return OTN_OK;
}

int otn_accept(otn_ctx* x, double alpha, double* u, const double* d_u, double* v,
               const double* d_v, const double* log_c, const double* trial, double* lc) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && u && d_u && v && d_v && log_c && trial && lc, "otn_accept: NULL argument");
  OTN_CUDA(otn::launch_accept(x, alpha, u, d_u, v, d_v, log_c, trial, lc, nullptr), "otn_accept");
  return OTN_OK;
}

int otn_reduce(otn_ctx* x, int op, const double* a, const double* b, const double* c,
               const double* d, double* host_out, int* host_flags) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && a && host_out, "otn_reduce: NULL argument");
  OTN_REQUIRE(op >= OTN_RED_ROW_STATS && op <= OTN_RED_L1_DOT, "otn_reduce: bad op");
  OTN_CUDA(cudaMemsetAsync(x->flags + 2, 0, sizeof(int), x->stream), "otn_reduce: flag");
  OTN_CUDA(otn::launch_reduce(x, op, x->n, a, b, c, d, x->scal + 8, x->flags + 2), "otn_reduce");
  OTN_CUDA(cudaMemcpyAsync(x->h_scal + 8, x->scal + 8, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                           x->stream), "otn_reduce: copy");
  OTN_CUDA(cudaMemcpyAsync(x->h_flags + 2, x->flags + 2, sizeof(int), cudaMemcpyDeviceToHost,
                           x->stream), "otn_reduce: copy");
  OTN_CUDA(stream_wait(x->stream), "otn_reduce: sync");
  host_out[0] = x->h_scal[8];
  host_out[1] = x->h_scal[9];
  if (host_flags) *host_flags = x->h_flags[2];
  return OTN_OK;
}

int otn_round_plan(otn_ctx* x, double* P, const double* C, const double* r, const double* c,
                   double* host_out, int* host_flags) {
  DeviceGuard dg_(x);
  OTN_REQUIRE(x && P && r && c && host_out, "otn_round_plan: NULL argument");
  OTN_CUDA(cudaMemsetAsync(x->flags + 3, 0, sizeof(int), x->stream), "otn_round_plan: flag");
  OTN_CUDA(otn::launch_round(x, P, C, r, c, x->scal + 16, x->flags + 3), "otn_round_plan");
  OTN_CUDA(cudaMemcpyAsync(x->h_scal + 16, x->scal + 16, 4 * sizeof(double),
                           cudaMemcpyDeviceToHost, x->stream), "otn_round_plan: copy");
  OTN_CUDA(cudaMemcpyAsync(x->h_flags + 3, x->flags + 3, sizeof(int), cudaMemcpyDeviceToHost,
                           x->stream), "otn_round_plan: copy");
  OTN_CUDA(stream_wait(x->stream), "otn_round_plan: sync");
  host_out[0] = x->h_scal[16 + 3];   // primal <P, C>
  host_out[1] = x->h_scal[16 + 2];   // deficit
  if (host_flags) *host_flags = x->h_flags[3];
  return OTN_OK;
}

}  // extern "C"
