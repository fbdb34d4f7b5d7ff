// O(n) projector / driver vector work, single-CTA deterministic reductions,
// and the final rounding of the plan onto U(r, c) with the primal cost.
#include "otn_common.cuh"
#include "otn_internal.h"

namespace otn {

// ---------------------------------------------------------------------------
// element-wise ops (operand order of the reference's numpy expressions)
// ---------------------------------------------------------------------------
__global__ void k_vec(int op, int64_t n, double s, const double* a, const double* b,
                      const double* c, const double* d, double* out, const int* gate) {
  __shared__ double2 s_exp[64];
  if (gate && *gate == 0) return;                   // uniform over the grid
  if (op == OTN_VEC_EXP) {                          // uniform: the table only where it is used
    exp_tab_load(s_exp);
    __syncthreads();
  }
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    double o;
    switch (op) {
      case OTN_VEC_ADD_SUB: o = __dsub_rn(__dadd_rn(a[i], b[i]), c[i]); break;
      case OTN_VEC_AXPY: o = __dadd_rn(a[i], __dmul_rn(s, b[i])); break;
      case OTN_VEC_STEP_V:
        o = __dadd_rn(__dadd_rn(a[i], __dmul_rn(s, b[i])), __dsub_rn(c[i], d[i]));
        break;
      case OTN_VEC_EXTRAP: o = __dadd_rn(a[i], __dmul_rn(s, __dsub_rn(a[i], b[i]))); break;
      case OTN_VEC_EXP: o = exp_tab(a[i], s_exp); break;
      case OTN_VEC_GRAD: o = __dsub_rn(exp_fast(a[i]), b[i]); break;
      case OTN_VEC_MUL_SUB: o = __dsub_rn(__dmul_rn(a[i], b[i]), __dmul_rn(s, c[i])); break;
      case OTN_VEC_DIV: o = __ddiv_rn(a[i], b[i]); break;
      case OTN_VEC_SUB: o = __dsub_rn(a[i], b[i]); break;
      case OTN_VEC_ADD: o = __dadd_rn(a[i], b[i]); break;
      case OTN_VEC_PRECOND: o = __dmul_rn(a[i], __dsub_rn(1.0, __dmul_rn(s, b[i]))); break;
      case OTN_VEC_NEG_DIV: o = __ddiv_rn(-a[i], b[i]); break;
      case OTN_VEC_RESCALE: o = __dmul_rn(a[i], exp_fast(__dsub_rn(b[i], c[i]))); break;
      case OTN_VEC_LSE_FIN: o = __dadd_rn(a[i], lse_value(b[i], c[i])); break;
      case OTN_VEC_LSE_FIN_SUB: o = __dsub_rn(a[i], lse_value(b[i], c[i])); break;
      case OTN_VEC_ROUND_SCALE: o = b[i] > 0.0 ? fmin(1.0, __ddiv_rn(a[i], b[i])) : 1.0; break;
      case OTN_VEC_SUB_MUL: o = __dsub_rn(a[i], __dmul_rn(b[i], c[i])); break;
      case OTN_VEC_MUL: o = __dmul_rn(a[i], b[i]); break;
      case OTN_VEC_COPY: o = a[i]; break;
      default: o = 0.0;
    }
    out[i] = o;
  }
}

// ---------------------------------------------------------------------------
// single-CTA reductions: thread t sums i = t, t+1024, ... then a fixed tree
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_reduce(int op, int64_t n, const double* a,
                                                 const double* b, const double* c,
                                                 const double* d, double* dst, int* flag,
                                                 const int* gate) {
  __shared__ double sh[33];
  if (gate && *gate == 0) return;
  double s0 = 0.0, s1 = 0.0;
  int f = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    switch (op) {
      case kRedRowStatsGrad:
      case OTN_RED_ROW_STATS: {
        const double x = exp_fast(a[i]), y = b[i];
        if (op == kRedRowStatsGrad) const_cast<double*>(c)[i] = __dsub_rn(x, y);   // VEC_GRAD
        s0 += fabs(__dsub_rn(x, y));
        s1 += __ddiv_rn(__dmul_rn(y, y), x);
        if (x <= 0.0) f |= 1;
        if (y < 0.0) f |= 2;
        break;
      }
      case OTN_RED_GRAD_L1:
        s0 += fabs(__dsub_rn(exp_fast(a[i]), b[i]));
        s1 += fabs(__dsub_rn(exp_fast(c[i]), d[i]));
        break;
      case OTN_RED_SUM_EXP: s0 += exp_fast(a[i]); break;
      case OTN_RED_DOT: s0 = fma(a[i], b[i], s0); break;
      case OTN_RED_L1: s0 += fabs(a[i]); break;
      case OTN_RED_L1_ADD: s0 += fabs(__dadd_rn(a[i], b[i])); break;
      case OTN_RED_NONPOS: if (a[i] <= 0.0) s0 += 1.0; break;
      case OTN_RED_L1_DOT: s0 += fabs(a[i]); s1 = fma(a[i], b[i], s1); break;
      case OTN_RED_OUTSIDE: if (!(a[i] >= 0x1p-700 && a[i] <= 0x1p+700)) s0 += 1.0; break;
      case OTN_RED_MAX: s1 = (i == threadIdx.x) ? a[i] : fmax(s1, a[i]); break;
      default: break;
    }
  }
  if (op == OTN_RED_MAX) {
    const double mx = block_max(n > threadIdx.x ? s1 : OTN_NINF, sh);
    if (threadIdx.x == 0) { dst[0] = mx; dst[1] = 0.0; }
    return;
  }
  s0 = block_sum(s0, sh);
  s1 = block_sum(s1, sh);
  if (f) atomicOr(flag, f);
  if (threadIdx.x == 0) {
    dst[0] = s0;
    dst[1] = s1;
  }
}

// ---------------------------------------------------------------------------
// rounding (driver.py:178-208) + primal cost (driver.py:306-310)
// ---------------------------------------------------------------------------
// Row pass: optionally scale columns in place (P_ij *= cs_j), then row sum and
// row minimum.  One warp per row.
__global__ void __launch_bounds__(256) k_round_rows(double* P, int64_t n, int64_t ld,
                                                   const double* cs, double* rsum,
                                                   double* rmin) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double* prow = P + row * ld;
  double s = 0.0, mn = OTN_INF;
  for (int64_t j = 2 * lane; j < n; j += 64) {
    double2 p = *reinterpret_cast<double2*>(prow + j);
    const bool two = j + 1 < n;
    if (cs) {
      p.x = __dmul_rn(p.x, cs[j]);
      if (two) p.y = __dmul_rn(p.y, cs[j + 1]);
      *reinterpret_cast<double2*>(prow + j) = p;
    }
    s += p.x;
    mn = fmin(mn, p.x);
    if (two) {
      s += p.y;
      mn = fmin(mn, p.y);
    }
  }
  s = warp_sum(s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if (lane == 0) {
    rsum[row] = s;
    if (rmin) rmin[row] = mn;
  }
}

// Column pass: optionally scale rows in place (P_ij *= rs_i), per-slab column
// partial sums.  CTA = 64 columns x one row slab.
__global__ void __launch_bounds__(256) k_round_cols(double* P, int64_t n, int64_t ld,
                                                   int64_t slab_rows, const double* rs,
                                                   double* part) {
  __shared__ double sm[8][kColTile];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = int64_t(blockIdx.x) * kColTile + 2 * lane;
  const int64_t i0 = int64_t(blockIdx.y) * slab_rows;
  const int64_t i1 = min(n, i0 + slab_rows);
  double a0 = 0.0, a1 = 0.0;
  if (j < n) {
    for (int64_t i = i0 + warp; i < i1; i += 8) {
      double2 p = *reinterpret_cast<double2*>(P + i * ld + j);
      if (rs) {
        const double sc = rs[i];
        p.x = __dmul_rn(p.x, sc);
        if (j + 1 < n) p.y = __dmul_rn(p.y, sc);
        *reinterpret_cast<double2*>(P + i * ld + j) = p;
      }
      a0 += p.x;
      if (j + 1 < n) a1 += p.y;
    }
  }
  sm[warp][2 * lane] = a0;
  sm[warp][2 * lane + 1] = a1;
  __syncthreads();
  if (threadIdx.x < kColTile) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += sm[w][threadIdx.x];
    const int64_t jj = int64_t(blockIdx.x) * kColTile + threadIdx.x;
    if (jj < ld) part[int64_t(blockIdx.y) * ld + jj] = t;
  }
}

// Single-CTA glue steps of the rounding.
//   stage 0: rs = where(rP > 0, min(1, r / rP), 1); flags (min < 0, total <= 0)
//   stage 1: cs = where(cP > 0, min(1, c / cP), 1) from slab partials
//   stage 2: er = r - rowsum, ec = c - colsum, deficit = sum(er)
//   stage 3: primal = sum_i rowdot_i
__global__ void __launch_bounds__(1024) k_round_glue(int stage, int64_t n, int64_t ld, int slabs,
                                                     const double* r, const double* c,
                                                     const double* rsum, const double* rmin,
                                                     const double* part, double* outv,
                                                     double* outv2, double* scal, int* flag) {
  __shared__ double sh[33];
  double acc = 0.0, mn = OTN_INF;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    if (stage == 0) {
      const double rp = rsum[i];
      acc += rp;
      mn = fmin(mn, rmin[i]);
      outv[i] = rp > 0.0 ? fmin(1.0, __ddiv_rn(r[i], rp)) : 1.0;
    } else if (stage == 1) {
      double t = 0.0;
      for (int k = 0; k < slabs; ++k) t += part[int64_t(k) * ld + i];
      outv[i] = t > 0.0 ? fmin(1.0, __ddiv_rn(c[i], t)) : 1.0;
    } else if (stage == 2) {
      const double er = __dsub_rn(r[i], rsum[i]);
      double t = 0.0;
      for (int k = 0; k < slabs; ++k) t += part[int64_t(k) * ld + i];
      outv[i] = er;
      outv2[i] = __dsub_rn(c[i], t);
      acc += er;
    } else {
      acc += rsum[i];
    }
  }
  acc = block_sum(acc, sh);
  if (stage == 0) {
    mn = -block_max(-mn, sh);
    if (threadIdx.x == 0) {
      int f = 0;
      if (mn < 0.0) f |= 1;
      if (!(acc > 0.0)) f |= 2;
      if (f) atomicOr(flag, f);
    }
  }
  if (threadIdx.x == 0) scal[stage] = acc;
}

// P_ij += (er_i * ec_j) / deficit (when deficit > 0), and rowdot_i = sum_j P_ij C_ij.
__global__ void __launch_bounds__(256) k_round_rank1(double* P, const double* C, int64_t n,
                                                    int64_t ld, const double* er,
                                                    const double* ec, const double* scal,
                                                    double* rowdot) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const double deficit = scal[2];
  const bool fix = deficit > 0.0;
  const double eri = er[row];
  double* prow = P + row * ld;
  double acc = 0.0;
  for (int64_t j = lane; j < n; j += 32) {
    double p = prow[j];
    if (fix) {
      p = __dadd_rn(p, __ddiv_rn(__dmul_rn(eri, ec[j]), deficit));
      prow[j] = p;
    }
    if (C) acc = fma(p, C[row * ld + j], acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) rowdot[row] = acc;
}

cudaError_t launch_vec(otn_ctx* x, int op, int64_t n, double s, const double* a, const double* b,
                       const double* c, const double* d, double* out, const int* gate) {
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 4 * x->num_sms);
  k_vec<<<unsigned(std::max<int64_t>(blocks, 1)), 256, 0, x->stream>>>(op, n, s, a, b, c, d, out,
                                                                       gate);
  return cudaGetLastError();
}

cudaError_t launch_reduce(otn_ctx* x, int op, int64_t n, const double* a, const double* b,
                          const double* c, const double* d, double* dst, int* flag,
                          const int* gate) {
  k_reduce<<<1, 1024, 0, x->stream>>>(op, n, a, b, c, d, dst, flag, gate);
  return cudaGetLastError();
}

__global__ void k_accept(int64_t n, int64_t ld, double s, double* u, const double* du, double* v,
                         const double* dv, const double* logc, const double* trial, double* lc,
                         const int* gate) {
  if (gate && *gate == 0) return;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < ld;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (i < n) {
      u[i] = __dadd_rn(u[i], __dmul_rn(s, du[i]));                                   // VEC_AXPY
      v[i] = __dadd_rn(__dadd_rn(v[i], __dmul_rn(s, dv[i])), __dsub_rn(logc[i], trial[i]));
    }
    lc[i] = logc[i];                                                                 // VEC_COPY
  }
}

cudaError_t launch_accept(otn_ctx* x, double s, double* u, const double* du, double* v,
                          const double* dv, const double* logc, const double* trial, double* lc,
                          const int* gate) {
  const int64_t blocks = std::min<int64_t>((x->ld + 255) / 256, 4 * x->num_sms);
  k_accept<<<unsigned(std::max<int64_t>(blocks, 1)), 256, 0, x->stream>>>(x->n, x->ld, s, u, du, v,
                                                                         dv, logc, trial, lc, gate);
  return cudaGetLastError();
}

// The projector's decisions after a Newton launch (projector.py:203-231),
// evaluated on the device so the accept path can be enqueued behind it:
// stage 0: the direction is usable (status OK, slope > 0: otherwise the host
// takes the Sinkhorn fallback or raises); stage 1: the full step passes the
// mass-form Armijo test, i.e. the backtracking loop would not run:
//   not (slope > floor and mass - 1 > ((1 - c1) * 1) * slope)
// with the host expression's operand order.
__global__ void k_step_gate(int stage, const DevResult* res, const double* mass,
                            double slope_floor, double c1, int* flags) {
  if (threadIdx.x != 0) return;
  if (stage == 0) {
    flags[0] = res->status == OTN_OK && res->slope > 0.0;
    flags[2] = 0;
  } else {
    const double slope = res->slope;
    const bool backtrack =
        slope > slope_floor && __dsub_rn(*mass, 1.0) > __dmul_rn(__dmul_rn(__dsub_rn(1.0, c1), 1.0), slope);
    flags[1] = flags[0] && !backtrack;
  }
}

cudaError_t launch_step_gate(otn_ctx* x, int stage, const DevResult* res, const double* mass,
                             double slope_floor, double armijo_c1, int* flags) {
  k_step_gate<<<1, 32, 0, x->stream>>>(stage, res, mass, slope_floor, armijo_c1, flags);
  return cudaGetLastError();
}

// scratch_scalars: >= 4 device doubles; uses ctx vectors vtmp0/vtmp1/r/z/q/sv as scratch.
cudaError_t launch_round(otn_ctx* x, double* P, const double* C, const double* r, const double* c,
                         double* scal, int* flag) {
  const int64_t n = x->n, ld = x->ld;
  const int slabs = x->lse_slabs;
  const int64_t slab_rows = (n + slabs - 1) / slabs;
  double* part = x->lse_part;            // slabs x ld (reuses the LSE partial area)
  double* rsum = x->vtmp0;
  double* rmin = x->vtmp1;
  double* rs = x->r;
  double* cs = x->z;
  double* er = x->q;
  double* ec = x->sv;
  const unsigned rgrid = unsigned((n + 7) / 8);
  dim3 cgrid(unsigned((ld + kColTile - 1) / kColTile), unsigned(slabs));
  // rP = P.sum(axis=1), min, total  -> row scale
  k_round_rows<<<rgrid, 256, 0, x->stream>>>(P, n, ld, nullptr, rsum, rmin);
  k_round_glue<<<1, 1024, 0, x->stream>>>(0, n, ld, slabs, r, c, rsum, rmin, part, rs, nullptr,
                                          scal, flag);
  // P *= rs[:, None]; cP = P.sum(axis=0) -> column scale
  k_round_cols<<<cgrid, 256, 0, x->stream>>>(P, n, ld, slab_rows, rs, part);
  k_round_glue<<<1, 1024, 0, x->stream>>>(1, n, ld, slabs, r, c, rsum, rmin, part, cs, nullptr,
                                          scal, flag);
  // P *= cs[None, :]; row sums; column sums; err_r, err_c, deficit
  k_round_rows<<<rgrid, 256, 0, x->stream>>>(P, n, ld, cs, rsum, nullptr);
  k_round_cols<<<cgrid, 256, 0, x->stream>>>(P, n, ld, slab_rows, nullptr, part);
  k_round_glue<<<1, 1024, 0, x->stream>>>(2, n, ld, slabs, r, c, rsum, rmin, part, er, ec, scal,
                                          flag);
  // rank-one repair + <P, C>
  k_round_rank1<<<rgrid, 256, 0, x->stream>>>(P, C, n, ld, er, ec, scal, rsum);
  k_round_glue<<<1, 1024, 0, x->stream>>>(3, n, ld, slabs, r, c, rsum, rmin, part, nullptr,
                                          nullptr, scal, flag);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// cost-matrix preparation (once per problem): (C == C^T).all() and C^T,
// 32 x 32 tiles through shared memory so both sides are read coalesced
// (dual.py:80-88 forms K^T as a contiguous copy unless C is symmetric)
// ---------------------------------------------------------------------------
constexpr int kTp = 32;

__global__ void __launch_bounds__(kTp * 8) k_symmetric(const double* C, int64_t n, int64_t ld,
                                                       int* flag) {
  __shared__ double tile[kTp][kTp + 1];
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (bj < bi) return;                               // upper-triangle tile pairs only
  const int tx = threadIdx.x & (kTp - 1), ty = threadIdx.x / kTp;
  // stage tile (bj, bi) transposed, compare with tile (bi, bj)
  for (int y = ty; y < kTp; y += 8) {
    const int64_t i = int64_t(bj) * kTp + y, j = int64_t(bi) * kTp + tx;
    tile[tx][y] = (i < n && j < n) ? C[i * ld + j] : 0.0;
  }
  __syncthreads();
  int bad = 0;
  for (int y = ty; y < kTp; y += 8) {
    const int64_t i = int64_t(bi) * kTp + y, j = int64_t(bj) * kTp + tx;
    if (i < n && j < n && !(C[i * ld + j] == tile[y][tx])) bad = 1;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

__global__ void __launch_bounds__(kTp * 8) k_transpose(double* out, const double* C, int64_t n,
                                                       int64_t ld) {
  __shared__ double tile[kTp][kTp + 1];
  const int tx = threadIdx.x & (kTp - 1), ty = threadIdx.x / kTp;
  for (int y = ty; y < kTp; y += 8) {
    const int64_t i = int64_t(blockIdx.y) * kTp + y, j = int64_t(blockIdx.x) * kTp + tx;
    tile[y][tx] = (i < n && j < n) ? C[i * ld + j] : 0.0;
  }
  __syncthreads();
  for (int y = ty; y < kTp; y += 8) {
    const int64_t i = int64_t(blockIdx.x) * kTp + y, j = int64_t(blockIdx.y) * kTp + tx;
    if (i < n && j < ld) out[i * ld + j] = tile[tx][y];   // padding columns get 0
  }
}

cudaError_t launch_symmetric(otn_ctx* x, const double* C, int* flag) {
  const unsigned t = unsigned((x->n + kTp - 1) / kTp);
  k_symmetric<<<dim3(t, t), kTp * 8, 0, x->stream>>>(C, x->n, x->ld, flag);
  return cudaGetLastError();
}

cudaError_t launch_transpose(otn_ctx* x, double* out, const double* C) {
  const unsigned tc = unsigned((x->ld + kTp - 1) / kTp);
  k_transpose<<<dim3(tc, tc), kTp * 8, 0, x->stream>>>(out, C, x->n, x->ld);
  return cudaGetLastError();
}

}  // namespace otn
