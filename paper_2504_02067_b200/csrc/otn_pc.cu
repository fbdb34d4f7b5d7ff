// On-the-fly point-cloud cost (D4/D5): every O(n^2) pass
// recomputes C_ij = (sum_k (x_ik - y_jk)^2) / C_max and the plan entry from the
// point coordinates instead of streaming a stored matrix.  The coordinate sum
// runs left to right with explicit roundings and the division is correctly
// rounded (reciprocal multiply + one FMA correction, Markstein), so C_ij
// is bit-identical to the host-materialized cost (PointCloudProblem.
// materialize_cost) and every exponent is formed with the stored path's
// operand order: results match the stored-C kernels up to summation order.
//
// One register-blocked "pair" kernel serves every pass.  A CTA owns RW*8 row
// points (RW per warp, in registers) and streams the column points in
// shared-memory tiles of 256; lane l takes columns l, l+32, ... of a tile, so
// each staged column is reused by all the CTA's rows.  Column passes (P^T x,
// column LSE) are the same kernel with the two point sets swapped
// (dist(x, y) == dist(y, x) exactly) and a flag that keeps the exponent's
// operand order ((ng*C + v_j) + u_i).  The point dimension D (1..4) is a
// template parameter so coordinates take exactly D registers per row.  FP64
// issue bounds it: ~30 FP64 instructions per entry (distance, division, exp).
#include "otn_common.cuh"
#include "otn_internal.h"

namespace otn {

constexpr int kPcThreads = 256;     // 8 warps
constexpr int kPcTile = 256;        // column points per shared-memory tile



// s / cmax, correctly rounded, as one multiply and two FMAs: with
// rc = RN(1/cmax), q0 = RN(s * rc) is within one ulp of s / cmax, the
// remainder e = s - q0 * cmax is exact in one FMA, and RN(q0 + e * rc) is the
// correctly rounded quotient (Markstein's theorem; it needs no underflow, so
// quotients near the subnormal range take __ddiv_rn).  Bit-identical to the
// host's IEEE division C /= C.max() (tests/test_gpu_pointcloud.py).
__device__ __forceinline__ double div_cmax(double s, double cmax, double rc) {
  const double q0 = __dmul_rn(s, rc);
  if (q0 < 0x1p-960) return __ddiv_rn(s, cmax);
  const double e = fma(-q0, cmax, s);
  return fma(e, rc, q0);
}

template <int D>
__device__ __forceinline__ double pc_cost(const double* a, const double* b, double cmax, double rc) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const double dk = __dsub_rn(a[k], b[k]);
    s = k == 0 ? __dmul_rn(dk, dk) : __dadd_rn(s, __dmul_rn(dk, dk));
  }
  return cmax > 0.0 ? div_cmax(s, cmax, rc) : s;
}

template <int D>
__device__ __forceinline__ double sep_exponent(const double* x, const double* y, double Ai,
                                               double Bj, double G) {
  double d = x[0] * y[0];
#pragma unroll
  for (int k = 1; k < D; ++k) d = fma(x[k], y[k], d);
  return fma(G, d, Ai + Bj);
}

// Plan exponent in separable form (SEP, the exp passes only): with
//   C_ij = (|x_i|^2 + |y_j|^2 - 2 x_i.y_j) / C_max,
//   e_ij = ng C_ij + v_j + u_i = (A_i + B_j) + G (x_i . y_j),
// A_i = (ng/C_max)|x_i|^2 + u_i per row (registers), B_j = (ng/C_max)|y_j|^2
// + v_j per column (staged with the tile), G = -2 ng/C_max: D FMAs, one add
// and one FMA per entry instead of the exact-cost path's ~14 FP64 operations
// (the exact path rounds C_ij itself to match a host-materialized cost
// bit for bit; the separable one differs from it by a few units in the last
// place of the exponent, ~1e-13 relative in a plan entry: inside every
// parity gate, tests/test_gpu_pointcloud.py).  OTN_PC_EXACT=1 selects the
// exact path for every pass.
template <int RW, int D, int OP, int MB = 2, bool SEP = false>
__global__ void __launch_bounds__(kPcThreads, MB) k_pair(PairArgs p) {
  __shared__ double sb[D][kPcTile];
  __shared__ double scp[kPcTile];
  __shared__ double svec[kPcTile];
  __shared__ double2 s_exp[64];
  exp_tab_load(s_exp);                               // made visible by the tile loop's barrier
  const double rc = p.cmax > 0.0 ? __drcp_rn(p.cmax) : 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i0 = (int64_t(blockIdx.x) * 8 + warp) * RW;
  const double ngc = __dmul_rn(p.ng, rc);            // SEP: ng / C_max
  const double G = -2.0 * ngc;
  double a[RW][D], rp[RW];
  double m[RW], s[RW];
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    const int64_t i = i0 + r;
#pragma unroll
    for (int k = 0; k < D; ++k) a[r][k] = i < p.na ? __ldg(p.A + k * p.lda + i) : 0.0;
    rp[r] = (p.rowpot && i < p.na) ? __ldg(p.rowpot + i) : 0.0;
    if (SEP) {                                       // rp becomes A_i
      double nx = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) nx = fma(a[r][k], a[r][k], nx);
      rp[r] = fma(ngc, nx, rp[r]);
    }
    m[r] = (OP == OTN_PC_LSE || OP == OTN_PC_LSE_PART || OP == OTN_PC_MAXD || OP == OTN_PC_DIAG)
               ? OTN_NINF : 0.0;
    if (OP == OTN_PC_LSE_SHIFT) m[r] = i < p.na ? __ldg(p.outer + i) : 0.0;   // fixed shift
    s[r] = 0.0;
  }
  for (int64_t j0 = 0; j0 < p.nb; j0 += kPcTile) {
    __syncthreads();
    for (int t = threadIdx.x; t < kPcTile; t += kPcThreads) {
      const int64_t j = j0 + t;
      const bool ok = j < p.nb;
#pragma unroll
      for (int k = 0; k < D; ++k) sb[k][t] = ok ? __ldg(p.B + k * p.ldb + j) : 0.0;
      double cp = 0.0;
      if (ok && p.colpot) {
        cp = __ldg(p.colpot + j);
        if (p.colpot_d) cp = __dadd_rn(cp, __dmul_rn(p.alpha, __ldg(p.colpot_d + j)));
      }
      if (SEP) {                                     // scp becomes B_j
        double ny = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) ny = fma(sb[k][t], sb[k][t], ny);
        cp = fma(ngc, ny, cp);
      }
      scp[t] = cp;
      svec[t] = (ok && p.vec) ? __ldg(p.vec + j) : 0.0;
    }
    __syncthreads();
    const int jn = int(p.nb - j0 < kPcTile ? p.nb - j0 : int64_t(kPcTile));
    if (OP == OTN_PC_LSE_SHIFT) {
      // against the known shift: no running max, no rescale; each staged
      // column point read once for all RW rows
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int t = lane + 32 * q;
        if (t < jn) {
          double bb[D];
#pragma unroll
          for (int k = 0; k < D; ++k) bb[k] = sb[k][t];
          const double cpt = scp[t];
#pragma unroll
          for (int r = 0; r < RW; ++r) {
            double e;
            if (SEP) {
              e = sep_exponent<D>(a[r], bb, rp[r], cpt, G);
            } else {
              const double c = pc_cost<D>(a[r], bb, p.cmax, rc);
              e = __dadd_rn(__dmul_rn(p.ng, c), cpt);
              if (p.rowpot) e = __dadd_rn(e, rp[r]);
            }
            s[r] += exp_tab(__dsub_rn(e, m[r]), s_exp);
          }
        }
      }
    } else if (OP == OTN_PC_LSE || OP == OTN_PC_LSE_PART) {
      // 8 columns per lane per tile: chunk max, one rescale, then exps; each
      // staged column point is read once for all RW rows (column-outer loop)
      double e[RW][8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int t = lane + 32 * q;
        if (t < jn) {
          double bb[D];
#pragma unroll
          for (int k = 0; k < D; ++k) bb[k] = sb[k][t];
          const double cpt = scp[t];
#pragma unroll
          for (int r = 0; r < RW; ++r) {
            if (SEP) {
              e[r][q] = sep_exponent<D>(a[r], bb, rp[r], cpt, G);
            } else {
              const double c = pc_cost<D>(a[r], bb, p.cmax, rc);
              e[r][q] = __dadd_rn(__dmul_rn(p.ng, c), cpt);
              if (p.rowpot) e[r][q] = __dadd_rn(e[r][q], rp[r]);
            }
          }
        } else {
#pragma unroll
          for (int r = 0; r < RW; ++r) e[r][q] = OTN_NINF;
        }
      }
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        double cm = OTN_NINF;
#pragma unroll
        for (int q = 0; q < 8; ++q) cm = fmax(cm, e[r][q]);
        if (cm > m[r]) {
          s[r] = s[r] * exp_tab_le0(m[r] - cm, s_exp);
          m[r] = cm;
        }
        if (m[r] != OTN_NINF) {
#pragma unroll
          for (int q = 0; q < 8; ++q) s[r] += exp_tab_le0(e[r][q] - m[r], s_exp);
        }
      }
    } else {
      for (int t = lane; t < jn; t += 32) {
        double bb[D];
#pragma unroll
        for (int k = 0; k < D; ++k) bb[k] = sb[k][t];
        const double cpj = scp[t], vj = svec[t];
#pragma unroll
        for (int r = 0; r < RW; ++r) {
          const double c = SEP ? 0.0 : pc_cost<D>(a[r], bb, p.cmax, rc);
          if (OP == OTN_PC_MAXD) {
            m[r] = fmax(m[r], c);
          } else if (OP == OTN_PC_CDOT) {
            s[r] = fma(c, vj, s[r]);
          } else {
            double e;
            if (SEP) {
              e = sep_exponent<D>(a[r], bb, rp[r], cpj, G);
            } else {
              const double kc = __dmul_rn(p.ng, c);
              e = p.order == 0 ? __dadd_rn(__dadd_rn(kc, cpj), rp[r])
                               : __dadd_rn(__dadd_rn(kc, rp[r]), cpj);
            }
            const double pe = exp_tab(e, s_exp);
            if (OP == OTN_PC_DOT) {
              s[r] = fma(pe, vj, s[r]);
            } else if (OP == OTN_PC_DOTC) {
              s[r] = fma(__dmul_rn(pe, c), vj, s[r]);
            } else {  // DIAG: sum P^2 vec, max exponent
              s[r] = fma(__dmul_rn(pe, pe), vj, s[r]);
              m[r] = fmax(m[r], e);
            }
          }
        }
      }
    }
  }
  // per-row warp reduction (fixed tree), lane 0 writes
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    const int64_t i = i0 + r;
    double mm = m[r], ss = s[r];
    if (OP == OTN_PC_LSE || OP == OTN_PC_LSE_PART) {
      warp_lse(mm, ss);
    } else {
      if (OP == OTN_PC_MAXD || OP == OTN_PC_DIAG) mm = warp_max(mm);
      if (OP != OTN_PC_MAXD) ss = warp_sum(ss);
    }
    if (lane == 0 && i < p.na) {
      if (OP == OTN_PC_LSE) {
        const double lse = lse_value(mm, ss);
        double o = 0.0;
        if (p.outer) {
          o = __ldg(p.outer + i);
          if (p.outer_d) o = __dadd_rn(o, __dmul_rn(p.alpha, __ldg(p.outer_d + i)));
        }
        p.out[i] = p.mode == 0 ? __dadd_rn(o, lse) : __dsub_rn(o, lse);
      } else if (OP == OTN_PC_LSE_PART) {
        p.out[i] = mm;
        p.out2[i] = ss;
      } else if (OP == OTN_PC_LSE_SHIFT) {
        p.out[i] = ss;
      } else if (OP == OTN_PC_MAXD) {
        p.out[i] = mm;
      } else {
        p.out[i] = ss;
        if (OP == OTN_PC_DIAG && p.out2) p.out2[i] = mm;
      }
    }
  }
}

template <int RW, int D, int OP, int MB = 2>
static cudaError_t launch_rw(const PairArgs& p, cudaStream_t st, bool sep) {
  const int64_t rows = 8 * RW;
  constexpr bool kSepOp = OP == OTN_PC_LSE || OP == OTN_PC_LSE_PART || OP == OTN_PC_LSE_SHIFT ||
                          OP == OTN_PC_DOT || OP == OTN_PC_DIAG;
  if (kSepOp && sep && p.cmax > 0.0)
    k_pair<RW, D, OP, MB, kSepOp><<<unsigned((p.na + rows - 1) / rows), kPcThreads, 0, st>>>(p);
  else
    k_pair<RW, D, OP, MB, false><<<unsigned((p.na + rows - 1) / rows), kPcThreads, 0, st>>>(p);
  return cudaGetLastError();
}

// Rows per warp / CTAs per SM (measured on B200, d = 3, n = 65536, 8192..65536
// rows): the log-sum-exp and product passes reuse each staged column point
// across 4 rows per warp at 2 CTAs per SM (LSE: 9.5 ms per pass against 9.9
// with 2 rows at 3 CTAs per SM), dropping to 2 rows when that leaves SMs
// idle.  8 rows per warp spills (the first choice, 1.6-1.8x slower).
template <int D, int OP>
static cudaError_t launch_d(const PairArgs& p, cudaStream_t st, int num_sms, bool sep) {
  if ((p.na + 31) / 32 < num_sms)
    return launch_rw<2, D, OP, 3>(p, st, sep);
  return launch_rw<4, D, OP, 2>(p, st, sep);
}

template <int OP>
static cudaError_t launch_pair_op(const PairArgs& p, cudaStream_t st, int num_sms, bool sep) {
  switch (p.d) {
    case 1: return launch_d<1, OP>(p, st, num_sms, sep);
    case 2: return launch_d<2, OP>(p, st, num_sms, sep);
    case 3: return launch_d<3, OP>(p, st, num_sms, sep);
    case 4: return launch_d<4, OP>(p, st, num_sms, sep);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_pair(otn_ctx* x, const PairArgs& p) {
  switch (p.op) {
    case OTN_PC_LSE: return launch_pair_op<OTN_PC_LSE>(p, x->stream, x->num_sms, !x->pc_exact);
    case OTN_PC_DOT: return launch_pair_op<OTN_PC_DOT>(p, x->stream, x->num_sms, !x->pc_exact);
    case OTN_PC_DIAG: return launch_pair_op<OTN_PC_DIAG>(p, x->stream, x->num_sms, !x->pc_exact);
    case OTN_PC_MAXD: return launch_pair_op<OTN_PC_MAXD>(p, x->stream, x->num_sms, !x->pc_exact);
    case OTN_PC_LSE_PART: return launch_pair_op<OTN_PC_LSE_PART>(p, x->stream, x->num_sms, !x->pc_exact);
    case OTN_PC_DOTC: return launch_pair_op<OTN_PC_DOTC>(p, x->stream, x->num_sms, !x->pc_exact);
    case OTN_PC_CDOT: return launch_pair_op<OTN_PC_CDOT>(p, x->stream, x->num_sms, !x->pc_exact);
    case OTN_PC_LSE_SHIFT: return launch_pair_op<OTN_PC_LSE_SHIFT>(p, x->stream, x->num_sms, !x->pc_exact);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace otn
