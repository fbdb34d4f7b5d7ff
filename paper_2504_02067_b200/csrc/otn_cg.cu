// Device-resident truncated-Newton direction solver (K6 + K7 + K8 and the
// CG / rho-annealing loops of newton.py:123-210) as ONE persistent
// cooperative kernel: one 512-thread CTA per SM, grid-wide barriers between
// the dependent phases, no host round trip until the direction is done.
//
// Data layout: CTA b owns the contiguous row block [r0, r1) of the plan P.
// A Hessian-vector product  q = rP*x - rho * P((P^T x)/cP)  is
//   phase A   per-CTA column partials  wpart[b][j] = sum_{i in block} P_ij x_i
//             (rows ascending, 16-byte streaming loads, FMA accumulate)
//   -- grid barrier --
//   phase A2  column slices: w_j = sum_b wpart[b][j] (fixed order); wc = w/cP
//   -- grid barrier --
//   phase B   own rows, DESCENDING (the rows phase A touched last are still
//             in L2): s_i = sum_j P_ij wc_j, then q_i = rP_i x_i - rho s_i.
// The thread -> column mapping is identical in phases A and B (thread t owns
// columns {2t, 2t+1} + k*1024 of every 4096-column tile), so each thread's
// wc values live in registers during phase B.  512 threads x 4 chunks of 16 B
// per row keep 64-128 KB of loads in flight per SM.
// CG vector updates are row-local; the dot products / L1 norms are grid
// reductions with fixed trees (deterministic, no FP64 atomics).
#include <cooperative_groups.h>

#include "otn_common.cuh"
#include "otn_internal.h"

namespace cg = cooperative_groups;

namespace otn {

constexpr int NT = kCoopThreads;
constexpr int NW = NT / 32;         // warps per CTA
constexpr int CH = 4;               // 16-byte chunks per thread per tile
constexpr int TILE = NT * 2 * CH;   // 4096 columns
constexpr int RB = 4;               // rows per phase-B group
constexpr int kRefresh = 50;        // newton.py:38 TRUE_RESIDUAL_REFRESH

struct Smem {
  double red[4][33];
  double gres[4];
  double a2[NW][33];
  double bpart[2][NW][RB];
};

__device__ __forceinline__ double2 ldcg2(const double* p) {
  return __ldcg(reinterpret_cast<const double2*>(p));
}

template <int K>
__device__ __forceinline__ void grid_reduce(cg::grid_group& grid, double (&v)[K], double* red,
                                            int& slot, Smem& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = gridDim.x;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) sh.red[k][warp] = v[k];
  }
  __syncthreads();
  if (warp == 0) {
    double* dst = red + (int64_t(slot) * G + blockIdx.x) * kRedWidth;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double t = warp_sum(lane < NW ? sh.red[k][lane] : 0.0);
      if (lane == 0) dst[k] = t;
    }
  }
  grid.sync();
  if (warp == 0) {
    const double* src = red + int64_t(slot) * G * kRedWidth;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double t = 0.0;
      for (int b = lane; b < G; b += 32) t += __ldcg(src + int64_t(b) * kRedWidth + k);
      t = warp_sum(t);
      if (lane == 0) sh.gres[k] = t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = sh.gres[k];
  slot ^= 1;
}

// Phase A: column partials of P^T x over this CTA's rows.
__device__ __noinline__ void phase_a(const CoopArgs& a, const double* x, int64_t r0, int64_t r1, double* wrow) {
  const int t = threadIdx.x;
  for (int64_t tile = 0; tile < a.ld; tile += TILE) {
    double2 acc[CH];
    bool ok[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      acc[c] = make_double2(0.0, 0.0);
      ok[c] = tile + c * NT * 2 + 2 * t < a.ld;
    }
    const double* base = a.P + tile + 2 * t;
    int64_t i = r0;
    for (; i + 1 < r1; i += 2) {
      const double x0 = x[i], x1 = x[i + 1];
      const double* p0 = base + i * a.ld;
      double2 v0[CH], v1[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (ok[c]) {
          v0[c] = ld_stream2(p0 + c * NT * 2);
          v1[c] = ld_stream2(p0 + a.ld + c * NT * 2);
        }
      }
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (ok[c]) {
          acc[c].x = fma(v0[c].x, x0, acc[c].x);
          acc[c].y = fma(v0[c].y, x0, acc[c].y);
          acc[c].x = fma(v1[c].x, x1, acc[c].x);
          acc[c].y = fma(v1[c].y, x1, acc[c].y);
        }
      }
    }
    if (i < r1) {
      const double x0 = x[i];
      const double* p0 = base + i * a.ld;
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (ok[c]) {
          const double2 v = ld_stream2(p0 + c * NT * 2);
          acc[c].x = fma(v.x, x0, acc[c].x);
          acc[c].y = fma(v.y, x0, acc[c].y);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (ok[c]) *reinterpret_cast<double2*>(wrow + tile + c * NT * 2 + 2 * t) = acc[c];
    }
  }
}

// Phase A2: reduce the per-CTA partials for 32-column slices.
//   kind 0: out = w / cP     (the HVP's inner vector, and apply_pc)
//   kind 1: out = -(w / cP)  (d_v, projector.py:201)
//   kind 2: out = w          (rmatvec)
__device__ __noinline__ void phase_a2(const CoopArgs& a, int kind, double* out, Smem& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = gridDim.x;
  for (int64_t s = blockIdx.x; s * 32 < a.ld; s += G) {
    const int64_t j = s * 32 + lane;
    double acc = 0.0;
    for (int bp = warp; bp < G; bp += NW) acc += __ldcg(a.wpart + int64_t(bp) * a.ld + j);
    sh.a2[warp][lane] = acc;
    __syncthreads();
    if (warp == 0) {
      double tot = 0.0;
#pragma unroll 8
      for (int w = 0; w < NW; ++w) tot += sh.a2[w][lane];
      double val = 0.0;
      if (j < a.n) {
        val = kind == 2 ? tot : __ddiv_rn(tot, __ldg(a.cP + j));
        if (kind == 1) val = -val;
      }
      out[j] = val;
    }
    __syncthreads();
  }
}

// Phase B: s_i = sum_j P_ij w_j for own rows (descending), into sv[i].
__device__ __noinline__ void phase_b(const CoopArgs& a, const double* w, int64_t r0, int64_t r1, double* sv,
                        Smem& sh) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int buf = 0;
  for (int64_t tile = 0; tile < a.ld; tile += TILE) {
    double2 wv[CH];
    bool ok[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int64_t j = tile + c * NT * 2 + 2 * t;
      ok[c] = j < a.ld;
      wv[c] = ok[c] ? ldcg2(w + j) : make_double2(0.0, 0.0);
    }
    const double* base = a.P + tile + 2 * t;
    for (int64_t hi = r1; hi > r0; hi -= RB) {
      double dot[RB];
      double2 v[RB][CH];
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        dot[k] = 0.0;
        const int64_t i = hi - 1 - k;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          if (i >= r0 && ok[c]) v[k][c] = ld_stream2(base + i * a.ld + c * NT * 2);
          else v[k][c] = make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int k = 0; k < RB; ++k) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          dot[k] = fma(v[k][c].x, wv[c].x, dot[k]);
          dot[k] = fma(v[k][c].y, wv[c].y, dot[k]);
        }
        dot[k] = warp_sum(dot[k]);
      }
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < RB; ++k) sh.bpart[buf][warp][k] = dot[k];
      }
      __syncthreads();
      if (t < RB) {
        const int64_t i = hi - 1 - t;
        if (i >= r0) {
          double tot = 0.0;
#pragma unroll 8
          for (int ww = 0; ww < NW; ++ww) tot += sh.bpart[buf][ww][t];
          sv[i] = tile == 0 ? tot : sv[i] + tot;
        }
      }
      buf ^= 1;
    }
  }
  __syncthreads();
}

// q = F(rho) x on own rows (newton.py:100-105; matvecs skipped when rho == 0).
__device__ void hvp(cg::grid_group& grid, const CoopArgs& a, const double* x, double rho,
                    double* q, int64_t r0, int64_t r1, Smem& sh, int64_t& nh) {
  if (rho != 0.0) {
    ++nh;
    __syncthreads();
    phase_a(a, x, r0, r1, a.wpart + int64_t(blockIdx.x) * a.ld);
    grid.sync();
    phase_a2(a, 0, a.wc, sh);
    grid.sync();
    phase_b(a, a.wc, r0, r1, a.sv, sh);
  }
  for (int64_t i = r0 + threadIdx.x; i < r1; i += NT) {
    double o = __dmul_rn(__ldg(a.rP + i), x[i]);
    if (rho != 0.0) o = __dsub_rn(o, __dmul_rn(rho, a.sv[i]));
    q[i] = o;
  }
  __syncthreads();
}

struct PcgOut {
  int status;
  int64_t iters;
  double resid;
};

// Jacobi-PCG, newton.py:123-172.  b == nullptr means b = -g.
__device__ PcgOut pcg(cg::grid_group& grid, const CoopArgs& a, double rho, const double* bvec,
                      double tol, double* x, bool has_x0, int64_t max_iters, int64_t r0,
                      int64_t r1, int& slot, Smem& sh, int64_t& nh) {
  PcgOut o{OTN_OK, 0, 0.0};
  if (has_x0) hvp(grid, a, x, rho, a.q, r0, r1, sh, nh);
  double loc[3] = {0.0, 0.0, 0.0};
  for (int64_t i = r0 + threadIdx.x; i < r1; i += NT) {
    const double Mi = __dmul_rn(__ldg(a.rP + i), __dsub_rn(1.0, __dmul_rn(rho, __ldg(a.mu + i))));
    a.M[i] = Mi;
    const double bi = bvec ? __ldg(bvec + i) : -__ldg(a.g + i);
    double ri;
    if (has_x0) {
      ri = __dsub_rn(bi, a.q[i]);
    } else {
      x[i] = 0.0;
      ri = bi;
    }
    a.r[i] = ri;
    const double zi = __ddiv_rn(ri, Mi);
    a.z[i] = zi;
    a.p[i] = zi;
    loc[0] += fabs(ri);
    loc[1] = fma(ri, zi, loc[1]);
    if (Mi <= 0.0) loc[2] += 1.0;
  }
  grid_reduce<3>(grid, loc, a.red, slot, sh);
  if (loc[2] > 0.0) { o.status = OTN_ST_PRECOND; return o; }
  if (loc[0] <= tol) { o.resid = loc[0]; return o; }
  double rz = loc[1];
  double norm = loc[0];
  for (int64_t k = 1; k <= max_iters; ++k) {
    hvp(grid, a, a.p, rho, a.q, r0, r1, sh, nh);
    double pq[1] = {0.0};
    for (int64_t i = r0 + threadIdx.x; i < r1; i += NT) pq[0] = fma(a.p[i], a.q[i], pq[0]);
    grid_reduce<1>(grid, pq, a.red, slot, sh);
    if (pq[0] <= 0.0) { o.status = OTN_ST_BREAKDOWN; o.iters = k; o.resid = pq[0]; return o; }
    const double alpha = rz / pq[0];
    for (int64_t i = r0 + threadIdx.x; i < r1; i += NT) {
      x[i] = __dadd_rn(x[i], __dmul_rn(alpha, a.p[i]));
      a.r[i] = __dsub_rn(a.r[i], __dmul_rn(alpha, a.q[i]));
    }
    if (k % kRefresh == 0) {
      hvp(grid, a, x, rho, a.q, r0, r1, sh, nh);
      for (int64_t i = r0 + threadIdx.x; i < r1; i += NT) {
        const double bi = bvec ? __ldg(bvec + i) : -__ldg(a.g + i);
        a.r[i] = __dsub_rn(bi, a.q[i]);
      }
    }
    double nz[2] = {0.0, 0.0};
    for (int64_t i = r0 + threadIdx.x; i < r1; i += NT) {
      const double ri = a.r[i];
      const double zi = __ddiv_rn(ri, a.M[i]);
      a.z[i] = zi;
      nz[0] += fabs(ri);
      nz[1] = fma(ri, zi, nz[1]);
    }
    grid_reduce<2>(grid, nz, a.red, slot, sh);
    norm = nz[0];
    if (norm <= tol) { o.iters = k; o.resid = norm; return o; }
    const double beta = nz[1] / rz;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += NT)
      a.p[i] = __dadd_rn(a.z[i], __dmul_rn(beta, a.p[i]));
    rz = nz[1];
  }
  o.status = OTN_ST_NONCONVERGENCE;
  o.iters = max_iters;
  o.resid = norm;
  return o;
}

__global__ void __launch_bounds__(NT, 1) k_coop(CoopArgs a) {
  __shared__ Smem sh;
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x;
  const int64_t r0 = (int64_t(blockIdx.x) * a.n) / G;
  const int64_t r1 = (int64_t(blockIdx.x + 1) * a.n) / G;
  int slot = 0;
  int64_t nh = 0;
  DevResult res{};
  res.status = OTN_OK;

  if (a.pre_flags) {
    // [0]: plan overflow (materialize), [1]: nonpositive sums (system prep);
    // checked in the reference's order (dual.py:155-169 then newton.py:76-77).
    const int f0 = ((volatile const int*)a.pre_flags)[0];
    const int f1 = ((volatile const int*)a.pre_flags)[1];
    if (f0) res.status = OTN_ST_PLAN_OVERFLOW;
    else if (f1) res.status = OTN_ST_NONPOSITIVE_SUMS;
    if (res.status != OTN_OK) {
      if (blockIdx.x == 0 && threadIdx.x == 0) *a.res = res;
      return;  // uniform across the grid: no barrier is skipped by only some CTAs
    }
  }

  if (a.mode == kModeNewton) {
    double gl[1] = {0.0};
    for (int64_t i = r0 + threadIdx.x; i < r1; i += NT) gl[0] += fabs(__ldg(a.g + i));
    grid_reduce<1>(grid, gl, a.red, slot, sh);
    const double gn = gl[0];
    res.rho_final = a.rho0;
    if (gn == 0.0) {
      for (int64_t i = r0 + threadIdx.x; i < r1; i += NT) a.d[i] = 0.0;
      __syncthreads();
    } else {
      for (int64_t i = r0 + threadIdx.x; i < r1; i += NT)
        a.d[i] = __ddiv_rn(-__ldg(a.g + i), __ldg(a.rP + i));
      double rho = a.rho0, used = a.rho0;
      int64_t total = 0;
      const double tol = __dmul_rn(__dmul_rn(0.25, a.eta), gn);
      const double target = __dmul_rn(a.eta, gn);
      while (true) {
        hvp(grid, a, a.d, 1.0, a.q, r0, r1, sh, nh);
        double rl[1] = {0.0};
        for (int64_t i = r0 + threadIdx.x; i < r1; i += NT)
          rl[0] += fabs(__dadd_rn(a.q[i], __ldg(a.g + i)));
        grid_reduce<1>(grid, rl, a.red, slot, sh);
        if (rl[0] <= target) { res.resid_l1 = rl[0]; break; }
        if (__dsub_rn(1.0, rho) < 1e-12) {
          res.status = OTN_ST_STAGNATION;
          res.resid_l1 = rl[0];
          res.diag_rho = rho;
          break;
        }
        ++res.pcg_calls;
        const PcgOut po = pcg(grid, a, rho, nullptr, tol, a.d, a.zero_init == 0, a.max_iters,
                              r0, r1, slot, sh, nh);
        if (po.status != OTN_OK) {
          res.status = po.status;
          res.diag_rho = rho;
          res.diag_resid = po.resid;
          total += po.iters;
          break;
        }
        total += po.iters;
        used = rho;
        rho = __dsub_rn(1.0, __ddiv_rn(__dsub_rn(1.0, rho), 4.0));
      }
      res.cg_iters = total;
      res.rho_final = used;
    }
    if (res.status == OTN_OK && a.dv) {
      __syncthreads();
      phase_a(a, a.d, r0, r1, a.wpart + int64_t(blockIdx.x) * a.ld);
      grid.sync();
      phase_a2(a, 1, a.dv, sh);
      double sl[1] = {0.0};
      for (int64_t i = r0 + threadIdx.x; i < r1; i += NT) sl[0] = fma(__ldg(a.g + i), a.d[i], sl[0]);
      grid_reduce<1>(grid, sl, a.red, slot, sh);
      res.slope = -sl[0];
    }
  } else if (a.mode == kModePcg) {
    res.pcg_calls = 1;
    const PcgOut po = pcg(grid, a, a.rho, a.b, a.tol, a.d, a.has_x0 != 0, a.max_iters, r0, r1,
                          slot, sh, nh);
    res.status = po.status;
    res.cg_iters = po.iters;
    res.resid_l1 = po.resid;
    res.diag_rho = a.rho;
    res.diag_resid = po.resid;
  } else if (a.mode == kModeHvp) {
    hvp(grid, a, a.xin, a.rho, a.d, r0, r1, sh, nh);
  } else if (a.mode == kModePc || a.mode == kModeRmatvec) {
    phase_a(a, a.xin, r0, r1, a.wpart + int64_t(blockIdx.x) * a.ld);
    grid.sync();
    phase_a2(a, a.mode == kModePc ? 0 : 2, a.wc, sh);
    grid.sync();
    for (int64_t i = int64_t(blockIdx.x) * NT + threadIdx.x; i < a.n; i += int64_t(G) * NT)
      a.d[i] = __ldcg(a.wc + i);
  } else if (a.mode == kModeMatvec) {
    // stage x into the padded workspace vector (phase B reads ld entries)
    for (int64_t j = int64_t(blockIdx.x) * NT + threadIdx.x; j < a.ld; j += int64_t(G) * NT)
      a.wc[j] = j < a.n ? __ldg(a.xin + j) : 0.0;
    grid.sync();
    phase_b(a, a.wc, r0, r1, a.sv, sh);
    for (int64_t i = r0 + threadIdx.x; i < r1; i += NT) a.d[i] = a.sv[i];
  }
  res.hvps = nh;
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.res = res;
}

cudaError_t launch_coop(otn_ctx* x, const CoopArgs& a) {
  void* args[] = {const_cast<CoopArgs*>(&a)};
  return cudaLaunchCooperativeKernel((void*)k_coop, dim3(x->coop_blocks), dim3(NT), args, 0,
                                     x->stream);
}

int coop_occupancy(int* blocks_per_sm) {
  return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_coop, NT, 0);
}

}  // namespace otn
