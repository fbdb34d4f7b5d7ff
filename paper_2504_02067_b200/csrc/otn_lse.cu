// Log-domain reductions over the stored cost (K1/K2/K3), plan materialization
// with the fused Jacobi diagonal (K4+K5), and the system prep vectors.
//
// All of these stream the n x n cost (or plan) once from HBM with 128-bit
// non-allocating loads and do their math in FP64 registers; they are HBM /
// FP64-pipe bound (exp costs ~20 FP64 instructions per entry).
#include "otn_common.cuh"
#include "otn_internal.h"

namespace otn {

struct LseArgs {
  const double* C;
  int64_t n, ld;
  double ng;                // -gamma
  const double* outer;      // nullable -> 0.0
  const double* outer_d;    // nullable; outer_eff = outer + alpha*outer_d
  const double* inner;
  const double* inner_d;    // nullable; inner_eff = inner + alpha*inner_d
  double alpha;
  int mode;                 // 0: out = outer + lse;  1: out = outer - lse
  double* out;
  const int* gate;          // nullable: skip the launch when *gate == 0
};

__device__ __forceinline__ double eff(const double* base, const double* dir, double alpha,
                                      int64_t j) {
  double b = __ldg(base + j);
  // numpy: base + alpha*dir, each operation rounded (dual.py:174-175)
  return dir ? __dadd_rn(b, __dmul_rn(alpha, __ldg(dir + j))) : b;
}

__device__ __forceinline__ double finish(const LseArgs& a, int64_t j, double lse) {
  double o = a.outer ? eff(a.outer, a.outer_d, a.alpha, j) : 0.0;
  return a.mode == 0 ? __dadd_rn(o, lse) : __dsub_rn(o, lse);
}

// ---------------------------------------------------------------------------
// Row LSE: one warp per row; each lane streams 8 entries (four 16-byte loads)
// per step, keeps an online (max, sum-exp) pair and rescales at most once per
// step, so the cost is ~1.1 exp per entry.
// ---------------------------------------------------------------------------
// 4 rows (warps) per 128-thread block: 1024 blocks keep the SMs evenly loaded,
// and the block stages each 256-column step of the inner vector (with its
// alpha * dir term, formed once per block instead of once per row) in shared
// memory, double-buffered with one barrier per step.
constexpr int kLseRowThreads = 128;

template <bool FULL>
__global__ void __launch_bounds__(kLseRowThreads) k_lse_rows(LseArgs a) {
  __shared__ double2 s_exp[64];
  __shared__ double s_in[2][256];
  if (a.gate && *a.gate == 0) return;               // uniform over the grid
  exp_tab_load(s_exp);
  const int64_t row = int64_t(blockIdx.x) * (kLseRowThreads / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const bool valid = FULL || row < a.n;
  const double* crow = a.C + (valid ? row : 0) * a.ld;
  const int64_t n = a.n;
  double m = OTN_NINF, s = 0.0;
  // C loads run one 256-column step ahead of the math (cur, nxt: a deeper
  // register prefetch costs occupancy and measured slower), as do the inner
  // vector's (raw values: the alpha * dir term is formed when staged)
  constexpr int kIn = 256 / kLseRowThreads;
  double2 cur[4], nxt[4];
  double ib[kIn], id[kIn];
  auto load_in = [&](int64_t base) {
#pragma unroll
    for (int q = 0; q < kIn; ++q) {
      const int64_t j = base + threadIdx.x + kLseRowThreads * q;
      ib[q] = FULL || j < n ? __ldg(a.inner + j) : 0.0;
      id[q] = a.inner_d && (FULL || j < n) ? __ldg(a.inner_d + j) : 0.0;
    }
  };
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t j = 64 * k + 2 * lane;
    cur[k] = valid && (FULL || j < n) ? ld_stream2(crow + j) : make_double2(0.0, 0.0);
  }
  load_in(0);
  int buf = 0;
  for (int64_t base = 0; base < n; base += 256) {
#pragma unroll
    for (int q = 0; q < kIn; ++q)   // numpy: base + alpha*dir, each operation rounded (dual.py:174-175)
      s_in[buf][threadIdx.x + kLseRowThreads * q] =
          a.inner_d ? __dadd_rn(ib[q], __dmul_rn(a.alpha, id[q])) : ib[q];
    __syncthreads();                                 // also publishes s_exp on the first step
    if (base + 256 < n) load_in(base + 256);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t j = base + 256 + 64 * k + 2 * lane;
      // (FULL: the last step has no next step; j < n covers that otherwise)
      nxt[k] = valid && (FULL ? base + 256 < n : j < n) ? ld_stream2(crow + j)
                                                        : make_double2(0.0, 0.0);
    }
    double b[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int jl = 64 * k + 2 * lane;
      const int64_t j = base + jl;
      const double2 in = *reinterpret_cast<const double2*>(&s_in[buf][jl]);
      b[2 * k] = FULL || j < n ? __dadd_rn(__dmul_rn(a.ng, cur[k].x), in.x) : OTN_NINF;
      b[2 * k + 1] = FULL || j + 1 < n ? __dadd_rn(__dmul_rn(a.ng, cur[k].y), in.y) : OTN_NINF;
    }
    double cm = b[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) cm = fmax(cm, b[k]);
    if (cm > m) {
      s = s * exp_tab(m - cm, s_exp);
      m = cm;
    }
    if (m != OTN_NINF) {
#pragma unroll
      for (int k = 0; k < 8; ++k) s = add_exp_le0(s, b[k] - m, s_exp);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) cur[k] = nxt[k];
    buf ^= 1;
  }
  warp_lse(m, s);
  if (valid && lane == 0) a.out[row] = finish(a, row, lse_value(m, s));
}

// ---------------------------------------------------------------------------
// Row LSE through the bulk-copy (TMA) engine, persistent (ld <= 4096).
//
// A 1-D cp.async.bulk request is served by the SM's copy engine one request
// after another (measured, tools/l2stream.cu: 4 KB requests stream at ~12
// GB/s per SM whatever the ring depth; whole 32 KB rows reach the SM's HBM
// share, tools/bulk_rows.cu: 6.7 TB/s chip-wide), so each request here is a
// WHOLE row of C (up to 32 KB, contiguous).  CTA b (one per SM) owns rows
// [b n / G, (b+1) n / G).  It stages the inner vector once (with its alpha *
// direction term for the trial sums, formed once); a producer lane streams
// the rows into a kRowStages-deep ring (full / empty mbarriers).  kRowGroups
// groups of 8 warps take the rows in turn (group g: rows g, g + kRowGroups,
// ...), warp w of a group holding 512 columns: the group first takes the row max
// (warp maxima through shared memory, a named barrier), then sums
// exp(b - max) over its entries (entries below -746 add an exact 0 and are
// skipped, as everywhere), and the group's first warp adds the 8 partial sums
// in warp order -- deterministic; numpy's own max-then-sum form
// (_kernels.py:33-40).
// ---------------------------------------------------------------------------
constexpr int kRowW = 4096;                         // columns staged per row (ld <= kRowW)
constexpr int kRowGroup = 8;                        // warps per row: 512 columns each
constexpr int kRowGroups = 3;                       // rows being reduced at once
constexpr int kRowStages = 6;                       // rows in flight (ring depth)
constexpr int kRowThreads = (kRowGroups * kRowGroup + 1) * 32;   // + the producer warp
constexpr size_t kRowSmem = size_t(kRowStages + 1) * kRowW * 8;  // ring + inner vector

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n"
      ::"r"(bar), "r"(phase) : "memory");
}
__device__ __forceinline__ void group_sync(int id) {   // the 8 warps of one stage
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kRowGroup * 32) : "memory");
}

template <bool DIR>
__global__ void __launch_bounds__(kRowThreads) k_lse_rows_bulk(LseArgs a) {
  extern __shared__ __align__(128) double s_dyn[];  // [kRowStages][kRowW] rows, [kRowW] inner
  __shared__ double2 s_exp[64];
  __shared__ __align__(8) uint64_t s_full[kRowStages], s_empty[kRowStages], s_inbar;
  __shared__ double s_pm[kRowGroups][kRowGroup], s_ps[kRowGroups][kRowGroup];
  if (a.gate && *a.gate == 0) return;               // uniform over the grid
  double* s_in = s_dyn + size_t(kRowStages) * kRowW;
  const int G = gridDim.x;
  const int64_t r0 = (int64_t(blockIdx.x) * a.n) / G, r1 = (int64_t(blockIdx.x + 1) * a.n) / G;
  const int rows = int(r1 - r0);
  const uint32_t bytes = uint32_t(a.ld) * 8u;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRowStages; ++s) {
      mbar_init(smem_addr(&s_full[s]), 1);
      mbar_init(smem_addr(&s_empty[s]), kRowGroup);
    }
    mbar_init(smem_addr(&s_inbar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the inner vector (and its direction, parked in stage 0 until combined)
    mbar_expect_tx(smem_addr(&s_inbar), bytes * (DIR ? 2u : 1u));
    bulk_load(smem_addr(s_in), a.inner, bytes, smem_addr(&s_inbar));
    if (DIR) bulk_load(smem_addr(s_dyn), a.inner_d, bytes, smem_addr(&s_inbar));
  }
  exp_tab_load(s_exp);
  __syncthreads();                                  // barriers initialized, table loaded
  mbar_wait(smem_addr(&s_inbar), 0);
  if (DIR) {                                        // numpy: base + alpha*dir (dual.py:174-175)
    for (int j = threadIdx.x; j < int(a.ld); j += kRowThreads)
      s_in[j] = __dadd_rn(s_in[j], __dmul_rn(a.alpha, s_dyn[j]));
    __syncthreads();                                // stage 0 free again
  }
  if (warp == kRowGroups * kRowGroup) {             // producer
    if (lane == 0) {
      for (int it = 0; it < rows; ++it) {
        const int s = it % kRowStages;
        if (it >= kRowStages) mbar_wait(smem_addr(&s_empty[s]), uint32_t(it / kRowStages - 1) & 1u);
        const uint32_t full = smem_addr(&s_full[s]);
        mbar_expect_tx(full, bytes);
        bulk_load(smem_addr(s_dyn + size_t(s) * kRowW), a.C + (r0 + it) * a.ld, bytes, full);
      }
    }
    return;
  }
  const int g = warp / kRowGroup, gw = warp % kRowGroup;   // group, warp within the group
  const int cb = gw * (kRowW / kRowGroup);                  // this warp's 512 columns
  for (int it = g; it < rows; it += kRowGroups) {
    const int s = it % kRowStages;
    const double* crow = s_dyn + size_t(s) * kRowW;
    mbar_wait(smem_addr(&s_full[s]), uint32_t(it / kRowStages) & 1u);
    double b[16];
    double wm = OTN_NINF;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = cb + 256 * h + 64 * k + 2 * lane;
        double2 c = make_double2(0.0, 0.0), in = make_double2(0.0, 0.0);
        if (j < int(a.ld)) {
          c = *reinterpret_cast<const double2*>(&crow[j]);
          in = *reinterpret_cast<const double2*>(&s_in[j]);
        }
        b[8 * h + 2 * k] = j < a.n ? __dadd_rn(__dmul_rn(a.ng, c.x), in.x) : OTN_NINF;
        b[8 * h + 2 * k + 1] = j + 1 < a.n ? __dadd_rn(__dmul_rn(a.ng, c.y), in.y) : OTN_NINF;
        wm = fmax(wm, fmax(b[8 * h + 2 * k], b[8 * h + 2 * k + 1]));
      }
    }
    wm = warp_max(wm);
    if (lane == 0) s_pm[g][gw] = wm;
    group_sync(1 + g);
    double M = s_pm[g][0];
#pragma unroll
    for (int w = 1; w < kRowGroup; ++w) M = fmax(M, s_pm[g][w]);
    double sum = 0.0;
    if (M != OTN_NINF) {
      // entries more than 707 below the row max add nothing (exp_m707); a
      // warp with no live entry in its 512 columns skips them all (late
      // stages: most warps), the others run the 16 exps straight-line
      bool any = false;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        b[k] = b[k] - M;
        any |= b[k] >= -707.0;
      }
      if (__any_sync(0xffffffffu, any)) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const bool live = b[k] >= -707.0;
          const double e = exp_m707(live ? b[k] : 0.0, s_exp);
          sum = live ? sum + e : sum;
        }
      }
    }
    sum = warp_sum(sum);
    if (lane == 0) s_ps[g][gw] = sum;
    group_sync(1 + g);
    if (gw == 0 && lane == 0) {
      double ss = s_ps[g][0];
#pragma unroll
      for (int w = 1; w < kRowGroup; ++w) ss += s_ps[g][w];
      const int64_t row = r0 + it;
      a.out[row] = finish(a, row, lse_value(M, ss));
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_addr(&s_empty[s]));    // row data released
    // (the next row's maxima overwrite s_pm only after this group's second
    // barrier, so s_ps / s_pm of this row are never read stale)
  }
}

// Persistent grid of the bulk-copy row LSE (one CTA per SM when it fits);
// 0 when the row is too wide or the kernel cannot be configured.
int lse_bulk_grid(int num_sms, int64_t n, int64_t ld, int* err) {
  if (ld > kRowW) return 0;
  cudaError_t e = cudaFuncSetAttribute(k_lse_rows_bulk<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(kRowSmem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_lse_rows_bulk<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(kRowSmem));
  int per = 0;
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_lse_rows_bulk<true>, kRowThreads,
                                                      kRowSmem);
  if (e != cudaSuccess || per < 1) {
    *err = e != cudaSuccess ? int(e) : -1;
    cudaGetLastError();
    return 0;
  }
  const int64_t g = int64_t(per) * num_sms;
  return int(g < n ? g : n);
}

// ---------------------------------------------------------------------------
// Column LSE (asymmetric C): CTA = 64 columns x one slab of rows; each warp
// walks rows 4 at a time (coalesced 512-byte row segments), lanes own 2
// columns.  Partial (max, sum) per slab go to the workspace and a finalize
// kernel merges the slabs in fixed order.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kLseThreads) k_lse_cols_part(LseArgs a, int64_t slab_rows,
                                                               double* part) {
  if (a.gate && *a.gate == 0) return;
  __shared__ double sm_m[8][kColTile];
  __shared__ double sm_s[8][kColTile];
  __shared__ double2 s_exp[64];
  exp_tab_load(s_exp);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = int64_t(blockIdx.x) * kColTile + 2 * lane;
  const int64_t i0 = int64_t(blockIdx.y) * slab_rows;
  const int64_t i1 = min(a.n, i0 + slab_rows);
  const bool c0 = j < a.n, c1 = j + 1 < a.n;
  double m0 = OTN_NINF, s0 = 0.0, m1 = OTN_NINF, s1 = 0.0;
  for (int64_t i = i0 + 4 * warp; i < i1; i += 32) {
    double b0[4], b1[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t ii = i + k;
      if (ii < i1 && c0) {
        const double2 c = ld_stream2(a.C + ii * a.ld + j);
        const double in = eff(a.inner, a.inner_d, a.alpha, ii);
        b0[k] = __dadd_rn(__dmul_rn(a.ng, c.x), in);
        b1[k] = c1 ? __dadd_rn(__dmul_rn(a.ng, c.y), in) : OTN_NINF;
      } else {
        b0[k] = OTN_NINF;
        b1[k] = OTN_NINF;
      }
    }
    double cm0 = fmax(fmax(b0[0], b0[1]), fmax(b0[2], b0[3]));
    double cm1 = fmax(fmax(b1[0], b1[1]), fmax(b1[2], b1[3]));
    if (cm0 > m0) { s0 = s0 * exp_tab(m0 - cm0, s_exp); m0 = cm0; }
    if (cm1 > m1) { s1 = s1 * exp_tab(m1 - cm1, s_exp); m1 = cm1; }
    if (m0 != OTN_NINF) {
#pragma unroll
      for (int k = 0; k < 4; ++k) s0 = add_exp_le0(s0, b0[k] - m0, s_exp);
    }
    if (m1 != OTN_NINF) {
#pragma unroll
      for (int k = 0; k < 4; ++k) s1 = add_exp_le0(s1, b1[k] - m1, s_exp);
    }
  }
  sm_m[warp][2 * lane] = m0;
  sm_s[warp][2 * lane] = s0;
  sm_m[warp][2 * lane + 1] = m1;
  sm_s[warp][2 * lane + 1] = s1;
  __syncthreads();
  if (threadIdx.x < kColTile) {
    const int t = threadIdx.x;
    double m = sm_m[0][t], s = sm_s[0][t];
#pragma unroll
    for (int w = 1; w < 8; ++w) lse_merge(m, s, sm_m[w][t], sm_s[w][t]);
    const int64_t jj = int64_t(blockIdx.x) * kColTile + t;
    if (jj < a.ld) {
      double* dst = part + (int64_t(blockIdx.y) * a.ld + jj) * 2;
      dst[0] = m;
      dst[1] = s;
    }
  }
}

__global__ void k_lse_cols_fin(LseArgs a, int slabs, const double* part) {
  if (a.gate && *a.gate == 0) return;
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= a.n) return;
  double m = OTN_NINF, s = 0.0;
  for (int k = 0; k < slabs; ++k) {
    const double* src = part + (int64_t(k) * a.ld + j) * 2;
    lse_merge(m, s, src[0], src[1]);
  }
  a.out[j] = finish(a, j, lse_value(m, s));
}

// ---------------------------------------------------------------------------
// Plan: P_ij = exp_tab((ng*C_ij + v_j) + u_i), one warp per row, 16-byte stores,
// zeros in the padding columns.  Fused K5: mu_i = (sum_j P_ij^2 icP_j)/rP_i.
// ---------------------------------------------------------------------------
// 4 rows (warps) per 128-thread block; each 256-column step of v and 1/cP is
// staged once per block in shared memory (double-buffered, loaded one step
// ahead), so a row's registers hold only its C prefetch.  FULL: n is a
// multiple of the step, no bounds predicates in the loop.
constexpr int kMatThreads = 128;

template <bool FULL>
__global__ void __launch_bounds__(kMatThreads) k_materialize(const double* __restrict__ C,
    int64_t n, int64_t ld, double ng, const double* __restrict__ u, const double* __restrict__ v,
    double* __restrict__ P, const double* __restrict__ icP, const double* __restrict__ rP,
    double* __restrict__ mu, int* __restrict__ flag, uint64_t* __restrict__ mask) {
  __shared__ double2 s_exp[64];
  __shared__ double s_v[2][256], s_ic[2][256];
  exp_tab_load(s_exp);
  const int64_t row = int64_t(blockIdx.x) * (kMatThreads / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const bool valid = FULL || row < n;               // every thread joins the block barriers
  const double* crow = C + (valid ? row : 0) * ld;
  double* prow = P + (valid ? row : 0) * ld;
  const double ui = valid ? __ldg(u + row) : 0.0;
  const int64_t mw = OTN_MASK_WORDS(ld);
  double acc = 0.0, mx = OTN_NINF;
  uint64_t bits = 0;
  int nnz = 0;
  constexpr int kIn = 256 / kMatThreads;
  double vb[kIn], ib[kIn];
  auto load_in = [&](int64_t base) {
#pragma unroll
    for (int q = 0; q < kIn; ++q) {
      const int64_t j = base + threadIdx.x + kMatThreads * q;
      vb[q] = FULL || j < n ? __ldg(v + j) : 0.0;
      ib[q] = icP && (FULL || j < n) ? __ldg(icP + j) : 0.0;
    }
  };
  double2 cur[4], nxt[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t j = 64 * k + 2 * lane;
    cur[k] = valid && (FULL || j < n) ? ld_stream2(crow + j) : make_double2(0.0, 0.0);
  }
  load_in(0);
  int buf = 0;
  for (int64_t base = 0; base < ld; base += 256) {
#pragma unroll
    for (int q = 0; q < kIn; ++q) {
      s_v[buf][threadIdx.x + kMatThreads * q] = vb[q];
      s_ic[buf][threadIdx.x + kMatThreads * q] = ib[q];
    }
    __syncthreads();                                 // also publishes s_exp on the first step
    if (base + 256 < ld) load_in(base + 256);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t j = base + 256 + 64 * k + 2 * lane;
      nxt[k] = valid && (FULL ? base + 256 < n : j < n) ? ld_stream2(crow + j)
                                                        : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int jl = 64 * k + 2 * lane;
      const int64_t j = base + jl;
      bool nz = false;
      if (valid && (FULL || j < ld)) {
        const double2 vv = *reinterpret_cast<const double2*>(&s_v[buf][jl]);
        double e0 = OTN_NINF, e1 = OTN_NINF;
        if (FULL || j < n) {
          e0 = __dadd_rn(__dadd_rn(__dmul_rn(ng, cur[k].x), vv.x), ui);
          if (FULL || j + 1 < n) e1 = __dadd_rn(__dadd_rn(__dmul_rn(ng, cur[k].y), vv.y), ui);
        }
        mx = fmax(mx, fmax(e0, e1));
        const double p0 = exp_tab(e0, s_exp), p1 = exp_tab(e1, s_exp);
        *reinterpret_cast<double2*>(prow + j) = make_double2(p0, p1);
        nz = (p0 != 0.0) || (p1 != 0.0);
        nnz += int(p0 != 0.0) + int(p1 != 0.0);
        if (icP) {
          const double2 ii = *reinterpret_cast<const double2*>(&s_ic[buf][jl]);
          if (FULL || j < n) acc = fma(__dmul_rn(p0, p0), ii.x, acc);
          if (FULL || j + 1 < n) acc = fma(__dmul_rn(p1, p1), ii.y, acc);
        }
      }
      // segment (64 columns = 512 B) occupancy bit for the HVP's zero skipping
      if (__ballot_sync(0xffffffffu, nz)) bits |= 1ull << (((base >> 6) + k) & 63);
    }
    if (mask && valid && (((base + 256) % kSegWordCols) == 0 || base + 256 >= ld)) {
      if (lane == 0) mask[row * mw + base / kSegWordCols] = bits;
      bits = 0;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) cur[k] = nxt[k];
    buf ^= 1;
  }
  if (!valid) return;
  mx = warp_max(mx);
  if (icP) acc = warp_sum(acc);
  if (mask) {
    nnz = warp_sum_int(nnz);
    if (lane == 0) mask[row * mw + mw - 1] = uint64_t(nnz);   // count word
  }
  if (lane == 0) {
    if (mx > 700.0) atomicOr(flag, 1);          // _kernels.py:53-58
    if (icP) mu[row] = __ddiv_rn(acc, __ldg(rP + row));
  }
}

// Segment occupancy mask of an externally supplied plan (same layout as the
// mask written by k_materialize).
__global__ void __launch_bounds__(kLseThreads) k_plan_mask(const double* __restrict__ P,
    int64_t n, int64_t ld, uint64_t* __restrict__ mask) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const int64_t mw = OTN_MASK_WORDS(ld);
  uint64_t bits = 0;
  int nnz = 0;
  for (int64_t base = 0; base < ld; base += 64) {
    const int64_t j = base + 2 * lane;
    bool nz = false;
    if (j < ld) {
      const double2 p = ld_stream2(P + row * ld + j);
      nz = (p.x != 0.0) || (p.y != 0.0);
      nnz += int(p.x != 0.0) + int(p.y != 0.0);
    }
    if (__ballot_sync(0xffffffffu, nz)) bits |= 1ull << ((base >> 6) & 63);
    if (((base + 64) % kSegWordCols) == 0 || base + 64 >= ld) {
      if (lane == 0) mask[row * mw + base / kSegWordCols] = bits;
      bits = 0;
    }
  }
  nnz = warp_sum_int(nnz);
  if (lane == 0) mask[row * mw + mw - 1] = uint64_t(nnz);   // count word
}

__global__ void k_sys_prep(int64_t n, const double* __restrict__ lr, const double* __restrict__ lc,
                           double* rP, double* cP, double* icP, int* flag) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double rp = exp_fast(lr[i]), cp = exp_fast(lc[i]);
  rP[i] = rp;
  cP[i] = cp;
  icP[i] = __ddiv_rn(1.0, cp);                  // newton.py:111: 1.0 / self.cP
  if (rp <= 0.0 || cp <= 0.0) atomicOr(flag, 2);  // newton.py:76-77
}

// (P*P) @ w — standalone seam operator (_kernels.py:64-74); the solver uses
// the copy fused into k_materialize.
__global__ void __launch_bounds__(kLseThreads) k_square_matvec(const double* __restrict__ P,
    int64_t n, int64_t ld, const double* __restrict__ w, double* __restrict__ out) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const double* prow = P + row * ld;
  double acc = 0.0;
  for (int64_t j = 2 * lane; j < n; j += 64) {
    const double2 p = ld_stream2(prow + j);
    acc = fma(__dmul_rn(p.x, p.x), __ldg(w + j), acc);
    if (j + 1 < n) acc = fma(__dmul_rn(p.y, p.y), __ldg(w + j + 1), acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) out[row] = acc;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static inline unsigned rows_grid(int64_t n, int threads = kLseThreads) {
  return unsigned((n + (threads / 32) - 1) / (threads / 32));
}

cudaError_t launch_lse_rows(otn_ctx* x, const double* C, double ng, const double* outer,
                            const double* outer_d, const double* inner, const double* inner_d,
                            double alpha, int mode, double* out, const int* gate) {
  LseArgs a{C, x->n, x->ld, ng, outer, outer_d, inner, inner_d, alpha, mode, out, gate};
  if (x->lse_bulk_ctas > 0) {                       // whole rows through the copy engine
    if (inner_d)
      k_lse_rows_bulk<true><<<x->lse_bulk_ctas, kRowThreads, kRowSmem, x->stream>>>(a);
    else
      k_lse_rows_bulk<false><<<x->lse_bulk_ctas, kRowThreads, kRowSmem, x->stream>>>(a);
    return cudaGetLastError();
  }
  // full tiles (n a multiple of the 256-column step and of the rows per block):
  // no bounds predicates in the streaming loop
  if (x->n % 256 == 0)
    k_lse_rows<true><<<rows_grid(x->n, kLseRowThreads), kLseRowThreads, 0, x->stream>>>(a);
  else
    k_lse_rows<false><<<rows_grid(x->n, kLseRowThreads), kLseRowThreads, 0, x->stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_lse_cols(otn_ctx* x, const double* C, double ng, const double* outer,
                            const double* outer_d, const double* inner, const double* inner_d,
                            double alpha, int mode, double* out, const int* gate) {
  LseArgs a{C, x->n, x->ld, ng, outer, outer_d, inner, inner_d, alpha, mode, out, gate};
  const int slabs = x->lse_slabs;
  const int64_t slab_rows = (x->n + slabs - 1) / slabs;
  dim3 grid(unsigned((x->ld + kColTile - 1) / kColTile), unsigned(slabs));
  k_lse_cols_part<<<grid, kLseThreads, 0, x->stream>>>(a, slab_rows, x->lse_part);
  k_lse_cols_fin<<<unsigned((x->n + 255) / 256), 256, 0, x->stream>>>(a, slabs, x->lse_part);
  return cudaGetLastError();
}

cudaError_t launch_materialize(otn_ctx* x, const double* C, double ng, const double* u,
                               const double* v, double* P, const double* icP, const double* rP,
                               double* mu, int* flag, uint64_t* mask) {
  const unsigned grid = rows_grid(x->n, kMatThreads);
  if (x->n == x->ld && x->n % 256 == 0)
    k_materialize<true><<<grid, kMatThreads, 0, x->stream>>>(C, x->n, x->ld, ng, u, v, P, icP, rP,
                                                             mu, flag, mask);
  else
    k_materialize<false><<<grid, kMatThreads, 0, x->stream>>>(C, x->n, x->ld, ng, u, v, P, icP, rP,
                                                              mu, flag, mask);
  return cudaGetLastError();
}

cudaError_t launch_plan_mask(otn_ctx* x, const double* P, uint64_t* mask) {
  k_plan_mask<<<rows_grid(x->n), kLseThreads, 0, x->stream>>>(P, x->n, x->ld, mask);
  return cudaGetLastError();
}

cudaError_t launch_sys_prep(otn_ctx* x, const double* lr, const double* lc, double* rP,
                            double* cP, double* icP, int* flag) {
  k_sys_prep<<<unsigned((x->n + 255) / 256), 256, 0, x->stream>>>(x->n, lr, lc, rP, cP, icP, flag);
  return cudaGetLastError();
}

cudaError_t launch_square_matvec(otn_ctx* x, const double* P, const double* w, double* out) {
  k_square_matvec<<<rows_grid(x->n), kLseThreads, 0, x->stream>>>(P, x->n, x->ld, w, out);
  return cudaGetLastError();
}

}  // namespace otn
