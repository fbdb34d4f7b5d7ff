// Device-resident truncated-Newton direction solver (K6 + K7 + K8 and the
// CG / rho-annealing loops of newton.py:123-210) as ONE persistent
// cooperative kernel: one 512-thread CTA per SM, grid-wide barriers between
// the dependent phases, no host round trip until the direction is done.
//
// Data layout: CTA b owns the contiguous row block [r0, r1) of the plan P
// (k_partition picks the blocks and the plan mode, below).  A Hessian-vector
// product  q = rP*x - rho * P((P^T x)/cP)  is
//   phase A   per-CTA column partials  wpart[b][j] = sum_{i in block} P_ij x_i
//   -- grid barrier --
//   phase A2  column slices: w_j = sum_b wpart[b][j] (fixed order); wc = w/cP
//   -- grid barrier --
//   phase B   own rows: s_i = sum_j P_ij wc_j, then q_i = rP_i x_i - rho s_i.
// Phases A / B stream the plan (dense plans: cp.async rings over per-CTA
// column windows) or walk compressed rows (sparse plans: CSR + local CSC in
// shared or global memory).  Inside the CG loop the barriers are merged with
// the CG-scalar reductions (pcg): 2 grid barriers per CG iteration.
// CG state lives in registers (one row per thread); dot products / L1 norms
// are grid reductions with fixed trees (deterministic, no FP64 atomics).
#include <cooperative_groups.h>
#include <type_traits>

#include "otn_common.cuh"
#include "otn_internal.h"

namespace cg = cooperative_groups;

namespace otn {

constexpr int NT = kCoopThreads;
constexpr int NW = NT / 32;         // warps per CTA
constexpr int CH = 4;               // 16-byte chunks per thread per tile
constexpr int TILE = NT * 2 * CH;   // 4096 columns
constexpr int kRows = 64;           // rows staged per chunk in phases A / B
constexpr int kRefresh = 50;        // newton.py:38 TRUE_RESIDUAL_REFRESH

struct Smem {
  double red[4][33];
  double gres[4];
  double a2[NW][33];
  double xs[NT];                    // phase A input: x of the CTA's rows (row - r0)
  double sv[NT];                    // phase B output: (P w) of the CTA's rows
  double bp[NW][kRows];             // phase B: per-warp partial row dots
};

__device__ __forceinline__ double2 ldcg2(const double* p) {
  return __ldcg(reinterpret_cast<const double2*>(p));
}

// Grid-wide barrier and deterministic sum of K values in one exchange.
//
// Every CTA reduces value k with warp k (fixed warp / block trees) and stores
// the CTA total into its slot of row k; thread 0 then arrives on the
// context's arrival counter (release) and spins until the counter reaches
// e * G for this exchange's epoch e (acquire); warp k reads the G totals of
// row k and sums them in a fixed order.  The counter and the epoch only ever
// increase (the last epoch is carried to the next launch, a.gs_epoch), so
// the counter is never reset; two slot sets alternate, so a fast CTA's next
// store never lands on a slot a slow CTA is still reading.  K = 0: barrier
// only.  Measured (tools/gsync_bench.cu, 148 x 512 threads): 2.06 us per
// 2-value exchange vs 3.61 us for cooperative groups' grid.sync() followed by
// the same loads (the bare barriers cost the same, 1.3 us).
// Summation order: lane l holds CTAs 64 m + 2 l + {0, 1}; sum over m of the
// pair sums, then the warp butterfly.
// All M slot loads of a lane are issued before the first add (measured: -1.3
// ms per D2 solve against load-add pairs).
__shared__ uint32_t s_ep;                           // last completed exchange (written by thread 0)

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// the arrival counter sits one 128-byte line after the epoch word
__device__ __forceinline__ uint32_t* gs_counter(const CoopArgs& a) { return a.gs_epoch + 32; }

template <int K>
__device__ __forceinline__ void gs_exchange(const CoopArgs& a, double* v, Smem& sh) {
  constexpr int M = kRedStride / 64;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = gridDim.x;
  const uint32_t e = s_ep + 1u;
  double* row = a.red + (size_t(e & 1u) * kRedWidth + warp) * kRedStride;
  if (K > 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < K; ++k) sh.red[k][warp] = v[k];
    }
    __syncthreads();
    if (warp < K) {
      const double t = warp_sum(lane < NW ? sh.red[warp][lane] : 0.0);
      if (lane == 0) __stcg(row + blockIdx.x, t);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t* cnt = gs_counter(a);
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
    const uint32_t target = e * uint32_t(G);
    while (int32_t(ld_acquire_u32(cnt) - target) < 0) {
    }
    s_ep = e;                                       // read again only after the next barrier
  }
  __syncthreads();
  if (K > 0) {
    double2 pr[M];
    if (warp < K) {
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int b = 64 * m + 2 * lane;
        pr[m] = b < G ? ldcg2(row + b) : make_double2(0.0, 0.0);
      }
    }
    if (warp < K) {
      double s = 0.0;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int b = 64 * m + 2 * lane;
        if (b + 1 == G) pr[m].y = 0.0;              // odd G: the pair's second slot is not a CTA
        s += pr[m].x + pr[m].y;
      }
      s = warp_sum(s);
      if (lane == 0) sh.gres[warp] = s;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = sh.gres[k];
  }
}

template <int K>
__device__ __forceinline__ void grid_reduce(double (&v)[K], const CoopArgs& a, Smem& sh) {
  gs_exchange<K>(a, v, sh);
}

// Grid barrier (no values).
__device__ __forceinline__ void grid_bar(const CoopArgs& a, Smem& sh) {
  gs_exchange<0>(a, nullptr, sh);
}

// ---------------------------------------------------------------------------
// Plan streaming (dense plans): per-CTA column windows + cp.async rings.
//
// A work item is one row i of one 4096-column tile T of the plan; its span
// [lo, hi) runs from the first to the last nonzero 64-column segment
// (seg_mask: exp underflow makes most of the plan exactly 0 at weak
// regularization; for pixel-grid costs a row's nonzero segments are one
// contiguous run).  At kernel start each CTA stages the spans of its rows and
// their union per tile — its column WINDOW — in shared memory.  Within a tile
// thread t owns window columns {2t, 2t+1} + c*1024, so for a sparse-ish plan
// all threads work on the few nonzero columns instead of most of them idling.
// Chunks outside the span are exact zeros and are neither loaded nor used:
// the results equal the dense computation.  (Register-batched
// ld.global.cg was the faster path for L2-resident spans in isolation,
// tools/l2stream.cu, but lost to the ring inside the kernel once the sparse
// modes below took the late stages; it was retired.)
// ---------------------------------------------------------------------------
constexpr int kSpanSmem = 8192;                     // (row, tile) spans staged per CTA (32 KB)
constexpr int kMaxTiles = 64;                       // ld <= 262144
__shared__ int s_win_lo[kMaxTiles], s_win_hi[kMaxTiles];
// Plan mode of this launch (chosen by k_partition, uniform over the grid):
//   kPlanRing    plan streamed from HBM through per-thread cp.async rings;
//   kPlanL2      (retired: register-batched direct loads of L2-resident
//                spans; measured no faster than the ring once the sparse
//                modes took the late stages, and its code cost I-cache)
//   kPlanSparse  each CTA compresses its rows' nonzeros into shared memory
//                once per launch (CSR for P w, a local CSC for P^T x);
//   kPlanSparseG the same compressed rows in a per-CTA slice of global memory
//                (L2-resident) when they exceed shared memory; the CSC then
//                holds the values themselves (contiguous reads, no gather).
enum PlanMode { kPlanRing = 0, kPlanL2 = 1, kPlanSparse = 2, kPlanSparseG = 3 };
__shared__ int s_mode;
__shared__ int s_nzc;                               // kPlanSparse: nonempty columns of the CTA
__shared__ int s_split;                             // kPlanSparse: threads splitting the CSC entries
__shared__ int s_direct2;                           // kPlanSparse: this CTA stores its CSC values directly
__shared__ uint16_t s_m0[kCoopThreads];             // kPlanSparse: column of each thread's first entry
__shared__ int s_kb[kCoopThreads + 1];              // kPlanSparse: first CSC entry of each thread

// Everything the streaming loops need, by value (registers, not the kernel's
// parameter copy in local memory).
struct PlanView {
  const double* P;
  const uint64_t* mask;     // global mask rows (nullptr = dense)
  int64_t ld, mw;
  int nt;                   // tiles
  int mode;                 // PlanMode
  uint32_t span_off;        // byte offset of the staged spans (lo | hi << 16) in s_ring
  void* sg;                 // kPlanSparseG buffer
};

// Plans too large for L2 (kPlanRing: streamed from HBM) use a per-thread
// cp.async ring instead: kRingDepth rows of all CH chunks in flight, refilled
// continuously (the register batches drain between batches, which costs HBM
// bandwidth; on L2-resident spans the ring is the slower one).
constexpr int kRingDepth = 5;
extern __shared__ __align__(128) double2 s_ring[];  // dynamic: ring or sparse rows, then spans
constexpr size_t kRingBytes = size_t(kRingDepth) * CH * NT * 16;

// kPlanSparse shared-memory layout (dynamic region; see the sparse section).
constexpr int kSparseRows = 512;                    // rows per CTA
constexpr int kSparseCols = TILE;                   // one tile (ld <= 4096)
constexpr int kSparseCap = 10600;                   // nonzeros per CTA (fits 227 KB with the statics)
constexpr size_t kSparseXs = 0;                     // double[kSparseCols]: x rows (A) / w window (B)
constexpr size_t kSparseRp = kSparseXs + kSparseCols * 8;               // int[kSparseRows + 1]
constexpr size_t kSparseCst = kSparseRp + (kSparseRows + 4) * 4;        // int[kSparseCols + 1]
constexpr size_t kSparseVal = kSparseCst + (kSparseCols + 4) * 4;       // double[cap]
constexpr size_t kSparseCol = kSparseVal + size_t(kSparseCap) * 8;      // u16[cap]
constexpr size_t kSparsePerm = kSparseCol + size_t(kSparseCap) * 2;     // u32[cap]: CSC (entry | row << 16)
constexpr size_t kSparseBytes = kSparsePerm + size_t(kSparseCap) * 4;
// the CSC is stored thread-interleaved (see stage_sparse): up to NT - 1 slots
// past the entry count, so a CTA's nonzeros must leave that much room
constexpr int kSparseNnzMax = kSparseCap - kCoopThreads;

// The (row, tile) spans live in the dynamic region after what the mode uses.
__device__ __forceinline__ uint32_t span_offset(int mode) {
  return uint32_t(mode == kPlanRing ? kRingBytes
                  : mode == kPlanSparse ? kSparseBytes
                  : mode == kPlanSparseG ? kSparseVal : 0);
}

// Spans are indexed off the extern __shared__ array itself so the compiler
// emits shared-memory loads (a pointer carried in a struct would be generic).
__device__ __forceinline__ uint32_t* span_ptr(uint32_t off) {
  return reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(s_ring) + off);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ int ntiles_of(int64_t ld) { return int((ld + TILE - 1) / TILE); }

// Span of global row i in tile ti straight from the global mask.
__device__ __forceinline__ void mask_span(const PlanView& v, int64_t i, int ti, int& lo, int& hi) {
  const int64_t T = int64_t(ti) * TILE;
  const int width = int(v.ld - T < TILE ? v.ld - T : int64_t(TILE));
  if (!v.mask) { lo = 0; hi = width; return; }
  const uint64_t bits = __ldg(v.mask + i * v.mw + T / kSegWordCols);
  if (!bits) { lo = hi = 0; return; }
  lo = (__ffsll(static_cast<long long>(bits)) - 1) * kSegCols;
  hi = min((64 - __clzll(static_cast<long long>(bits))) * kSegCols, width);
}

// Span of row r0 + il (il = row index within the CTA) in tile ti.
__device__ __forceinline__ void get_span(const PlanView& v, int il, int ti, int& lo, int& hi) {
  const uint32_t s = span_ptr(v.span_off)[il * v.nt + ti];
  lo = int(s & 0xffffu);
  hi = int(s >> 16);
}

// col in [lo, hi) with one compare (lo <= hi): outside-span chunks and the
// chunks past the window end (col >= uhi >= hi) both fail it.
__device__ __forceinline__ bool in_span(int col, int lo, int hi) {
  return unsigned(col - lo) < unsigned(hi - lo);
}

__device__ PlanView plan_view(const CoopArgs& a, int64_t r0, int64_t r1) {
  PlanView v;
  v.P = a.P;
  v.mask = a.mask;
  v.ld = a.ld;
  v.mw = a.mw;
  v.nt = ntiles_of(a.ld);
  v.mode = s_mode;
  v.span_off = span_offset(v.mode);
  v.sg = a.sg;
  return v;
}

// Stage spans and windows; zero this CTA's column-partial row outside its
// windows (phase A writes only inside them, A2 reads the whole row).
__device__ void stage_layout(const CoopArgs& a, int64_t r0, int64_t r1, double* wrow) {
  const PlanView v = plan_view(a, r0, r1);
  const int t = threadIdx.x;
  const int64_t items = (r1 - r0) * v.nt;
  if (t < v.nt) { s_win_lo[t] = 1 << 30; s_win_hi[t] = 0; }
  __syncthreads();
  for (int64_t k = t; k < items; k += NT) {
    const int ti = int(k % v.nt);
    int lo, hi;
    mask_span(v, r0 + k / v.nt, ti, lo, hi);
    span_ptr(v.span_off)[k] = uint32_t(lo) | (uint32_t(hi) << 16);
    if (lo < hi) {
      atomicMin(&s_win_lo[ti], lo);
      atomicMax(&s_win_hi[ti], hi);
    }
  }
  __syncthreads();
  if (t < v.nt && s_win_lo[t] >= s_win_hi[t]) s_win_lo[t] = s_win_hi[t] = 0;
  __syncthreads();
  for (int64_t j = 2 * int64_t(t); j < a.ld; j += 2 * NT) {
    const int ti = int(j / TILE), rel = int(j - int64_t(ti) * TILE);
    if (rel < s_win_lo[ti] || rel >= s_win_hi[ti])
      *reinterpret_cast<double2*>(wrow + j) = make_double2(0.0, 0.0);
  }
  __syncthreads();
}

// Issue this thread's chunks of row il into the ring slot at smem byte
// address `dst`, then commit one group (possibly empty).
__device__ __forceinline__ void ring_fill(const PlanView& v, const double* src_row, int il, int ti,
                                          int col0, uint32_t dst) {
  int lo, hi;
  get_span(v, il, ti, lo, hi);
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int col = col0 + c * NT * 2;
    if (in_span(col, lo, hi)) cp_async16(dst + c * NT * 16, src_row + col);
  }
  cp_commit();
}

constexpr uint32_t kSlotBytes = CH * NT * 16;

// Phase A over one tile through the ring.
__device__ __forceinline__ void phase_a_ring(const PlanView& v, const double* fill_row, int c0,
                                             int m, int ti, int col0, double2 (&acc)[CH],
                                             const Smem& sh) {
  const uint32_t ring0 = smem_u32(s_ring) + 16u * threadIdx.x;
#pragma unroll
  for (int d = 0; d < kRingDepth - 1; ++d) {
    if (d < m) ring_fill(v, fill_row, c0 + d, ti, col0, ring0 + d * kSlotBytes);
    else cp_commit();
    fill_row += v.ld;
  }
  int slot = 0;
  uint32_t fdst = ring0 + (kRingDepth - 1) * kSlotBytes;
  for (int q = 0; q < m; ++q) {
    if (q + kRingDepth - 1 < m) ring_fill(v, fill_row, c0 + q + kRingDepth - 1, ti, col0, fdst);
    else cp_commit();
    fill_row += v.ld;
    fdst = fdst == ring0 + (kRingDepth - 1) * kSlotBytes ? ring0 : fdst + kSlotBytes;
    cp_wait<kRingDepth - 1>();
    int lo, hi;
    get_span(v, c0 + q, ti, lo, hi);
    const double xi = sh.xs[c0 + q];
    const double2* row = s_ring + slot * CH * NT + threadIdx.x;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (in_span(col0 + c * NT * 2, lo, hi)) {
        const double2 pv = row[c * NT];
        acc[c].x = fma(pv.x, xi, acc[c].x);
        acc[c].y = fma(pv.y, xi, acc[c].y);
      }
    }
    slot = slot + 1 == kRingDepth ? 0 : slot + 1;
  }
}

// ---------------------------------------------------------------------------
// kPlanSparse / kPlanSparseG: compressed rows.
//
// At weak regularization a row of the plan holds tens to hundreds of
// nonzeros (the rest underflow to exact 0), far fewer than its segment span.
// Each CTA then extracts its rows' nonzeros once per launch (warp per row,
// ballot compaction, column order) into a CSR — in the dynamic shared memory
// the ring would otherwise use, or in a per-CTA slice of global memory — plus
// a local CSC (rows ascending within a column, built by a counting sort and
// stored thread-interleaved: in shared memory as (CSR entry, row) pairs, in
// the global mode holding the values themselves).  Phase A splits
// the CSC entries evenly over the threads (sums per column in row order,
// column pieces joined left to right); phase B walks the CSR, warp per row.
// k_partition chooses these modes and a row partition balanced on nonzeros,
// and guarantees the capacities below.
// ---------------------------------------------------------------------------

struct SparseView {
  double* xs;
  int* rp;
  int* cst;
  double* val;                                      // CSR values (row-major, columns ascending)
  uint16_t* col;
  uint32_t* perm;                                   // mode 2: CSC slot -> CSR entry | row << 16
  double* cval;                                     // mode 3: CSC values
  uint16_t* crow;                                   // mode 3: CSC rows
  double* scval;                                    // CSC slots [0, gs) in shared memory
  uint16_t* scrow;
  int gs;                                           // slots held in shared memory
  bool direct;                                      // mode 3, or mode 2 with few nonzeros
};

// Mode 3 keeps the first kSparseGS slots of its (thread-interleaved) CSC in
// the shared memory mode 2 uses for its compressed rows -- every thread's
// first entries, read without an L2 round trip -- past the staged spans.
constexpr size_t kSparseGSmem = (kSparseVal + size_t(kSparseRows) * 4 + 15) / 16 * 16;
constexpr int kSparseGS = int((kSparseBytes + size_t(kSparseRows) * 4 - kSparseGSmem) / 10) / 8 * 8;

// Mode 2 with at most kSparseDCap nonzeros stores its CSC values and rows
// directly (like mode 3, all slots in shared memory: no CSR-entry indirection,
// contiguous reads in phase A), in the same region: CSR values + columns
// [kSparseDCap], then CSC values + rows [kSparseDCap + NT] (interleaving slack).
constexpr int kSparseDCap = int((kSparseCap * 14 - 10 * kCoopThreads) / 20);
constexpr size_t kSparseDCol = kSparseVal + size_t(kSparseDCap) * 8;
constexpr size_t kSparseDSv = kSparseDCol + size_t(kSparseDCap) * 2;
constexpr size_t kSparseDSr = kSparseDSv + size_t(kSparseDCap + kCoopThreads) * 8;
static_assert(kSparseDSr + size_t(kSparseDCap + kCoopThreads) * 2 <= kSparseBytes,
              "mode-2 direct CSC fits the compressed-rows region");

// Per-CTA slice of the global compressed-rows buffer (kPlanSparseG):
// val [cap] + cval [slot] doubles, then col [cap] + crow [slot] u16.
constexpr int kSparseGCap = 49152;                  // nonzeros per CTA (u16 CSC offsets)
constexpr int kSparseGSlot = kSparseGCap + kCoopThreads;   // interleaved CSC: + one row of padding
constexpr size_t kSparseGBytes = size_t(kSparseGCap) * (8 + 2) + size_t(kSparseGSlot) * (8 + 2);

__device__ __forceinline__ SparseView sparse_view(void* sg) {
  char* b = reinterpret_cast<char*>(s_ring);
  SparseView v;
  v.xs = reinterpret_cast<double*>(b + kSparseXs);
  v.rp = reinterpret_cast<int*>(b + kSparseRp);
  v.cst = reinterpret_cast<int*>(b + kSparseCst);
  if (s_mode == kPlanSparseG) {
    char* g = reinterpret_cast<char*>(sg) + size_t(blockIdx.x) * kSparseGBytes;
    v.val = reinterpret_cast<double*>(g);
    v.cval = v.val + kSparseGCap;
    v.col = reinterpret_cast<uint16_t*>(v.cval + kSparseGSlot);
    v.crow = v.col + kSparseGCap;
    v.perm = nullptr;
    v.scval = reinterpret_cast<double*>(b + kSparseGSmem);
    v.scrow = reinterpret_cast<uint16_t*>(b + kSparseGSmem + size_t(kSparseGS) * 8);
    v.gs = kSparseGS;
    v.direct = true;
  } else if (s_direct2) {
    v.val = reinterpret_cast<double*>(b + kSparseVal);
    v.col = reinterpret_cast<uint16_t*>(b + kSparseDCol);
    v.perm = nullptr;
    v.cval = nullptr;
    v.crow = nullptr;
    v.scval = reinterpret_cast<double*>(b + kSparseDSv);
    v.scrow = reinterpret_cast<uint16_t*>(b + kSparseDSr);
    v.gs = 1 << 30;
    v.direct = true;
  } else {
    v.val = reinterpret_cast<double*>(b + kSparseVal);
    v.col = reinterpret_cast<uint16_t*>(b + kSparseCol);
    v.perm = reinterpret_cast<uint32_t*>(b + kSparsePerm);
    v.cval = nullptr;
    v.crow = nullptr;
    v.scval = nullptr;
    v.scrow = nullptr;
    v.gs = 0;
    v.direct = false;
  }
  return v;
}

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// In-place inclusive prefix sum of a[0, len), len <= NT * 8 (one CTA).
__device__ void block_incl_scan(int* a, int len, Smem& sh) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int loc[8], sum = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = t * 8 + k;
    sum += i < len ? a[i] : 0;
    loc[k] = sum;
  }
  const int incl = warp_incl_scan(sum, lane);
  int* wsum = reinterpret_cast<int*>(sh.red);         // 16 ints (free outside grid_reduce)
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int off = incl - sum;
  for (int w = 0; w < warp; ++w) off += wsum[w];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = t * 8 + k;
    if (i < len) a[i] = loc[k] + off;
  }
  __syncthreads();
}

// Extract this CTA's nonzeros (CSR, column order) and build the local CSC.
__device__ void stage_sparse(const CoopArgs& a, int64_t r0, int64_t r1, double* wrow, Smem& sh) {
  if (threadIdx.x == 0) s_direct2 = 0;
  __syncthreads();
  SparseView sp = sparse_view(a.sg);
  const PlanView v = plan_view(a, r0, r1);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int rows = int(r1 - r0);
  if (warp == 0) {                                  // row pointers from the mask count words
    int run = 0;
    for (int b = 0; b < rows; b += 32) {
      const int r = b + lane;
      const int c = r < rows ? int(__ldg(v.mask + (r0 + r) * v.mw + v.mw - 1)) : 0;
      const int incl = warp_incl_scan(c, lane);
      if (r < rows) sp.rp[r + 1] = run + incl;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
      sp.rp[0] = 0;
      if (s_mode == kPlanSparse && run <= kSparseDCap) s_direct2 = 1;
    }
  }
  __syncthreads();
  sp = sparse_view(a.sg);                           // the layout s_direct2 selects
  const unsigned lt = (1u << lane) - 1u;
  constexpr int U = 8;                              // 64-column steps loaded at once
  for (int r = warp; r < rows; r += NW) {           // warp per row, columns ascending
    int lo, hi;
    get_span(v, r, 0, lo, hi);
    const double* prow = v.P + (r0 + r) * v.ld;
    int pos = sp.rp[r];
    const int end = sp.rp[r + 1];
    for (int j0 = lo; j0 < hi; j0 += 64 * U) {
      double2 pv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + 64 * u + 2 * lane;
        pv[u] = j < hi ? ldcg2(prow + j) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + 64 * u + 2 * lane;
        const bool nx = pv[u].x != 0.0, ny = pv[u].y != 0.0;
        const unsigned bx = __ballot_sync(0xffffffffu, nx), by = __ballot_sync(0xffffffffu, ny);
        int q = pos + __popc(bx & lt) + __popc(by & lt);
        if (nx) {
          if (q < end) { sp.val[q] = pv[u].x; sp.col[q] = uint16_t(j); }
          ++q;
        }
        if (ny && q < end) { sp.val[q] = pv[u].y; sp.col[q] = uint16_t(j + 1); }
        pos += __popc(bx) + __popc(by);
      }
    }
  }
  const int ulo = s_win_lo[0], W = s_win_hi[0] - ulo;
  for (int d = t; d <= W; d += NT) sp.cst[d] = 0;
  __syncthreads();
  const int E = sp.rp[rows];
  for (int e = t; e < E; e += NT) atomicAdd(&sp.cst[sp.col[e] - ulo], 1);
  __syncthreads();
  block_incl_scan(sp.cst, W, sh);                   // cst[d] = end of column d
  // phase A splits the CSC entries over `split` threads, >= 8 entries each
  // (fewer, longer pieces: a column cut in many pieces is summed serially);
  // thread t takes entries [s_kb[t], s_kb[t+1])
  {
    const int split = E / 8 < 1 ? 1 : (E / 8 < NT ? E / 8 : NT);
    if (t == 0) s_split = split;
    s_kb[t] = t < split ? int((int64_t(t) * E) / split) : E;
    if (t == 0) s_kb[NT] = E;
    __syncthreads();
  }
  {
    // CSC placement: rows descending, each row's (distinct) columns in
    // parallel, cst[] as a decrementing cursor -> rows ascending within every
    // column, deterministically.  Stored thread-interleaved: entry k of
    // thread t's range at (k - s_kb[t]) * split + t, so phase A's loads are
    // consecutive across a warp.  Mode 3 stores the values themselves (global
    // memory), mode 2 the CSR entry and its row (shared memory).
    const int split = s_split;
    for (int r = rows - 1; r >= 0; --r) {
      for (int e = sp.rp[r] + t; e < sp.rp[r + 1]; e += NT) {
        const int k = --sp.cst[sp.col[e] - ulo];
        int o = int((int64_t(k) * split) / E);
        while (o + 1 < split && s_kb[o + 1] <= k) ++o;
        while (s_kb[o] > k) --o;
        const int addr = (k - s_kb[o]) * split + o;
        if (sp.direct) {
          if (addr < sp.gs) {
            sp.scval[addr] = sp.val[e];
            sp.scrow[addr] = uint16_t(r);
          } else {
            sp.cval[addr] = sp.val[e];
            sp.crow[addr] = uint16_t(r);
          }
        } else {
          sp.perm[addr] = uint32_t(e) | (uint32_t(r) << 16);
        }
      }
      __syncthreads();
    }
    if (t == 0) sp.cst[W] = E;                      // cst[d] = start of column d
    __syncthreads();
  }
  // Compact the nonempty columns in place of cst: cptr[m] (u16 start of the
  // m-th nonempty column, cptr[nzc] = E) and ccol[m] (its window column).
  int st[9], nonempty = 0;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const int d = t * 8 + k;
    st[k] = d < W ? sp.cst[d] : E;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) nonempty += st[k + 1] > st[k];
  const int incl = warp_incl_scan(nonempty, lane);
  int* wsum = reinterpret_cast<int*>(sh.red);
  __syncthreads();                                  // all cst reads done
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int m = incl - nonempty;
  for (int w = 0; w < warp; ++w) m += wsum[w];
  uint16_t* cptr = reinterpret_cast<uint16_t*>(sp.cst);
  uint16_t* ccol = cptr + (kSparseCols + 2);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int d = t * 8 + k;
    if (d < W && st[k + 1] > st[k]) { cptr[m] = uint16_t(st[k]); ccol[m] = uint16_t(d); ++m; }
    else if (d < W) wrow[ulo + d] = 0.0;            // empty column: phase A never writes it
  }
  if (t == NT - 1) s_nzc = m;                       // last thread holds the total
  __syncthreads();
  if (t == 0) cptr[s_nzc] = uint16_t(E);
  // thread t's first CSC entry (s_kb) -> its first column (s_m0)
  const int split = s_split;
  if (t < split) {
    const int kb = int((int64_t(t) * E) / split);
    int lo = 0, hi = s_nzc;                         // cptr[lo] <= kb < cptr[lo + 1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (cptr[mid] <= kb) lo = mid; else hi = mid;
    }
    s_m0[t] = uint16_t(lo);
  }
  __syncthreads();
}

// Phase A (sparse): w_j = sum over own rows of P_ij x_i.  The CSC entries are
// split evenly over the threads (a few columns hold most entries of a CTA, so
// a thread per column would serialize on them); each thread sums its entries
// column by column (rows ascending); a column cut by thread boundaries is the
// left-to-right sum of its pieces, finished by the thread holding its start.
// Deterministic: the split depends only on the entry count.
__device__ void phase_a_sparse(void* sg, int64_t r0, int64_t r1, double* wrow, Smem& sh) {
  const SparseView sp = sparse_view(sg);
  const int t = threadIdx.x;
  const uint16_t* cptr = reinterpret_cast<const uint16_t*>(sp.cst);
  const uint16_t* ccol = cptr + (kSparseCols + 2);
  double* head = &sh.bp[0][0];                      // per-thread piece of a column begun earlier
  const double* xs = sh.xs;
  const int ulo = s_win_lo[0];
  // (no initialization of head: every head[u] the joins below read is written
  // in this call — a thread whose range starts inside a column always ends
  // with `begun` set or closes that column; the caller's stage_x barrier
  // orders this call after the previous readers)
  const int kb = s_kb[t], ke = s_kb[t + 1];
  double tail = 0.0;
  int tail_m = -1;
  if (kb < ke) {
    // entries are loaded 8 at a time regardless of column boundaries (columns
    // are short: a load per column would expose the full L2 / shared-memory
    // latency), then consumed in order with the column bookkeeping in registers
    // the current column's end and window column are kept in registers, the
    // next ones loaded as soon as a column closes (the store never waits)
    int m = s_m0[t], mend = cptr[m + 1], mcol = ccol[m];
    bool begun = cptr[m] < kb;                      // column started in an earlier thread
    double acc = 0.0;
    const int S = s_split;
    // entries [k0, min(k0 + 8, kend)); mode 3 reads its shared-memory slots
    // (SMEM) and its global ones in separate loops (no per-entry choice)
    auto batch = [&](int k0, int kend, auto smem_tag) {
      constexpr bool SMEM = decltype(smem_tag)::value;
      double pv[8], xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = k0 + u;
        pv[u] = 0.0;
        xv[u] = 0.0;
        if (k < kend) {
          const int ad = (k - kb) * S + t;
          if (SMEM) {
            pv[u] = sp.scval[ad];
            xv[u] = xs[sp.scrow[ad]];
          } else if (sp.direct) {
            pv[u] = sp.cval[ad];
            xv[u] = xs[sp.crow[ad]];
          } else {
            const uint32_t pe = sp.perm[ad];
            pv[u] = sp.val[pe & 0xffffu];
            xv[u] = xs[pe >> 16];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = k0 + u;
        if (k >= kend) break;
        if (k == mend) {                            // column m ended inside this thread
          if (begun) head[t] = acc;
          else wrow[ulo + mcol] = acc;
          begun = false;
          acc = 0.0;
          ++m;
          mend = cptr[m + 1];
          mcol = ccol[m];
        }
        acc = fma(pv[u], xv[u], acc);
      }
    };
    int k0 = kb;
    if (sp.direct) {
      // this thread's slots (k - kb) * S + t below sp.gs sit in shared memory
      const int ks = t < sp.gs ? min(ke, kb + (sp.gs - 1 - t) / S + 1) : kb;
      for (; k0 < ks; k0 += 8) batch(k0, ks, std::true_type{});
      k0 = ks;
    }
    for (; k0 < ke; k0 += 8) batch(k0, ke, std::false_type{});
    if (begun) head[t] = acc;                       // piece of a column begun earlier
    else if (mend <= ke) wrow[ulo + mcol] = acc;    // whole column inside this thread
    else { tail = acc; tail_m = m; }                // column continues in later threads
  }
  __syncthreads();
  if (tail_m >= 0) {
    const int cend = cptr[tail_m + 1];
    double s = tail;
    for (int u = t + 1; s_kb[u] < cend; ++u) s += head[u];   // s_kb[split..NT] = E
    wrow[ulo + ccol[tail_m]] = s;
  }
}

// Phase B (sparse): s_i = sum_j P_ij w_j.  The CTA's window of w is staged in
// shared memory first (one coalesced read); then warp per row, lanes strided
// over the row's entries, a fixed-tree warp sum.
__device__ void phase_b_sparse(void* sg, const double* w, int64_t r0, int64_t r1,
                               double* sv) {   // sv: sh.sv
  const SparseView sp = sparse_view(sg);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, rows = int(r1 - r0);
  const int ulo = s_win_lo[0], W = s_win_hi[0] - ulo;
  double* ws = sp.xs - ulo;                         // ws[j] for window columns j
  __syncthreads();
  {
    // all of this thread's window loads in flight at once (W <= TILE = 8 NT)
    double wv[TILE / NT];
#pragma unroll
    for (int u = 0; u < TILE / NT; ++u) {
      const int d = t + u * NT;
      wv[u] = d < W ? __ldcg(w + ulo + d) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < TILE / NT; ++u) {
      const int d = t + u * NT;
      if (d < W) sp.xs[d] = wv[u];
    }
  }
  __syncthreads();
  for (int r = warp; r < rows; r += NW) {
    double dot = 0.0;
    const int e1 = sp.rp[r + 1];
    int e = sp.rp[r] + lane;
    for (; e + 224 < e1; e += 256) {                // eight loads in flight (global mode)
      double pv[8], wv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) { pv[u] = sp.val[e + 32 * u]; wv[u] = ws[sp.col[e + 32 * u]]; }
#pragma unroll
      for (int u = 0; u < 8; ++u) dot = fma(pv[u], wv[u], dot);
    }
    for (; e + 96 < e1; e += 128) {
      double pv[4], wv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { pv[u] = sp.val[e + 32 * u]; wv[u] = ws[sp.col[e + 32 * u]]; }
#pragma unroll
      for (int u = 0; u < 4; ++u) dot = fma(pv[u], wv[u], dot);
    }
    for (; e < e1; e += 32) dot = fma(sp.val[e], ws[sp.col[e]], dot);
    dot = warp_sum(dot);
    if (lane == 0) sv[r] = dot;
  }
  __syncthreads();
}

// Phase A: column partials of P^T x over this CTA's rows (ascending).
// Input: sh.xs[row - r0] (filled by the caller, followed by a barrier).
__device__ __noinline__ void phase_a(const PlanView v, int64_t r0, int64_t r1, double* wrow,
                                     Smem& sh) {
  if (v.mode >= kPlanSparse) {
    phase_a_sparse(v.sg, r0, r1, wrow, sh);
    return;
  }
  const int t = threadIdx.x;
  const int rows = int(r1 - r0);
  for (int ti = 0; ti < v.nt; ++ti) {
    const int64_t T = int64_t(ti) * TILE;
    const int ulo = s_win_lo[ti], W = s_win_hi[ti] - ulo;
    if (W <= 0) continue;
    const int col0 = ulo + 2 * t;
    double2 acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = make_double2(0.0, 0.0);
    for (int c0 = 0; c0 < rows; c0 += kRows) {
      const int m = min(rows - c0, kRows);
      const double* row0 = v.P + (r0 + c0) * v.ld + T;
      phase_a_ring(v, row0, c0, m, ti, col0, acc, sh);
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int rel = c * NT * 2 + 2 * t;
      if (rel < W) *reinterpret_cast<double2*>(wrow + T + ulo + rel) = acc[c];
    }
  }
}

// Phase A2: reduce the per-CTA partials for 32-column slices.
//   kind 0: out = w / cP     (the HVP's inner vector, and apply_pc)
//   kind 1: out = -(w / cP)  (d_v, projector.py:201)
//   kind 2: out = w          (rmatvec)
//   wprev / wkeep (CG pipelining, pcg below): w = sum_b wpart[b] + beta * wprev
//   before the kind is applied, and w is kept in wkeep (may alias wprev).
// Returns this thread's share of sum_j w_j * out_j over its columns (warp 0
// lanes; 0 elsewhere) -- for kind 0 that is sum_j w_j^2 / cP_j = p^T P (P^T p / cP),
// the matvec part of p.q (see pcg).
__device__ __noinline__ double phase_a2(const CoopArgs& a, int kind, double* out, Smem& sh,
                                        const double* wprev = nullptr, double beta = 0.0,
                                        double* wkeep = nullptr) {
  double wq = 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = gridDim.x;
  for (int64_t s = blockIdx.x; s * 32 < a.ld; s += G) {
    const int64_t j = s * 32 + lane;
    double acc = 0.0;
    // issue all of this warp's partial loads before summing (latency-bound otherwise)
    for (int b0 = warp; b0 < G; b0 += NW * 16) {
      double v[16];
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const int bp = b0 + m * NW;
        v[m] = bp < G ? __ldcg(a.wpart + int64_t(bp) * a.ld + j) : 0.0;
      }
#pragma unroll
      for (int m = 0; m < 16; ++m) acc += v[m];
    }
    sh.a2[warp][lane] = acc;
    __syncthreads();
    if (warp == 0) {
      double tot = 0.0;
#pragma unroll 8
      for (int w = 0; w < NW; ++w) tot += sh.a2[w][lane];
      if (wprev) tot = __dadd_rn(tot, __dmul_rn(beta, __ldcg(wprev + j)));
      if (wkeep) wkeep[j] = tot;
      double val = 0.0;
      if (j < a.n) {
        val = kind == 2 ? tot : __ddiv_rn(tot, __ldg(a.cP + j));
        if (kind == 1) val = -val;
        wq = fma(tot, val, wq);
      }
      out[j] = val;
    }
    __syncthreads();
  }
  return wq;
}

// Phase A2 split for the CG pipeline (used when every CTA owns at most one
// 32-column slice, ld <= 32 G): a2_sums loads and sums the partials of the
// CTA's slice per warp (no scalar needed yet); a2_tail (warp 0) finishes
// the slice once beta is known.  Same arithmetic as phase_a2.
__device__ __forceinline__ bool a2_single_slice(const CoopArgs& a) {
  return a.ld <= int64_t(32) * gridDim.x;
}

__device__ __forceinline__ void a2_sums(const CoopArgs& a, Smem& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = gridDim.x;
  const int64_t s = blockIdx.x;
  if (s * 32 >= a.ld) return;
  const int64_t j = s * 32 + lane;
  double acc = 0.0;
  // 10 loads per batch (one batch for up to 160 CTAs; the padding zeros end in
  // the +0.0 the slice total starts from, as phase_a2's 16 do)
  for (int b0 = warp; b0 < G; b0 += NW * 10) {
    double v[10];
#pragma unroll
    for (int m = 0; m < 10; ++m) {
      const int bp = b0 + m * NW;
      v[m] = bp < G ? __ldcg(a.wpart + int64_t(bp) * a.ld + j) : 0.0;
    }
#pragma unroll
    for (int m = 0; m < 10; ++m) acc += v[m];
  }
  sh.a2[warp][lane] = acc;
}

// After a2_sums and a barrier: out_j = w_j / cP_j with w = sum + beta * wreg,
// for warp 0's lanes (column j = 32 * blockIdx.x + lane).  wreg holds the
// previous w_j in a register (the same thread formed it last iteration) and
// receives the new one, which is also kept in a.q; cPj is 1/cP's divisor,
// loaded once per launch.  Returns w_j * out_j.  Same arithmetic as phase_a2.
__device__ __forceinline__ double a2_tail(const CoopArgs& a, double* out, Smem& sh, double beta,
                                          double& wreg, double cPj) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t s = blockIdx.x;
  double wq = 0.0;
  if (warp == 0 && s * 32 < a.ld) {
    const int64_t j = s * 32 + lane;
    double tot = 0.0;
#pragma unroll 8
    for (int w = 0; w < NW; ++w) tot += sh.a2[w][lane];
    tot = __dadd_rn(tot, __dmul_rn(beta, wreg));
    a.q[j] = tot;
    wreg = tot;
    double val = 0.0;
    if (j < a.n) {
      val = __ddiv_rn(tot, cPj);
      wq = fma(tot, val, wq);
    }
    out[j] = val;
  }
  return wq;
}

// Sum eight per-lane values over the warp with a transpose-reduction (fixed
// butterfly, 9 shuffles instead of 8 x 5): on return lane l holds the total of
// value ((l>>4)&1)*4 + ((l>>3)&1)*2 + ((l>>2)&1).
__device__ __forceinline__ double warp_reduce8(const double (&d)[8], int lane) {
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
  double w4[4], w2[2];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double keep = h16 ? d[k + 4] : d[k], give = h16 ? d[k] : d[k + 4];
    w4[k] = keep + __shfl_xor_sync(0xffffffffu, give, 16);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double keep = h8 ? w4[k + 2] : w4[k], give = h8 ? w4[k] : w4[k + 2];
    w2[k] = keep + __shfl_xor_sync(0xffffffffu, give, 8);
  }
  const double keep = h4 ? w2[1] : w2[0], give = h4 ? w2[0] : w2[1];
  double s = keep + __shfl_xor_sync(0xffffffffu, give, 4);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  return s;
}

// Phase B over one tile through the ring, rows descending: per-lane dots of 8
// rows, one transpose-reduction, per-warp partials in sh.bp[warp][row - c0].
__device__ __forceinline__ void phase_b_ring(const PlanView& v, const double* fill_row, int e,
                                             int m, int c0, int ti, int col0,
                                             const double2 (&wv)[CH], Smem& sh) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int row_of_lane = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
  const uint32_t ring0 = smem_u32(s_ring) + 16u * t;
#pragma unroll
  for (int d = 0; d < kRingDepth - 1; ++d) {
    if (d < m) ring_fill(v, fill_row, e - 1 - d, ti, col0, ring0 + d * kSlotBytes);
    else cp_commit();
    fill_row -= v.ld;
  }
  int slot = 0;
  uint32_t fdst = ring0 + (kRingDepth - 1) * kSlotBytes;
  double d8[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) d8[k] = 0.0;
  for (int q = 0; q < m; ++q) {
    if (q + kRingDepth - 1 < m) ring_fill(v, fill_row, e - kRingDepth - q, ti, col0, fdst);
    else cp_commit();
    fill_row -= v.ld;
    fdst = fdst == ring0 + (kRingDepth - 1) * kSlotBytes ? ring0 : fdst + kSlotBytes;
    cp_wait<kRingDepth - 1>();
    int lo, hi;
    get_span(v, e - 1 - q, ti, lo, hi);
    const double2* row = s_ring + slot * CH * NT + t;
    double dot = 0.0;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (in_span(col0 + c * NT * 2, lo, hi)) {
        const double2 pv = row[c * NT];
        dot = fma(pv.x, wv[c].x, dot);
        dot = fma(pv.y, wv[c].y, dot);
      }
    }
    const int b = q & 7;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k == b) d8[k] = dot;
    if (b == 7 || q == m - 1) {
      const double s = warp_reduce8(d8, lane);
      if ((lane & 3) == 0 && row_of_lane <= b) sh.bp[warp][e - 1 - (q - b + row_of_lane) - c0] += s;
#pragma unroll
      for (int k = 0; k < 8; ++k) d8[k] = 0.0;
    }
    slot = slot + 1 == kRingDepth ? 0 : slot + 1;
  }
}

// Phase B: s_i = sum_j P_ij w_j for own rows (DESCENDING: the rows phase A
// streamed last are the likeliest L2 hits), into sv[i].  Per-warp partials
// accumulate in shared memory; one fixed-order sum over warps per chunk.
// Output: sh.sv[row - r0] (complete after the closing barrier).
__device__ __noinline__ void phase_b(const PlanView v, const double* w, int64_t r0, int64_t r1,
                                     Smem& sh) {
  if (v.mode >= kPlanSparse) {
    phase_b_sparse(v.sg, w, r0, r1, sh.sv);
    return;
  }
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int rows = int(r1 - r0);
  for (int e = rows; e > 0; e -= kRows) {          // chunk [e - m, e) of CTA rows
    const int m = min(e, kRows), c0 = e - m;
    for (int k = lane; k < m; k += 32) sh.bp[warp][k] = 0.0;
    __syncwarp();
    for (int ti = 0; ti < v.nt; ++ti) {
      const int64_t T = int64_t(ti) * TILE;
      const int ulo = s_win_lo[ti], W = s_win_hi[ti] - ulo;
      if (W <= 0) continue;
      const int col0 = ulo + 2 * t;
      double2 wv[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int rel = c * NT * 2 + 2 * t;
        wv[c] = rel < W ? ldcg2(w + T + ulo + rel) : make_double2(0.0, 0.0);
      }
      const double* row_top = v.P + (r0 + e - 1) * v.ld + T;
      phase_b_ring(v, row_top, e, m, c0, ti, col0, wv, sh);
    }
    __syncthreads();
    if (t < m) {
      double tot = 0.0;
#pragma unroll
      for (int ww = 0; ww < NW; ++ww) tot += sh.bp[ww][t];
      sh.sv[c0 + t] = tot;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// CG state in registers.  Every CTA owns at most NT rows (k_partition and
// launch_coop guarantee it), so thread t holds row r0 + t of every CG vector
// (x, r, z, p, q, the Jacobi diagonal) in registers for the whole launch; only
// the plan phases exchange data, through sh.xs / sh.sv and the column
// workspace.  Threads without a row hold zeros (and M = 1): they add nothing
// to any reduction.
// ---------------------------------------------------------------------------
struct Row {
  bool own;
  int64_t i;                                        // global row (valid when own)
};

// A^T x partials of the CTA rows for x held one value per thread.
__device__ __forceinline__ void stage_x(double xv, Smem& sh) {
  __syncthreads();                                  // previous readers of sh.xs are done
  sh.xs[threadIdx.x] = xv;
  __syncthreads();
}

// q = F(rho) x for the thread's row (newton.py:100-105; matvecs skipped when
// rho == 0): q = rP x - rho * P((P^T x) / cP).
__device__ double hvp(cg::grid_group& grid, const CoopArgs& a, double xv, double rho, double rPi,
                      int64_t r0, int64_t r1, Smem& sh, int64_t& nh) {
  double o = __dmul_rn(rPi, xv);
  if (rho != 0.0) {
    ++nh;
    stage_x(xv, sh);
    phase_a(plan_view(a, r0, r1), r0, r1, a.wpart + int64_t(blockIdx.x) * a.ld, sh);
    grid_bar(a, sh);
    phase_a2(a, 0, a.wc, sh);
    grid_bar(a, sh);
    phase_b(plan_view(a, r0, r1), a.wc, r0, r1, sh);   // ends with a barrier
    if (int64_t(threadIdx.x) < r1 - r0) o = __dsub_rn(o, __dmul_rn(rho, sh.sv[threadIdx.x]));
    else o = 0.0;                                   // no row: sh.sv is not written there
  }
  return o;
}

struct PcgOut {
  int status;
  int64_t iters;
  double resid;
};

// Jacobi-PCG, newton.py:123-172, on register rows.  b == nullptr means b = -g.
// x: in (if has_x0) / out.
//
// Pipelined matvec: the phase-A partials of the next direction are formed
// from z BEFORE the r.z reduction, and phase A2 combines them as
// P^T p_new = P^T z + beta * P^T p (the previous direction's column sums are
// kept in a.q, and for the single-slice split in a register of warp 0), so
// the r.z barrier doubles as the HVP's partials barrier; p.q is reduced with
// the A2 -> phase B barrier (see the loop): 2 grid barriers per CG iteration
// instead of 4, both reductions split around independent work.  The CG
// recurrences (x, r, z, p, alpha, beta and the stopping tests) are the
// reference's, operation for operation; only the column sums of P^T p and
// the matvec part of p.q are formed by linearity.
__device__ PcgOut pcg(cg::grid_group& grid, const CoopArgs& a, const Row& row, double rPi, double rho,
                      const double* bvec, double tol, double& x, bool has_x0, int64_t max_iters,
                      int64_t r0, int64_t r1, Smem& sh, int64_t& nh) {
  PcgOut o{OTN_OK, 0, 0.0};
  const bool mv = rho != 0.0;                       // F(0) = diag(rP): no plan passes
  double q = 0.0;
  if (has_x0) q = hvp(grid, a, x, rho, rPi, r0, r1, sh, nh);
  double M = 1.0, bi = 0.0, r = 0.0, z = 0.0, p = 0.0;
  double loc[3] = {0.0, 0.0, 0.0};
  if (row.own) {
    M = __dmul_rn(rPi, __dsub_rn(1.0, __dmul_rn(rho, __ldg(a.mu + row.i))));
    bi = bvec ? __ldg(bvec + row.i) : -__ldg(a.g + row.i);
    if (has_x0) {
      r = __dsub_rn(bi, q);
    } else {
      x = 0.0;
      r = bi;
    }
    z = __ddiv_rn(r, M);
    p = z;
    loc[0] = fabs(r);
    loc[1] = fma(r, z, 0.0);
    if (M <= 0.0) loc[2] = 1.0;
  } else {
    x = 0.0;
  }
  double* wrow = a.wpart + int64_t(blockIdx.x) * a.ld;
  if (mv) {                                         // partials of the first direction p = z
    stage_x(p, sh);
    phase_a(plan_view(a, r0, r1), r0, r1, wrow, sh);
  }
  grid_reduce<3>(loc, a, sh);
  if (loc[2] > 0.0) { o.status = OTN_ST_PRECOND; return o; }
  if (loc[0] <= tol) { o.resid = loc[0]; return o; }
  double rz = loc[1];
  double norm = loc[0];
  double beta = 0.0;
  bool fresh = true;                                // no previous direction yet
  const bool split = mv && a2_single_slice(a);      // overlap the r.z reduction with A2's loads
  // split A2: warp 0's lanes own column slice_j of P^T p; its previous value
  // and cP stay in registers
  const int64_t slice_j = int64_t(blockIdx.x) * 32 + (threadIdx.x & 31);
  const bool slice_lane = (threadIdx.x >> 5) == 0 && slice_j < a.ld;
  double wreg = 0.0;
  const double cPj = split && slice_lane && slice_j < a.n ? __ldg(a.cP + slice_j) : 1.0;
  bool pending = false;                             // an r.z reduction begun, not finished
  double nz[2] = {0.0, 0.0};
  for (int64_t k = 1; k <= max_iters; ++k) {
    // p.q = sum_i rP_i p_i^2 - rho * sum_j w_j (w_j / cP_j), w = P^T p: both
    // sums are known once A2 has run, so their reduction IS the barrier
    // between A2 and phase B (one barrier fewer than p.q after phase B).
    double wq = 0.0;
    if (pending) {
      // the previous iteration's r.z exchange is complete (nz holds the sums)
      a2_sums(a, sh);
      __syncthreads();                              // publishes sh.a2
      pending = false;
      norm = nz[0];
      if (norm <= tol) { o.iters = k - 1; o.resid = norm; return o; }
      beta = nz[1] / rz;
      p = __dadd_rn(z, __dmul_rn(beta, p));
      rz = nz[1];
      ++nh;
      wq = a2_tail(a, a.wc, sh, beta, wreg, cPj);
    }
    q = __dmul_rn(rPi, p);
    double pq;
    if (mv) {
      if (!split || fresh) {
        ++nh;
        wq = phase_a2(a, 0, a.wc, sh, fresh ? nullptr : a.q, beta, a.q);
        if (split && slice_lane) wreg = __ldcg(a.q + slice_j);   // just written by this thread
      }
      double sums[2] = {fma(p, q, 0.0), wq};
      grid_reduce<2>(sums, a, sh);             // also publishes a.wc
      phase_b(plan_view(a, r0, r1), a.wc, r0, r1, sh);   // ends with a barrier
      pq = __dsub_rn(sums[0], __dmul_rn(rho, sums[1]));
      q = row.own ? __dsub_rn(q, __dmul_rn(rho, sh.sv[threadIdx.x])) : 0.0;
    } else {
      double pq1[1] = {fma(p, q, 0.0)};
      grid_reduce<1>(pq1, a, sh);
      pq = pq1[0];
    }
    fresh = false;
    if (pq <= 0.0) { o.status = OTN_ST_BREAKDOWN; o.iters = k; o.resid = pq; return o; }
    const double alpha = rz / pq;
    x = __dadd_rn(x, __dmul_rn(alpha, p));
    r = __dsub_rn(r, __dmul_rn(alpha, q));
    if (k % kRefresh == 0) {
      const double qx = hvp(grid, a, x, rho, rPi, r0, r1, sh, nh);
      r = __dsub_rn(bi, qx);
    }
    if (!row.own) r = 0.0;
    z = __ddiv_rn(r, M);
    // With the true residual (every kRefresh iterations) P^T p is re-anchored
    // too: the next direction's column sums are formed directly instead of by
    // the recurrence P^T z + beta P^T p, whose rounding drifts over long CG
    // runs (residual replacement; the partials of z are not needed then).
    const bool anchor = mv && k % kRefresh == 0;
    if (mv && !anchor) {                            // partials of z, read after the barrier
      stage_x(z, sh);
      phase_a(plan_view(a, r0, r1), r0, r1, wrow, sh);
    }
    nz[0] = fabs(r);
    nz[1] = fma(r, z, 0.0);
    if (split && !anchor) {
      grid_reduce<2>(nz, a, sh);
      pending = true;
      continue;                                     // finished at the top of the next iteration
    }
    grid_reduce<2>(nz, a, sh);
    norm = nz[0];
    if (norm <= tol) { o.iters = k; o.resid = norm; return o; }
    beta = nz[1] / rz;
    p = __dadd_rn(z, __dmul_rn(beta, p));
    rz = nz[1];
    if (anchor) {                                   // partials of p itself; A2 sums them directly
      stage_x(p, sh);
      phase_a(plan_view(a, r0, r1), r0, r1, wrow, sh);
      grid_bar(a, sh);
      fresh = true;
    }
  }
  if (pending) {                                    // the budget ran out on a begun reduction
    // (nz was completed by its exchange)
    norm = nz[0];
    if (norm <= tol) { o.iters = max_iters; o.resid = norm; return o; }
  }
  o.status = OTN_ST_NONCONVERGENCE;
  o.iters = max_iters;
  o.resid = norm;
  return o;
}

// Column pass of the CTA rows for x held one value per thread (phase A + A2).
__device__ void column_pass(cg::grid_group& grid, const CoopArgs& a, double xv, int kind,
                            double* out, int64_t r0, int64_t r1, Smem& sh) {
  stage_x(xv, sh);
  phase_a(plan_view(a, r0, r1), r0, r1, a.wpart + int64_t(blockIdx.x) * a.ld, sh);
  grid_bar(a, sh);
  phase_a2(a, kind, out, sh);
}

// The launch result; for otn_newton_step also its first gate (the direction
// is usable: status OK and slope > 0), which k_step_gate stage 0 would compute.
__device__ __forceinline__ void publish_result(const CoopArgs& a, const DevResult& res) {
  *a.res = res;
  if (a.step_flags) {
    a.step_flags[0] = res.status == OTN_OK && res.slope > 0.0;
    a.step_flags[2] = 0;
  }
}

// The arguments stay in the kernel's parameter space (__grid_constant__): the
// device functions take them by reference, which would otherwise copy the
// struct to local memory and turn every field read in the CG loop into a
// local load (measured: D2 solve 73.1 -> 70.3 ms, bit-identical).
__global__ void __launch_bounds__(NT, 1) k_coop(const __grid_constant__ CoopArgs a) {
  __shared__ Smem sh;
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x;
  const int64_t r0 = a.part[blockIdx.x];             // rows [r0, r1): k_partition
  const int64_t r1 = a.part[blockIdx.x + 1];
  if (threadIdx.x == 0) {
    s_mode = a.part[G + 1];
    s_ep = *reinterpret_cast<volatile const uint32_t*>(a.gs_epoch);   // the previous launch's last
  }
  int64_t nh = 0;
  DevResult res{};
  res.status = OTN_OK;
  const Row row{int64_t(threadIdx.x) < r1 - r0, r0 + threadIdx.x};
  const double rPi = row.own && a.rP ? __ldg(a.rP + row.i) : 0.0;
  __syncthreads();
  stage_layout(a, r0, r1, a.wpart + int64_t(blockIdx.x) * a.ld);
  if (s_mode >= kPlanSparse) stage_sparse(a, r0, r1, a.wpart + int64_t(blockIdx.x) * a.ld, sh);

  if (a.pre_flags) {
    // [0]: plan overflow (materialize), [1]: nonpositive sums (system prep);
    // checked in the reference's order (dual.py:155-169 then newton.py:76-77).
    const int f0 = ((volatile const int*)a.pre_flags)[0];
    const int f1 = ((volatile const int*)a.pre_flags)[1];
    if (f0) res.status = OTN_ST_PLAN_OVERFLOW;
    else if (f1) res.status = OTN_ST_NONPOSITIVE_SUMS;
    if (res.status != OTN_OK) {
      if (blockIdx.x == 0 && threadIdx.x == 0) publish_result(a, res);
      return;  // uniform across the grid: no barrier is skipped by only some CTAs
    }
  }

  if (a.mode == kModeNewton) {
    const double gi = row.own ? __ldg(a.g + row.i) : 0.0;
    double gl[1] = {fabs(gi)};
    grid_reduce<1>(gl, a, sh);
    const double gn = gl[0];
    res.rho_final = a.rho0;
    double d = 0.0;
    if (gn != 0.0) {
      if (row.own) d = __ddiv_rn(-gi, rPi);
      double rho = a.rho0, used = a.rho0;
      int64_t total = 0;
      const double tol = __dmul_rn(__dmul_rn(0.25, a.eta), gn);
      const double target = __dmul_rn(a.eta, gn);
      while (true) {
        const double q = hvp(grid, a, d, 1.0, rPi, r0, r1, sh, nh);
        double rl[1] = {row.own ? fabs(__dadd_rn(q, gi)) : 0.0};
        grid_reduce<1>(rl, a, sh);
        if (rl[0] <= target) { res.resid_l1 = rl[0]; break; }
        if (__dsub_rn(1.0, rho) < 1e-12) {
          res.status = OTN_ST_STAGNATION;
          res.resid_l1 = rl[0];
          res.diag_rho = rho;
          break;
        }
        ++res.pcg_calls;
        const PcgOut po = pcg(grid, a, row, rPi, rho, nullptr, tol, d, a.zero_init == 0,
                              a.max_iters, r0, r1, sh, nh);
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
    if (row.own) a.d[row.i] = d;
    if (res.status == OTN_OK && a.dv) {
      column_pass(grid, a, d, 1, a.dv, r0, r1, sh);
      double sl[1] = {fma(gi, d, 0.0)};
      grid_reduce<1>(sl, a, sh);
      res.slope = -sl[0];
    }
  } else if (a.mode == kModePcg) {
    res.pcg_calls = 1;
    double x = row.own && a.has_x0 ? a.d[row.i] : 0.0;
    const PcgOut po = pcg(grid, a, row, rPi, a.rho, a.b, a.tol, x, a.has_x0 != 0, a.max_iters,
                          r0, r1, sh, nh);
    if (row.own) a.d[row.i] = x;
    res.status = po.status;
    res.cg_iters = po.iters;
    res.resid_l1 = po.resid;
    res.diag_rho = a.rho;
    res.diag_resid = po.resid;
  } else if (a.mode == kModeHvp) {
    const double q = hvp(grid, a, row.own ? a.xin[row.i] : 0.0, a.rho, rPi, r0, r1, sh, nh);
    if (row.own) a.d[row.i] = q;
  } else if (a.mode == kModePc || a.mode == kModeRmatvec) {
    column_pass(grid, a, row.own ? a.xin[row.i] : 0.0, a.mode == kModePc ? 0 : 2, a.wc, r0, r1, sh);
    grid_bar(a, sh);
    for (int64_t i = int64_t(blockIdx.x) * NT + threadIdx.x; i < a.n; i += int64_t(G) * NT)
      a.d[i] = __ldcg(a.wc + i);
  } else if (a.mode == kModeProbe) {
    // Diagnostic: repeat one building block max_iters times (bench tooling).
    const int what = a.has_x0;
    const double xv = row.own ? a.xin[row.i] : 0.0;
    stage_x(xv, sh);
    for (int64_t k = 0; k < a.max_iters; ++k) {
      if (what == 0) {
        grid_bar(a, sh);
      } else if (what == 1) {
        double v[2] = {1.0, 2.0};
        grid_reduce<2>(v, a, sh);
      } else if (what == 2) {
        phase_a(plan_view(a, r0, r1), r0, r1, a.wpart + int64_t(blockIdx.x) * a.ld, sh);
        __syncthreads();
      } else if (what == 3) {
        phase_b(plan_view(a, r0, r1), a.xin, r0, r1, sh);
      } else if (what == 4) {
        column_pass(grid, a, xv, 0, a.wc, r0, r1, sh);
        grid_bar(a, sh);
      } else {
        const double q = hvp(grid, a, xv, 0.5, rPi, r0, r1, sh, nh);
        if (row.own) a.d[row.i] = q;
      }
    }
  } else if (a.mode == kModeMatvec) {
    // stage x into the padded workspace vector (phase B reads ld entries)
    for (int64_t j = int64_t(blockIdx.x) * NT + threadIdx.x; j < a.ld; j += int64_t(G) * NT)
      a.wc[j] = j < a.n ? __ldg(a.xin + j) : 0.0;
    grid_bar(a, sh);
    phase_b(plan_view(a, r0, r1), a.wc, r0, r1, sh);
    if (row.own) a.d[row.i] = sh.sv[threadIdx.x];
  }
  res.hvps = nh;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t* st = reinterpret_cast<const int64_t*>(a.part + ((G + 2 + 1) & ~1));
    res.plan_mode = s_mode;
    res.plan_nnz = st[0];
    res.plan_span = st[1];
    int rmax = 0;
    for (int b = 0; b < G; ++b) rmax = max(rmax, a.part[b + 1] - a.part[b]);
    res.plan_rows_max = rmax;
    *a.gs_epoch = s_ep;                             // this thread completed the last exchange
    publish_result(a, res);
  }
}

static_assert(kRingBytes == size_t(kRingDepth) * kSlotBytes, "ring layout");
static_assert(kSparseGSmem + size_t(kSparseGS) * 10 <= kSparseBytes + size_t(kSparseRows) * 4,
              "mode-3 shared CSC slots fit the dynamic region");
constexpr size_t kDynRing = kRingBytes + size_t(kSpanSmem) * 4;
constexpr size_t kDynSparse = kSparseBytes + size_t(kSparseRows) * 4;
constexpr size_t kDynBytes = kDynRing > kDynSparse ? kDynRing : kDynSparse;

// ---------------------------------------------------------------------------
// k_partition: one CTA picks the plan mode of the next k_coop launch and its
// row partition (integer arithmetic only: deterministic).
//   part[0..G] = row boundaries of the G CTAs, part[G+1] = PlanMode.
// Sparse (one tile, ld <= 4096): rows balanced on cost_i = nnz_i + 32, row i
// going to CTA floor(prefix_i * G / total); used if every CTA's rows and
// nonzeros fit its shared (kPlanSparse) or global (kPlanSparseG) slice.
// Otherwise equal rows (the streaming phases cost ~ rows x window chunks; a
// span-balanced split measured slower) and the ring.
// ---------------------------------------------------------------------------
constexpr int kPartThreads = 1024;
constexpr int kPartRows = kSparseCols;               // rows handled in shared memory

template <typename T>
__device__ T block_sum_part(T v, T* buf) {                // all threads get the total
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) buf[warp] = v;
  __syncthreads();
  T tot = 0;
  for (int w = 0; w < kPartThreads / 32; ++w) tot += buf[w];
  return tot;
}

__global__ void __launch_bounds__(kPartThreads) k_partition(const uint64_t* mask, int64_t n,
                                                            int64_t ld, int64_t mw, int G,
                                                            int sg_ok, int* part) {
  __shared__ int s_pref[kPartRows + 1];      // inclusive prefix of the sparse row costs
  __shared__ int64_t s_buf[32];
  __shared__ int s_ibuf[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int mode = kPlanRing;
  bool sparse = false;
  int64_t s_nz = 0;                                  // nonzeros of the plan (all threads)
  int64_t span = n * ld;                             // entries the ring streams per pass
  if (mask) {
    int64_t nz = 0, sp = 0;
    const int nt = int((ld + TILE - 1) / TILE);
    for (int64_t i = t; i < n; i += kPartThreads) {
      nz += int64_t(__ldg(mask + i * mw + mw - 1));
      for (int ti = 0; ti < nt; ++ti) {               // [first, last] nonzero segment per tile
        const uint64_t bits = __ldg(mask + i * mw + ti);
        if (!bits) continue;
        const int width = int(ld - int64_t(ti) * TILE < TILE ? ld - int64_t(ti) * TILE : TILE);
        const int lo = (__ffsll(static_cast<long long>(bits)) - 1) * kSegCols;
        const int hi = min((64 - __clzll(static_cast<long long>(bits))) * kSegCols, width);
        sp += hi - lo;
      }
    }
    nz = block_sum_part<int64_t>(nz, s_buf);
    sp = block_sum_part<int64_t>(sp, s_buf);
    s_nz = nz;
    span = sp;
    const int64_t cap = sg_ok ? kSparseGCap : kSparseCap;
    // compressed rows pay 10 B per nonzero per pass (value + column) against
    // 8 B per span column: only below half density
    sparse = ld <= kSparseCols && n <= kPartRows && nz * 5 <= int64_t(G) * cap * 4 &&
             nz * 2 <= n * ld;
  }
  if (sparse) {
    // inclusive prefix of cost_i over rows: 4 contiguous rows per thread
    constexpr int R = kPartRows / kPartThreads;
    int c[R], run = 0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int64_t i = int64_t(t) * R + k;
      c[k] = i < n ? int(__ldg(mask + i * mw + mw - 1)) + 32 : 0;
      run += c[k];
    }
    int incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) s_ibuf[warp] = incl;
    __syncthreads();
    int off = incl - run;
    for (int w = 0; w < warp; ++w) off += s_ibuf[w];
    if (t == 0) s_pref[0] = 0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      off += c[k];
      const int64_t i = int64_t(t) * R + k;
      if (i < n) s_pref[i + 1] = off;
    }
    __syncthreads();
    const int64_t total = s_pref[n] > 0 ? s_pref[n] : 1;
    // CTA of row i: floor(pref_excl(i) * G / total); part[b] = first row of CTA >= b
    for (int64_t i = t; i < n; i += kPartThreads) {
      const int cb = int(int64_t(s_pref[i]) * G / total);
      const int pb = i == 0 ? -1 : int(int64_t(s_pref[i - 1]) * G / total);
      for (int k = pb + 1; k <= cb; ++k) part[k] = int(i);
    }
    const int last = int(int64_t(s_pref[n - 1]) * G / total);
    for (int k = last + 1 + t; k <= G; k += kPartThreads) part[k] = int(n);
    __syncthreads();
    int bad_smem = 0, bad_glob = 0;
    for (int b = t; b < G; b += kPartThreads) {
      const int r0 = part[b], r1 = part[b + 1];
      const int rows = r1 - r0, nnz = s_pref[r1] - s_pref[r0] - 32 * rows;
      if (rows > kSparseRows || nnz > kSparseNnzMax) bad_smem = 1;
      if (rows > kSparseRows || nnz > kSparseGCap || !sg_ok) bad_glob = 1;
    }
    const int no_smem = block_sum_part<int>(bad_smem, s_ibuf);
    const int no_glob = block_sum_part<int>(bad_glob, s_ibuf);
    // the global-memory CSR/CSC pays 20 B per nonzero per HVP through L2
    // (CSR for phase B, CSC for phase A): above ~25% density the dense ring
    // is faster (measured: 33% density 63 us vs ~34 us per HVP)
    const bool glob_ok = no_glob == 0 && s_nz * 4 <= int64_t(n) * ld;
    sparse = no_smem == 0 || glob_ok;
    if (sparse) mode = no_smem == 0 ? kPlanSparse : kPlanSparseG;
  }
  __syncthreads();
  if (t == 0) {                                      // statistics for the launch record
    int64_t* st = reinterpret_cast<int64_t*>(part + ((G + 2 + 1) & ~1));
    st[0] = mask ? s_nz : n * ld;
    st[1] = span;
  }
  if (sparse) {
    if (t == 0) part[G + 1] = mode;
    return;
  }
  for (int b = t; b <= G; b += kPartThreads) part[b] = int((int64_t(b) * n) / G);
  if (t == 0) part[G + 1] = mode;
}

cudaError_t launch_coop(otn_ctx* x, const CoopArgs& a0) {
  // CG vectors live one row per thread: at most NT rows per CTA (n <= 75776 on 148 SMs)
  if ((a0.n + x->coop_blocks - 1) / x->coop_blocks > NT) return cudaErrorInvalidValue;
  CoopArgs a = a0;
  a.stages = kRingDepth;
  a.part = x->part;
  a.sg = x->sg;
  if (x->time_coop) cudaEventRecord(x->ev_coop[0], x->stream);
  k_partition<<<1, kPartThreads, 0, x->stream>>>(a.mask, a.n, a.ld, a.mw, x->coop_blocks,
                                                 x->sg != nullptr, x->part);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  void* args[] = {&a};
  e = cudaLaunchCooperativeKernel((void*)k_coop, dim3(x->coop_blocks), dim3(NT), args, kDynBytes,
                                  x->stream);
  if (e == cudaSuccess && x->time_coop) e = cudaEventRecord(x->ev_coop[1], x->stream);
  return e;
}

size_t sparse_g_bytes_per_cta() { return kSparseGBytes; }

int coop_occupancy(int* blocks_per_sm) {
  cudaError_t e = cudaFuncSetAttribute(k_coop, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kDynBytes));
  if (e != cudaSuccess) return int(e);
  return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_coop, NT,
                                                            kDynBytes);
}

}  // namespace otn
