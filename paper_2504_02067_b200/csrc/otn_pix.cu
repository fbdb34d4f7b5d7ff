// Cost construction for 8-bit point sets on the tensor cores (K10: the setup
// GEMM of problems.py:87-111 for d = 784 pixel sets, SURVEY §8 / BASELINE D3).
//
//   C_ij = max(|x_i|^2 + |y_j|^2 - 2 x_i . y_j, 0) / max_ij(...)
//
// Pixel intensities are integers 0..255, so every dot product is an exact
// integer (<= d * 255^2 < 2^31 for d < 33025): the products run as
// u8 x u8 -> s32 tcgen05 MMAs and every entry before the final division is
// the exact integer numpy's float64 GEMM also produces (all partial sums
// < 2^53) -- the cost equals the host's bit for bit, independent of
// summation order.
//
//   k_pix_pack   X, Y (float64, n x d) -> u8 rows padded to KP = 128k bytes,
//                exact squared norms; flags any entry that is not an integer
//                in [0, 255]
//   k_pix_tc     the tensor-core product, pass 1 (maximum) and pass 2
//                (cost / maximum, written once)
#include "otn_common.cuh"
#include "otn_internal.h"

namespace otn {

namespace {

__global__ void __launch_bounds__(256) k_pix_pack(const double* X, const double* Y, int64_t n,
                                                  int64_t d, int64_t kp, uint8_t* packed,
                                                  int* norms, int* err) {
  const int lane = threadIdx.x & 31;
  const int64_t r = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (r >= 2 * n) return;
  const double* src = r < n ? X + r * d : Y + (r - n) * d;
  uint8_t* dst = packed + r * kp;
  int sum = 0, bad = 0;
  for (int64_t k = lane; k < kp; k += 32) {
    const double v = k < d ? src[k] : 0.0;
    const bool ok = v >= 0.0 && v <= 255.0 && v == floor(v);
    bad |= !ok;
    const int q = ok ? int(v) : 0;
    dst[k] = uint8_t(q);
    sum += q * q;
  }
  sum = warp_sum_int(sum);
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, 1);
  if (lane == 0) norms[r] = sum;
}

__device__ __forceinline__ uint32_t smem_u32addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0) : "memory");
}
// ---------------------------------------------------------------------------
// The product on the 5th-generation tensor cores: tcgen05.mma kind::i8
// (u8 x u8 -> s32) with the accumulator tile in tensor memory.
//
// CTA tile 128 (X rows) x 256 (Y rows), two CTAs per SM.  All 128 threads
// stage the 128-byte K slices with cp.async into a 2-stage ring in the
// canonical K-major 128-byte-swizzle layout (8-row atoms of 1024 B, 16-byte
// chunk c of row r at chunk c ^ (r % 8)); one elected thread issues the MMAs
// (M = 128, N = 256, K = 32, 4 per slice) and tcgen05.commit on a per-stage
// mbarrier hands each slot back once the MMAs that read it completed.  The
// epilogue (thread t = TMEM lane t = tile row t) reads its row with
// tcgen05.ld 32x32b.x16, forms the exact integer cost and either reduces the
// maximum (pass 1) or writes cost / max through a shared-memory transpose
// (pass 2) -- two passes, so the normalized cost is written once, without a
// separate scale pass.  (Measured against an mma.sync m16n8k32 kernel and a
// warp-specialized variant fed by 16 KB bulk copies of pre-swizzled slices:
// DESIGN.md section 3.3.)
// ---------------------------------------------------------------------------
constexpr int kTcM = 128, kTcN = 256, kTcKB = 128, kTcStages = 2;   // 2 CTAs per SM
constexpr int kTcThreads = 128;
constexpr uint32_t kTcABytes = kTcM * kTcKB, kTcBBytes = kTcN * kTcKB;
constexpr uint32_t kTcStageBytes = kTcABytes + kTcBBytes;
constexpr size_t kTcSmem = size_t(kTcStages) * kTcStageBytes + 1024;   // + 1024 B alignment slack

__device__ __forceinline__ uint64_t tc_smem_desc(uint32_t saddr) {
  // K-major, SWIZZLE_128B: LBO 16 B (unused), SBO 1024 B (8-row atoms), version 1
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
// instruction descriptor: s32 accumulator, u8 A and B, both K-major, N = 256, M = 128
constexpr uint32_t kTcIdesc = (2u << 4) | (uint32_t(kTcN >> 3) << 17) | (uint32_t(kTcM >> 4) << 24);

__device__ __forceinline__ void tc_mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void tc_mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar), "r"(parity) : "memory");
}
template <bool WRITE>
__global__ void __launch_bounds__(kTcThreads, 1) k_pix_tc(const uint8_t* A8, const uint8_t* B8,
                                                          const int* na, const int* nb, int64_t n,
                                                          int64_t ld, int64_t kp, double* C,
                                                          unsigned long long* cmax_bits) {
  extern __shared__ __align__(1024) uint8_t s_tc_raw[];
  __shared__ __align__(8) unsigned long long s_empty[kTcStages], s_acc;   // slot free, tile done
  __shared__ uint32_t s_tmem;
  __shared__ unsigned long long s_max[kTcThreads / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(s_tc_raw));
  const uint32_t base = (raw + 1023u) & ~1023u;      // 128-byte swizzle atoms need 1024-B alignment
  const int64_t i0 = int64_t(blockIdx.y) * kTcM, j0 = int64_t(blockIdx.x) * kTcN;
  const int nkb = int(kp / kTcKB);
  const uint32_t empty0 = static_cast<uint32_t>(__cvta_generic_to_shared(&s_empty[0]));
  const uint32_t accb = static_cast<uint32_t>(__cvta_generic_to_shared(&s_acc));
  if (t == 0) {
    for (int s = 0; s < kTcStages; ++s) tc_mbar_init(empty0 + 8u * s, 1);
    tc_mbar_init(accb, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {                                   // 256 TMEM columns: the 128 x 256 s32 tile
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&s_tmem));
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(dst), "n"(kTcN) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;

  auto issue = [&](int kb) {                         // K slice kb -> ring slot kb % stages
    const uint32_t sa = base + uint32_t(kb % kTcStages) * kTcStageBytes, sb = sa + kTcABytes;
#pragma unroll
    for (int i = 0; i < (kTcM * 8) / kTcThreads; ++i) {
      const int q = t + kTcThreads * i, row = q >> 3, c = q & 7;
      const bool ok = i0 + row < n;
      const uint8_t* src = A8 + (ok ? i0 + row : 0) * kp + int64_t(kb) * kTcKB + 16 * c;
      cp16(sa + (row >> 3) * 1024 + (row & 7) * 128 + ((c ^ (row & 7)) << 4), src, ok);
    }
#pragma unroll
    for (int i = 0; i < (kTcN * 8) / kTcThreads; ++i) {
      const int q = t + kTcThreads * i, row = q >> 3, c = q & 7;
      const bool ok = j0 + row < n;
      const uint8_t* src = B8 + (ok ? j0 + row : 0) * kp + int64_t(kb) * kTcKB + 16 * c;
      cp16(sb + (row >> 3) * 1024 + (row & 7) * 128 + ((c ^ (row & 7)) << 4), src, ok);
    }
  };
#pragma unroll
  for (int s = 0; s < kTcStages - 1; ++s) {
    if (s < nkb) issue(s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int kb = 0; kb < nkb; ++kb) {
    const int nk = kb + kTcStages - 1;               // refill the slot slice kb - 1 used
    if (nk < nkb) {
      if (nk >= kTcStages) tc_mbar_wait(empty0 + 8u * (nk % kTcStages), ((nk / kTcStages) - 1) & 1);
      issue(nk);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(kTcStages - 1) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> MMA reads
    __syncthreads();
    if (warp == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const uint32_t sa = base + uint32_t(kb % kTcStages) * kTcStageBytes, sb = sa + kTcABytes;
#pragma unroll
        for (int k = 0; k < kTcKB / 32; ++k) {
          const uint64_t da = tc_smem_desc(sa + 32u * k), db = tc_smem_desc(sb + 32u * k);
          const uint32_t acc = (kb | k) != 0;
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}"
              ::"r"(tmem), "l"(da), "l"(db), "r"(kTcIdesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u),
                "r"(0u) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(empty0 + 8u * (kb % kTcStages)) : "memory");
        if (kb == nkb - 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                       ::"r"(accb) : "memory");
      }
      __syncwarp();
    }
  }
  tc_mbar_wait(accb, 0);                             // the accumulator tile is complete
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // epilogue: thread t holds tile row t (TMEM lane t), 16 columns per load
  const int64_t i = i0 + t;
  const int64_t ni = i < n ? na[i] : 0;
  const double cmax = WRITE ? __longlong_as_double(static_cast<long long>(*cmax_bits)) : 0.0;
  double vmax = 0.0;
#pragma unroll 1
  for (int c0 = 0; c0 < kTcN; c0 += 16) {
    uint32_t v[16];
    const uint32_t taddr = tmem + (uint32_t(warp * 32) << 16) + uint32_t(c0);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int64_t jb = j0 + c0;
    if (jb >= ld) continue;                          // (uniform over the CTA)
    double o[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int64_t j = jb + q;
      // exact integers: |x|^2 + |y|^2 - 2 x.y (every term and sum < 2^53)
      const int64_t e = i < n && j < n ? ni + nb[j] - 2 * int64_t(static_cast<int32_t>(v[q])) : 0;
      o[q] = e > 0 ? double(e) : 0.0;
      vmax = fmax(vmax, o[q]);
      if (WRITE && j < n) o[q] = __ddiv_rn(o[q], cmax);   // numpy: C /= C.max()
    }
    if (WRITE) {
      // through shared memory (the idle ring): the warp's 32 rows x 16 columns,
      // then 8 lanes per row write its 128 contiguous bytes
      double* tile = reinterpret_cast<double*>(s_tc_raw + (base - raw)) + warp * (32 * 17);
#pragma unroll
      for (int q = 0; q < 16; ++q) tile[lane * 17 + q] = o[q];
      __syncwarp();
#pragma unroll
      for (int rr = 0; rr < 32; rr += 4) {
        const int row = rr + (lane >> 3), col = 2 * (lane & 7);
        const int64_t gi = i0 + warp * 32 + row;
        if (gi < n)
          *reinterpret_cast<double2*>(C + gi * ld + jb + col) =
              make_double2(tile[row * 17 + col], tile[row * 17 + col + 1]);
      }
      __syncwarp();
    }
  }
  if (!WRITE) {
    unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(vmax));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, bits, o);
      bits = other > bits ? other : bits;
    }
    if (lane == 0) s_max[warp] = bits;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (!WRITE && t == 0) {
    unsigned long long m = s_max[0];
    for (int w = 1; w < kTcThreads / 32; ++w) m = s_max[w] > m ? s_max[w] : m;
    atomicMax(cmax_bits, m);                         // non-negative doubles order as their bits
  }
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTcN)
                 : "memory");
  }
}

}  // namespace

cudaError_t launch_pixel_cost(otn_ctx* x, const double* X, const double* Y, int64_t d, double* C,
                              unsigned long long* cmax_bits, int* err) {
  const int64_t n = x->n, ld = x->ld, kp = (d + kTcKB - 1) / kTcKB * kTcKB;
  const size_t packed_bytes = size_t(2 * n) * size_t(kp);
  const size_t need = (packed_bytes + 255) / 256 * 256 + size_t(2 * n) * sizeof(int);
  if (x->pix_scratch_bytes < need) {                // grown once, kept with the context
    if (x->pix_scratch) cudaFree(x->pix_scratch);
    x->pix_scratch = nullptr;
    x->pix_scratch_bytes = 0;
    cudaError_t e = cudaMalloc(&x->pix_scratch, need);
    if (e != cudaSuccess) return e;
    x->pix_scratch_bytes = need;
  }
  uint8_t* packed = static_cast<uint8_t*>(x->pix_scratch);
  int* norms = reinterpret_cast<int*>(packed + (packed_bytes + 255) / 256 * 256);
  cudaMemsetAsync(cmax_bits, 0, sizeof(unsigned long long), x->stream);
  cudaMemsetAsync(err, 0, sizeof(int), x->stream);
  k_pix_pack<<<unsigned((2 * n + 7) / 8), 256, 0, x->stream>>>(X, Y, n, d, kp, packed, norms, err);
  const uint8_t* A8 = packed;
  const uint8_t* B8 = packed + size_t(n) * kp;
  static bool attr = false;                          // (per process; the attribute is per function)
  if (!attr) {
    cudaFuncSetAttribute(k_pix_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTcSmem));
    cudaFuncSetAttribute(k_pix_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTcSmem));
    attr = true;
  }
  const dim3 grid(unsigned((ld + kTcN - 1) / kTcN), unsigned((n + kTcM - 1) / kTcM));
  k_pix_tc<false><<<grid, kTcThreads, kTcSmem, x->stream>>>(A8, B8, norms, norms + n, n, ld, kp,
                                                            C, cmax_bits);
  k_pix_tc<true><<<grid, kTcThreads, kTcSmem, x->stream>>>(A8, B8, norms, norms + n, n, ld, kp,
                                                           C, cmax_bits);
  return cudaGetLastError();
}

}  // namespace otn
