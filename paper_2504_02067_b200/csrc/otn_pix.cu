// Cost construction for 8-bit point sets on the tensor cores (K10: the setup
// GEMM of problems.py:87-111 for d = 784 pixel sets, SURVEY §8 / BASELINE D3).
//
//   C_ij = max(|x_i|^2 + |y_j|^2 - 2 x_i . y_j, 0) / max_ij(...)
//
// Pixel intensities are integers 0..255, so every dot product is an exact
// integer (<= 784 * 255^2 < 2^31): the products run as u8 x u8 -> s32 MMAs
// (mma.sync m16n8k32) and every entry before the final division is the exact
// integer numpy's float64 GEMM also produces (all partial sums < 2^53) -- the
// cost equals the host's bit for bit, independent of summation order.
//
//   k_pix_pack   X, Y (float64, n x d) -> u8 rows padded to KP = 32k bytes,
//                exact squared norms; flags any entry that is not an integer
//                in [0, 255]
//   k_pix_gemm   128 x 128 tiles of X8 . Y8^T, 3-stage cp.async ring of
//                32-byte K slices, ldmatrix + mma.sync; epilogue forms the
//                unnormalized cost, writes it (padding columns 0) and reduces
//                the maximum (non-negative doubles order as their bits)
//   k_pix_scale  C /= max over the n x n block
#include "otn_common.cuh"
#include "otn_internal.h"

namespace otn {

namespace {

constexpr int kPixTile = 128;            // output tile (rows and columns)
constexpr int kPixThreads = 256;         // 8 warps: 2 (rows) x 4 (columns)
constexpr int kPixStages = 3;
constexpr int kPixPitch = 48;            // bytes per staged row (32 + 16: ldmatrix conflict-free)
constexpr int kPixStageBytes = kPixTile * kPixPitch;

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
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma_u8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                       uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__global__ void __launch_bounds__(kPixThreads) k_pix_gemm(const uint8_t* A8, const uint8_t* B8,
                                                          const int* na, const int* nb,
                                                          int64_t n, int64_t ld, int64_t kp,
                                                          double* C,
                                                          unsigned long long* cmax_bits) {
  __shared__ __align__(128) uint8_t sA[kPixStages][kPixStageBytes];
  __shared__ __align__(128) uint8_t sB[kPixStages][kPixStageBytes];
  __shared__ unsigned long long s_max[kPixThreads / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wm = warp & 1, wn = warp >> 1;          // warp tile: 64 rows x 32 columns
  const int64_t i0 = int64_t(blockIdx.y) * kPixTile, j0 = int64_t(blockIdx.x) * kPixTile;
  const int nk = int(kp / 32);
  // staging: thread t copies row t/2, 16-byte half t%2, of the A and B slices
  const int srow = t >> 1, shalf = t & 1;
  const bool avalid = i0 + srow < n, bvalid = j0 + srow < n;
  const uint8_t* asrc = A8 + (avalid ? i0 + srow : 0) * kp + 16 * shalf;
  const uint8_t* bsrc = B8 + (bvalid ? j0 + srow : 0) * kp + 16 * shalf;
  const uint32_t adst = smem_u32addr(&sA[0][0]) + srow * kPixPitch + 16 * shalf;
  const uint32_t bdst = smem_u32addr(&sB[0][0]) + srow * kPixPitch + 16 * shalf;
  auto issue = [&](int kt) {
    const int st = kt % kPixStages;
    cp16(adst + st * kPixStageBytes, asrc + int64_t(kt) * 32, avalid);
    cp16(bdst + st * kPixStageBytes, bsrc + int64_t(kt) * 32, bvalid);
  };
#pragma unroll
  for (int s = 0; s < kPixStages - 1; ++s) {
    if (s < nk) issue(s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  int acc[4][4][4];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[mi][ni][q] = 0;
  // ldmatrix row addresses: A matrices (rows 0-7 | 8-15) x (k 0-15 | 16-31),
  // B matrices (k 0-15 | 16-31) x (n tile 0 | 1)
  const int q = lane >> 3, rr = lane & 7;
  const uint32_t a_off = (wm * 64 + (q & 1) * 8 + rr) * kPixPitch + (q >> 1) * 16;
  const uint32_t b_off = (wn * 32 + (q >> 1) * 8 + rr) * kPixPitch + (q & 1) * 16;
  for (int kt = 0; kt < nk; ++kt) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kPixStages - 2) : "memory");
    __syncthreads();                                 // slice kt visible; slice kt-1 consumed
    if (kt + kPixStages - 1 < nk) issue(kt + kPixStages - 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const int st = kt % kPixStages;
    const uint32_t abase = smem_u32addr(&sA[st][0]) + a_off;
    const uint32_t bbase = smem_u32addr(&sB[st][0]) + b_off;
    uint32_t a[4][4], b[4][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
      ldsm_x4(abase + mi * 16 * kPixPitch, a[mi][0], a[mi][1], a[mi][2], a[mi][3]);
#pragma unroll
    for (int np = 0; np < 2; ++np)
      ldsm_x4(bbase + np * 16 * kPixPitch, b[2 * np][0], b[2 * np][1], b[2 * np + 1][0],
              b[2 * np + 1][1]);
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) mma_u8(acc[mi][ni], a[mi], b[ni][0], b[ni][1]);
  }
  // epilogue: rows g, g + 8 and columns 2 tq, 2 tq + 1 of every m16 x n8 tile
  const int g = lane >> 2, tq = lane & 3;
  double vmax = 0.0;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t i = i0 + wm * 64 + mi * 16 + g + 8 * h;
      if (i >= n) continue;
      const int64_t ni_ = na[i];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int64_t j = j0 + wn * 32 + ni * 8 + 2 * tq;
        if (j >= ld) continue;
        double2 o;
        // exact integers: |x|^2 + |y|^2 - 2 x.y (every term and sum < 2^53)
        const int64_t e0 = j < n ? ni_ + nb[j] - 2 * int64_t(acc[mi][ni][2 * h]) : 0;
        const int64_t e1 = j + 1 < n ? ni_ + nb[j + 1] - 2 * int64_t(acc[mi][ni][2 * h + 1]) : 0;
        o.x = e0 > 0 ? double(e0) : 0.0;
        o.y = e1 > 0 ? double(e1) : 0.0;
        vmax = fmax(vmax, fmax(o.x, o.y));
        *reinterpret_cast<double2*>(C + i * ld + j) = o;
      }
    }
  }
  unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(vmax));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, bits, o);
    bits = other > bits ? other : bits;
  }
  if (lane == 0) s_max[warp] = bits;
  __syncthreads();
  if (t == 0) {
    unsigned long long m = s_max[0];
    for (int w = 1; w < kPixThreads / 32; ++w) m = s_max[w] > m ? s_max[w] : m;
    atomicMax(cmax_bits, m);                         // non-negative doubles order as their bits
  }
}

__global__ void __launch_bounds__(256) k_pix_scale(double* C, int64_t n, int64_t ld,
                                                   const unsigned long long* cmax_bits) {
  const double cmax = __longlong_as_double(static_cast<long long>(*cmax_bits));
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    double* row = C + i * ld;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x)
      row[j] = __ddiv_rn(row[j], cmax);              // numpy: C /= C.max()
  }
}

}  // namespace

cudaError_t launch_pixel_cost(otn_ctx* x, const double* X, const double* Y, int64_t d, double* C,
                              unsigned long long* cmax_bits, int* err) {
  const int64_t n = x->n, ld = x->ld, kp = (d + 31) / 32 * 32;
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
  void* scratch = x->pix_scratch;
  uint8_t* packed = static_cast<uint8_t*>(scratch);
  int* norms = reinterpret_cast<int*>(packed + (packed_bytes + 255) / 256 * 256);
  cudaMemsetAsync(cmax_bits, 0, sizeof(unsigned long long), x->stream);
  cudaMemsetAsync(err, 0, sizeof(int), x->stream);
  k_pix_pack<<<unsigned((2 * n + 7) / 8), 256, 0, x->stream>>>(X, Y, n, d, kp, packed, norms, err);
  const dim3 grid(unsigned((ld + kPixTile - 1) / kPixTile), unsigned((n + kPixTile - 1) / kPixTile));
  k_pix_gemm<<<grid, kPixThreads, 0, x->stream>>>(packed, packed + size_t(n) * kp, norms,
                                                  norms + n, n, ld, kp, C, cmax_bits);
  k_pix_scale<<<unsigned(n < 65535 ? n : 65535), 256, 0, x->stream>>>(C, n, ld, cmax_bits);
  return cudaGetLastError();
}

}  // namespace otn
