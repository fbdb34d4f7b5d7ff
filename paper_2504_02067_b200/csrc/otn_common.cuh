// Shared device helpers for the B200 truncated-Newton EOT kernels (sm_100a).
//
// Conventions
//  * Every matrix is row-major float64 with leading dimension `ld` (a multiple
//    of 32, i.e. 256-byte rows); columns n <= j < ld are padding.  Matrices
//    written by these kernels (the plan P) carry zeros in the padding.
//  * Vectors have length n; kernels never read past n.
//  * Wherever the reference rounds an intermediate (numpy evaluates one ufunc
//    at a time), the kernels use explicit __dmul_rn/__dadd_rn/__ddiv_rn so the
//    compiler cannot contract the pair into an FMA and change the rounding.
//    Inner-product accumulations may use FMA (the reference's BLAS does too).
//  * All reductions use fixed trees; no floating-point atomics anywhere, so
//    every run is bit-reproducible.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#define OTN_INF (__longlong_as_double(0x7ff0000000000000ULL))
#define OTN_NINF (__longlong_as_double(0xfff0000000000000ULL))

namespace otn {

__device__ __forceinline__ double2 ldg2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

// Streaming 128-bit load that does not allocate in L1 (plan / cost tiles are
// touched once per pass; keep L1 for the broadcast vectors).
__device__ __forceinline__ double2 ld_stream2(const double* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

// Branch-free float64 exp (max error ~1 ulp), used for every plan entry.
// CUDA's exp(double) takes a divergent slow path for |x| > 708, which is where
// most plan exponents live at weak regularization (they underflow to 0).
// Cody-Waite reduction x = k ln2 + r, |r| <= ln2/2, degree-13 Taylor
// polynomial in Horner form, and 2^k applied as two exact power-of-two factors
// so subnormal results are rounded once and underflow / overflow come out as
// 0 / inf.  x < -746 -> 0, x > 710 -> inf, NaN -> NaN.
__device__ __forceinline__ double pow2i(int e) {        // 2^e, -1022 <= e <= 1023
  return __hiloint2double((e + 1023) << 20, 0);
}
// Coefficients live in the constant bank so DFMA reads them directly (a
// double immediate would cost two uniform moves per use inside hot loops).
__constant__ double kExpPoly[14] = {
    1.6059043836821614599e-10, 2.0876756987868098979e-09, 2.5052108385441718775e-08,
    2.7557319223985890653e-07, 2.7557319223985890653e-06, 2.4801587301587301587e-05,
    1.9841269841269841270e-04, 1.3888888888888888889e-03, 8.3333333333333333333e-03,
    4.1666666666666666667e-02, 1.6666666666666666667e-01, 0.5, 1.0, 1.0};
__constant__ double kExpRed[3] = {1.4426950408889634, 6.93147180369123816490e-01,
                                  1.90821492927058770002e-10};

__device__ __forceinline__ double exp_fast(double x) {
  x = x < -746.0 ? -746.0 : (x > 710.0 ? 710.0 : x);
  // k = round(x / ln2) via the 1.5*2^52 shifter: no FRND / F2I conversions
  const double t = fma(x, kExpRed[0], 6755399441055744.0);
  const int k = __double2loint(t);
  const double kd = t - 6755399441055744.0;
  double r = fma(-kd, kExpRed[1], x);                     // ln2_hi (exact product)
  r = fma(-kd, kExpRed[2], r);                            // ln2_lo
  double p = kExpPoly[0];                                 // 1/13! ... 1/0! (Horner)
#pragma unroll
  for (int i = 1; i < 14; ++i) p = fma(p, r, kExpPoly[i]);
  const int k1 = k >> 1;
  return (p * pow2i(k1)) * pow2i(k - k1);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Merge (m2, s2) into the running log-sum-exp state (m, s), where the state
// represents m + log(s) and m = -inf encodes an empty / all -inf set.
__device__ __forceinline__ void lse_merge(double& m, double& s, double m2, double s2) {
  if (m2 > m) {
    s = __dadd_rn(__dmul_rn(s, exp_fast(m - m2)), s2);
    m = m2;
  } else if (m2 != OTN_NINF) {
    s = __dadd_rn(s, __dmul_rn(s2, exp_fast(m2 - m)));
  }
}

__device__ __forceinline__ void warp_lse(double& m, double& s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double m2 = __shfl_xor_sync(0xffffffffu, m, o);
    double s2 = __shfl_xor_sync(0xffffffffu, s, o);
    lse_merge(m, s, m2, s2);
  }
}

// The reference maps every non-finite row maximum to -inf (_kernels.py:36-41).
__device__ __forceinline__ double lse_value(double m, double s) {
  return isfinite(m) ? __dadd_rn(m, log(s)) : OTN_NINF;
}

// Block-wide sum over blockDim.x threads (multiple of 32, <= 1024); the result
// is returned to every thread.  `sh` needs 33 doubles.  Fixed tree.
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < nw ? sh[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) sh[32] = t;
  }
  __syncthreads();
  return sh[32];
}

__device__ __forceinline__ double block_max(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < nw ? sh[lane] : OTN_NINF;
    t = warp_max(t);
    if (lane == 0) sh[32] = t;
  }
  __syncthreads();
  return sh[32];
}

}  // namespace otn
