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

__device__ __forceinline__ double warp_sum(double v) {
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
    s = __dadd_rn(__dmul_rn(s, exp(m - m2)), s2);
    m = m2;
  } else if (m2 != OTN_NINF) {
    s = __dadd_rn(s, __dmul_rn(s2, exp(m2 - m)));
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
