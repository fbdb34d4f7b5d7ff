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

// Table-driven float64 exp for the n^2-entry hot loops (LSE, plan, on-the-fly
// pair passes): x = (64 e + j) ln2/64 + r with |r| <= ln2/128, so a degree-5
// polynomial is enough; 2^(j/64) comes from a 64-entry double-double table
// that each kernel stages in shared memory (exp_tab_load; indexed by data, so
// a constant-bank table would serialize); 2^e is applied as
// two exact power-of-two factors (one rounding for subnormal results).  About
// 15 FP64 instructions instead of exp_fast's 21; max error <= 1 ulp (tested
// against numpy, tests/test_gpu_kernels.py::test_exp_tab_accuracy).
__device__ const double2 kExp2Tab[64] = {
    {1.0, 0.0}, {1.0108892860517005, -1.5234778603368577e-17},
    {1.0218971486541166, 5.109225028973444e-17}, {1.0330248790212284, 7.600838874027088e-18},
    {1.0442737824274138, 8.551889705537965e-17}, {1.0556451783605572, 1.759325738772092e-18},
    {1.0671404006768237, -7.899853966841582e-17}, {1.0787607977571199, -6.656660436056593e-17},
    {1.0905077326652577, -3.046782079812471e-17}, {1.102382583307841, 5.2660368715706944e-17},
    {1.1143867425958924, 1.0410278456845571e-16}, {1.1265216186082418, 5.165856758795457e-17},
    {1.1387886347566916, 8.912812676025408e-17}, {1.1511892299529827, 3.250710218863827e-17},
    {1.1637248587775775, 3.8292048369240935e-17}, {1.1763969916502812, 5.554203254218079e-17},
    {1.189207115002721, 3.982015231465646e-17}, {1.202156731452703, 6.644981499252301e-17},
    {1.215247359980469, -7.712630692681488e-17}, {1.22848053610687, -1.89878163130253e-17},
    {1.241857812073484, 4.658027591836937e-17}, {1.255380757024691, -6.7113898212968784e-18},
    {1.2690509571917332, 2.667932131342186e-18}, {1.2828700160787783, 1.713594918243561e-17},
    {1.2968395546510096, 2.5382502794888315e-17}, {1.3109612115247644, -7.181536135519454e-17},
    {1.3252366431597413, -2.8587312100388614e-17}, {1.339667524053303, 8.927282594831732e-17},
    {1.3542555469368927, 7.70094837980299e-17}, {1.3690024229745905, 9.593797919118849e-17},
    {1.383909881963832, -6.770511658794786e-17}, {1.3989796725383112, -9.614213209051323e-17},
    {1.4142135623730951, -9.667293313452913e-17}, {1.42961333839197, -1.2031642489053655e-17},
    {1.4451808069770467, -3.0237581349939873e-17}, {1.460917794180647, -5.600377186075216e-17},
    {1.4768261459394993, -3.483994556892796e-17}, {1.4929077282912648, 1.4192920154284036e-17},
    {1.5091644275934228, -1.016455327754295e-16}, {1.5255981507445384, -1.1024941712342561e-16},
    {1.5422108254079407, 7.949834809697621e-17}, {1.559004400237837, 3.7812070533575275e-17},
    {1.5759808451078865, -1.0136916471278304e-17}, {1.593142151342267, -1.0094406542311964e-16},
    {1.6104903319492543, 2.4707192569797888e-17}, {1.6280274218573478, -6.712955084707084e-17},
    {1.645755478153965, -1.0125679913674773e-16}, {1.6636765803267364, 5.8909926967131e-17},
    {1.681792830507429, 8.199010020581497e-17}, {1.7001063537185235, -8.0237193703977e-18},
    {1.718619298122478, -1.851380418263111e-17}, {1.7373338352737062, 3.164389299292957e-17},
    {1.7562521603732995, 2.960140695448873e-17}, {1.7753764925265212, 6.429731796556572e-17},
    {1.7947090750031072, 1.8227458427912087e-17}, {1.8142521755003989, -9.969531538920349e-17},
    {1.8340080864093424, 3.283107224245627e-17}, {1.8539791250833855, 9.761887490727594e-17},
    {1.8741676341103, -6.122763413004143e-17}, {1.8945759815869656, 3.4034035352165297e-17},
    {1.9152065613971474, -1.0619946056195963e-16}, {1.9360617934922943, 1.0332385960676326e-16},
    {1.9571441241754002, 8.960767791036668e-17}, {1.978456026387951, 4.0388753109278167e-17},
};

__constant__ double kExpTabC[6] = {92.332482616893658, 0.01083042468962958, 6.619564634077006e-12,
                                   1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0};

__device__ __forceinline__ void exp_tab_load(double2* tab) {
  // global (not __constant__): the 64 distinct addresses are one coalesced read
  for (int i = threadIdx.x; i < 64; i += blockDim.x) tab[i] = __ldg(&kExp2Tab[i]);
}

// exp_tab without the range clamp: x in [-746, 710] (or NaN).  Callers that
// already know x >= -746 (they skip x < -746, whose exp is exactly 0: a
// warp whose entries all underflow issues no exp at all) and x <= 710.
__device__ __forceinline__ double exp_tab_nc(double x, const double2* __restrict__ tab) {
  const double t = fma(x, kExpTabC[0], 6755399441055744.0);   // 64/ln2, 1.5*2^52 shifter
  const int k = __double2loint(t);
  const double kd = t - 6755399441055744.0;
  double r = fma(-kd, kExpTabC[1], x);               // ln2/64 high part (30 bits: exact product)
  r = fma(-kd, kExpTabC[2], r);                      // ln2/64 low part
  // q = e^r - 1 = r (1 + r/2 + r^2/6 + r^3/24 + r^4/120)
  double q = fma(r, kExpTabC[3], kExpTabC[4]);
  q = fma(q, r, kExpTabC[5]);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  q = q * r;
  const double2 tj = tab[k & 63];
  const double y = tj.x + fma(tj.x, q, tj.y);        // 2^(j/64) e^r, one final rounding
  const int e = k >> 6, e1 = e >> 1;
  return (y * pow2i(e1)) * pow2i(e - e1);
}

// exp(x) for -707 <= x <= 0, the log-sum-exp terms against the row maximum:
// exp_tab_nc's reduction and polynomial, but the result is normal, so 2^e is
// applied by adding e to the exponent field (one integer add instead of two
// power-of-two multiplies; identical bits).  Terms below -707 are < 1e-307
// next to the maximum's own exp(0) = 1 and are skipped by the callers (the
// per-lane sums they would enter are >= 1 or are merged into one that is:
// adding them changes no bit).
__device__ __forceinline__ double exp_m707(double x, const double2* __restrict__ tab) {
  const double t = fma(x, kExpTabC[0], 6755399441055744.0);   // 64/ln2, 1.5*2^52 shifter
  const int k = __double2loint(t);
  const double kd = t - 6755399441055744.0;
  double r = fma(-kd, kExpTabC[1], x);
  r = fma(-kd, kExpTabC[2], r);
  double q = fma(r, kExpTabC[3], kExpTabC[4]);
  q = fma(q, r, kExpTabC[5]);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  q = q * r;
  const double2 tj = tab[k & 63];
  const double y = tj.x + fma(tj.x, q, tj.y);
  return __hiloint2double(__double2hiint(y) + ((k >> 6) << 20), __double2loint(y));
}

__device__ __forceinline__ double exp_tab(double x, const double2* __restrict__ tab) {
  return exp_tab_nc(x < -746.0 ? -746.0 : (x > 710.0 ? 710.0 : x), tab);
}

// exp_tab for x <= 0 (a term against its running maximum): the upper clamp
// cannot trigger, so it is dropped -- the same bits, NaN included.
__device__ __forceinline__ double exp_tab_le0(double x, const double2* __restrict__ tab) {
  return exp_tab_nc(x < -746.0 ? -746.0 : x, tab);
}

// s + exp(x) for x <= 0 (log-sum-exp accumulation against a running max):
// entries below -746 add an exact 0 and are skipped; NaN propagates.
__device__ __forceinline__ double add_exp_le0(double s, double x, const double2* __restrict__ tab) {
  if (!(x < -746.0)) s += exp_tab_nc(x, tab);
  return s;
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
