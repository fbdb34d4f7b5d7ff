// Grid barrier + 2-value reduction latency on one B200 (148 CTAs x 512 threads,
// cooperative launch): the variants considered for k_coop's exchanges.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/gsync_bench.cu -o build/gsync_bench
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

constexpr int NT = 512, NW = 16, STR = 256;

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ void st2(uint64_t* p, uint64_t a, uint64_t b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld2(const uint64_t* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t ld_rlx(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct Buf {
  double* red;        // [2][2][STR] doubles
  uint64_t* gs;       // [2][2][STR][2]
  uint32_t* cnt;      // counters
  double* out;
};

__shared__ double s_red[2][33];
__shared__ double s_res[2];

// variant 0: cg grid.sync + partial loads (the current k_coop reduction)
__device__ void red_cg(cg::grid_group& grid, const Buf& b, double* v, int& slot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x;
  double* base = b.red + slot * 2 * STR;
  for (int k = 0; k < 2; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) for (int k = 0; k < 2; ++k) s_red[k][warp] = v[k];
  __syncthreads();
  if (warp < 2) {
    double t = warp_sum(lane < NW ? s_red[warp][lane] : 0.0);
    if (lane == 0) base[warp * STR + blockIdx.x] = t;
  }
  grid.sync();
  if (warp < 2) {
    double t = 0.0;
    for (int m = 0; m < STR / 64; ++m) {
      int bb = 64 * m + 2 * lane;
      double2 p = bb < G ? __ldcg(reinterpret_cast<const double2*>(base + warp * STR + bb)) : make_double2(0, 0);
      t += p.x + p.y;
    }
    t = warp_sum(t);
    if (lane == 0) s_res[warp] = t;
  }
  __syncthreads();
  v[0] = s_res[0]; v[1] = s_res[1];
  slot ^= 1;
}

// variant 1/2: epoch-tagged slots polled by the reading warps (sleep_ns between polls)
template <int SLEEP>
__device__ void red_flag(const Buf& b, double* v, uint32_t& ep) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x;
  for (int k = 0; k < 2; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) for (int k = 0; k < 2; ++k) s_red[k][warp] = v[k];
  __syncthreads();
  const uint32_t e = ep + 1;
  if (warp < 2) {
    double t = warp_sum(lane < NW ? s_red[warp][lane] : 0.0);
    uint64_t* row = b.gs + ((e & 1) * 2 + warp) * STR * 2;
    uint64_t tag = uint64_t(e) << 32;
    if (lane == 0) {
      uint64_t bits = __double_as_longlong(t);
      __threadfence();
      st2(row + 2 * blockIdx.x, tag | (bits & 0xffffffffull), tag | (bits >> 32));
    }
    double part[8];
    bool ok;
    do {
      ok = true;
      for (int q = 0; q < 8; ++q) {
        int bb = 64 * (q >> 1) + 2 * lane + (q & 1);
        part[q] = 0.0;
        if (bb < G) {
          uint64_t lo, hi;
          ld2(row + 2 * bb, lo, hi);
          ok &= (lo >> 32) == e && (hi >> 32) == e;
          part[q] = __longlong_as_double((hi << 32) | (lo & 0xffffffffull));
        }
      }
      if (SLEEP && !__all_sync(0xffffffffu, ok)) __nanosleep(SLEEP);
    } while (!__all_sync(0xffffffffu, ok));
    __threadfence();
    double s = 0.0;
    for (int m = 0; m < 4; ++m) s += part[2 * m] + part[2 * m + 1];
    s = warp_sum(s);
    if (lane == 0) s_res[warp] = s;
  }
  __syncthreads();
  v[0] = s_res[0]; v[1] = s_res[1];
  ep = e;
}

// variant 3: arrival counter (one atomic per CTA, lane 0 spins on it) + one read of the slots
__device__ void red_cnt(const Buf& b, double* v, uint32_t& ep) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x;
  for (int k = 0; k < 2; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) for (int k = 0; k < 2; ++k) s_red[k][warp] = v[k];
  __syncthreads();
  const uint32_t e = ep + 1;
  double* base = b.red + (e & 1) * 2 * STR;
  if (warp < 2) {
    double t = warp_sum(lane < NW ? s_red[warp][lane] : 0.0);
    if (lane == 0) base[warp * STR + blockIdx.x] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(b.cnt, 1u);
    const uint32_t target = e * uint32_t(G);
    while (int32_t(ld_acq(b.cnt) - target) < 0) {}
  }
  __syncthreads();
  if (warp < 2) {
    double t = 0.0;
    for (int m = 0; m < STR / 64; ++m) {
      int bb = 64 * m + 2 * lane;
      double2 p = bb < G ? __ldcg(reinterpret_cast<const double2*>(base + warp * STR + bb)) : make_double2(0, 0);
      t += p.x + p.y;
    }
    t = warp_sum(t);
    if (lane == 0) s_res[warp] = t;
  }
  __syncthreads();
  v[0] = s_res[0]; v[1] = s_res[1];
  ep = e;
}

// variant 6: counter + loads, release atomic (no separate fence); 7: barrier only
template <bool DATA>
__device__ void red_cnt_rel(const Buf& b, double* v, uint32_t& ep) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x;
  const uint32_t e = ep + 1;
  double* base = b.red + (e & 1) * 2 * STR;
  if (DATA) {
    for (int k = 0; k < 2; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0) for (int k = 0; k < 2; ++k) s_red[k][warp] = v[k];
    __syncthreads();
    if (warp < 2) {
      double t = warp_sum(lane < NW ? s_red[warp][lane] : 0.0);
      if (lane == 0) base[warp * STR + blockIdx.x] = t;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(b.cnt) : "memory");
    const uint32_t target = e * uint32_t(G);
    while (int32_t(ld_acq(b.cnt) - target) < 0) {}
  }
  __syncthreads();
  if (DATA) {
    if (warp < 2) {
      double t = 0.0;
      for (int m = 0; m < STR / 64; ++m) {
        int bb = 64 * m + 2 * lane;
        double2 p = bb < G ? __ldcg(reinterpret_cast<const double2*>(base + warp * STR + bb)) : make_double2(0, 0);
        t += p.x + p.y;
      }
      t = warp_sum(t);
      if (lane == 0) s_res[warp] = t;
    }
    __syncthreads();
    v[0] = s_res[0]; v[1] = s_res[1];
  }
  ep = e;
}

// variant 9/10: warp 0 alone does totals, arrive, wait, loads (9: lane 0 spins, the
// other lanes wait at __syncwarp; 10: the whole warp polls the counter)
template <bool WARP_POLL>
__device__ void red_w0(const Buf& b, double* v, uint32_t& ep) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x;
  for (int k = 0; k < 2; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) for (int k = 0; k < 2; ++k) s_red[k][warp] = v[k];
  __syncthreads();
  const uint32_t e = ep + 1;
  double* base = b.red + (e & 1) * 2 * STR;
  if (warp == 0) {
    for (int k = 0; k < 2; ++k) {
      double t = warp_sum(lane < NW ? s_red[k][lane] : 0.0);
      if (lane == 0) __stcg(base + k * STR + blockIdx.x, t);
    }
    __syncwarp();
    const uint32_t target = e * uint32_t(G);
    if (WARP_POLL) {
      if (lane == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(b.cnt) : "memory");
      while (true) {
        const uint32_t c = ld_acq(b.cnt);
        if (__all_sync(0xffffffffu, int32_t(c - target) >= 0)) break;
      }
    } else {
      if (lane == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(b.cnt) : "memory");
        while (int32_t(ld_acq(b.cnt) - target) < 0) {}
      }
      __syncwarp();
    }
    double2 p[2][4];
    for (int k = 0; k < 2; ++k)
      for (int m = 0; m < 4; ++m) {
        int bb = 64 * m + 2 * lane;
        p[k][m] = bb < G ? __ldcg(reinterpret_cast<const double2*>(base + k * STR + bb)) : make_double2(0, 0);
      }
    for (int k = 0; k < 2; ++k) {
      double t = 0.0;
      for (int m = 0; m < 4; ++m) t += p[k][m].x + p[k][m].y;
      t = warp_sum(t);
      if (lane == 0) s_res[k] = t;
    }
  }
  __syncthreads();
  v[0] = s_res[0]; v[1] = s_res[1];
  ep = e;
}

// variant 11/12: the arrival counter split over K lines (CTA b arrives on line
// b % K, K lanes of warp 0 poll the K lines) + one read of the slots
template <int K>
__device__ void red_cntk(const Buf& b, double* v, uint32_t& ep) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x;
  for (int k = 0; k < 2; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) for (int k = 0; k < 2; ++k) s_red[k][warp] = v[k];
  __syncthreads();
  const uint32_t e = ep + 1;
  double* base = b.red + (e & 1) * 2 * STR;
  if (warp < 2) {
    double t = warp_sum(lane < NW ? s_red[warp][lane] : 0.0);
    if (lane == 0) base[warp * STR + blockIdx.x] = t;
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0)
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(b.cnt + 32 * (blockIdx.x % K)) : "memory");
    // line k receives the CTAs b = k mod K: ceil((G - k) / K) per exchange
    const uint32_t per = lane < K ? uint32_t((G - lane + K - 1) / K) : 0u;
    const uint32_t target = e * per;
    while (true) {
      const uint32_t c = lane < K ? ld_acq(b.cnt + 32 * lane) : 0u;
      if (__all_sync(0xffffffffu, int32_t(c - target) >= 0)) break;
    }
  }
  __syncthreads();
  if (warp < 2) {
    double t = 0.0;
    for (int m = 0; m < STR / 64; ++m) {
      int bb = 64 * m + 2 * lane;
      double2 p = bb < G ? __ldcg(reinterpret_cast<const double2*>(base + warp * STR + bb)) : make_double2(0, 0);
      t += p.x + p.y;
    }
    t = warp_sum(t);
    if (lane == 0) s_res[warp] = t;
  }
  __syncthreads();
  v[0] = s_res[0]; v[1] = s_res[1];
  ep = e;
}

// variant 14/15/16: counter + loads (as 6, slot loads issued before the adds),
// thread 0 polling with D relaxed loads in flight, issued S cycles apart, then
// an acq_rel fence (17: D = 4 with ld.acquire polls, no fence)
template <int D, int S, bool ACQ>
__device__ void red_cnt_pipe(const Buf& b, double* v, uint32_t& ep) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x;
  const uint32_t e = ep + 1;
  double* base = b.red + (e & 1) * 2 * STR;
  for (int k = 0; k < 2; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) for (int k = 0; k < 2; ++k) s_red[k][warp] = v[k];
  __syncthreads();
  if (warp < 2) {
    double t = warp_sum(lane < NW ? s_red[warp][lane] : 0.0);
    if (lane == 0) __stcg(base + warp * STR + blockIdx.x, t);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(b.cnt) : "memory");
    const uint32_t target = e * uint32_t(G);
    uint32_t c[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      c[d] = ACQ ? ld_acq(b.cnt) : ld_rlx(b.cnt);
      if (d + 1 < D) {
        const long long t0 = clock64();
        while (clock64() - t0 < S) {}
      }
    }
    bool done = false;
    while (!done) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        if (!done) {
          if (int32_t(c[d] - target) >= 0) done = true;
          else c[d] = ACQ ? ld_acq(b.cnt) : ld_rlx(b.cnt);
        }
      }
    }
    if (!ACQ) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
  if (warp < 2) {
    double2 p[STR / 64];
    for (int m = 0; m < STR / 64; ++m) {
      int bb = 64 * m + 2 * lane;
      p[m] = bb < G ? __ldcg(reinterpret_cast<const double2*>(base + warp * STR + bb)) : make_double2(0, 0);
    }
    double t = 0.0;
    for (int m = 0; m < STR / 64; ++m) t += p[m].x + p[m].y;
    t = warp_sum(t);
    if (lane == 0) s_res[warp] = t;
  }
  __syncthreads();
  v[0] = s_res[0]; v[1] = s_res[1];
  ep = e;
}

// variant 20/21: the product's exchange (acquire poll, loads before the adds)
// with each CTA's slot padded to its own 32-byte sector (20) / 128-byte line (21)
// (no write sharing of slot lines between CTAs)
template <int PAD>
__device__ void red_cnt_pad(const Buf& b, double* v, uint32_t& ep) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x;
  const uint32_t e = ep + 1;
  double* base = b.red + (e & 1) * 2 * STR * PAD;
  for (int k = 0; k < 2; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) for (int k = 0; k < 2; ++k) s_red[k][warp] = v[k];
  __syncthreads();
  if (warp < 2) {
    double t = warp_sum(lane < NW ? s_red[warp][lane] : 0.0);
    if (lane == 0) __stcg(base + (warp * STR + blockIdx.x) * PAD, t);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(b.cnt) : "memory");
    const uint32_t target = e * uint32_t(G);
    while (int32_t(ld_acq(b.cnt) - target) < 0) {}
  }
  __syncthreads();
  if (warp < 2) {
    double p[STR / 32];
#pragma unroll
    for (int m = 0; m < STR / 32; ++m) {
      const int bb = 32 * m + lane;
      p[m] = bb < G ? __ldcg(base + (warp * STR + bb) * PAD) : 0.0;
    }
    double t = 0.0;
#pragma unroll
    for (int m = 0; m < STR / 32; ++m) t += p[m];
    t = warp_sum(t);
    if (lane == 0) s_res[warp] = t;
  }
  __syncthreads();
  v[0] = s_res[0]; v[1] = s_res[1];
  ep = e;
}

// variant 4: arrival counter; the last arriver sums and broadcasts (value + epoch) in one line
__device__ void red_last(const Buf& b, double* v, uint32_t& ep) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x;
  __shared__ int s_last;
  for (int k = 0; k < 2; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) for (int k = 0; k < 2; ++k) s_red[k][warp] = v[k];
  __syncthreads();
  const uint32_t e = ep + 1;
  double* base = b.red + (e & 1) * 2 * STR;
  uint64_t* bc = b.gs + (e & 1) * 4;                // broadcast: 2 values x (lo, hi)
  if (warp < 2) {
    double t = warp_sum(lane < NW ? s_red[warp][lane] : 0.0);
    if (lane == 0) base[warp * STR + blockIdx.x] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t old = atomicAdd(b.cnt, 1u);
    s_last = old == e * uint32_t(G) - 1;
  }
  __syncthreads();
  if (s_last) {
    if (warp < 2) {
      __threadfence();
      double t = 0.0;
      for (int m = 0; m < STR / 64; ++m) {
        int bb = 64 * m + 2 * lane;
        double2 p = bb < G ? __ldcg(reinterpret_cast<const double2*>(base + warp * STR + bb)) : make_double2(0, 0);
        t += p.x + p.y;
      }
      t = warp_sum(t);
      if (lane == 0) s_res[warp] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t tag = uint64_t(e) << 32;
      uint64_t b0 = __double_as_longlong(s_res[0]), b1 = __double_as_longlong(s_res[1]);
      __threadfence();
      st2(bc, tag | (b0 & 0xffffffffull), tag | (b0 >> 32));
      st2(bc + 2, tag | (b1 & 0xffffffffull), tag | (b1 >> 32));
    }
  } else if (threadIdx.x == 0) {
    uint64_t a0, a1, c0, c1;
    do {
      ld2(bc, a0, a1);
      ld2(bc + 2, c0, c1);
    } while ((a0 >> 32) != e || (a1 >> 32) != e || (c0 >> 32) != e || (c1 >> 32) != e);
    __threadfence();
    s_res[0] = __longlong_as_double((a1 << 32) | (a0 & 0xffffffffull));
    s_res[1] = __longlong_as_double((c1 << 32) | (c0 & 0xffffffffull));
  }
  __syncthreads();
  v[0] = s_res[0]; v[1] = s_res[1];
  ep = e;
}

__global__ void __launch_bounds__(NT, 1) k(Buf b, int variant, int reps) {
  cg::grid_group grid = cg::this_grid();
  int slot = 0;
  uint32_t ep = 0;
  double acc = 0.0;
  for (int r = 0; r < reps; ++r) {
    double v[2] = {1.0 + threadIdx.x, 2.0};
    if (variant == 0) red_cg(grid, b, v, slot);
    else if (variant == 1) red_flag<0>(b, v, ep);
    else if (variant == 2) red_flag<64>(b, v, ep);
    else if (variant == 3) red_cnt(b, v, ep);
    else if (variant == 5) red_flag<256>(b, v, ep);
    else if (variant == 6) red_cnt_rel<true>(b, v, ep);
    else if (variant == 7) red_cnt_rel<false>(b, v, ep);
    else if (variant == 8) grid.sync();
    else if (variant == 9) red_w0<false>(b, v, ep);
    else if (variant == 10) red_w0<true>(b, v, ep);
    else if (variant == 11) red_cntk<4>(b, v, ep);
    else if (variant == 12) red_cntk<8>(b, v, ep);
    else if (variant == 13) red_cntk<16>(b, v, ep);
    else if (variant == 14) red_cnt_pipe<1, 0, false>(b, v, ep);
    else if (variant == 15) red_cnt_pipe<2, 300, false>(b, v, ep);
    else if (variant == 16) red_cnt_pipe<4, 150, false>(b, v, ep);
    else if (variant == 17) red_cnt_pipe<4, 150, true>(b, v, ep);
    else if (variant == 18) red_cnt_pipe<8, 80, false>(b, v, ep);
    else if (variant == 19) red_cnt_pipe<1, 0, true>(b, v, ep);
    else if (variant == 20) red_cnt_pad<4>(b, v, ep);
    else if (variant == 21) red_cnt_pad<16>(b, v, ep);
    else red_last(b, v, ep);
    acc += v[0] + v[1];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) b.out[0] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  Buf b;
  cudaMalloc(&b.red, 2 * 2 * STR * 8 * 16);
  cudaMalloc(&b.gs, 2 * 2 * STR * 16);
  cudaMalloc(&b.cnt, 32 * 4 * 16);
  cudaMalloc(&b.out, 64);
  const char* names[] = {"cg grid.sync + loads", "flag poll", "flag poll + sleep 64", "counter + loads",
                         "counter, last arriver broadcasts", "flag poll + sleep 256",
                         "counter (release red) + loads", "counter barrier only", "cg grid.sync only",
                         "warp 0: lane 0 spins", "warp 0: whole warp polls",
                         "counter over 4 lines + loads", "counter over 8 lines + loads",
                         "counter over 16 lines + loads",
                         "pipe: 1 relaxed poll + fence", "pipe: 2 relaxed polls + fence",
                         "pipe: 4 relaxed polls + fence", "pipe: 4 acquire polls",
                         "pipe: 8 relaxed polls + fence", "pipe: 1 acquire poll (product)",
                         "product, slots padded to 32 B", "product, slots padded to 128 B"};
  for (int variant : {19, 20, 21}) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(b.gs, 0, 2 * 2 * STR * 16);
      cudaMemset(b.cnt, 0, 32 * 4 * 16);
      int reps = 2000;
      void* args[] = {&b, &variant, &reps};
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)k, dim3(sms), dim3(NT), args, 0, 0);
      cudaEventRecord(e1);
      cudaError_t err = cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double out;
      cudaMemcpy(&out, b.out, 8, cudaMemcpyDeviceToHost);
      if (rep == 2)
        printf("%-34s %6.2f us per reduce  (check %.6g, %s)\n", names[variant], ms * 1e3 / reps, out,
               cudaGetErrorString(err));
    }
  }
  return 0;
}
