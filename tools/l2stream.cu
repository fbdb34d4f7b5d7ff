// Microbenchmark: per-SM streaming rate of short strided row spans that sit in
// L2 (the k_coop phase-A access pattern of a sparse plan), by copy mechanism.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/l2stream.cu -o build/l2stream
//   build/l2stream [span_doubles=768] [rows=28]
// Each CTA (one per SM) sums `rows` rows of `span` doubles (row stride 4096
// doubles) `reps` times; the sum is written out so nothing is elided.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int NT = 512;
constexpr int LD = 4096;

__device__ __forceinline__ void cp_async16(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

extern __shared__ __align__(128) double2 ring[];

// K1: per-thread cp.async ring, D rows deep, 16 B per thread per chunk.
template <int D>
__global__ void __launch_bounds__(NT, 1) k_cpasync(const double* P, int span, int rows, int reps, double* out) {
  const int t = threadIdx.x;
  const double* base = P + size_t(blockIdx.x) * rows * LD + 1024;
  const int nch = (span / 2 + NT - 1) / NT;            // <= 4
  const unsigned r0 = unsigned(__cvta_generic_to_shared(ring)) + 16u * t;
  const unsigned slot = 4u * NT * 16u;
  double2 acc = make_double2(0, 0);
  for (int rep = 0; rep < reps; ++rep) {
    auto fill = [&](int q, int s) {
      const double* src = base + size_t(q) * LD;
      for (int c = 0; c < nch; ++c) {
        const int j = 2 * (t + c * NT);
        if (j < span) cp_async16(r0 + s * slot + c * NT * 16, src + j);
      }
      cp_commit();
    };
    for (int d = 0; d < D - 1; ++d) { if (d < rows) fill(d, d); else cp_commit(); }
    for (int q = 0; q < rows; ++q) {
      if (q + D - 1 < rows) fill(q + D - 1, (q + D - 1) % D); else cp_commit();
      cp_wait<D - 1>();
      for (int c = 0; c < nch; ++c) {
        const int j = 2 * (t + c * NT);
        if (j < span) {
          const double2 v = ring[(q % D) * 4 * NT + c * NT + t];
          acc.x += v.x; acc.y += v.y;
        }
      }
    }
    __syncthreads();
  }
  out[blockIdx.x * NT + t] = acc.x + acc.y;
}

// K2: plain 16-byte loads, U rows in flight per thread (registers).
template <int U>
__global__ void __launch_bounds__(NT, 1) k_ldg(const double* P, int span, int rows, int reps, double* out) {
  const int t = threadIdx.x;
  const double* base = P + size_t(blockIdx.x) * rows * LD + 1024;
  double2 acc = make_double2(0, 0);
  for (int rep = 0; rep < reps; ++rep) {
    for (int c = 0; 2 * c * NT < span; ++c) {
      const int j = 2 * (t + c * NT);
      if (j >= span) continue;
      for (int q0 = 0; q0 < rows; q0 += U) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          v[u] = q0 + u < rows ? __ldcg(reinterpret_cast<const double2*>(base + size_t(q0 + u) * LD + j))
                               : make_double2(0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; }
      }
    }
  }
  out[blockIdx.x * NT + t] = acc.x + acc.y;
}

// K3: one bulk async copy per row (elected thread), mbarrier per slot, D deep.
__device__ __forceinline__ void mbar_init(unsigned bar, int cnt) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(bar), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}\n"
      ::"r"(bar), "r"(phase) : "memory");
}

template <int D>
__global__ void __launch_bounds__(NT, 1) k_bulk(const double* P, int span, int rows, int reps, double* out) {
  __shared__ __align__(8) unsigned long long bars[D];
  const int t = threadIdx.x;
  const double* base = P + size_t(blockIdx.x) * rows * LD + 1024;
  const unsigned ring0 = unsigned(__cvta_generic_to_shared(ring));
  const unsigned slot = unsigned(span) * 8u;
  if (t < D) mbar_init(unsigned(__cvta_generic_to_shared(&bars[t])), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int issued = 0, consumed = 0;
  const int total = reps * rows;
  auto issue = [&](int k) {
    const int s = k % D;
    const unsigned bar = unsigned(__cvta_generic_to_shared(&bars[s]));
    mbar_expect(bar, slot);
    bulk_g2s(ring0 + s * slot, base + size_t(k % rows) * LD, slot, bar);
  };
  if (t == 0) for (; issued < D && issued < total; ++issued) issue(issued);
  for (; consumed < total; ++consumed) {
    const int s = consumed % D;
    mbar_wait(unsigned(__cvta_generic_to_shared(&bars[s])), (consumed / D) & 1);
    const double2* row = ring + s * (span / 2);
    for (int j = t; j < span / 2; j += NT) { const double2 v = row[j]; acc.x += v.x; acc.y += v.y; }
    __syncthreads();   // slot free
    if (t == 0 && issued < total) { issue(issued); ++issued; }
  }
  out[blockIdx.x * NT + t] = acc.x + acc.y;
}


// K4: bulk-copy ring with full/empty mbarriers (producer = thread 0; each of
// the 16 consumer warps releases a slot after reading it).
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(bar) : "memory");
}
template <int D>
__global__ void __launch_bounds__(NT, 1) k_bulk2(const double* P, int span, int rows, int reps, double* out) {
  __shared__ __align__(8) unsigned long long full[D], empty[D];
  const int t = threadIdx.x, lane = t & 31;
  const double* base = P + size_t(blockIdx.x) * rows * LD + 1024;
  const unsigned ring0 = unsigned(__cvta_generic_to_shared(ring));
  const unsigned slot = unsigned(span) * 8u;
  if (t < D) {
    mbar_init(unsigned(__cvta_generic_to_shared(&full[t])), 1);
    mbar_init(unsigned(__cvta_generic_to_shared(&empty[t])), NT / 32);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int total = reps * rows;
  int issued = 0;
  auto issue = [&](int k) {
    const int s = k % D;
    if (k >= D) mbar_wait(unsigned(__cvta_generic_to_shared(&empty[s])), ((k / D) - 1) & 1);
    const unsigned bar = unsigned(__cvta_generic_to_shared(&full[s]));
    mbar_expect(bar, slot);
    bulk_g2s(ring0 + s * slot, base + size_t(k % rows) * LD, slot, bar);
  };
  if (t == 0) for (; issued < D - 1 && issued < total; ++issued) issue(issued);
  double2 acc = make_double2(0, 0);
  for (int c = 0; c < total; ++c) {
    if (t == 0 && issued < total) { issue(issued); ++issued; }
    const int s = c % D;
    mbar_wait(unsigned(__cvta_generic_to_shared(&full[s])), (c / D) & 1);
    const double2* row = ring + s * (span / 2);
    for (int j = t; j < span / 2; j += NT) { const double2 v = row[j]; acc.x += v.x; acc.y += v.y; }
    __syncwarp();
    if (lane == 0) mbar_arrive(unsigned(__cvta_generic_to_shared(&empty[s])));
  }
  out[blockIdx.x * NT + t] = acc.x + acc.y;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main(int argc, char** argv) {
  const int span = argc > 1 ? atoi(argv[1]) : 768;
  const int rows = argc > 2 ? atoi(argv[2]) : 28;
  const int G = 148, reps = 200;
  double *P, *out;
  cudaMalloc(&P, size_t(G) * rows * LD * 8 + (1 << 20));
  cudaMemset(P, 0, size_t(G) * rows * LD * 8);
  cudaMalloc(&out, G * NT * 8);
  const double bytes = double(G) * rows * span * 8.0 * reps;
  const int smem = 200 * 1024;
  auto rep = [&](const char* name, float ms) {
    printf("%-14s span=%5d rows=%3d  %8.2f us/pass  %7.2f TB/s  %6.1f GB/s/SM  err=%s\n", name, span, rows,
           ms * 1e3 / reps, bytes / (ms * 1e-3) / 1e12, bytes / (ms * 1e-3) / 1e9 / G,
           cudaGetErrorString(cudaGetLastError()));
  };
#define CPA(D)                                                                                  \
  cudaFuncSetAttribute(k_cpasync<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);       \
  rep("cpasync D=" #D, timeit([&] { k_cpasync<D><<<G, NT, smem>>>(P, span, rows, reps, out); }));
  CPA(2) CPA(3) CPA(5) CPA(6)
#define LDG(U) rep("ldg U=" #U, timeit([&] { k_ldg<U><<<G, NT>>>(P, span, rows, reps, out); }));
  LDG(1) LDG(4) LDG(8) LDG(16)
#define BULK(D)                                                                                 \
  if (D * span * 8 <= smem) {                                                                   \
    cudaFuncSetAttribute(k_bulk<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);        \
    rep("bulk D=" #D, timeit([&] { k_bulk<D><<<G, NT, smem>>>(P, span, rows, reps, out); }));  \
  }
  BULK(4) BULK(16)
#define BULK2(D)                                                                                \
  if (D * span * 8 <= smem) {                                                                   \
    cudaFuncSetAttribute(k_bulk2<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);       \
    rep("bulk2 D=" #D, timeit([&] { k_bulk2<D><<<G, NT, smem>>>(P, span, rows, reps, out); })); \
  }
  BULK2(2) BULK2(4) BULK2(6) BULK2(8) BULK2(16) BULK2(24)
  return 0;
}
