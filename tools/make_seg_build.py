"""Build build/ab/libotn_seg.so: otn_cg.cu with clock64 probes between the
segments of the CG iteration (CTA 0, thread 0, accumulated per plan mode),
read back by tools/seg_run.py (OTN_LIB_AB=build/ab/libotn_seg.so).
Diagnostic only; the probes add a few global read-modify-writes per iteration."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
s = open(os.path.join(ROOT, "paper_2504_02067_b200/csrc/otn_cg.cu")).read()


def rep(old, new):
    global s
    if s.count(old) != 1:
        sys.exit(f"anchor not found once: {old[:60]!r}")
    s = s.replace(old, new)


rep("struct PcgOut {", '''__device__ unsigned long long g_seg[4][12];       // [plan mode][segment] cycles
extern "C" int otn_dbg_seg(unsigned long long* host) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host, g_seg, sizeof(g_seg));
  static unsigned long long z[4][12];
  cudaMemcpyToSymbol(g_seg, z, sizeof(z));
  return 0;
}
#define SEG(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) { const long long _t = clock64(); \\
  g_seg[s_mode][i] += _t - tseg; tseg = _t; } } while (0)

struct PcgOut {''')
rep('''  for (int64_t k = 1; k <= max_iters; ++k) {
    // p.q = sum_i rP_i p_i^2''', '''  long long tseg = clock64();
  for (int64_t k = 1; k <= max_iters; ++k) {
    SEG(0);
    // p.q = sum_i rP_i p_i^2''')
rep('''      a2_sums(a, sh);
      __syncthreads();                              // publishes sh.a2''', '''      a2_sums(a, sh);
      SEG(1);
      __syncthreads();                              // publishes sh.a2
      SEG(2);''')
rep('''      wq = a2_tail(a, a.wc, sh, beta, wreg, cPj);
    }''', '''      wq = a2_tail(a, a.wc, sh, beta, wreg, cPj);
      SEG(3);
    }''')
rep('''      grid_reduce<2>(sums, a, sh);             // also publishes a.wc
      phase_b(plan_view(a, r0, r1), a.wc, r0, r1, sh);   // ends with a barrier''', '''      grid_reduce<2>(sums, a, sh);             // also publishes a.wc
      SEG(4);
      phase_b(plan_view(a, r0, r1), a.wc, r0, r1, sh);   // ends with a barrier
      SEG(5);''')
rep('''    if (mv && !anchor) {                            // partials of z, read after the barrier
      stage_x(z, sh);
      phase_a(plan_view(a, r0, r1), r0, r1, wrow, sh);
    }''', '''    SEG(7);
    if (mv && !anchor) {                            // partials of z, read after the barrier
      stage_x(z, sh);
      SEG(8);
      phase_a(plan_view(a, r0, r1), r0, r1, wrow, sh);
      SEG(9);
    }''')
rep('''    if (split && !anchor) {
      grid_reduce<2>(nz, a, sh);
      pending = true;''', '''    if (split && !anchor) {
      grid_reduce<2>(nz, a, sh);
      SEG(10);
      pending = true;''')
# per-CTA work between exchanges and wait inside them (thread 0), per plan mode
rep('''__shared__ uint32_t s_ep;''', '''__shared__ uint32_t s_ep;
__shared__ long long s_tdone;
__shared__ int s_dbgm;
__device__ unsigned long long g_work[4][256], g_wait[4][256], g_nex[4][256];
extern "C" int otn_dbg_cta(unsigned long long* host) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host, g_work, sizeof(g_work));
  cudaMemcpyFromSymbol(host + 1024, g_wait, sizeof(g_wait));
  cudaMemcpyFromSymbol(host + 2048, g_nex, sizeof(g_nex));
  static unsigned long long z[4][256];
  cudaMemcpyToSymbol(g_work, z, sizeof(z));
  cudaMemcpyToSymbol(g_wait, z, sizeof(z));
  cudaMemcpyToSymbol(g_nex, z, sizeof(z));
  return 0;
}''')
rep('''    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
    const uint32_t target = e * uint32_t(G);
    while (int32_t(ld_acquire_u32(cnt) - target) < 0) {
    }''', '''    const long long _ta = clock64();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
    const uint32_t target = e * uint32_t(G);
    while (int32_t(ld_acquire_u32(cnt) - target) < 0) {
    }
    const long long _td = clock64();
    if (s_tdone != 0 && s_dbgm >= 0 && s_dbgm < 4) {
      g_work[s_dbgm][blockIdx.x] += _ta - s_tdone;
      g_wait[s_dbgm][blockIdx.x] += _td - _ta;
      g_nex[s_dbgm][blockIdx.x] += 1;
    }
    s_tdone = _td;''')
rep('''    s_mode = a.part[G + 1];''', '''    s_mode = a.part[G + 1];
    s_tdone = 0;
    s_dbgm = s_mode;''')
out = "/tmp/otn_cg_seg.cu"
open(out, "w").write(s)
subprocess.check_call([os.path.join(ROOT, "tools/build_ab.sh"), "seg", out])
