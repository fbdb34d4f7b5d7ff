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
rep('''    if (mv) {                                       // partials of z, read after the barrier
      stage_x(z, sh);
      phase_a(plan_view(a, r0, r1), r0, r1, wrow, sh);
    }''', '''    SEG(7);
    if (mv) {                                       // partials of z, read after the barrier
      stage_x(z, sh);
      SEG(8);
      phase_a(plan_view(a, r0, r1), r0, r1, wrow, sh);
      SEG(9);
    }''')
rep('''      grid_reduce<2>(nz, a, sh);
      pending = true;''', '''      grid_reduce<2>(nz, a, sh);
      SEG(10);
      pending = true;''')
out = "/tmp/otn_cg_seg.cu"
open(out, "w").write(s)
subprocess.check_call([os.path.join(ROOT, "tools/build_ab.sh"), "seg", out])
