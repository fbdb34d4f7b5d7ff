"""Build build/ab/libotn_stage.so: otn_cg.cu with clock64 probes between the
sub-steps of a persistent launch's staging (CTA 0, thread 0, per plan mode),
read back by tools/stage_run.py (OTN_LIB_AB=build/ab/libotn_stage.so).
Diagnostic only."""
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


rep("__shared__ int s_mode;", '''__shared__ int s_mode;
__shared__ long long s_tst;
__device__ unsigned long long g_stage[4][10];
extern "C" int otn_dbg_stage(unsigned long long* host) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host, g_stage, sizeof(g_stage));
  static unsigned long long z[4][10];
  cudaMemcpyToSymbol(g_stage, z, sizeof(z));
  return 0;
}
#define STG(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) { const long long _t = clock64(); \\
  if (s_mode >= 0 && s_mode < 4) g_stage[s_mode][i] += _t - s_tst; s_tst = _t; } } while (0)''')
rep('''  stage_layout(a, r0, r1, a.wpart + int64_t(blockIdx.x) * a.ld);
  if (s_mode >= kPlanSparse) stage_sparse(a, r0, r1, a.wpart + int64_t(blockIdx.x) * a.ld, sh);''',
    '''  if (blockIdx.x == 0 && threadIdx.x == 0) s_tst = clock64();
  stage_layout(a, r0, r1, a.wpart + int64_t(blockIdx.x) * a.ld);
  STG(0);
  if (s_mode >= kPlanSparse) stage_sparse(a, r0, r1, a.wpart + int64_t(blockIdx.x) * a.ld, sh);
  STG(7);''')
rep('''  const int ulo = s_win_lo[0], W = s_win_hi[0] - ulo;
  for (int d = t; d <= W; d += NT) sp.cst[d] = 0;''', '''  STG(1);
  const int ulo = s_win_lo[0], W = s_win_hi[0] - ulo;
  for (int d = t; d <= W; d += NT) sp.cst[d] = 0;''')
rep('''  block_incl_scan(sp.cst, W, sh);                   // cst[d] = end of column d''',
    '''  block_incl_scan(sp.cst, W, sh);                   // cst[d] = end of column d
  STG(2);''')
rep('''    if (t == 0) sp.cst[W] = E;                      // cst[d] = start of column d''',
    '''    STG(3);
    if (t == 0) sp.cst[W] = E;                      // cst[d] = start of column d''')
rep('''  if (t == 0) cptr[s_nzc] = uint16_t(E);''', '''  STG(4);
  if (t == 0) cptr[s_nzc] = uint16_t(E);''')
out = "/tmp/otn_cg_stage.cu"
open(out, "w").write(s)
subprocess.check_call([os.path.join(ROOT, "tools/build_ab.sh"), "stage", out])
