"""Per-sub-step cycles of the persistent launch's staging (CTA 0), per plan
mode, over one D2 solve:
    python tools/make_stage_build.py && OTN_LIB_AB=build/ab/libotn_stage.so python tools/stage_run.py"""
import ctypes
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402
from paper_2504_02067_b200 import _lib  # noqa: E402

lib = _lib.load()
p = ot.workload("grid:64:l2sq:0")
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
ot.mdot(dp, 2.0 ** 5, 2.0 ** 16)
buf = (ctypes.c_ulonglong * 40)()
lib.otn_dbg_stage(buf)
ot.mdot(dp, 2.0 ** 5, 2.0 ** 16)
lib.otn_dbg_stage(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(4, 10).astype(float) / 1.965e3   # us
names = ["stage_layout", "CSR extraction", "column counts + scan", "CSC placement",
         "compaction", "-", "-", "split / thread starts"]
launches = {0: 27, 2: 11, 3: 7}
for m in (0, 2, 3):
    print(f"mode {m}: per launch (us)")
    for i, nm in enumerate(names):
        if a[m][i] > 0:
            print(f"   {nm:24s} {a[m][i] / launches[m]:8.1f}")
