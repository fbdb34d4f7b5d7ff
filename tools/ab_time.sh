#!/bin/bash
# Interleaved D2-L2^2 solve timing of library builds (wall clock around mdot
# with synchronizes, median of 10 after 2 warm-up solves, two rounds):
#   tools/ab_time.sh build/ab/libotn_base.so ""     ("" = the in-tree build)
for i in 1 2; do
for lib in "$@"; do OTN_LIB_AB=$lib timeout 300 python - <<'PY'
import os, sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_2504_02067_b200 as ot
p = ot.workload("grid:64:l2sq:0")
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
ts = []
for k in range(12):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ot.mdot(dp, 2.0**5, 2.0**16)
    torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print("lib", os.environ.get("OTN_LIB_AB") or "in-tree", "median ms", round(1e3 * float(np.median(ts[2:])), 2),
      "min", round(1e3 * min(ts[2:]), 2))
PY
done; done
