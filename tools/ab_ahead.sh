for i in 1 2; do
for a in 0 1; do OTN_NO_AHEAD=$a timeout 300 python - <<'PY'
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
print("OTN_NO_AHEAD", os.environ["OTN_NO_AHEAD"], "median ms", round(1e3 * float(np.median(ts[2:])), 2), "min", round(1e3 * min(ts[2:]), 2))
PY
done; done
