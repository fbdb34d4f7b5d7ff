"""cProfile of one D2 L2^2 solve (device-resident cost): where host time goes."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402

p = ot.workload("grid:64:l2sq:0")
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
for _ in range(2):
    ot.mdot(dp, 2.0 ** 5, 2.0 ** 16)
torch.cuda.synchronize()
t0 = time.perf_counter()
ot.mdot(dp, 2.0 ** 5, 2.0 ** 16)
torch.cuda.synchronize()
print("wall", time.perf_counter() - t0)
pr = cProfile.Profile()
pr.enable()
ot.mdot(dp, 2.0 ** 5, 2.0 ** 16)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats(os.environ.get("SORT", "tottime")).print_stats(int(os.environ.get("TOP", "45")))
