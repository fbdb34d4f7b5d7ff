"""One D2 L2^2 n=4096 solve for ncu (the k_coop launches are the profiled kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "grid:64:l2sq:0"
gf = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0 ** 16
p = ot.workload(spec)
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
sol = ot.mdot(dp, 2.0 ** 5, gf)
torch.cuda.synchronize()
print("stages", len(sol.iterations), "cg", sum(i.stats.cg_iters for i in sol.iterations))
