import time, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2504_02067_b200 as ot
from paper_2504_02067_b200 import problems
for spec in ["grid:64:l2sq:0", "grid:64:l1:0"]:
    p = problems.workload(spec)
    pd = problems.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
    for k in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        sol = ot.mdot(pd, 2.0**5, 2.0**16)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        st = sol.final_state; st.set_targets(p.r, p.c)
        print(spec, f"{t1-t0:.4f}s", "stages", len(sol.iterations), "cg", sum(i.stats.cg_iters for i in sol.iterations), "err", st.grad_norm_l1(), flush=True)
