"""On-the-fly pair kernel pass times at n = 65536 (3-D points, gamma 2^10):
row LSE, column LSE, row P.w -- median of 7 after warm-up (A/B helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_02067_b200 import _lib, problems  # noqa: E402
from paper_2504_02067_b200.pointcloud import PointCloudCost  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
dev = torch.device("cuda", 0)
pc = problems.points_problem(n, 3, 0)
cost = PointCloudCost(pc, dev)
rng = np.random.default_rng(0)
u = cost.upload(np.log(pc.r) + 0.01 * rng.standard_normal(n))
v = cost.upload(np.log(pc.c) + 0.01 * rng.standard_normal(n))
w = cost.upload(rng.standard_normal(n))
out = cost.zeros(n)
for name, kw in (("row_lse", dict(op=_lib.PC_LSE, rows_first=True, colpot=v, rowpot=None)),
                 ("col_lse", dict(op=_lib.PC_LSE, rows_first=False, colpot=u, rowpot=None)),
                 ("row_dot", dict(op=_lib.PC_DOT, rows_first=True, colpot=v, rowpot=u, vec=w))):
    ts = []
    for rep in range(9):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cost.pass_(out=out, ng=-(2.0 ** 10), **kw)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts[2:]))
    print(f"{name}: {ms:.3f} ms  {float(n) * n / ms / 1e6:.0f} G entries/s")
