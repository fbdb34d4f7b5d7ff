"""Pair-kernel pass time by row count (the rows-per-warp choice in otn_pc.cu
launch_d was measured with this; rows are a prefix of the point set)."""
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
for na in (n, n // 2, n // 4, n // 8):
    for op, nm in ((_lib.PC_LSE, "lse"), (_lib.PC_DOT, "dot")):
        kw = dict(op=op, rowpot=u, colpot=v, vec=w, ng=-1024.0)
        cost.be.pass_(op, cost.Xt, na, cost.Yt, n, 3, cost.cmax, -1024.0, 0, v, None, 0.0, u, w,
                      None, None, 0, out, None)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            cost.be.pass_(op, cost.Xt, na, cost.Yt, n, 3, cost.cmax, -1024.0, 0, v, None, 0.0, u,
                          w, None, None, 0, out, None)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"na={na} {nm}: {ms:.3f} ms "
              f"{na * n / ms / 1e6:.1f} G/s", flush=True)
