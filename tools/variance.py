"""Per-solve wall-time variance of the D2 headline solve (diagnostic)."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402
from paper_2504_02067_b200._device import TELEMETRY  # noqa: E402

p = ot.workload("grid:64:l2sq:0")
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
for _ in range(3):
    ot.mdot(dp, 2.0 ** 5, 2.0 ** 16)
for mode in ("gc-on", "gc-off"):
    if mode == "gc-off":
        gc.disable()
    ts, cs = [], []
    for _ in range(8):
        TELEMETRY.reset()
        TELEMETRY.time_coop = True
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ot.mdot(dp, 2.0 ** 5, 2.0 ** 16)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
        cs.append(sum(ms for (ms, *_r) in TELEMETRY.coop))
        TELEMETRY.time_coop = False
    print(mode, "wall", [f"{t:.0f}" for t in ts], "coop", [f"{c:.0f}" for c in cs], flush=True)
gc.enable()
