"""Row log-sum-exp pass time on the D2 cost (n = 4096, 134 MB): cold (L2
flushed before each pass) and warm, at a dense and a sparse plan's
potentials; HBM GB/s over the 8 n^2 bytes a pass must read.  Run once per
build (OTN_LSE_BULK=1 selects the bulk-copy kernel; LSE_BENCH_NOSOLVE=1 skips
the solves that provide realistic potentials)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json  # noqa: E402

import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402
from paper_2504_02067_b200._device import vptr  # noqa: E402

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") \
    else 6650.0
p = ot.workload("grid:64:l2sq:0")
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
flush = torch.empty(512 << 20 >> 2, dtype=torch.float32, device="cuda")
print("config", ot.DualState(dp, 1.0)._ctx.config, flush=True)
for lg in (5, 10, 16):
    if os.environ.get("LSE_BENCH_NOSOLVE"):          # (kernel variants that cannot solve)
        import numpy as np
        st = ot.DualState(dp, 2.0 ** lg, u=np.log(p.r), v=np.log(p.c))
    else:
        st = ot.mdot(dp, 2.0 ** 5, 2.0 ** lg).final_state
    k = st._ctx
    out = k.vec()
    args = (st._dc.ptr(), st._ng, vptr(st._u), vptr(st._v), vptr(out))
    for cold in (True, False):
        ts = []
        for rep in range(30):
            if cold:
                flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            k.call("otn_lse_rows", *args)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts = sorted(ts)[5:-5]
        us = sum(ts) / len(ts)
        gbs = 8.0 * k.n * k.n / (us * 1e-6) / 1e9
        print(f"gamma=2^{lg} {'cold' if cold else 'warm'}: {us:6.1f} us  {gbs:7.0f} GB/s "
              f"({gbs / peak:.0%} of {peak:.0f})", flush=True)
