"""Time grid-level building blocks (probe modes) on a real plan (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2504_02067_b200 as ot
from paper_2504_02067_b200._device import vptr
p = ot.workload("grid:64:l2sq:0")
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
st = ot.mdot(dp, 2.0 ** 5, 2.0 ** 10).final_state
s = ot.DiscountedSystem.from_state(st)
k = s._ctx
x = torch.randn(k.ld, dtype=torch.float64, device="cuda")
out = k.vec()
for what in [int(a) for a in sys.argv[1:]]:
    reps = 2000
    def go():
        k.call("otn_probe", vptr(s._P), vptr(s._mask), vptr(s._cP), vptr(s._rP), vptr(x), vptr(out), what, reps)
    go(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); go(); e1.record(); e1.synchronize()
    print(f"what={what}: {e0.elapsed_time(e1) / reps * 1e3:.3f} us", flush=True)
if os.environ.get("DUMP"):
    import numpy as np
    d = out.cpu().numpy()[: 148 * 4].reshape(148, 4)
    print("per-reduce cycles [pre, sync, read, final-sync]: mean", d.mean(0).round(0).tolist(),
          "max", d.max(0).round(0).tolist(), "min", d.min(0).round(0).tolist())
