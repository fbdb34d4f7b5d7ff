"""One probe launch (for ncu): python tools/probe_one.py <what> <masked 0|1> <log2 gamma>."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402
from paper_2504_02067_b200._device import vptr  # noqa: E402

what, masked, lg = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
p = ot.workload("grid:64:l2sq:0")
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
from paper_2504_02067_b200._device import TELEMETRY  # noqa: E402
st = ot.mdot(dp, 2.0 ** 5, 2.0 ** lg).final_state
ncoop = sum(TELEMETRY.calls.get(k_, 0) for k_ in ("otn_newton", "otn_pcg", "otn_apply_F",
                                                   "otn_apply_pc", "otn_matvec", "otn_rmatvec"))
s = ot.DiscountedSystem.from_state(st)
k = s._ctx
x = torch.randn(k.ld, dtype=torch.float64, device="cuda")
out = k.vec()
mask = s._mask if masked else None
for _ in range(3):
    k.call("otn_probe", vptr(s._P), vptr(mask), vptr(s._cP), vptr(s._rP), vptr(x), vptr(out), what,
           int(os.environ.get("PROBE_REPS", "20")))
torch.cuda.synchronize()
print("coop_launches_before_probe", ncoop)
