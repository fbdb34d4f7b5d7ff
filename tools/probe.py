"""Time the persistent solver's building blocks on a real D2 plan (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402
from paper_2504_02067_b200._device import vptr  # noqa: E402

p = ot.workload(sys.argv[1] if len(sys.argv) > 1 else "grid:64:l2sq:0")
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
NAMES = ["grid.sync", "grid_reduce<2>", "phase A", "phase B", "A+sync+A2+sync", "full HVP"]
for lg in [int(a) for a in (sys.argv[2:] or ["10", "16"])]:
    st = ot.mdot(dp, 2.0 ** 5, 2.0 ** lg).final_state
    s = ot.DiscountedSystem.from_state(st)
    k = s._ctx
    x = torch.randn(k.ld, dtype=torch.float64, device="cuda")
    out = k.vec()
    for mask in (s._mask, None):
        row = []
        for what in range(6):
            reps = 400
            def go():
                k.call("otn_probe", vptr(s._P), vptr(mask), vptr(s._cP), vptr(s._rP), vptr(x),
                       vptr(out), what, reps)
            go()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            go()
            e1.record()
            e1.synchronize()
            row.append(e0.elapsed_time(e1) / reps * 1e3)
        print(f"gamma=2^{lg} {'masked' if mask is not None else 'dense '}: " +
              "  ".join(f"{n} {t:6.2f}us" for n, t in zip(NAMES, row)), flush=True)
