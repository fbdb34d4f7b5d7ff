"""Per-launch profile of the persistent solver over one solve: plan mode, rows
per CTA, HVPs and microseconds per HVP (diagnostic; synchronizes per launch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402
from paper_2504_02067_b200._device import TELEMETRY  # noqa: E402
from paper_2504_02067_b200 import newton as nt  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "grid:64:l2sq:0"
gf = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0 ** 16
p = ot.workload(spec)
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
ot.mdot(dp, 2.0 ** 5, gf)          # warm
rows = []


def wrap(orig, sys_pos):
    def wrapped(*a, **kw):
        TELEMETRY.time_coop = True
        n0 = len(TELEMETRY.coop)
        res = orig(*a, **kw)
        ms, h, dv, n, *_ = TELEMETRY.coop[n0]
        sys_ = a[sys_pos]
        k = sys_._ctx
        lay = np.zeros(k.coop_blocks + 2, dtype=np.int32)
        k.call("otn_coop_layout", lay.ctypes.data)
        m = sys_._mask.cpu().numpy()
        rows.append((int(lay[-1]), int(np.diff(lay[:-1]).max()), int(m[:, -1].sum()), h, ms * 1e3))
        return res
    return wrapped


nt._newton_device = wrap(nt._newton_device, 1)            # (grad_u, sys, ...)
nt._newton_step_device = wrap(nt._newton_step_device, 1)  # (state, sys, ...)
sol = ot.mdot(dp, 2.0 ** 5, gf)
tot = sum(r[4] for r in rows)
print(f"{'mode':>4} {'maxrows':>7} {'nnz':>9} {'hvps':>5} {'us':>9} {'us/hvp':>7}")
for r in rows:
    print(f"{r[0]:4d} {r[1]:7d} {r[2]:9d} {r[3]:5d} {r[4]:9.1f} {r[4] / max(r[3], 1):7.2f}")
for mode in (0, 1, 2, 3):
    sel = [r for r in rows if r[0] == mode]
    if sel:
        h = sum(r[3] for r in sel)
        us = sum(r[4] for r in sel)
        print(f"mode {mode}: launches {len(sel)} hvps {h} total {us / 1e3:.2f} ms  "
              f"{us / max(h, 1):.2f} us/hvp")
print(f"total k_coop {tot / 1e3:.2f} ms over {len(rows)} launches")
