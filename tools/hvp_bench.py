"""Micro-benchmark of the persistent HVP kernel on real D2 plans (per gamma).

For each gamma in the annealing schedule of the D2 L2^2 s0 solve: snapshot the
plan, report segment density, and time single-HVP launches (apply_F) and a
fixed-iteration PCG with / without zero-segment skipping.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402
from paper_2504_02067_b200 import newton  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "grid:64:l2sq:0"
p = ot.workload(spec)
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
n = p.n
nn8 = n * n * 8.0


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


for lg in (8, 10, 12, 13, 14, 15, 16):
    st = ot.mdot(dp, 2.0 ** 5, 2.0 ** lg).final_state
    sysd = ot.DiscountedSystem.from_state(st)
    mask = sysd._mask
    m = mask.cpu().numpy().view(np.uint64)
    bits = sum(bin(int(w)).count("1") for w in m.ravel())
    dens = bits / (n * ((n + 63) // 64))
    d = torch.randn(sysd._ctx.ld, dtype=torch.float64, device="cuda")
    d[n:] = 0
    out = []
    for use_mask in (True, False):
        sysd._mask = mask if use_mask else None
        t_hvp = timed(lambda: sysd.apply_F(0.9, d), 20)
        b = d.clone()
        t0 = time.perf_counter()
        try:
            x, k = newton.pcg_solve(sysd, 0.999, b, 1e-300, max_iters=200)
        except ot.errors.NonconvergenceError:
            k = 200
        torch.cuda.synchronize()
        t_cg = (time.perf_counter() - t0) * 1e3
        out.append((t_hvp, t_cg / 200))
    print(f"gamma=2^{lg:2d} seg_density={dens:5.3f}  apply_F masked {out[0][0]*1e3:7.1f} us "
          f"dense {out[1][0]*1e3:7.1f} us | CG iter masked {out[0][1]*1e3:7.1f} us dense "
          f"{out[1][1]*1e3:7.1f} us | dense GB/s {2*nn8/out[1][1]/1e6:7.0f}", flush=True)
