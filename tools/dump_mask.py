"""Save the plan segment mask (and row spans) of the D2 system at one gamma (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402

spec = sys.argv[1]
os.makedirs("gpurun_out", exist_ok=True)
p = ot.workload(spec)
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
out = {}
for lg in [int(a) for a in sys.argv[2:]]:
    st = ot.mdot(dp, 2.0 ** 5, 2.0 ** lg).final_state
    s = ot.DiscountedSystem.from_state(st)
    out[f"mask_{lg}"] = s._mask.cpu().numpy()
    out[f"P_{lg}"] = s._P[:, : p.n].cpu().numpy().astype(np.float32)
np.savez_compressed(f"gpurun_out/mask_{spec.replace(':', '_')}.npz", **out)
print("saved")
