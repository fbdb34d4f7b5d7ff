"""Bitwise A/B of two library builds on full solves: writes u, v, P row sums
and the CG counts of D2-L2^2 / D2-L1 / D3 / a point cloud solve to an .npz
(run once per build via OTN_LIB_AB, then compare the files)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402

out = {}
for spec in ("grid:64:l2sq:0", "grid:64:l1:0", "pix:4096:784:0", "pts:1024:2:0", "grid:32:l2sq:0"):
    p = ot.workload(spec)
    dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
    sol = ot.mdot(dp, 2.0 ** 5, 2.0 ** 16 if spec.startswith(("grid:64", "pix")) else 2.0 ** 12)
    st = sol.final_state
    out[spec + ":u"] = np.asarray(st.u)
    out[spec + ":v"] = np.asarray(st.v)
    out[spec + ":cg"] = np.array([i.stats.cg_iters for i in sol.iterations])
    out[spec + ":P"] = sol.P.sum(dim=1).cpu().numpy() if torch.is_tensor(sol.P) else sol.P.sum(axis=1)
np.savez(sys.argv[1], **out)
if len(sys.argv) > 2:
    a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
    diff = [k for k in a.files if not np.array_equal(a[k], b[k])]
    print("bitwise identical:", not diff, diff[:6])
