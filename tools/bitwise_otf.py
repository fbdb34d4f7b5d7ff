"""Bitwise A/B of two library builds on on-the-fly (point-cloud) solves:
u, v and CG counts of 2-D / 3-D problems to an .npz (run per build via
OTN_LIB_AB, compare with the second argument when given)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402

out = {}
for n, d, gf in ((4096, 3, 2.0 ** 10), (2048, 2, 2.0 ** 12), (1000, 4, 2.0 ** 9)):
    pc = ot.points_problem(n, d, 0)
    sol = ot.mdot(pc, 2.0 ** 5, gf)
    key = f"otf{n}x{d}"
    out[key + ":u"] = np.asarray(sol.final_state.u)
    out[key + ":v"] = np.asarray(sol.final_state.v)
    out[key + ":cg"] = np.array([i.stats.cg_iters for i in sol.iterations])
    out[key + ":primal"] = np.array([sol.primal_cost])
np.savez(sys.argv[1], **out)
if len(sys.argv) > 2:
    a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
    diff = [k for k in a.files if not np.array_equal(a[k], b[k])]
    print("bitwise identical:", not diff, diff[:6])
