"""Print the stage trajectory of one golden case on the GPU next to the reference's."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402

name = sys.argv[1]
z = np.load(f"tests/golden/traj_{name}.npz", allow_pickle=True)
meta = json.loads(str(z["meta"]))
p = ot.workload(meta["spec"])
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
sol = ot.mdot(dp, meta["gamma_i"], meta["gamma_f"])
ref = [(s["gamma"], s["newton_steps"], s["cg_iters"]) for s in meta["stages"]]
got = [(it.gamma, it.stats.newton_steps, it.stats.cg_iters) for it in sol.iterations]
for k in range(max(len(ref), len(got))):
    a = ref[k] if k < len(ref) else ("", "", "")
    b = got[k] if k < len(got) else ("", "", "")
    print(f"{k:3d}  ref {a}   got {b}")
st = sol.final_state
print("du", float(np.abs(st.u - z["u"]).max() / np.abs(z["u"]).max()))
