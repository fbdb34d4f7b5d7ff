import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import load_traj
from paper_2504_02067_b200 import mdot, problems, MdotOptions
for name in sys.argv[1:]:
    meta, arr = load_traj(name)
    p = problems.workload(meta["spec"])
    dp = problems.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
    sol = mdot(dp, meta["gamma_i"], meta["gamma_f"])
    u, v = sol.final_state.u, sol.final_state.v
    du = u - arr["u"]; dv = v - arr["v"]
    sc = np.abs(arr["u"]).max()
    print(name, "raw du", np.abs(du).max() / sc, "dv", np.abs(dv).max() / np.abs(arr["v"]).max())
    print("  du mean", du.mean(), "du std", du.std(), "dv mean", dv.mean(), "dv std", dv.std())
    s = np.median(du)
    print("  gauge-fixed du", np.abs(du - s).max() / sc, "dv", np.abs(dv + s).max() / np.abs(arr["v"]).max())
    g = meta["stages"][-1]["gamma"]
    # log-plan difference on the support: (du_i + dv_j)
    print("  max |du_i + dv_j| (log-plan shift)", np.abs(du[:, None] + dv[None, :]).max())
    print("  ref P rowsum err vs ours", np.abs(sol.P.cpu().numpy().sum(1) - arr["P_rowsum"]).max() if hasattr(sol.P, 'cpu') else None)
