"""D5 on ONE GPU: a full on-the-fly solve at n = 2^20 3-D uniform
points, gamma 2^5 -> 2^10, with the true-marginal error and the rounded
plan's primal cost checked after return; writes gpurun_out/r01_d5_solve.json
(kept as profiles/r01_d5_solve.json).  ~10-15 min of GPU time."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402
from paper_2504_02067_b200._device import TELEMETRY  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 20
lg = int(sys.argv[2]) if len(sys.argv) > 2 else 10
pc = ot.points_problem(n, 3, 0)
TELEMETRY.reset()
torch.cuda.synchronize()
t0 = time.perf_counter()
sol = ot.mdot(pc, 2.0 ** 5, 2.0 ** lg)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
st = sol.final_state
st.set_targets(pc.r, pc.c)
err = st.grad_norm_l1()
res = {"n": n, "dim": 3, "gamma": [2.0 ** 5, 2.0 ** lg], "gpus": 1, "solve_s": dt,
       "stages": len(sol.iterations), "newton": sum(i.stats.newton_steps for i in sol.iterations),
       "cg": sum(i.stats.cg_iters for i in sol.iterations),
       "pair_passes": TELEMETRY.calls.get("otn_pc_pass", 0), "true_marginal_err": err,
       "eps_target_final_stage": sol.iterations[-1].eps_d, "primal_cost": sol.primal_cost,
       "error_bound": sol.error_bound,
       "per_stage": [{"gamma": it.gamma, "newton": it.stats.newton_steps, "cg": it.stats.cg_iters,
                      "wall_ms": it.wall_ms} for it in sol.iterations]}
print(json.dumps(res, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open(os.environ.get("D5_OUT", "gpurun_out/r02_d5_solve.json"), "w"), indent=1)
