"""D5 evidence: per-pass time of the on-the-fly pair kernel
at n = 2^20 (3-D uniform points) on ONE GPU -- the exact-C_max pass, a row
LSE pass, a row P.w pass, a column LSE pass.  A D5 solve is ~230 such passes
(D4's call pattern); on G GPUs each pass splits by rows with one n-vector
allreduce per column product (8 MB at n = 2^20, ~10-20 us over NVLink), so
the per-pass time over G is the scaling model.  Writes gpurun_out/r01_d5_pass.json
(kept as profiles/r01_d5_pass.json)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_02067_b200 import _lib, problems  # noqa: E402
from paper_2504_02067_b200.pointcloud import PointCloudCost  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 20
gamma = 2.0 ** 10
dev = torch.device("cuda", 0)
pc = problems.points_problem(n, 3, 0)
t0 = time.perf_counter()
cost = PointCloudCost(pc, dev)                 # one MAXD pass for the exact C_max
torch.cuda.synchronize()
t_cmax = time.perf_counter() - t0
rng = np.random.default_rng(0)
u = cost.upload(np.log(pc.r) + 0.01 * rng.standard_normal(n))
v = cost.upload(np.log(pc.c) + 0.01 * rng.standard_normal(n))
w = cost.upload(rng.standard_normal(n))
out = cost.zeros(n)
res = {"n": n, "dim": 3, "gamma": gamma, "entries_per_pass": float(n) * n, "cmax_pass_s": t_cmax}
for name, kw in (("row_lse", dict(op=_lib.PC_LSE, rows_first=True, colpot=v, rowpot=None)),
                 ("row_dot", dict(op=_lib.PC_DOT, rows_first=True, colpot=v, rowpot=u, vec=w)),
                 ("col_lse", dict(op=_lib.PC_LSE, rows_first=False, colpot=u, rowpot=None))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cost.pass_(out=out, ng=-gamma, **kw)
    e1.record()
    e1.synchronize()
    s = e0.elapsed_time(e1) / 1e3
    res[name + "_s"] = s
    res[name + "_entries_per_s"] = float(n) * n / s
    print(f"{name}: {s:.3f} s  {float(n) * n / s / 1e9:.1f} G entries/s", flush=True)
passes = 232                                   # D4 (n=65536, gamma 2^5 -> 2^10) pass count
per = np.mean([res["row_lse_s"], res["row_dot_s"], res["col_lse_s"]])
res["model"] = {"passes_per_solve_d4_pattern": passes, "solve_1gpu_s": passes * per,
                "solve_8gpu_s_compute_only": passes * per / 8}
print(json.dumps(res, indent=1))
os.makedirs("profiles", exist_ok=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/r01_d5_pass.json", "w"), indent=1)   # copied to profiles/
