"""Time the on-the-fly point-cloud solve (D4-style) on one GPU."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402
from paper_2504_02067_b200 import problems  # noqa: E402
from paper_2504_02067_b200._device import TELEMETRY  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
lg = int(sys.argv[2]) if len(sys.argv) > 2 else 10
pc = problems.points_problem(n, 3, 0)
torch.cuda.synchronize()
TELEMETRY.reset()
t0 = time.perf_counter()
sol = ot.mdot(pc, 2.0 ** 5, 2.0 ** lg)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
st = sol.final_state
st.set_targets(pc.r, pc.c)
calls = TELEMETRY.calls
print(f"n={n} gamma_f=2^{lg}: {dt:.2f}s stages={len(sol.iterations)} "
      f"newton={sum(i.stats.newton_steps for i in sol.iterations)} "
      f"cg={sum(i.stats.cg_iters for i in sol.iterations)} passes={calls.get('otn_pc_pass', 0)} "
      f"err={st.grad_norm_l1():.3g} primal={sol.primal_cost:.10g}", flush=True)
# per-pass timing of one row DOT pass
from paper_2504_02067_b200 import _lib  # noqa: E402
cost = st._pc
w = cost.zeros(n)
out = cost.zeros(cost.rows)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for op, name in ((_lib.PC_DOT, "dot"), (_lib.PC_LSE, "lse")):
    cost.pass_(op, rows_first=True, out=out, ng=-2.0 ** lg, colpot=st._v, rowpot=st._u, vec=w)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        cost.pass_(op, rows_first=True, out=out, ng=-2.0 ** lg, colpot=st._v, rowpot=st._u, vec=w)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"  {name} pass: {ms:.2f} ms = {n * n / ms / 1e6:.1f} G entries/s", flush=True)
