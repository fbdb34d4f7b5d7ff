"""Record the reference's primitive-call mix for a bench workload (test infra).

    python oracle/callmix.py grid:64:l2sq:0 32 65536 > tests/golden/callmix_D2_grid64_l2sq_s0.json

Runs the bit-exact oracle once (the reference's own call pattern) and counts
calls of each dense primitive: LSE passes, plan materializations, (P*P)w,
dgemv-N, dgemv-T, rounding.  bench.py's CPU baseline times a bounded sample
of each primitive on the host cores and scales by these counts.
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import otn_oracle as orc  # noqa: E402
from paper_2504_02067_b200 import problems  # noqa: E402


def main():
    spec, gi, gf = sys.argv[1], float(sys.argv[2]), float(sys.argv[3])
    p = problems.workload(spec)
    orc.CALLS.clear()
    t0 = time.monotonic()
    run = orc.mdot(p.C, p.r, p.c, gi, gf)
    wall = time.monotonic() - t0
    st = run.state
    st.r, st.c = p.r, p.c
    print(json.dumps({"spec": spec, "gamma_i": gi, "gamma_f": gf, "n": p.n,
                      "calls": dict(orc.CALLS), "oracle_wall_s": wall,
                      "host_cores": os.cpu_count(), "true_marginal_err": st.gnorm(),
                      "stages": len(run.stages),
                      "cg": sum(pr.cg_iters for (_, _, _, _, pr) in run.stages)}, indent=1))


if __name__ == "__main__":
    main()
