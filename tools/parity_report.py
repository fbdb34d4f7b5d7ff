"""Parity report of the device solver against the reference's golden
trajectories (tests/golden/traj_*.npz): per-stage CG counts side by side,
u / v inf-norm-relative differences, primal, true-marginal error.

    python tools/parity_report.py [name-substring ...] [--json out.json]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import load_traj, traj_names  # noqa: E402


def rel_inf(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def main(argv):
    import torch

    import paper_2504_02067_b200 as ot
    out_json = None
    if "--json" in argv:
        i = argv.index("--json")
        out_json = argv[i + 1]
        argv = argv[:i] + argv[i + 2:]
    names = [n for n in traj_names() if not argv or any(a in n for a in argv)]
    rows = {}
    for name in names:
        meta, arr = load_traj(name)
        p = ot.workload(meta["spec"])
        prob = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c) if p.n >= 1024 else p
        sol = ot.mdot(prob, meta["gamma_i"], meta["gamma_f"],
                      opts=ot.MdotOptions(projector=meta.get("projector", "newton")))
        st = sol.final_state
        du, dv = rel_inf(st.u, arr["u"]), rel_inf(st.v, arr["v"])
        got = [it.stats.cg_iters for it in sol.iterations]
        ref = [s["cg_iters"] for s in meta["stages"]]
        ss = meta.get("self_spread", {})
        st.set_targets(p.r, p.c)
        err = st.grad_norm_l1()
        rows[name] = dict(stages=[len(got), len(ref)], cg_total=[sum(got), sum(ref)],
                          cg_ours=got, cg_ref=ref, cg_ref_det=ss.get("cg"),
                          newton=[sum(it.stats.newton_steps for it in sol.iterations),
                                  sum(s["newton_steps"] for s in meta["stages"])],
                          du=du, dv=dv, self_du=ss.get("du"), self_dv=ss.get("dv"),
                          primal_rel=abs(sol.primal_cost - meta["primal"]) / abs(meta["primal"]),
                          true_marginal_err=err, ops_equal=sol.report.ops == meta["ops"])
        r = rows[name]
        print(f"{name}: stages {r['stages']} cg {r['cg_total']} newton {r['newton']} "
              f"du={du:.3e} dv={dv:.3e} (ref self {ss.get('du', float('nan')):.1e}) "
              f"primal_rel={r['primal_rel']:.2e} err={err:.3e} ops_eq={r['ops_equal']}")
        if got != ref:
            diff = [(i, a, b) for i, (a, b) in enumerate(zip(got, ref)) if a != b]
            print("   differing stages (i, ours, ref):", diff)
    if out_json:
        with open(out_json, "w") as fh:
            json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
