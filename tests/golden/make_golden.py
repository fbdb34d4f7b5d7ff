"""Generate golden vectors from the REFERENCE solver (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--large]

Imports ``otnewton`` from ``/root/reference/pkg/src`` (read-only) and records,
for each workload spec, the reference's full trajectory (per-stage and
per-Newton-step counts, step sizes, discounts), its final potentials, costs
and op tallies, plus kernel-level outputs on seeded inputs.  Inputs are NOT
stored: tests regenerate them from the spec with
``paper_2504_02067_b200.problems.workload`` and this script asserts that those
generators reproduce the reference's inputs bit for bit (sha256 recorded).

With ``--verify-oracle`` it also runs ``oracle/otn_oracle.py`` on every case
and records whether the oracle reproduces the reference bit for bit.

``/root/reference`` does not exist on the GPU box; the outputs
(``tests/golden/*.npz``) are committed and travel with the repo.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import otnewton as ref  # noqa: E402
from otnewton import opcount as ref_opcount  # noqa: E402

from oracle import otn_oracle as orc  # noqa: E402
from paper_2504_02067_b200 import problems as mine  # noqa: E402

SMALL = [
    # (name, spec, gamma_i, gamma_f)
    ("grid4_l1_s0", "grid:4:l1:0", 2.0 ** 4, 2.0 ** 10),
    ("grid6_l2sq_s5", "grid:6:l2sq:5", 2.0 ** 4, 2.0 ** 10),
    ("grid8_l1_s3", "grid:8:l1:3", 2.0 ** 4, 2.0 ** 12),
    ("grid16_l1_s1", "grid:16:l1:1", 2.0 ** 5, 2.0 ** 14),
    ("grid16_l2sq_s1", "grid:16:l2sq:1", 2.0 ** 5, 2.0 ** 14),
    ("pts256_2d_s0", "pts:256:2:0", 2.0 ** 5, 2.0 ** 12),
    ("pts1024_2d_s0_fixed", "pts:1024:2:0", 2.0 ** 10, 2.0 ** 10),   # D1 (fixed gamma)
    ("pts1024_2d_s1_fixed", "pts:1024:2:1", 2.0 ** 10, 2.0 ** 10),
    ("pts1024_2d_s0_anneal", "pts:1024:2:0", 2.0 ** 5, 2.0 ** 14),   # D1 annealed
    ("pts1024_3d_s0", "pts:1024:3:0", 2.0 ** 5, 2.0 ** 10),
    ("grid32_l1_s0", "grid:32:l1:0", 2.0 ** 5, 2.0 ** 12),
    ("grid32_l2sq_s0", "grid:32:l2sq:0", 2.0 ** 5, 2.0 ** 12),
    ("pix256_784_s0", "pix:256:784:0", 2.0 ** 5, 2.0 ** 14),
]

# MdotOptions(projector="sinkhorn"): the log-domain Sinkhorn baseline branch
# (driver.py:218-223,277-279 -> oracles.py:243-265), several gamma stages each
SINKHORN = [
    ("sk_grid16_l1_s1", "grid:16:l1:1", 2.0 ** 5, 2.0 ** 10),
    ("sk_grid16_l2sq_s1", "grid:16:l2sq:1", 2.0 ** 5, 2.0 ** 12),
    ("sk_pts256_2d_s0", "pts:256:2:0", 2.0 ** 5, 2.0 ** 10),
    ("sk_pts1024_3d_s0", "pts:1024:3:0", 2.0 ** 5, 2.0 ** 9),
]

# ragged, mid-size cases (n = 1000 ... 3000, not a multiple of the 32-column
# padding or of the CTA counts); oracle-verified, GPU-checked, not re-run by
# the CPU suite (names start with "M")
MEDIUM = [
    ("M_grid45_l2sq_s2", "grid:45:l2sq:2", 2.0 ** 5, 2.0 ** 13),
    ("M_grid40_l1_s4", "grid:40:l1:4", 2.0 ** 5, 2.0 ** 12),
    ("M_pts2000_3d_s1", "pts:2000:3:1", 2.0 ** 5, 2.0 ** 11),
    ("M_pix1000_784_s1", "pix:1000:784:1", 2.0 ** 5, 2.0 ** 12),
    ("M_pts3000_2d_s2", "pts:3000:2:2", 2.0 ** 5, 2.0 ** 12),
]

LARGE = [
    ("D2_grid64_l1_s0", "grid:64:l1:0", 2.0 ** 5, 2.0 ** 16),
    ("D2_grid64_l2sq_s0", "grid:64:l2sq:0", 2.0 ** 5, 2.0 ** 16),
    ("D2_grid64_l2sq_s1", "grid:64:l2sq:1", 2.0 ** 5, 2.0 ** 16),
    ("D2_grid64_l2sq_s2", "grid:64:l2sq:2", 2.0 ** 5, 2.0 ** 16),
    ("D2_grid64_l2sq_s3", "grid:64:l2sq:3", 2.0 ** 5, 2.0 ** 16),
    ("D3_pix4096_784_s0", "pix:4096:784:0", 2.0 ** 5, 2.0 ** 16),
    ("D2_grid64_l1_s1", "grid:64:l1:1", 2.0 ** 5, 2.0 ** 16),
    ("D3_pix4096_784_s1", "pix:4096:784:1", 2.0 ** 5, 2.0 ** 16),
]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def ref_problem(spec):
    """Build the inputs with the reference's own generators where it has them."""
    kind, *rest = spec.split(":")
    if kind == "grid":
        side, metric, seed = int(rest[0]), rest[1], int(rest[2])
        n = side * side
        return ref.Problem(C=ref.gen_grid_cost(side, metric),
                           r=ref.gen_marginal(n, "smooth-random", seed),
                           c=ref.gen_marginal(n, "smooth-random", seed + 1))
    # point clouds: the reference has no generator; use ours, wrapped in its Problem
    p = mine.workload(spec)
    return ref.Problem(C=p.C, r=p.r, c=p.c)


def trajectory(sol):
    stages = []
    for it in sol.iterations:
        s = it.stats
        stages.append(dict(
            t=it.t, gamma=it.gamma, eps_d=it.eps_d, q_next=it.q_next,
            newton_steps=s.newton_steps, cg_iters=s.cg_iters,
            sinkhorn_steps=s.sinkhorn_steps, backtracks=s.backtracks,
            rho_final=s.rho_final, delta_min=s.delta_min,
            grad_norm_final=s.grad_norm_final, ops_n2=it.ops_n2,
            steps=[dict(cg_iters=st.cg_iters, alpha=st.alpha, backtracks=st.backtracks,
                        rho_final=st.rho_final, eta=st.eta, grad_before=st.grad_before,
                        grad_after=st.grad_after, delta=st.delta)
                   for st in s.steps]))
    return stages


def oracle_trajectory(run):
    stages = []
    for (t, g, eps, q, pr) in run.stages:
        stages.append(dict(
            t=t, gamma=g, eps_d=eps, q_next=q, newton_steps=pr.newton_steps,
            cg_iters=pr.cg_iters, sinkhorn_steps=pr.sinkhorn_steps,
            backtracks=pr.backtracks, rho_final=pr.rho_final, delta_min=pr.delta_min,
            grad_norm_final=pr.grad_norm_final,
            steps=[dict(cg_iters=s.cg_iters, alpha=s.alpha, backtracks=s.backtracks,
                        rho_final=s.rho_final, eta=s.eta, grad_before=s.grad_before,
                        grad_after=s.grad_after, delta=s.delta) for s in pr.steps]))
    return stages


def strip_ops(stages):
    return [{k: v for k, v in s.items() if k != "ops_n2"} for s in stages]


def run_case(name, spec, gi, gf, verify_oracle, projector="newton"):
    prob = ref_problem(spec)
    opts = ref.MdotOptions(projector=projector)
    p2 = mine.workload(spec)
    gens_equal = (np.array_equal(prob.C, p2.C) and np.array_equal(prob.r, p2.r)
                  and np.array_equal(prob.c, p2.c))
    assert gens_equal, f"{spec}: package generators differ from the reference's"
    ref_opcount.reset()
    t0 = time.monotonic()
    sol = ref.mdot(prob, gi, gf, opts=opts)
    wall = time.monotonic() - t0
    st = sol.final_state
    st.set_targets(prob.r, prob.c)
    true_err = st.grad_norm_l1()
    meta = dict(
        name=name, spec=spec, gamma_i=gi, gamma_f=gf, n=prob.n, projector=projector,
        sha_C=sha(prob.C), sha_r=sha(prob.r), sha_c=sha(prob.c),
        primal=sol.primal_cost, error_bound=sol.error_bound,
        dual_value=sol.report.dual_value_final, grad_norm_final=sol.report.grad_norm_final,
        true_marginal_err=true_err, ops=sol.report.ops, ref_wall_s=wall,
        stages=trajectory(sol),
        totals=dict(stages=len(sol.iterations),
                    newton=sum(i.stats.newton_steps for i in sol.iterations),
                    cg=sum(i.stats.cg_iters for i in sol.iterations),
                    backtracks=sum(i.stats.backtracks for i in sol.iterations)),
    )
    arrays = dict(u=st.u.copy(), v=st.v.copy(),
                  P_rowsum=sol.P.sum(axis=1), P_colsum=sol.P.sum(axis=0))
    # The reference's own reduction-order noise floor: rerun with
    # OTN_DETERMINISTIC=1 (fixed-order matvecs instead of BLAS, opcount.py:89-91)
    # and record how far the trajectory and potentials move.
    os.environ["OTN_DETERMINISTIC"] = "1"
    try:
        ref_opcount.reset()
        det = ref.mdot(ref.Problem(C=prob.C, r=prob.r, c=prob.c), gi, gf, opts=opts)
    finally:
        del os.environ["OTN_DETERMINISTIC"]
    du_det = float(np.abs(det.final_state.u - st.u).max() / np.abs(st.u).max())
    dv_det = float(np.abs(det.final_state.v - st.v).max() / np.abs(st.v).max())
    meta["self_spread"] = dict(
        stages=len(det.iterations),
        newton=[i.stats.newton_steps for i in det.iterations],
        cg=[i.stats.cg_iters for i in det.iterations],
        cg_total=sum(i.stats.cg_iters for i in det.iterations),
        du=du_det, dv=dv_det, primal=det.primal_cost)
    print(f"  self-spread (BLAS vs deterministic): stages {len(det.iterations)} "
          f"cg {meta['self_spread']['cg_total']} vs {meta['totals']['cg']}, du={du_det:.2e}")
    if prob.n <= 64:
        arrays["P"] = sol.P.copy()
    if verify_oracle:
        run = orc.mdot(prob.C, prob.r, prob.c, gi, gf, projector=projector)
        same = (np.array_equal(run.state.u, st.u) and np.array_equal(run.state.v, st.v)
                and run.primal == sol.primal_cost and run.ops == sol.report.ops
                and oracle_trajectory(run) == strip_ops(meta["stages"]))
        meta["oracle_bitwise"] = bool(same)
        print(f"  oracle bitwise identical: {same}")
    np.savez_compressed(os.path.join(HERE, f"traj_{name}.npz"),
                        meta=np.array(json.dumps(meta)), **arrays)
    print(f"{name}: n={prob.n} stages={meta['totals']['stages']} "
          f"newton={meta['totals']['newton']} cg={meta['totals']['cg']} "
          f"err={true_err:.3g} wall={wall:.2f}s")


def kernel_goldens():
    """Reference kernel outputs on seeded inputs (inputs regenerated in tests)."""
    from otnewton._kernels import log_plan_row_sums, materialize_plan, square_matvec
    from otnewton.newton import DiscountedSystem, newton_solve, pcg_solve
    out = {}
    rng = np.random.default_rng(9)
    n = 256 + 17
    K = rng.normal(size=(n, n)) * 10
    u = rng.normal(size=n)
    v = rng.normal(size=n)
    out["lse_K273"] = log_plan_row_sums(K, u, v)
    rng = np.random.default_rng(10)
    P = rng.random((259, 259))
    w = rng.random(259)
    out["sqmv_259"] = square_matvec(P, w)
    rng = np.random.default_rng(11)
    K = rng.normal(size=(7, 7))
    u = rng.normal(size=7)
    v = rng.normal(size=7)
    out["plan_7"] = materialize_plan(K, u, v)
    # discounted systems from seeded dual states on grid problems
    for n_, seed in ((32, 33), (64, 3), (256, 5)):
        C = ref.grid_points_cost(n_, "l1")
        r = ref.gen_marginal(n_, "smooth-random", seed)
        c = ref.gen_marginal(n_, "spiky-random", seed + 100)
        rs = np.random.default_rng(seed + 7)
        st = ref.DualState(ref.Problem(C=C, r=r, c=c), 4.0,
                           u=np.log(r) + 0.3 * rs.standard_normal(n_),
                           v=np.log(c) + 0.3 * rs.standard_normal(n_))
        out[f"sys{n_}_logr"] = st.log_rP.copy()
        out[f"sys{n_}_logc"] = st.log_cP.copy()
        sys_ = DiscountedSystem.from_state(st)
        out[f"sys{n_}_mu"] = sys_.diag_prc().copy()
        b = np.random.default_rng(seed + 1).standard_normal(n_) * 0.01
        for rho in (0.0, 0.9, 0.99):
            d, it = pcg_solve(sys_, rho, b, tol_l1=1e-12)
            out[f"sys{n_}_pcg{rho}_x"] = d
            out[f"sys{n_}_pcg{rho}_iters"] = np.array([it])
        g = b - b.mean()
        res = newton_solve(g, sys_, eta=0.05)
        out[f"sys{n_}_newton_d"] = res.d_u
        out[f"sys{n_}_newton_meta"] = np.array([res.rho_final, res.cg_iters,
                                                res.undiscounted_residual_l1])
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)
    print("kernels.npz:", len(out), "arrays")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--large", action="store_true", help="also the n=4096 D2/D3 cases")
    ap.add_argument("--medium", action="store_true", help="also the ragged mid-size cases")
    ap.add_argument("--only", default=None)
    ap.add_argument("--verify-oracle", action="store_true")
    args = ap.parse_args()
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count()))
    orc.set_threads(os.cpu_count())       # slab-parallel oracle: bit-identical results
    kernel_goldens()
    cases = ([c + ("newton",) for c in SMALL] + [c + ("sinkhorn",) for c in SINKHORN]
             + ([c + ("newton",) for c in MEDIUM] if args.medium else [])
             + ([c + ("newton",) for c in LARGE] if args.large else []))
    for name, spec, gi, gf, projector in cases:
        if args.only and args.only not in name:
            continue
        run_case(name, spec, gi, gf, args.verify_oracle, projector)


if __name__ == "__main__":
    main()
