"""End-to-end parity of the B200 ``mdot`` against the reference's own trajectories.

Golden trajectories come from the reference package (tests/golden/make_golden.py).
Gates:
  strict  — wherever the reference reproduces itself (BLAS vs its deterministic
            mode: identical per-stage counts, potentials within 1e-9): identical
            stage count, identical per-stage Newton-step and CG-iteration counts,
            identical op tallies, u and v within max(1e-10, SPREAD_X x the
            reference's own spread) (inf-norm relative);
  spread  — where the reference does not reproduce itself to 1e-9, and the
            order-sensitive D2-L2^2 class (seed 0:
            789 vs 785 CG in stage 14, u within 3.4e-11): identical gamma
            schedule and Newton counts, each stage's CG count within that stage's
            det-vs-BLAS difference or, for the D2-L2^2 class, within the class's
            largest relative det-vs-BLAS difference (per stage and in total, over
            every seed of the class), u and v within max(1e-10, SPREAD_X x
            its self-spread),
            primal within 1e-9 relative, true-marginal error <= 1e-6 at full size.
"""

import numpy as np
import pytest

from conftest import load_traj, traj_names
from paper_2504_02067_b200 import MdotOptions, mdot, opcount, problems

pytestmark = pytest.mark.gpu

# Potentials are compared within SPREAD_X times the reference's own
# reduction-order spread (BLAS vs OTN_DETERMINISTIC=1, meta['self_spread']).
# The device is a third summation order (fixed trees, pipelined CG with the
# column sums re-anchored every kRefresh iterations); the achieved multiples
# are logged per case (profiles/r02_parity_gates.txt) -- most are below 10.
SPREAD_X = 100

# Configuration classes whose CG counts move under any change of summation
# order (SURVEY.md §6 "Measured noise floor": the n = 4096 squared-L2 grid --
# the reference's own reorderings differ by up to 4 CG in a stage at n = 4096
# and 7 at n = 1024, even where a given seed's two runs happen to agree).
# Their goldens are held to the spread gate, with the class's spread: the
# largest relative BLAS-vs-deterministic difference the reference shows on any
# seed of the class (per stage and in total).
ORDER_SENSITIVE = ("grid:64:l2sq",)


def config_class(meta):
    return meta["spec"].rsplit(":", 1)[0]


def class_spread(cls):
    """(per-stage, total) relative CG spread of the reference over every golden
    of the class: max |det - BLAS| / BLAS."""
    rel_stage, rel_total = 0.0, 0.0
    for name in traj_names():
        meta, _ = load_traj(name)
        ss = meta.get("self_spread")
        if config_class(meta) != cls or ss is None:
            continue
        ref = [s["cg_iters"] for s in meta["stages"]]
        for a, b in zip(ss["cg"], ref):
            rel_stage = max(rel_stage, abs(a - b) / max(b, 1))
        rel_total = max(rel_total, abs(ss["cg_total"] - sum(ref)) / max(sum(ref), 1))
    return rel_stage, rel_total


def gate(meta):
    """strict iff the reference is reproducible against itself on this case
    (BLAS vs OTN_DETERMINISTIC=1 give identical per-stage counts and potentials
    within 1e-9, meta['self_spread']) and the configuration is not an
    order-sensitive class."""
    ss = meta.get("self_spread")
    if ss is None or config_class(meta) in ORDER_SENSITIVE:
        return "spread"
    same = (ss["stages"] == len(meta["stages"])
            and ss["cg"] == [s["cg_iters"] for s in meta["stages"]]
            and ss["newton"] == [s["newton_steps"] for s in meta["stages"]])
    if same and ss["du"] < 1e-9 and ss["dv"] < 1e-9:
        return "strict"
    # the reference's trajectory is not reproducible against itself (e.g. L1
    # grids near the frozen-link regime, README "Numerical envelope"): only the
    # solution quality is comparable
    return "chaotic" if max(ss["du"], ss["dv"]) > 1e-6 else "spread"


def rel_inf(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def device_problem(prob):
    import torch
    return problems.Problem(C=torch.from_numpy(prob.C).cuda(), r=prob.r, c=prob.c,
                            label=prob.label)


def run_case(name, on_device=False):
    meta, arr = load_traj(name)
    prob = problems.workload(meta["spec"])
    if on_device:
        prob = device_problem(prob)
    opcount.reset()
    sol = mdot(prob, meta["gamma_i"], meta["gamma_f"],
               opts=MdotOptions(projector=meta.get("projector", "newton")))
    return meta, arr, prob, sol


def check(meta, arr, sol, name):
    g = gate(meta)
    print(f"{name}: gate={g}")
    ss = meta.get("self_spread", {})
    st = sol.final_state
    if g != "chaotic":
        assert len(sol.iterations) == len(meta["stages"]), "stage count"
    got_cg = [it.stats.cg_iters for it in sol.iterations]
    ref_cg = [s["cg_iters"] for s in meta["stages"]]
    got_newton = [it.stats.newton_steps for it in sol.iterations]
    ref_newton = [s["newton_steps"] for s in meta["stages"]]
    du, dv = rel_inf(st.u, arr["u"]), rel_inf(st.v, arr["v"])
    if g == "strict":
        # identical discrete trajectory, potentials to 1e-10 (or SPREAD_X x the
        # reference's own spread where that is larger, e.g. 2e-9 on grid16_l2sq)
        tol = max(1e-10, SPREAD_X * ss.get("du", 0.0), SPREAD_X * ss.get("dv", 0.0))
        assert [it.gamma for it in sol.iterations] == [s["gamma"] for s in meta["stages"]]
        assert got_newton == ref_newton, (got_newton, ref_newton)
        assert got_cg == ref_cg, (got_cg, ref_cg)
        got_sk = [it.stats.sinkhorn_steps for it in sol.iterations]
        assert got_sk == [s["sinkhorn_steps"] for s in meta["stages"]], got_sk
        assert sol.report.ops == meta["ops"]
        assert du <= tol and dv <= tol, (du, dv, tol)
        assert sol.primal_cost == pytest.approx(meta["primal"], rel=1e-9, abs=1e-14)
    elif g == "chaotic":
        # The reference does not reproduce itself here (BLAS vs deterministic:
        # per-stage Newton/CG counts differ from the first frozen-link stage on,
        # potentials by > 1e-6), and the adaptive annealing step then picks a
        # different gamma schedule (grid32_l1_s0: 16 stages in both reference
        # runs, 16-19 on the device depending on the reduction trees).  Only
        # solution quality is comparable: the same final gamma, the cost within
        # the annealing guarantee of the reference's, the true-marginal error no
        # worse than the last stage's projection tolerance.
        assert sol.iterations[-1].gamma == meta["stages"][-1]["gamma"]
        assert abs(sol.primal_cost - meta["primal"]) <= meta["error_bound"]
        eps_last = meta["stages"][-1]["eps_d"]
        st.set_targets(sol.final_state.problem.r, sol.final_state.problem.c)
        assert st.grad_norm_l1() <= max(eps_last, 2 * meta["true_marginal_err"])
    else:
        # inside the reference's own BLAS-vs-deterministic spread (BASELINE.md
        # section 2): the same gamma schedule and Newton-step counts, every
        # stage's CG count within that stage's det-vs-BLAS difference (0 where
        # the reference reproduces itself), the CG total within the reference's
        # own total difference, u and v within SPREAD_X x the reference's own spread.
        assert [it.gamma for it in sol.iterations] == [s["gamma"] for s in meta["stages"]]
        assert got_newton == ref_newton, (got_newton, ref_newton)
        det_cg = ss["cg"]
        rel_stage, rel_total = (class_spread(config_class(meta))
                                if config_class(meta) in ORDER_SENSITIVE else (0.0, 0.0))
        for k, (a, b, c) in enumerate(zip(got_cg, ref_cg, det_cg)):
            tol_k = max(abs(c - b), int(np.ceil(rel_stage * b)))
            assert abs(a - b) <= tol_k, ("stage", k, a, b, c, tol_k)
        tol_t = max(abs(ss["cg_total"] - sum(ref_cg)), int(np.ceil(rel_total * sum(ref_cg))))
        assert abs(sum(got_cg) - sum(ref_cg)) <= tol_t, (sum(got_cg), sum(ref_cg), ss["cg_total"],
                                                          tol_t)
        tol = max(1e-10, SPREAD_X * ss["du"], SPREAD_X * ss["dv"])
        assert du <= tol and dv <= tol, (du, dv, tol)
        assert sol.primal_cost == pytest.approx(meta["primal"], rel=1e-9, abs=1e-14)
    print(f"{name}: gate={g} stages={len(got_cg)} cg={sum(got_cg)} (ref {sum(ref_cg)}, "
          f"ref det-vs-BLAS {ss.get('cg_total')}) du={du:.3e} dv={dv:.3e} "
          f"(ref self-spread {ss.get('du', float('nan')):.2e}/{ss.get('dv', float('nan')):.2e}; "
          f"x{_mult(du, ss.get('du'))}/x{_mult(dv, ss.get('dv'))})")


def _mult(d, ref):
    return f"{d / ref:.1f}" if ref else "-"


@pytest.mark.parametrize("name", [n for n in traj_names() if not n.startswith("D")])
def test_small_trajectories(name):
    meta, arr, prob, sol = run_case(name)
    check(meta, arr, sol, name)
    # rounded plan is exactly feasible (test_driver.py:203-208)
    np.testing.assert_allclose(sol.P.sum(axis=1), prob.r, atol=1e-12)
    np.testing.assert_allclose(sol.P.sum(axis=0), prob.c, atol=1e-12)
    # the rank-one repair can leave roundoff-level negatives: the reference
    # itself returns min(P) = -2.9e-19 on grid16_l1_s1
    assert sol.P.min() >= -1e-15


@pytest.mark.parametrize("name", [n for n in traj_names() if n.startswith("D")])
def test_full_size_trajectories(name):
    """n = 4096 bench configurations, device-resident cost."""
    meta, arr, prob, sol = run_case(name, on_device=True)
    check(meta, arr, sol, name)
    st = sol.final_state
    st.set_targets(prob.r, prob.c)
    assert st.grad_norm_l1() <= 1e-6          # the metric's precision target
    P = sol.P
    np.testing.assert_allclose(P.sum(dim=1).cpu().numpy(), prob.r, atol=1e-12)
    np.testing.assert_allclose(P.sum(dim=0).cpu().numpy(), prob.c, atol=1e-12)


def test_deterministic_bit_identical():
    """Fixed reduction trees: two runs are bit-identical (test_cli.py:190-204)."""
    prob = problems.workload("grid:16:l2sq:1")
    a = mdot(prob, 2.0 ** 5, 2.0 ** 12)
    b = mdot(prob, 2.0 ** 5, 2.0 ** 12)
    np.testing.assert_array_equal(a.P, b.P)
    assert a.report.ops == b.report.ops


def test_sinkhorn_projector_path():
    prob = problems.grid_problem(4, "l1", 6)
    sol = mdot(prob, 2.0 ** 4, 2.0 ** 8, opts=MdotOptions(projector="sinkhorn"))
    assert sol.report.solver == "mdot-sinkhorn"
    np.testing.assert_allclose(sol.P.sum(axis=1), prob.r, atol=1e-12)
    assert sol.report.ops.get("sinkhorn", 0) > 0


@pytest.mark.parametrize("spec", ["grid:32:l2sq:0", "grid:32:l1:1"])
def test_fused_newton_step_matches_per_call_path(spec, monkeypatch):
    """otn_newton_step (Newton + alpha = 1 trial + gated accept path, one
    host sync) against the per-call path otn_newton -> otn_trial_cols ->
    accept -> row LSE -> row statistics: the same kernels in the same order,
    so the solves are bit-identical, with identical op tallies, including
    steps that backtrack (device gate closed, host loop takes over)."""
    from paper_2504_02067_b200.dual import DualState
    prob = problems.workload(spec)
    a = mdot(prob, 2.0 ** 5, 2.0 ** 14)
    monkeypatch.setattr(DualState, "_newton_step", None)
    b = mdot(prob, 2.0 ** 5, 2.0 ** 14)
    np.testing.assert_array_equal(a.final_state.u, b.final_state.u)
    np.testing.assert_array_equal(a.final_state.v, b.final_state.v)
    np.testing.assert_array_equal(a.P, b.P)
    assert a.report.ops == b.report.ops
    sa = [(it.stats.newton_steps, it.stats.cg_iters, it.stats.backtracks) for it in a.iterations]
    sb = [(it.stats.newton_steps, it.stats.cg_iters, it.stats.backtracks) for it in b.iterations]
    assert sa == sb
    print(spec, "backtracks", sum(x[2] for x in sa), "steps", sum(x[0] for x in sa))


@pytest.mark.parametrize("n", [1, 2, 3, 5, 33])
def test_tiny_problems_match_oracle(n):
    """Edge sizes against the oracle restatement of the reference: n = 1 fails
    the same way (a zero-entropy marginal makes eps_d 0: DomainError), n = 2,
    3, 5, 33 give the same stage-by-stage CG counts and potentials."""
    from oracle import otn_oracle as orc
    from paper_2504_02067_b200.errors import DomainError
    rng = np.random.default_rng(n)
    C = rng.random((n, n))
    C = C / C.max() if n > 1 else np.zeros((1, 1))
    r = np.full(n, 1.0 / n)
    c = rng.random(n) + 0.5
    c /= c.sum()
    prob = problems.Problem(C=C, r=r, c=c)
    if n == 1:
        with pytest.raises(DomainError):
            mdot(prob, 2.0 ** 2, 2.0 ** 8)
        with pytest.raises(orc.OracleFailure):
            orc.mdot(C, r, c, 2.0 ** 2, 2.0 ** 8)
        return
    sol = mdot(prob, 2.0 ** 2, 2.0 ** 8)
    run = orc.mdot(C, r, c, 2.0 ** 2, 2.0 ** 8)
    assert [i.stats.cg_iters for i in sol.iterations] == [pr.cg_iters for (*_, pr) in run.stages]
    assert [i.gamma for i in sol.iterations] == [g for (_t, g, *_rest) in run.stages]
    assert rel_inf(sol.final_state.u, run.state.u) <= 1e-10
    assert rel_inf(sol.final_state.v, run.state.v) <= 1e-10
