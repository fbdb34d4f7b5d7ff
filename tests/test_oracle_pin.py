"""Pin the CPU oracle (oracle/otn_oracle.py) to the reference (CPU-only).

The golden vectors were produced by the reference package itself
(tests/golden/make_golden.py); the oracle must reproduce them BIT FOR BIT —
same per-stage and per-step counts, same potentials, same op tallies — and
must satisfy the reference's own known-answer tests.
"""

import math

import numpy as np
import pytest

from conftest import load_traj, traj_names
from oracle import otn_oracle as orc
from paper_2504_02067_b200 import problems

FAST = [n for n in traj_names() if not n.startswith(("D", "M"))]   # (M, D: GPU-checked only)


def _trajectory(run):
    out = []
    for (t, g, eps, q, pr) in run.stages:
        out.append(dict(t=t, gamma=g, eps_d=eps, q_next=q, newton_steps=pr.newton_steps,
                        cg_iters=pr.cg_iters, sinkhorn_steps=pr.sinkhorn_steps,
                        backtracks=pr.backtracks, rho_final=pr.rho_final,
                        delta_min=pr.delta_min, grad_norm_final=pr.grad_norm_final,
                        steps=[dict(cg_iters=s.cg_iters, alpha=s.alpha, backtracks=s.backtracks,
                                    rho_final=s.rho_final, eta=s.eta,
                                    grad_before=s.grad_before, grad_after=s.grad_after,
                                    delta=s.delta) for s in pr.steps]))
    return out


@pytest.mark.parametrize("name", FAST)
def test_oracle_matches_reference_bitwise(name):
    meta, arr = load_traj(name)
    prob = problems.workload(meta["spec"])
    run = orc.mdot(prob.C, prob.r, prob.c, meta["gamma_i"], meta["gamma_f"],
                   projector=meta.get("projector", "newton"))
    assert np.array_equal(run.state.u, arr["u"])
    assert np.array_equal(run.state.v, arr["v"])
    assert run.primal == meta["primal"]
    assert run.ops == meta["ops"]
    ref = [{k: v for k, v in s.items() if k != "ops_n2"} for s in meta["stages"]]
    got = _trajectory(run)
    # json turns inf into Infinity -> float('inf'); compare as floats
    assert json_norm(got) == json_norm(ref)


@pytest.mark.parametrize("name", traj_names())
def test_every_golden_records_a_bitwise_oracle(name):
    """make_golden.py --verify-oracle ran the oracle beside the reference on
    every case, the n = 4096 D2 / D3 solves included (too slow for this
    suite), and recorded whether it reproduced the reference bit for bit."""
    meta, _ = load_traj(name)
    assert meta.get("oracle_bitwise") is True


def test_slab_threads_do_not_change_bits():
    """The slab-parallel oracle (bench.py's CPU baseline) is bit-identical to
    the serial one: every 256-row slab is an independent computation."""
    prob = problems.workload("grid:32:l2sq:0")
    runs = []
    for k in (1, 4):
        orc.set_threads(k)
        try:
            runs.append(orc.mdot(prob.C, prob.r, prob.c, 2.0 ** 5, 2.0 ** 10))
        finally:
            orc.set_threads(1)
    assert np.array_equal(runs[0].state.u, runs[1].state.u)
    assert np.array_equal(runs[0].P, runs[1].P)
    assert runs[0].ops == runs[1].ops


def json_norm(obj):
    import json
    return json.loads(json.dumps(obj))


def test_oracle_kernels_match_reference(kernels_golden):
    g = kernels_golden
    rng = np.random.default_rng(9)
    n = 273
    K = rng.normal(size=(n, n)) * 10
    u = rng.normal(size=n)
    v = rng.normal(size=n)
    assert np.array_equal(orc.tiled_row_lse(K, u, v), g["lse_K273"])
    rng = np.random.default_rng(10)
    P = rng.random((259, 259))
    w = rng.random(259)
    assert np.array_equal(orc.tiled_square_mv(P, w), g["sqmv_259"])
    rng = np.random.default_rng(11)
    K = rng.normal(size=(7, 7))
    u = rng.normal(size=7)
    v = rng.normal(size=7)
    assert np.array_equal(orc.tiled_plan(K, u, v), g["plan_7"])


@pytest.mark.parametrize("n_,seed", [(32, 33), (64, 3), (256, 5)])
def test_oracle_cg_and_newton_match_reference(kernels_golden, n_, seed):
    g = kernels_golden
    C = problems.grid_points_cost(n_, "l1")
    r = problems.gen_marginal(n_, "smooth-random", seed)
    c = problems.gen_marginal(n_, "spiky-random", seed + 100)
    rs = np.random.default_rng(seed + 7)
    st = orc.Dual(C, 4.0, np.log(r) + 0.3 * rs.standard_normal(n_),
                  np.log(c) + 0.3 * rs.standard_normal(n_), r, c, orc.Tally())
    assert np.array_equal(st.log_r, g[f"sys{n_}_logr"])
    assert np.array_equal(st.log_c, g[f"sys{n_}_logc"])
    sysm = orc.System.of(st)
    assert np.array_equal(sysm.mu(), g[f"sys{n_}_mu"])
    b = np.random.default_rng(seed + 1).standard_normal(n_) * 0.01
    for rho in (0.0, 0.9, 0.99):
        x, it = orc.cg(sysm, rho, b, 1e-12)
        assert np.array_equal(x, g[f"sys{n_}_pcg{rho}_x"])
        assert it == int(g[f"sys{n_}_pcg{rho}_iters"][0])
    res = orc.newton_direction(b - b.mean(), sysm, 0.05)
    assert np.array_equal(res.d_u, g[f"sys{n_}_newton_d"])
    meta = g[f"sys{n_}_newton_meta"]
    assert (res.rho_final, res.cg_iters, res.resid) == (meta[0], int(meta[1]), meta[2])


# ---- the reference's own known-answer tests, run against the oracle --------

def test_closed_form_two_point_plan():
    """projector tests: off-diagonal mass 1/(1+e^4) at gamma=4 (test_projector.py:147-153)."""
    C = np.array([[0.0, 1.0], [1.0, 0.0]])
    r = c = np.array([0.5, 0.5])
    st = orc.Dual(C, 4.0, np.log(r), np.log(c), r, c, orc.Tally())
    orc.project(st, r, c, 1e-10)
    P = st.plan()
    assert P[0, 1] + P[1, 0] == pytest.approx(1.0 / (1.0 + math.exp(4.0)), abs=1e-10)


def test_jacobi_exact_direction():
    """test_newton.py:204-213: d = [0.2, -0.2], no CG."""
    sysm = orc.System(np.full((2, 2), 0.25), np.array([0.5, 0.5]), np.array([0.5, 0.5]),
                      orc.Tally())
    res = orc.newton_direction(np.array([-0.1, 0.1]), sysm, 0.25)
    np.testing.assert_allclose(res.d_u, [0.2, -0.2], rtol=1e-14)
    assert res.cg_iters == 0


def test_diag_hand_value():
    """test_newton.py:90-93: mu = [0.5, 0.5]."""
    sysm = orc.System(np.full((2, 2), 0.25), np.array([0.5, 0.5]), np.array([0.5, 0.5]),
                      orc.Tally())
    np.testing.assert_allclose(sysm.mu(), [0.5, 0.5], rtol=1e-15)


def test_schedule_constants():
    u = np.full(4096, 1.0 / 4096)
    assert orc.eps_rule(2.0 ** 5, 1.5, u, u) == pytest.approx(0.045949, rel=1e-4)
    bound = 2.0 * min(orc.entropy(u), orc.entropy(u)) / 2.0 ** 18
    assert bound == pytest.approx(6.3459e-5, rel=1e-4)


def test_rounding_hand_example():
    """test_driver.py:139-143."""
    P = np.array([[0.3, 0.3], [0.2, 0.2]])
    r = c = np.array([0.5, 0.5])
    np.testing.assert_allclose(orc.round_to_polytope(P, r, c, orc.Tally()),
                               np.full((2, 2), 0.25), atol=1e-15)
