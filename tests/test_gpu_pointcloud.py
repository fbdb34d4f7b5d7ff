"""On-the-fly point-cloud path (D4/D5 kernels) on the B200: the cost recomputed
from coordinates must reproduce the stored-cost path and the reference."""

import numpy as np
import pytest

from conftest import load_traj
from paper_2504_02067_b200 import DualState, mdot, opcount, problems
from paper_2504_02067_b200.pointcloud import PointCloudCost, PointCloudState

pytestmark = pytest.mark.gpu


def _pair(n, d, seed):
    pc = problems.points_problem(n, d, seed)
    dense = problems.Problem(C=pc.materialize_cost(), r=pc.r, c=pc.c)
    return pc, dense


@pytest.mark.parametrize("n,d", [(300, 2), (257, 3), (1024, 3)])
def test_otf_lse_and_plan_match_stored(n, d):
    import torch
    pc, dense = _pair(n, d, 5)
    cost = PointCloudCost(pc, torch.device("cuda", 0))
    assert cost.cmax == pc.raw_cost_rows(0, n).max()
    rng = np.random.default_rng(1)
    u = np.log(pc.r) + 0.3 * rng.standard_normal(n)
    v = np.log(pc.c) + 0.3 * rng.standard_normal(n)
    gamma = 40.0
    a = PointCloudState(cost, gamma, u, v, pc.r, pc.c)
    b = DualState(dense, gamma, u=u, v=v)
    a.refresh()
    np.testing.assert_allclose(a._lr.cpu().numpy(), b.log_rP, rtol=1e-13)
    np.testing.assert_allclose(a._lc.cpu().numpy(), b.log_cP, rtol=1e-13)
    sa, sb = a._system(), b._system()
    np.testing.assert_allclose(sa._mu.cpu().numpy(), sb.diag_prc(), rtol=1e-12)
    x = torch.from_numpy(rng.standard_normal(n)).cuda()
    from paper_2504_02067_b200.pointcloud import _Result
    qa = cost.zeros(n)
    sa._hvp(0.9, x, qa, _Result())
    qb = sb.apply_F(0.9, x.cpu().numpy())
    np.testing.assert_allclose(qa.cpu().numpy(), qb, rtol=1e-11, atol=1e-15)


@pytest.mark.parametrize("name", ["pts256_2d_s0", "pts1024_2d_s0_fixed", "pts1024_3d_s0"])
def test_otf_mdot_matches_reference_trajectory(name):
    """Strict gate: same stages / Newton steps / CG counts / op
    tally as the reference on the materialized cost, potentials to 1e-10."""
    meta, arr = load_traj(name)
    _, n, d, seed = meta["spec"].split(":")
    pc = problems.points_problem(int(n), int(d), int(seed))
    opcount.reset()
    sol = mdot(pc, meta["gamma_i"], meta["gamma_f"])
    assert [it.stats.cg_iters for it in sol.iterations] == [s["cg_iters"] for s in meta["stages"]]
    assert [it.stats.newton_steps for it in sol.iterations] == \
        [s["newton_steps"] for s in meta["stages"]]
    assert sol.report.ops == meta["ops"]
    st = sol.final_state
    du = np.abs(st.u - arr["u"]).max() / np.abs(arr["u"]).max()
    dv = np.abs(st.v - arr["v"]).max() / np.abs(arr["v"]).max()
    assert du <= 1e-10 and dv <= 1e-10, (du, dv)
    assert sol.P is None
    assert sol.primal_cost == pytest.approx(meta["primal"], rel=1e-9)
    st.set_targets(pc.r, pc.c)
    assert st.grad_norm_l1() <= 2 * meta["true_marginal_err"] + 1e-12


@pytest.mark.parametrize("n,d,scale", [(2048, 2, 1.0), (1500, 3, 1e-3), (777, 4, 1e4)])
def test_otf_cost_bitwise(n, d, scale):
    """The pair kernel's C_ij = D_ij / C_max (a reciprocal multiply plus an
    FMA correction in place of a division) is bit-identical to the host's IEEE
    division, read out through C . e_k (PC_CDOT with a one-hot vector)."""
    import torch
    from paper_2504_02067_b200 import _lib
    pc = problems.points_problem(n, d, 11)
    pc.X = pc.X * scale
    pc.Y = pc.Y * scale
    cost = PointCloudCost(pc, torch.device("cuda", 0))
    C = pc.materialize_cost()
    assert cost.cmax == pc.raw_cost_rows(0, n).max()
    out = cost.zeros(n)
    e = cost.zeros(n)
    for k in np.random.default_rng(0).choice(n, 24, replace=False):
        e.zero_()
        e[int(k)] = 1.0
        cost.pass_(_lib.PC_CDOT, rows_first=True, out=out, vec=e)
        got = out.cpu().numpy()
        np.testing.assert_array_equal(got.view(np.int64), C[:, k].view(np.int64))


def test_separable_exponent_matches_exact_cost_path():
    """The separable plan exponent of the on-the-fly exp passes (the default)
    against the exact-cost path (OTN_PC_EXACT=1, read when a context is
    created: a fresh process): same trajectory, potentials within 1e-11."""
    import json
    import os
    import subprocess
    import sys
    code = r'''
import json, sys
sys.path.insert(0, ".")
from paper_2504_02067_b200 import mdot, problems
pc = problems.points_problem(2048, 3, 4)
sol = mdot(pc, 2.0 ** 5, 2.0 ** 11)
st = sol.final_state
print(json.dumps(dict(u=st.u.tolist(), v=st.v.tolist(), primal=sol.primal_cost,
                      cg=[it.stats.cg_iters for it in sol.iterations])))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    runs = []
    for exact in ("0", "1"):
        out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True,
                             text=True, env=dict(os.environ, OTN_PC_EXACT=exact), timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        runs.append(json.loads(out.stdout.strip().splitlines()[-1]))
    sep, exact = runs
    assert sep["cg"] == exact["cg"]
    for k in ("u", "v"):
        a, b = np.array(sep[k]), np.array(exact[k])
        assert np.abs(a - b).max() <= 1e-11 * np.abs(b).max()
    assert sep["primal"] == pytest.approx(exact["primal"], rel=1e-11)
