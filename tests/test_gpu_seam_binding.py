"""The reference-side binding of INTEGRATION.md §2 (integration/otnewton_b200.py),
executed: the five operator-seam functions of otnewton (_kernels.py:22-74,
newton.py:43-56), computed by libotn_b200.so, drive a complete MDOT solve of
the reference's algorithm.  /root/reference does not exist on the GPU box, so
the driver is the oracle's restatement of the same code (oracle/otn_oracle.py,
bit-identical to the reference), whose seam functions are rebound exactly as
a maintainer would rebind otnewton's; the result is held to the strict gate
against the reference's own golden trajectories."""

import os
import sys

import numpy as np
import pytest

from conftest import load_traj
from oracle import otn_oracle as orc
from paper_2504_02067_b200 import _lib, problems

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "integration"))


@pytest.fixture
def seam(monkeypatch):
    from otnewton_b200 import Seam
    s = Seam(_lib.LIB_PATH, device=0,
             overflow_error=lambda msg: orc.OracleFailure("PlanOverflowError", msg))
    monkeypatch.setattr(orc, "tiled_row_lse", s.log_plan_row_sums)
    monkeypatch.setattr(orc, "tiled_plan", s.materialize_plan)
    monkeypatch.setattr(orc, "tiled_square_mv", s.square_matvec)

    def mv(P, x, tally):
        tally.bump(1)
        return s.matvec(P, x)

    def rmv(P, x, tally):
        tally.bump(1)
        return s.rmatvec(P, x)
    monkeypatch.setattr(orc, "mv", mv)
    monkeypatch.setattr(orc, "rmv", rmv)
    return s


@pytest.mark.parametrize("name", ["grid16_l1_s1", "pts256_2d_s0", "pts1024_2d_s0_fixed"])
def test_reference_driver_on_the_b200_seam(seam, name):
    meta, arr = load_traj(name)
    p = problems.workload(meta["spec"])
    run = orc.mdot(p.C, p.r, p.c, meta["gamma_i"], meta["gamma_f"])
    got = [(pr.newton_steps, pr.cg_iters) for (*_, pr) in run.stages]
    want = [(s["newton_steps"], s["cg_iters"]) for s in meta["stages"]]
    assert got == want
    assert run.ops == meta["ops"]
    du = np.abs(run.state.u - arr["u"]).max() / np.abs(arr["u"]).max()
    dv = np.abs(run.state.v - arr["v"]).max() / np.abs(arr["v"]).max()
    assert du <= 1e-10 and dv <= 1e-10, (du, dv)
    assert run.primal == pytest.approx(meta["primal"], rel=1e-9)


def test_seam_contract_details(seam):
    """Scalar outer term (dual.py:182 passes 0.0), the out= buffer, and the
    overflow rejection (_kernels.py:53-58)."""
    rng = np.random.default_rng(3)
    n = 70
    K = -rng.random((n, n)) * 5
    v = rng.standard_normal(n)
    np.testing.assert_allclose(seam.log_plan_row_sums(K, 0.0, v), _ref_lse(K, v), rtol=1e-13)
    buf = np.empty((n, n))
    out = seam.materialize_plan(K, v, v, out=buf)
    assert out is buf
    np.testing.assert_allclose(buf, np.exp((K + v[None, :]) + v[:, None]), rtol=2e-15)
    with pytest.raises(orc.OracleFailure):
        seam.materialize_plan(K, v + 800.0, v)


def _ref_lse(K, v):
    t = K + v[None, :]
    m = t.max(axis=1)
    return m + np.log(np.exp(t - m[:, None]).sum(axis=1))
