"""Input validation and error classes of the public API, CPU-only (the
reference's test_problems.py / test_driver.py / test_io.py idioms): every
check fires before any device work, with the reference's exception class."""

import numpy as np
import pytest

import paper_2504_02067_b200 as ot
from paper_2504_02067_b200 import errors


def tiny():
    return ot.grid_problem(3, "l1", 0)


@pytest.mark.parametrize("kw,msg", [
    (dict(gamma_i=0.0, gamma_f=1.0), "positive"),
    (dict(gamma_i=1.0, gamma_f=-1.0), "positive"),
    (dict(gamma_i=1.0, gamma_f=2.0, p=0.5), "p must"),
    (dict(gamma_i=1.0, gamma_f=2.0, q_init=1.0), "q_init"),
])
def test_mdot_rejects_bad_schedule_before_device(kw, msg):
    with pytest.raises(errors.DomainError, match=msg):
        ot.mdot(tiny(), **kw)


def test_mdot_rejects_unknown_projector():
    with pytest.raises(errors.DomainError, match="projector"):
        ot.mdot(tiny(), 1.0, 2.0, opts=ot.MdotOptions(projector="lbfgs"))


def test_problem_validation():
    C = np.full((3, 3), 0.5)
    r = np.full(3, 1 / 3)
    with pytest.raises(errors.DimensionError):
        ot.Problem(C=np.zeros((2, 3)), r=r, c=r)
    with pytest.raises(errors.DimensionError):
        ot.Problem(C=C, r=np.full(2, 0.5), c=r)
    with pytest.raises(errors.DomainError, match="negative"):
        ot.Problem(C=C, r=np.array([0.5, 0.6, -0.1]), c=r)
    with pytest.raises(errors.DomainError, match="sums"):
        ot.Problem(C=C, r=np.array([0.5, 0.5, 0.5]), c=r)
    with pytest.raises(errors.DomainError, match=r"\[0, 1\]"):
        ot.Problem(C=C * 3.0, r=r, c=r)
    bad = C.copy()
    bad[0, 0] = np.nan
    with pytest.raises(errors.DomainError, match="finite"):
        ot.Problem(C=bad, r=r, c=r)


def test_schedule_rule_errors():
    with pytest.raises(errors.DomainError):
        ot.eps_rule(0.0, 1.5, np.full(4, 0.25), np.full(4, 0.25))
    with pytest.raises(errors.DomainError):
        ot.adjust_schedule(1.0, 0.9)
    with pytest.raises(errors.DomainError):
        ot.smooth_marginals(np.full(4, 0.25), np.full(4, 0.25), 1.5)


def test_generator_errors():
    with pytest.raises(errors.DomainError):
        ot.gen_grid_cost(4, "l3")
    with pytest.raises(errors.DomainError):
        ot.gen_marginal(4, "lumpy", 0)
    with pytest.raises(errors.DimensionError):
        ot.gen_marginal(0, "uniform", 0)
    with pytest.raises(errors.DomainError):
        ot.workload("cube:4")


def test_otp_parse_errors(tmp_path):
    f = tmp_path / "bad.otp"
    f.write_text("")
    with pytest.raises(errors.ParseError, match="empty"):
        ot.load_problem(str(f))
    f.write_text("OTP x\n")
    with pytest.raises(errors.ParseError, match="dimension"):
        ot.load_problem(str(f))
    f.write_text("OTP 2\n0 1\n1 0\n0.5 0.5\n")
    with pytest.raises(errors.ParseError):
        ot.load_problem(str(f))


def test_eta_and_armijo_rules():
    assert ot.eta_rule(0.5, 0.1) == pytest.approx(0.5)
    assert ot.eta_rule(2.0, 0.1) == pytest.approx(0.99)
    with pytest.raises(errors.DomainError):
        ot.eta_rule(0.0, 0.1)
    with pytest.raises(errors.DomainError):
        ot.eta_rule(0.1, 0.2)
    with pytest.raises(errors.DomainError):
        ot.armijo_accept(1.0, 1.0, np.array([1.0]), np.array([1.0]))   # not a descent direction
    with pytest.raises(errors.DomainError):
        ot.delta_ratio(0.0, 0.0, 0.5)
