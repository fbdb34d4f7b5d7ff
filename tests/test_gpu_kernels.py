"""Kernel-level parity on the B200: each C-ABI operator vs the CPU oracle on the
same seeded inputs (tolerances written per test: float64, different but fixed
reduction trees, so agreement is at the 1e-15..1e-13 relative level)."""

import math

import numpy as np
import pytest

from oracle import otn_oracle as orc
from paper_2504_02067_b200 import DiscountedSystem, DualState, newton_solve, pcg_solve, problems
from paper_2504_02067_b200.errors import (
    ConditioningError,
    NonconvergenceError,
    PlanOverflowError,
)

pytestmark = pytest.mark.gpu

LSE_RTOL = 1e-13   # log-sum-exp: online (max, sum) merge vs numpy pairwise sum


def make_state(n, seed=0, gamma=4.0, spread=0.5, metric="l1", symmetric=True):
    if symmetric:
        C = problems.grid_points_cost(n, metric)
    else:
        rng = np.random.default_rng(seed + 99)
        C = rng.random((n, n))
    r = problems.gen_marginal(n, "smooth-random", seed)
    c = problems.gen_marginal(n, "spiky-random", seed + 100)
    prob = problems.Problem(C=C, r=r, c=c)
    rng = np.random.default_rng(seed + 1)
    u = np.log(r) + spread * rng.standard_normal(n)
    v = np.log(c) + spread * rng.standard_normal(n)
    return prob, u, v


def oracle_state(prob, gamma, u, v):
    return orc.Dual(prob.C, gamma, u, v, prob.r, prob.c, orc.Tally())


@pytest.mark.parametrize("n,sym", [(1, True), (5, True), (33, True), (273, True), (273, False),
                                   (1000, False), (4096, True)])
def test_row_and_column_lse(n, sym):
    prob, u, v = make_state(n, seed=n, symmetric=sym)
    gamma = 37.5
    st = DualState(prob, gamma, u=u, v=v)
    ref = oracle_state(prob, gamma, u, v)
    np.testing.assert_allclose(st.log_rP, ref.log_r, rtol=LSE_RTOL, atol=1e-300)
    np.testing.assert_allclose(st.log_cP, ref.log_c, rtol=LSE_RTOL, atol=1e-300)


def test_lse_large_magnitude_and_tail():
    """No overflow at |x| ~ 1000 (test_core.py:17-19); n not a tile multiple."""
    n = 257
    prob, u, v = make_state(n, seed=3)
    u = u + 1000.0
    st = DualState(prob, 2.0, u=u, v=v)
    ref = oracle_state(prob, 2.0, u, v)
    np.testing.assert_allclose(st.log_rP, ref.log_r, rtol=LSE_RTOL)
    np.testing.assert_allclose(st.log_cP, ref.log_c, rtol=LSE_RTOL)


def test_rebalance_and_exit_scaling():
    prob, u, v = make_state(300, seed=7, symmetric=False)
    st = DualState(prob, 8.0, u=u, v=v)
    ref = oracle_state(prob, 8.0, u, v)
    st.rebalance_columns()
    ref.balance_cols()
    np.testing.assert_allclose(st.v, ref.v, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(st.log_rP, ref.log_r, rtol=1e-13, atol=1e-13)
    st.scale_rows_to_target()
    ref.balance_rows_exit()
    np.testing.assert_allclose(st.u, ref.u, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(st.log_cP, ref.log_c, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("sym", [True, False])
def test_trial_column_sums_and_mass(sym):
    n = 500
    prob, u, v = make_state(n, seed=11, symmetric=sym)
    st = DualState(prob, 6.0, u=u, v=v)
    ref = oracle_state(prob, 6.0, u, v)
    rng = np.random.default_rng(0)
    du, dv = rng.standard_normal(n), rng.standard_normal(n)
    got = st.trial_log_col_sums(du, dv, 0.3)
    want = ref.trial_log_c(du, dv, 0.3)
    np.testing.assert_allclose(got, want, rtol=LSE_RTOL)


def test_materialize_and_mu():
    n = 700
    prob, u, v = make_state(n, seed=5)
    st = DualState(prob, 12.0, u=u, v=v)
    ref = oracle_state(prob, 12.0, u, v)
    P = st.materialize_plan()
    np.testing.assert_allclose(P, ref.plan(), rtol=2e-15, atol=0)
    sysd = DiscountedSystem.from_state(st)
    sysr = orc.System.of(ref)
    np.testing.assert_allclose(sysd.diag_prc(), sysr.mu(), rtol=1e-13)
    np.testing.assert_allclose(sysd.rP, sysr.rP, rtol=1e-13)


def test_overflow_rejected():
    prob, u, v = make_state(3)
    st = DualState(prob, 4.0, u=u + 800.0, v=v)
    with pytest.raises(PlanOverflowError):
        st.materialize_plan()


@pytest.mark.parametrize("n", [8, 300, 4096])
def test_hvp_operators(n):
    prob, u, v = make_state(n, seed=2, gamma=4.0)
    st = DualState(prob, 4.0, u=u, v=v)
    sysd = DiscountedSystem.from_state(st)
    P, rP, cP = sysd.P, sysd.rP, sysd.cP
    d = np.random.default_rng(1).standard_normal(n)
    for rho in (0.0, 0.5, 1.0):
        want = rP * d - rho * (P @ ((P.T @ d) / cP))
        np.testing.assert_allclose(sysd.apply_F(rho, d), want, rtol=1e-12, atol=1e-14 * np.abs(want).max())
    np.testing.assert_allclose(sysd.apply_pc(d), (P.T @ d) / cP, rtol=1e-12)
    np.testing.assert_allclose(sysd.apply_prc(d), (P @ ((P.T @ d) / cP)) / rP, rtol=1e-12)


@pytest.mark.parametrize("n_,seed", [(32, 33), (64, 3), (256, 5)])
def test_pcg_and_newton_vs_reference(kernels_golden, n_, seed):
    """CG iteration counts exact, solutions to 1e-10 relative vs the reference."""
    g = kernels_golden
    C = problems.grid_points_cost(n_, "l1")
    r = problems.gen_marginal(n_, "smooth-random", seed)
    c = problems.gen_marginal(n_, "spiky-random", seed + 100)
    rs = np.random.default_rng(seed + 7)
    st = DualState(problems.Problem(C=C, r=r, c=c), 4.0,
                   u=np.log(r) + 0.3 * rs.standard_normal(n_),
                   v=np.log(c) + 0.3 * rs.standard_normal(n_))
    sysd = DiscountedSystem.from_state(st)
    np.testing.assert_allclose(sysd.diag_prc(), g[f"sys{n_}_mu"], rtol=1e-13)
    b = np.random.default_rng(seed + 1).standard_normal(n_) * 0.01
    for rho in (0.0, 0.9, 0.99):
        x, it = pcg_solve(sysd, rho, b, 1e-12)
        ref = g[f"sys{n_}_pcg{rho}_x"]
        assert it == int(g[f"sys{n_}_pcg{rho}_iters"][0])
        assert np.abs(x - ref).max() <= 1e-10 * np.abs(ref).max()
    res = newton_solve(b - b.mean(), sysd, 0.05)
    meta = g[f"sys{n_}_newton_meta"]
    assert res.cg_iters == int(meta[1])
    assert res.rho_final == meta[0]
    ref = g[f"sys{n_}_newton_d"]
    assert np.abs(res.d_u - ref).max() <= 1e-10 * np.abs(ref).max()


def test_pcg_warm_start_and_budget():
    prob, u, v = make_state(32, seed=35)
    sysd = DiscountedSystem.from_state(DualState(prob, 4.0, u=u, v=v))
    b = np.random.default_rng(36).standard_normal(32)
    d, _ = pcg_solve(sysd, 0.7, b, tol_l1=1e-12)
    d2, iters = pcg_solve(sysd, 0.7, b, tol_l1=1e-10, d0=d)
    assert iters == 0
    np.testing.assert_array_equal(d2, d)
    with pytest.raises(NonconvergenceError) as err:
        pcg_solve(sysd, 0.9999, b, tol_l1=1e-15, max_iters=2)
    assert err.value.best is not None and err.value.best.shape == (32,)
    with pytest.raises(ConditioningError):
        pcg_solve(sysd, 1.0, b, tol_l1=1e-10)


def test_jacobi_exact_direction_and_hand_mu():
    sysd = DiscountedSystem(np.full((2, 2), 0.25), np.array([0.5, 0.5]), np.array([0.5, 0.5]))
    np.testing.assert_allclose(sysd.diag_prc(), [0.5, 0.5], rtol=1e-15)
    res = newton_solve(np.array([-0.1, 0.1]), sysd, eta=0.25, rho0=0.0)
    np.testing.assert_allclose(res.d_u, [0.2, -0.2], rtol=1e-14)
    assert res.cg_iters == 0 and res.rho_final == 0.0


def test_rho_anneals_on_quarter_grid():
    prob, u, v = make_state(16, seed=41)
    sysd = DiscountedSystem.from_state(DualState(prob, 16.0, u=u, v=v))
    grad = np.random.default_rng(42).standard_normal(16) * 0.01
    grad -= grad.mean()
    res = newton_solve(grad, sysd, eta=0.01)
    k = math.log(1.0 - res.rho_final) / math.log(4.0)
    assert k == pytest.approx(round(k), abs=1e-9)
    resid = sysd.apply_F(1.0, res.d_u) + grad
    assert np.abs(resid).sum() <= 0.01 * np.abs(grad).sum() + 1e-15


@pytest.mark.parametrize("op", ["VEC_EXP", "VEC_GRAD"])
def test_exp_fast_accuracy(op):
    """The kernels' two branch-free exps vs numpy: <= 1 ulp over the whole
    range, exact 0 / inf / NaN at the ends.  VEC_EXP runs exp_tab (the
    table-driven exp of every LSE / plan / pair entry); VEC_GRAD with b = 0
    runs exp_fast (the polynomial one used for O(n) work and LSE merges)."""
    from paper_2504_02067_b200 import _lib
    from paper_2504_02067_b200._device import Context, require_cuda, vptr
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(-750, 712, 200000), rng.uniform(-1, 1, 50000),
                        rng.uniform(-746, -700, 50000),
                        [0.0, -0.0, 1.0, -1.0, -745.1, -745.2, -744.4, 709.78, 709.79, 710.0,
                         -np.inf, np.inf, np.nan, 1e-300, -1e-300]])
    n = 8192
    x = np.concatenate([x, np.zeros((-x.size) % n)])
    ctx = Context.get(n, require_cuda())
    got = np.empty_like(x)
    for k in range(0, x.size, n):
        a = ctx.vec(x[k:k + n])
        out = ctx.vec()
        zero = ctx.vec(np.zeros(n))
        ctx.call("otn_vec", getattr(_lib, op), 0.0, vptr(a), vptr(zero), None, None, vptr(out))
        got[k:k + n] = ctx.download(out)
    want = np.exp(x)
    both_nan = np.isnan(got) & np.isnan(want)
    assert np.all(both_nan == np.isnan(want))
    ok = ~np.isnan(want)
    g, w = got[ok], want[ok]
    # ulp distance on the IEEE bit patterns (monotone for non-negative doubles)
    ulps = np.abs(g.view(np.int64) - w.view(np.int64))
    assert ulps.max() <= 1, (ulps.max(), x[ok][np.argmax(ulps)])


def _layout(sysd):
    k = sysd._ctx
    G = k.coop_blocks
    lay = np.zeros(G + 2, dtype=np.int32)
    k.call("otn_coop_layout", lay.ctypes.data)
    return lay[: G + 1], int(lay[G + 1])


def _sparse_plan(n, per_row, seed, heavy=0):
    """Banded-random sparse plan with exact zeros elsewhere (+ a few heavy rows)."""
    rng = np.random.default_rng(seed)
    P = np.zeros((n, n))
    for i in range(n):
        k = per_row if i >= heavy else min(n, 40 * per_row)
        cols = np.unique((i + rng.integers(-3 * per_row, 3 * per_row + 1, size=k)) % n)
        P[i, cols] = rng.random(len(cols)) * 10.0 ** rng.uniform(-300, 0, len(cols))
    P[np.arange(n), np.arange(n)] += 1.0           # positive row / column sums
    return P


@pytest.mark.parametrize("n,per_row,heavy,mode", [
    (64, 3, 0, 2), (300, 8, 0, 2), (1024, 20, 5, 2), (4096, 12, 9, 2),
    (1024, 1024, 0, 0), (4096, 600, 0, 3), (2048, 1400, 0, 0), (2048, 2048, 0, 0),
    (4096, 4096, 0, 0),
    # wider than one 4096-column tile (ld 6016, 9024): the streamed ring over
    # several tiles and the multi-slice column pass (ld > 32 x 148)
    (6000, 6000, 0, 0), (9000, 60, 0, 0)])
def test_hvp_plan_modes(n, per_row, heavy, mode):
    """Every plan mode (0 streamed ring, 2 sparse shared-memory rows, 3 sparse
    global-memory rows; mode 1 is retired) against numpy on the same plan; the
    sparse modes also on heavy rows."""
    if per_row >= n:
        rng = np.random.default_rng(n)
        P = rng.random((n, n)) + 0.01
    else:
        P = _sparse_plan(n, per_row, seed=n + heavy, heavy=heavy)
    rP, cP = P.sum(1), P.sum(0)
    sysd = DiscountedSystem(P, rP, cP)
    d = np.random.default_rng(7).standard_normal(n)
    got_pc = sysd.apply_pc(d)
    part, got_mode = _layout(sysd)
    assert got_mode == mode
    assert part[0] == 0 and part[-1] == n and np.all(np.diff(part) >= 0)
    want_pc = (P.T @ d) / cP
    np.testing.assert_allclose(got_pc, want_pc, rtol=1e-12, atol=1e-14 * np.abs(want_pc).max())
    for rho in (0.5, 1.0):
        want = rP * d - rho * (P @ ((P.T @ d) / cP))
        np.testing.assert_allclose(sysd.apply_F(rho, d), want, rtol=1e-11,
                                   atol=1e-13 * np.abs(want).max())
    want_prc = (P @ ((P.T @ d) / cP)) / rP
    np.testing.assert_allclose(sysd.apply_prc(d), want_prc, rtol=1e-12,
                               atol=1e-14 * np.abs(want_prc).max())
    x, _ = pcg_solve(sysd, 0.9, -d, 1e-10 * np.abs(d).sum())
    F = np.diag(rP) - 0.9 * (P / cP) @ P.T
    np.testing.assert_allclose(F @ x, -d, rtol=1e-6, atol=1e-9 * np.abs(d).max())


class TestLambda2:
    """lambda2 (newton.py:220-236) by device Lanczos vs the reference's dense
    eigensolve (test_newton.py:258-283 idioms)."""

    def test_independence_is_rank_one(self):
        from paper_2504_02067_b200 import lambda2
        r, c = np.array([0.25, 0.35, 0.4]), np.array([0.3, 0.3, 0.4])
        P = np.outer(r, c)
        sysd = DiscountedSystem(P, P.sum(1), P.sum(0))
        assert lambda2(sysd) == pytest.approx(0.0, abs=1e-10)

    @pytest.mark.parametrize("n,seed", [(10, 60), (64, 1), (700, 2)])
    def test_matches_dense_eigh(self, n, seed):
        from paper_2504_02067_b200 import lambda2
        rng = np.random.default_rng(seed)
        P = rng.random((n, n)) ** 4
        P /= P.sum()
        rP, cP = P.sum(1), P.sum(0)
        G = P / (np.sqrt(rP)[:, None] * np.sqrt(cP)[None, :])
        ev = np.linalg.eigvalsh(G @ G.T)
        assert ev[-1] == pytest.approx(1.0, abs=1e-10)
        assert lambda2(DiscountedSystem(P, rP, cP)) == pytest.approx(ev[-2], abs=1e-9)

    def test_near_decoupled_blocks_push_lambda2_to_one(self):
        from paper_2504_02067_b200 import lambda2
        A = np.full((2, 2), 0.25)
        eps = 1e-8
        P = np.block([[A, np.full((2, 2), eps)], [np.full((2, 2), eps), A]])
        assert lambda2(DiscountedSystem(P, P.sum(axis=1), P.sum(axis=0))) > 1.0 - 1e-6

    def test_size_guard(self):
        from paper_2504_02067_b200 import lambda2
        from paper_2504_02067_b200.errors import RefusalError
        n = 2049
        P = np.full((n, n), 1.0 / (n * n))
        with pytest.raises(RefusalError):
            lambda2(DiscountedSystem(P, P.sum(axis=1), P.sum(axis=0)))


def test_bulk_copy_row_lse_matches_oracle():
    """The opt-in bulk-copy (TMA) row LSE (OTN_LSE_BULK=1, read when a context
    is created: a fresh process) against the oracle, plain and with the
    trial direction, at a full and a ragged size."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_gpu_kernels import make_state, oracle_state
from oracle import otn_oracle as orc
from paper_2504_02067_b200 import DualState
for n, sym in ((4096, True), (1000, False), (33, True)):
    prob, u, v = make_state(n, seed=n, symmetric=sym)
    st = DualState(prob, 4.0, u=u, v=v)
    assert st._ctx.config["lse_bulk_ctas"] > 0, st._ctx.config
    ref = oracle_state(prob, 4.0, u, v)
    np.testing.assert_allclose(st.log_rP, ref.log_r, rtol=1e-13)
    du = np.random.default_rng(1).standard_normal(n) * 0.1
    dv = np.random.default_rng(2).standard_normal(n) * 0.1
    got = st.trial_log_col_sums(du, dv, 0.5)
    want = ref.trial_log_c(du, dv, 0.5)
    np.testing.assert_allclose(got, want, rtol=1e-13)
print("bulk ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env=dict(os.environ, OTN_LSE_BULK="1"), timeout=600)
    assert out.returncode == 0 and "bulk ok" in out.stdout, out.stderr[-3000:]


def test_wide_mdot_matches_oracle():
    """A full mdot on a cost wider than one tile (n = 5184 > 4096: several
    column tiles, the multi-slice column pass, residual replacement there)
    against the oracle restatement of the reference, same seeded problem."""
    spec, gi, gf = "grid:72:l2sq:0", 2.0 ** 5, 2.0 ** 8
    prob = problems.workload(spec)
    import os
    orc.set_threads(os.cpu_count() or 1)               # bit-identical for any thread count
    run = orc.mdot(prob.C, prob.r, prob.c, gi, gf)
    import torch
    from paper_2504_02067_b200 import mdot
    dp = problems.Problem(C=torch.from_numpy(prob.C).cuda(), r=prob.r, c=prob.c)
    sol = mdot(dp, gi, gf)
    got = [(it.gamma, it.stats.newton_steps, it.stats.cg_iters) for it in sol.iterations]
    want = [(g, pr.newton_steps, pr.cg_iters) for (_t, g, _eps, _q, pr) in run.stages]
    assert got == want
    du = np.abs(sol.final_state.u - run.state.u).max() / np.abs(run.state.u).max()
    dv = np.abs(sol.final_state.v - run.state.v).max() / np.abs(run.state.v).max()
    assert du <= 1e-10 and dv <= 1e-10, (du, dv)
