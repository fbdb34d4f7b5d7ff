"""The fused projector step (otn_newton_step) and the asynchronous read-back
(otn_reduce_async) against the per-call C-ABI path they replace, on one
state: same bits when the step is accepted, state untouched when it is not."""
import ctypes

import numpy as np
import pytest

from paper_2504_02067_b200 import _lib, problems
from paper_2504_02067_b200._device import vptr
from paper_2504_02067_b200.dual import DualState
from paper_2504_02067_b200.newton import _newton_device, _newton_step_device
from paper_2504_02067_b200.projector import ARMIJO_C1, ARMIJO_SLOPE_FLOOR

pytestmark = pytest.mark.gpu


def _state(spec="grid:16:l2sq:1", gamma=2.0 ** 8, seed=0):
    prob = problems.workload(spec)
    rng = np.random.default_rng(seed)
    u = np.log(prob.r) + 0.05 * rng.standard_normal(prob.n)
    v = np.log(prob.c) + 0.05 * rng.standard_normal(prob.n)
    st = DualState(prob, gamma, u=u, v=v)
    st.rebalance_columns()
    return prob, st


def _dev(st):
    return [t.clone() for t in (st._u, st._v, st._lr, st._lc, st._g, st._trial_vec)]


@pytest.mark.parametrize("spec,gamma", [("grid:16:l2sq:1", 2.0 ** 8), ("grid:24:l1:0", 2.0 ** 10),
                                        ("pix:256:784:0", 2.0 ** 9)])
def test_newton_step_matches_per_call_path(spec, gamma):
    _, a = _state(spec, gamma)
    _, b = _state(spec, gamma)
    eta = 0.5
    for st in (a, b):
        st._row_grad_norm()                           # leaves g in st._g
    da, dva = a._dir_bufs()
    db, dvb = b._dir_bufs()
    sa, sb = a._system(), b._system()
    res_a, mass_a, rowstat_a, = _newton_step_device(a, sa, a._g, eta, 0.0, False, None, da, dva,
                                                    ARMIJO_C1, ARMIJO_SLOPE_FLOOR)
    res_b = _newton_device(b._g, sb, eta, 0.0, False, None, db, dvb)
    assert (res_a.status, res_a.cg_iters, res_a.hvps) == (res_b.status, res_b.cg_iters, res_b.hvps)
    assert res_a.slope == res_b.slope and res_a.slope > 0.0
    np.testing.assert_array_equal(da.cpu().numpy(), db.cpu().numpy())
    mass_b = b._trial(db, dvb, 1.0, b._trial_buf())
    assert mass_a == mass_b
    np.testing.assert_array_equal(a._trial_vec.cpu().numpy(), b._trial_vec.cpu().numpy())
    accept = not (res_b.slope > ARMIJO_SLOPE_FLOOR and
                  mass_b - 1.0 > (1.0 - ARMIJO_C1) * 1.0 * res_b.slope)
    assert (rowstat_a is not None) == accept
    if accept:
        b._accept(1.0, db, dvb)
        b.refresh_rows_only()
        assert rowstat_a == b._row_stats()
        for x, y in zip(_dev(a)[:5], _dev(b)[:5]):
            np.testing.assert_array_equal(x.cpu().numpy(), y.cpu().numpy())


def test_rejected_step_leaves_the_state_untouched():
    """A full step the Armijo test rejects leaves u, v and the caches as they
    were (the host then backtracks from the returned trial mass).  Rejection
    is forced with c1 = 1 + 1e300: mass - 1 > (1 - c1) * slope always holds."""
    _, st = _state()
    st._row_grad_norm()
    before = _dev(st)[:5]
    d, dv = st._dir_bufs()
    sys_ = st._system()
    res, mass, rowstat = _newton_step_device(st, sys_, st._g, 0.5, 0.0, False, None, d, dv,
                                             1.0 + 1e300, 0.0)
    assert res.status == _lib.OTN_OK and mass is not None and rowstat is None
    for x, y in zip(before, _dev(st)[:5]):
        np.testing.assert_array_equal(x.cpu().numpy(), y.cpu().numpy())


def test_failed_newton_runs_nothing_after_it():
    """A Newton launch that fails (CG budget of 1 iteration) gates off the trial
    and the accept path: no trial mass, state untouched."""
    _, st = _state("grid:16:l2sq:1", 2.0 ** 12)
    st._row_grad_norm()
    before = _dev(st)
    d, dv = st._dir_bufs()
    res, mass, rowstat = _newton_step_device(st, st._system(), st._g, 1e-6, 0.0, False, 1, d, dv,
                                             ARMIJO_C1, ARMIJO_SLOPE_FLOOR)
    assert res.status != _lib.OTN_OK and mass is None and rowstat is None
    for x, y in zip(before, _dev(st)):
        np.testing.assert_array_equal(x.cpu().numpy(), y.cpu().numpy())


def test_async_reduce_equals_sync_reduce():
    _, st = _state()
    k = st._ctx
    for op, args in ((_lib.RED_GRAD_L1, (st._lr, st._r, st._lc, st._c)),
                     (_lib.RED_ROW_STATS, (st._lr, st._r, None, None)),
                     (_lib.RED_SUM_EXP, (st._lr, None, None, None))):
        out = (ctypes.c_double * 2)()
        fl = ctypes.c_int(0)
        k.call("otn_reduce", op, *(vptr(x) for x in args), out, ctypes.byref(fl))
        import torch
        host = torch.empty(2, dtype=torch.float64, pin_memory=True)
        k.call("otn_reduce_async", op, *(vptr(x) for x in args), ctypes.c_void_p(host.data_ptr()))
        torch.cuda.current_stream().synchronize()
        assert (host[0].item(), host[1].item()) == (out[0], out[1])
    g = st._grad_norm_l1_deferred()
    assert g.value() == st.grad_norm_l1()


def test_row_stats_and_accept_equal_their_component_ops():
    """otn_row_stats == otn_vec(GRAD) + otn_reduce(ROW_STATS) and otn_accept ==
    otn_vec(AXPY) + otn_vec(STEP_V) + copy, bit for bit."""
    import torch
    _, st = _state()
    k = st._ctx
    g1, g2 = k.vec(), k.vec()
    out1, out2 = (ctypes.c_double * 2)(), (ctypes.c_double * 2)()
    f1, f2 = ctypes.c_int(0), ctypes.c_int(0)
    k.call("otn_row_stats", vptr(st._lr), vptr(st._r), vptr(g1), out1, ctypes.byref(f1))
    k.call("otn_vec", _lib.VEC_GRAD, 0.0, vptr(st._lr), vptr(st._r), None, None, vptr(g2))
    k.call("otn_reduce", _lib.RED_ROW_STATS, vptr(st._lr), vptr(st._r), None, None, out2,
           ctypes.byref(f2))
    assert (out1[0], out1[1], f1.value) == (out2[0], out2[1], f2.value)
    np.testing.assert_array_equal(g1.cpu().numpy(), g2.cpu().numpy())
    rng = np.random.default_rng(3)
    du, dv, tr = (torch.from_numpy(rng.standard_normal(k.ld)).cuda() for _ in range(3))
    u1, v1, u2, v2 = st._u.clone(), st._v.clone(), st._u.clone(), st._v.clone()
    lc1, lc2 = k.vec(), k.vec()
    k.call("otn_accept", 0.375, vptr(u1), vptr(du), vptr(v1), vptr(dv), vptr(st._log_c), vptr(tr),
           vptr(lc1))
    k.call("otn_vec", _lib.VEC_AXPY, 0.375, vptr(u2), vptr(du), None, None, vptr(u2))
    k.call("otn_vec", _lib.VEC_STEP_V, 0.375, vptr(v2), vptr(dv), vptr(st._log_c), vptr(tr),
           vptr(v2))
    k.copy(lc2, st._log_c)
    for x, y in ((u1, u2), (v1, v2), (lc1, lc2)):
        np.testing.assert_array_equal(x.cpu().numpy(), y.cpu().numpy())


def test_newton_step_column_kernels_path():
    """otn_newton_step with symmetric = 0 (the trial through the two-kernel
    column LSE on C itself, gated) equals the per-call path on the same
    asymmetric cost."""
    _, a = _state("pix:256:784:0", 2.0 ** 9)
    _, b = _state("pix:256:784:0", 2.0 ** 9)
    for st in (a, b):
        st._row_grad_norm()
        C = st._dc.C
        st._dc.col_args = (lambda C=C: (vptr(C), 0))     # no transpose: column kernels
    da, dva = a._dir_bufs()
    db, dvb = b._dir_bufs()
    res_a, mass_a, _ = _newton_step_device(a, a._system(), a._g, 0.5, 0.0, False, None, da, dva,
                                           ARMIJO_C1, ARMIJO_SLOPE_FLOOR)
    res_b = _newton_device(b._g, b._system(), 0.5, 0.0, False, None, db, dvb)
    assert res_a.status == res_b.status == _lib.OTN_OK
    mass_b = b._trial(db, dvb, 1.0, b._trial_buf())
    assert mass_a == mass_b
    np.testing.assert_array_equal(a._trial_vec.cpu().numpy(), b._trial_vec.cpu().numpy())


def test_persistent_launch_timing():
    """otn_set_timing / otn_coop_ms: device time of the last persistent launch
    (the bench's roofline source); an error while timing is off."""
    from paper_2504_02067_b200._device import TELEMETRY
    from paper_2504_02067_b200.errors import OTNError
    _, st = _state()
    st._row_grad_norm()
    d, dv = st._dir_bufs()
    TELEMETRY.reset()
    TELEMETRY.time_coop = True
    try:
        res, _, _ = _newton_step_device(st, st._system(), st._g, 0.5, 0.0, False, None, d, dv,
                                        ARMIJO_C1, ARMIJO_SLOPE_FLOOR)
        ms, hvps, dvflag, n, mode, nnz, span, cg = TELEMETRY.coop[-1]
        assert ms > 0.0 and hvps == res.hvps and n == st.n
        assert mode == res.plan_mode and cg == res.cg_iters
        assert 0 < nnz <= span <= n * st._ctx.ld
    finally:
        TELEMETRY.time_coop = False
    k = st._ctx
    assert k.coop_timing() is False
    with pytest.raises(OTNError):
        k.coop_ms()
