"""Context hygiene of the C-ABI: calls from another host
thread, stale device flags after a failed solve, and the ownership of
``Solution.P`` on device problems."""

import threading

import numpy as np
import pytest

from paper_2504_02067_b200 import DiscountedSystem, DualState, mdot, pcg_solve, problems
from paper_2504_02067_b200.errors import PlanOverflowError

pytestmark = pytest.mark.gpu


def _state(n, shift=0.0):
    C = problems.grid_points_cost(n, "l1")
    r = problems.gen_marginal(n, "smooth-random", 3)
    c = problems.gen_marginal(n, "smooth-random", 4)
    return DualState(problems.Problem(C=C, r=r, c=c), 4.0, u=np.log(r) + shift, v=np.log(c))


def test_calls_from_a_second_host_thread():
    """Every entry point makes its context's device current (static runtime:
    the current device is per host thread)."""
    st = _state(64)
    sysd = DiscountedSystem.from_state(st)
    b = np.random.default_rng(0).standard_normal(64) * 1e-3
    want, it_main = pcg_solve(sysd, 0.5, b, 1e-12)
    out = {}

    def worker():
        import torch
        torch.cuda.set_device(0)
        out["x"], out["it"] = pcg_solve(sysd, 0.5, b, 1e-12)
    th = threading.Thread(target=worker)
    th.start()
    th.join()
    assert out["it"] == it_main
    np.testing.assert_array_equal(out["x"], want)


def test_direct_system_after_an_overflowing_solve():
    """A PlanOverflow on a cached (device, n) context must not leak into a
    later system built directly from caller arrays."""
    bad = _state(64, shift=800.0)
    with pytest.raises(PlanOverflowError):
        DiscountedSystem.from_state(bad)
    good = DiscountedSystem(np.full((64, 64), 1.0 / 64 ** 2), np.full(64, 1.0 / 64),
                            np.full(64, 1.0 / 64))
    b = np.random.default_rng(1).standard_normal(64) * 1e-3
    x, _ = pcg_solve(good, 0.5, b, 1e-12)
    assert np.all(np.isfinite(x))


def test_device_solution_plan_is_not_overwritten():
    import torch
    p = problems.workload("grid:16:l1:1")
    dp = problems.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
    sol = mdot(dp, 2.0 ** 5, 2.0 ** 10)
    keep = sol.P.clone()
    st = sol.final_state
    st.u = st.u + 0.01                       # a different plan
    DiscountedSystem.from_state(st)          # materializes into the state's buffer
    assert torch.equal(sol.P, keep)


def test_device_solve_launches_only_library_kernels():
    """A solve of a device-resident problem (after the first, which prepares
    the cost) runs no framework kernels: every launch is the library's
    (buffers are zeroed by memsets, the symmetry test and transpose are
    library kernels, the prepared cost is reused)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    p = problems.workload("pix:1024:784:0")                     # asymmetric: transpose path
    dp = problems.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
    mdot(dp, 2.0 ** 5, 2.0 ** 9)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        mdot(dp, 2.0 ** 5, 2.0 ** 9)
        torch.cuda.synchronize()
    kernels = {e.name for e in prof.events() if e.device_type.name == "CUDA"
               and not e.name.lower().startswith(("memcpy", "memset"))}
    foreign = sorted(k for k in kernels if "otn::" not in k)
    assert kernels and not foreign, foreign
