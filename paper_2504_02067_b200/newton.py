"""The discounted Newton system and its device-resident solvers (mirrors ``newton.py``).

``F(rho) = D(rP) (I - rho P_rc)`` with ``P_rc = D(rP)^-1 P D(cP)^-1 P^T`` is
applied as two streaming passes over the plan in HBM (K6, K7).  ``pcg_solve``
and ``newton_solve`` each run as ONE persistent cooperative kernel
(``otn_pcg`` / ``otn_newton``): the CG loop, the 50-iteration true-residual
refresh, the L1 stopping test, the forcing test and the rho annealing all
happen on the device; the host reads back only the outcome record.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib, opcount
from ._device import TELEMETRY, Context, is_tensor, require_cuda, torch, vptr
from .errors import ConditioningError, NonconvergenceError, RefusalError, StagnationError

RHO_CAP = 1e-12               # newton.py:32
RHO_DECAY = 4.0               # newton.py:34
CG_TOL_FRACTION = 0.25        # newton.py:36
TRUE_RESIDUAL_REFRESH = 50    # newton.py:38 (compiled into the kernel)
LAMBDA2_MAX_N = 2048          # newton.py:40


@dataclass
class NewtonResult:
    """Outcome of one annealed truncated-Newton direction solve (newton.py:59-66)."""

    d_u: object
    rho_final: float
    cg_iters: int
    undiscounted_residual_l1: float


def _as_host(like, dev_vec, ctx):
    """Return dev_vec in the caller's array type (numpy in -> numpy out)."""
    if is_tensor(like):
        return dev_vec[: ctx.n].clone()
    return ctx.download(dev_vec)


class DiscountedSystem:
    """Plan snapshot realizing P_rc, P_c and F(rho) as device operators.

    Constructed either from host/device arrays (API parity with newton.py:72-79)
    or, on the solver path, from a DualState via :meth:`from_state`, which
    materializes the plan into the state's reusable HBM buffer together with
    the Jacobi diagonal (one fused pass, K4 + K5).
    """

    def __init__(self, P, rP, cP, *, _ctx=None, _mu=None, _icP=None, _mask=None):
        if _ctx is None:
            rP_h = rP.detach().cpu().numpy() if is_tensor(rP) else np.asarray(rP, dtype=np.float64)
            cP_h = cP.detach().cpu().numpy() if is_tensor(cP) else np.asarray(cP, dtype=np.float64)
            if np.any(rP_h <= 0.0) or np.any(cP_h <= 0.0):
                raise ConditioningError("plan row/column sums must be strictly positive")
            n = int(P.shape[0])
            ctx = Context.get(n, require_cuda(P.device if is_tensor(P) else None))
            Pd = ctx.mat()
            if is_tensor(P):
                Pd[:, : min(P.shape[1], ctx.ld)].copy_(P[:, : ctx.ld])
            else:
                from ._device import torch
                Pd[:, :n].copy_(torch().from_numpy(np.ascontiguousarray(P, dtype=np.float64)))
            self._ctx = ctx
            self._P = Pd
            self._rP = ctx.vec(rP_h)
            self._cP = ctx.vec(cP_h)
            self._icP = ctx.vec(1.0 / cP_h)
            self._mu_dev = None
            self._mask = ctx.seg_mask()
            ctx.call("otn_plan_mask", vptr(Pd), vptr(self._mask))
        else:
            self._ctx = _ctx
            self._P, self._rP, self._cP = P, rP, cP
            self._icP = _icP
            self._mu_dev = _mu
            self._mask = _mask
        self.n = self._ctx.n
        self._mu_counted = False

    @classmethod
    def from_state(cls, state, check_flags=True):
        """Snapshot the current plan (newton.py:81-90): rP, cP from the log-domain
        caches, P into the state's reusable buffer, mu fused into that pass.

        check_flags=False skips the host round trip for the overflow /
        nonpositive-sum flags: the persistent solver reads them first and
        returns the same statuses (same order), so the projector's Newton
        launch raises the same errors without an extra synchronization."""
        ctx = state._ctx
        bufs = getattr(state, "_sysbufs", None)
        if bufs is None:
            bufs = tuple(ctx.vec() for _ in range(4))
            state._sysbufs = bufs
        rP, cP, icP, mu = bufs
        lr, lc = state._lr_dev(), state._lc_dev()
        ctx.call("otn_system_prep", vptr(lr), vptr(lc), vptr(rP), vptr(cP), vptr(icP), None)
        P, mask = state._materialize(reuse_buffer=True, icP=icP, rP=rP, mu=mu, check=False)
        if check_flags:
            flags = (ctypes.c_int * 4)()
            ctx.call("otn_read_flags", flags)
            if flags[0]:
                _lib.raise_for_status(_lib.OTN_ST_PLAN_OVERFLOW, "materialize_plan")
            if flags[1]:
                _lib.raise_for_status(_lib.OTN_ST_NONPOSITIVE_SUMS, "DiscountedSystem")
        return cls(P, rP, cP, _ctx=ctx, _mu=mu, _icP=icP, _mask=mask)

    # -- host views for API parity ---------------------------------------------
    @property
    def P(self):
        return self._P[:, : self.n].cpu().numpy()

    @property
    def rP(self):
        return self._ctx.download(self._rP)

    @property
    def cP(self):
        return self._ctx.download(self._cP)

    def _in(self, d):
        if is_tensor(d):
            if d.shape[0] >= self._ctx.ld and d.is_contiguous():
                return d
            return self._ctx.vec(d)
        return self._ctx.vec(d)

    # -- operators (newton.py:92-112) ------------------------------------------------
    def apply_pc(self, d):
        """P_c d = (P^T d)/cP (newton.py:96-98)."""
        opcount.add(1)
        out = self._ctx.vec()
        self._ctx.call("otn_apply_pc", vptr(self._P), vptr(self._mask), vptr(self._cP),
                       vptr(self._in(d)), vptr(out))
        return _as_host(d, out, self._ctx)

    def apply_prc(self, d):
        """P_rc d = P((P^T d)/cP)/rP (newton.py:92-94)."""
        opcount.add(2)
        k = self._ctx
        w = k.vec()
        k.call("otn_apply_pc", vptr(self._P), vptr(self._mask), vptr(self._cP), vptr(self._in(d)),
               vptr(w))
        s = k.vec()
        k.call("otn_matvec", vptr(self._P), vptr(self._mask), vptr(w), vptr(s))
        out = s / self._rP.clamp_min(np.finfo(np.float64).tiny)
        return _as_host(d, out, k)

    def apply_F(self, rho, d):
        """F(rho) d = rP*d - rho*P((P^T d)/cP) (newton.py:100-105)."""
        if rho != 0.0:
            opcount.add(2)
        out = self._ctx.vec()
        self._ctx.call("otn_apply_F", vptr(self._P), vptr(self._mask), vptr(self._rP),
                       vptr(self._cP), float(rho), vptr(self._in(d)), vptr(out))
        return _as_host(d, out, self._ctx)

    def _newton_dir(self, grad_u, eta, rho0, zero_init, max_cg_iters, d_u, d_v):
        """newton_solve + d_v = -apply_pc(d_u) + slope in one device launch
        (newton.py:175-210, projector.py:196-205); op tally included."""
        res = _newton_device(grad_u, self, eta, rho0, zero_init, max_cg_iters, d_u, d_v)
        opcount.add(1)                       # d_v = -apply_pc(d_u)  (projector.py:201)
        return res

    def _tally_mu(self):
        if not self._mu_counted:
            opcount.add(2)
            self._mu_counted = True

    def _mu(self):
        if self._mu_dev is None:
            k = self._ctx
            self._mu_dev = k.vec()
            sq = k.vec()
            k.call("otn_square_matvec", vptr(self._P), vptr(self._icP), vptr(sq))
            self._mu_dev[: self.n] = sq[: self.n] / self._rP[: self.n]
        return self._mu_dev

    def diag_prc(self):
        """mu = diag(P_rc) = ((P*P) @ (1/cP)) / rP (newton.py:107-112)."""
        self._tally_mu()
        return self._ctx.download(self._mu())

    def dense_prc(self):
        """Dense P_rc for small-n validation (newton.py:116-117); host numpy."""
        P, rP, cP = self.P, self.rP, self.cP
        return (P / rP[:, None]) @ (P.T / cP[:, None])

    def dense_F(self, rho):
        return np.diag(self.rP) @ (np.eye(self.n) - rho * self.dense_prc())


def _finish(res, what, best, rho_for_msg=None, eta_gn=None):
    rc = res.status
    if rc == _lib.OTN_OK:
        return
    diag = {"rho": res.diag_rho, "residual_l1": res.diag_resid}
    if rc == _lib.OTN_ST_NONCONVERGENCE:
        raise NonconvergenceError("CG did not reach its tolerance within the iteration budget",
                                  best=best() if best else None, diagnostics=diag)
    if rc == _lib.OTN_ST_STAGNATION:
        raise StagnationError(
            f"discount reached {res.diag_rho} without meeting the forcing test "
            f"(residual {res.resid_l1:.3g} > {eta_gn:.3g})")
    if rc == _lib.OTN_ST_BREAKDOWN:
        raise ConditioningError(f"CG breakdown: curvature {res.diag_resid:.3g} along search direction")
    _lib.raise_for_status(rc, what)


def pcg_solve(sys, rho, b, tol_l1, d0=None, max_iters=None):
    """Jacobi-PCG for F(rho) d = b on the device (newton.py:123-172).

    Returns ``(d, iterations)`` in the caller's array type.
    """
    if not 0.0 <= rho < 1.0:
        raise ConditioningError(f"pcg_solve needs rho in [0, 1), got {rho}")
    if tol_l1 <= 0.0:
        raise ConditioningError("tol_l1 must be positive")
    if max_iters is None:
        max_iters = 10 * sys.n
    k = sys._ctx
    sys._tally_mu()
    mu = sys._mu()
    bd = sys._in(b)
    x = k.vec(d0) if d0 is not None else k.vec()
    res = _lib.SolveResult()
    rc = k.call("otn_pcg", vptr(sys._P), vptr(sys._mask), vptr(sys._rP), vptr(sys._cP), vptr(mu),
                float(rho),
                vptr(bd), float(tol_l1), vptr(x), int(d0 is not None), int(max_iters),
                ctypes.byref(res))
    opcount.add(2 * int(res.hvps))
    like = b if d0 is None else d0
    _finish(res if rc == res.status else res, "pcg_solve",
            best=lambda: _as_host(like, x, k))
    return _as_host(like, x, k), int(res.cg_iters)


def _newton_device(grad_u, sys, eta, rho0, zero_init, max_cg_iters, d_u, d_v):
    """One otn_newton launch; op tally as the reference's call pattern."""
    k = sys._ctx
    if max_cg_iters is None:
        max_cg_iters = 10 * sys.n
    res = _lib.SolveResult()
    timed = k.coop_timing()
    k.call("otn_newton", vptr(sys._P), vptr(sys._mask), vptr(sys._rP), vptr(sys._cP),
           vptr(sys._mu()),
           vptr(grad_u), float(eta), float(rho0), int(bool(zero_init)), int(max_cg_iters),
           vptr(d_u), vptr(d_v), ctypes.byref(res))
    if timed:
        TELEMETRY.coop.append((k.coop_ms(), int(res.hvps), int(d_v is not None), k.n,
                               int(res.plan_mode), int(res.plan_nnz), int(res.plan_span),
                               int(res.cg_iters)))
    if res.pcg_calls > 0:
        sys._tally_mu()
    opcount.add(2 * int(res.hvps))
    return res


def _newton_step_device(state, sys, grad_u, eta, rho0, zero_init, max_cg_iters, d_u, d_v,
                        armijo_c1, slope_floor, prework=None):
    """One otn_newton_step launch sequence for a DualState: the Newton
    direction, its trial at alpha = 1 and, when the Armijo test passes there,
    the accept path, with one host synchronization.  Returns
    (res, mass or None, row statistics or None); the op tally of the Newton
    part is added here, the trial's and the refresh's by the caller."""
    k = sys._ctx
    if max_cg_iters is None:
        max_cg_iters = 10 * sys.n
    res = _lib.SolveResult()
    out = (ctypes.c_double * 5)()
    fl = ctypes.c_int(0)
    timed = k.coop_timing()
    # every buffer is a persistent one of the state (its plan / system buffers,
    # direction buffers, potentials, caches): their pointers are built once
    key = (sys._P.data_ptr(), sys._rP.data_ptr(), d_u.data_ptr(), d_v.data_ptr(),
           grad_u.data_ptr())
    cached = getattr(state, "_nstep_ptrs", None)
    if cached is None or cached[0] != key:
        ccols, sym = state._dc.col_args()
        head = (vptr(sys._P), vptr(sys._mask), vptr(sys._rP), vptr(sys._cP), vptr(sys._mu()),
                vptr(grad_u))
        mid = (vptr(d_u), vptr(d_v), state._dc.ptr(), ccols, sym)
        tail = (vptr(state._u), vptr(state._v), vptr(state._r), vptr(state._log_c),
                vptr(state._trial_vec), vptr(state._lc), vptr(state._lr), vptr(state._g))
        cached = state._nstep_ptrs = (key, head, mid, tail)
    _, head, mid, tail = cached
    if prework is None:
        k.call("otn_newton_step", *head, float(eta), float(rho0), int(bool(zero_init)),
               int(max_cg_iters), *mid, state._ng, *tail,
               float(armijo_c1), float(slope_floor), ctypes.byref(res), out, ctypes.byref(fl))
    else:
        # enqueue, do the caller's host work while the GPU runs the step, collect
        k.call("otn_newton_step", *head, float(eta), float(rho0), int(bool(zero_init)),
               int(max_cg_iters), *mid, state._ng, *tail,
               float(armijo_c1), float(slope_floor), None, None, None)
        prework()
        k.call("otn_newton_step_wait", ctypes.byref(res), out, ctypes.byref(fl))
    if timed:
        TELEMETRY.coop.append((k.coop_ms(), int(res.hvps), 1, k.n, int(res.plan_mode),
                               int(res.plan_nnz), int(res.plan_span), int(res.cg_iters)))
    if res.pcg_calls > 0:
        sys._tally_mu()
    opcount.add(2 * int(res.hvps))
    opcount.add(1)                           # d_v = -apply_pc(d_u)  (projector.py:201)
    mass = float(out[0]) if out[3] else None
    rowstat = (float(out[1]), float(out[2]), int(fl.value)) if out[4] else None
    return res, mass, rowstat


def newton_solve(grad_u, sys, eta, rho0=0.0, zero_init=False, max_cg_iters=None):
    """Annealed discounted solve for the truncated Newton direction (newton.py:175-210)."""
    if eta <= 0.0:
        raise ConditioningError(f"eta must be positive, got {eta}")
    if not 0.0 <= rho0 < 1.0:
        raise ConditioningError(f"rho0 must be in [0, 1), got {rho0}")
    k = sys._ctx
    g = sys._in(grad_u)
    d = k.vec()
    res = _newton_device(g, sys, eta, rho0, zero_init, max_cg_iters, d, None)
    gn = float(np.abs(k.download(g)).sum()) if res.status == _lib.OTN_ST_STAGNATION else 0.0
    _finish(res, "newton_solve", best=lambda: _as_host(grad_u, d, k), eta_gn=eta * gn)
    return NewtonResult(_as_host(grad_u, d, k), float(res.rho_final), int(res.cg_iters),
                        float(res.resid_l1))


def next_rho0(rho_old):
    """Warm-start discount for the next solve (newton.py:213-217)."""
    if not 0.0 <= rho_old < 1.0:
        raise ConditioningError(f"rho_old must be in [0, 1), got {rho_old}")
    return max(0.0, 1.0 - (1.0 - rho_old) * RHO_DECAY)


def lambda2(sys, tol=1e-13):
    """Second-largest eigenvalue of P_rc (newton.py:220-236).

    The reference eigendecomposes the dense symmetric form
    S = D(rP)^-1/2 P D(cP)^-1 P^T D(rP)^-1/2 (similar to P_rc).  Here S is
    never formed: Lanczos with full reorthogonalization runs on the device
    operators (S x = D(rP)^-1/2 P ((P^T D(rP)^-1/2 x) / cP): one apply_pc and
    one matvec launch per step), restarting from a fresh vector orthogonal to
    the basis if the Krylov space closes, until the two largest Ritz values'
    residual bounds are below ``tol`` (or the basis spans R^n, where they are
    exact).  Same guard, leading-eigenvalue check and clamp as the reference.
    """
    n = sys.n
    if n > LAMBDA2_MAX_N:
        raise RefusalError(f"lambda2 needs a dense eigensolve; n={n} exceeds {LAMBDA2_MAX_N}")
    t = torch()
    k = sys._ctx
    isr = 1.0 / t.sqrt(sys._rP[:n])
    w = k.vec()
    s_vec = k.vec()
    xin = k.vec()

    def apply_S(x):
        xin[:n] = x * isr
        k.call("otn_apply_pc", vptr(sys._P), vptr(sys._mask), vptr(sys._cP), vptr(xin), vptr(w))
        k.call("otn_matvec", vptr(sys._P), vptr(sys._mask), vptr(w), vptr(s_vec))
        return s_vec[:n] * isr

    gen = t.Generator(device=k.device).manual_seed(2504)
    Q = t.zeros((n, n), dtype=t.float64, device=k.device)
    alphas, betas = [], []
    q = t.rand(n, dtype=t.float64, device=k.device, generator=gen) + 0.5
    q /= t.linalg.vector_norm(q)
    m = 0
    evals = np.zeros(1)
    while m < n:
        Q[:, m] = q
        r = apply_S(q)
        a = float(t.dot(q, r))
        r -= a * q
        if m > 0 and betas[-1] > 0.0:
            r -= betas[-1] * Q[:, m - 1]
        for _ in range(2):                         # full reorthogonalization (twice is enough)
            r -= Q[:, : m + 1] @ (Q[:, : m + 1].T @ r)
        alphas.append(a)
        b = float(t.linalg.vector_norm(r))
        m += 1
        T = np.diag(alphas) + np.diag(betas[: m - 1], 1) + np.diag(betas[: m - 1], -1)
        evals, vecs = np.linalg.eigh(T)
        scale = max(abs(evals[-1]), 1.0)
        if m == n:
            break
        if m >= 2 and b * max(abs(vecs[-1, -1]), abs(vecs[-1, -2])) <= tol * scale and m >= min(n, 8):
            break
        if b <= 1e-14 * scale:                     # invariant subspace: restart orthogonally
            betas.append(0.0)
            for _ in range(10):
                q = t.rand(n, dtype=t.float64, device=k.device, generator=gen) - 0.5
                for _ in range(2):
                    q -= Q[:, :m] @ (Q[:, :m].T @ q)
                nq = float(t.linalg.vector_norm(q))
                if nq > 1e-8:
                    break
            q = q / nq
        else:
            betas.append(b)
            q = r / b
    opcount.add(2 * m)
    lead = float(evals[-1])
    if abs(lead - 1.0) > 1e-8:
        raise ConditioningError(f"leading eigenvalue of P_rc is {lead}, expected 1")
    if n == 1:
        return 0.0
    return float(min(evals[-2], 1.0 - 1e-16))
