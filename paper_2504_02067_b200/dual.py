"""Dual potentials and the log-domain plan, resident in HBM (mirrors ``dual.py:22-219``).

The plan implied by potentials (u, v) at inverse temperature gamma is
``P_ij = exp(u_i + v_j - gamma*C_ij)``.  Row and column sums are always
log-domain reductions over the stored cost (kernels K1/K2 of the C-ABI), never
sums of the linear plan, and are cached until u, v or gamma is reassigned —
the same invalidation contract as the reference.

Every vector lives on the GPU in a padded buffer.  The public attributes
(``u``, ``v``, ``log_rP``, ``row_sums()`` ...) return host numpy copies so code
written against the reference keeps working; the solver itself only touches
the device buffers (``_u``, ``_lr`` ...).  The op tally is incremented at the
reference's call sites (``dual.py:73,87,95,97,163,173,181,191,205``).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib, opcount
from ._device import DeviceCost, is_tensor, require_cuda, torch, vptr
from .errors import DomainError


def device_cost(problem, device=None):
    """The problem's device-resident cost, created once per problem object."""
    dc = getattr(problem, "_otn_state_cost", None)
    dev = require_cuda(device)
    if dc is None or dc.ctx.device != dev:
        dc = DeviceCost.of(problem, dev)
        try:
            problem._otn_state_cost = dc
        except AttributeError:
            pass
    else:
        dc.ctx.sync_stream()
    return dc


class DeferredScalar:
    """A device reduction result in flight: value() = out[0] + out[1] once the
    stream has passed the copy (telemetry the control flow does not branch on).
    A fresh 64-slot block is allocated when one fills, so a slot is never
    reused while a value in it is pending."""

    __slots__ = ("_host", "_stream")

    def __init__(self, host, stream):
        self._host, self._stream = host, stream

    def value(self):
        self._stream.synchronize()
        h = self._host.numpy()
        return float(h[0] + h[1])


class DualState:
    """Single-owner mutable dual state at one temperature (dual.py:22-46)."""

    def __init__(self, problem, gamma, u=None, v=None, r=None, c=None, *, cost=None):
        if not np.isfinite(gamma) or gamma <= 0.0:
            raise DomainError(f"gamma must be positive and finite, got {gamma}")
        self.problem = problem
        self._dc = cost if cost is not None else device_cost(problem)
        self._ctx = self._dc.ctx
        k = self._ctx
        self._gamma = float(gamma)
        # u and v as the two rows of one device block, filled by one
        # stream-ordered copy from page-locked staging (no host stall)
        self._uv = k.zeros((2, k.ld))
        self._u, self._v = self._uv.unbind(0)
        init = [np.zeros(self.n) if x is None else x for x in (u, v)]
        if any(is_tensor(x) for x in init):
            k.upload(self._u, init[0])
            k.upload(self._v, init[1])
        else:
            k.upload_rows_async(self._uv, init, "uv")
        self._lr = k.vec()
        self._lc = k.vec()
        self._g = k.vec()
        self._trial_vec = k.vec()
        self._tmp = k.vec()
        self._cache_valid = False
        self._rowstat = None
        self._K_formed = False
        self._KT_formed = False
        self._plan_buf = None
        self.set_targets(problem.r if r is None else r, problem.c if c is None else c)

    # -- invalidating attributes (dual.py:48-54) ----------------------------
    @property
    def n(self):
        return self.problem.n

    @property
    def gamma(self):
        return self._gamma

    @gamma.setter
    def gamma(self, value):
        self._gamma = float(value)
        self._cache_valid = False
        self._rowstat = None
        self._K_formed = False
        self._KT_formed = False

    @property
    def u(self):
        return self._ctx.download(self._u)

    @u.setter
    def u(self, value):
        self._ctx.upload(self._u, value)
        self._invalidate()

    @property
    def v(self):
        return self._ctx.download(self._v)

    @v.setter
    def v(self, value):
        self._ctx.upload(self._v, value)
        self._invalidate()

    def _invalidate(self):
        self._cache_valid = False
        self._rowstat = None

    @property
    def cache_valid(self):
        return self._cache_valid

    def set_targets(self, r, c, _logs=None):
        """Swap the target marginals (dual.py:64-67); logs are taken on the host
        with numpy, exactly as the reference's np.log(r) / np.log(c) (mdot may
        pass them precomputed: ``_logs`` = (np.log(r), np.log(c))).  The four
        device vectors are rewritten in place by stream-ordered copies from
        page-locked staging (no host stall); the same arrays again are a no-op."""
        r = np.asarray(r, dtype=np.float64)
        c = np.asarray(c, dtype=np.float64)
        prev = getattr(self, "_targets_copy", None)
        if prev is not None and np.array_equal(prev[0], r) and np.array_equal(prev[1], c):
            self.r, self.c = r, c                   # same values (copy kept: safe if mutated)
            return
        self.r = r
        self.c = c
        k = self._ctx
        if getattr(self, "_tgt", None) is None:
            # r, c, log r, log c as rows of one device block: one H2D copy
            self._tgt = k.zeros((4, k.ld))
            self._r, self._c, self._log_r, self._log_c = self._tgt.unbind(0)
        with np.errstate(divide="ignore", invalid="ignore"):
            lr, lc = _logs if _logs is not None else (np.log(self.r), np.log(self.c))
            k.upload_rows_async(self._tgt, (self.r, self.c, lr, lc), "targets")
        self._targets_copy = (self.r.copy(), self.c.copy())
        self._rowstat = None

    # -- op tally for the implicit K = -gamma C and its transpose -----------
    @property
    def _ng(self):
        return -self._gamma

    def _touch_K(self):
        if not self._K_formed:
            opcount.add(1)          # dual.py:73
            self._K_formed = True

    def _touch_KT(self):
        if not self._KT_formed:
            self._touch_K()
            if not self._dc.symmetric:
                opcount.add(1)      # dual.py:87
            self._KT_formed = True

    # -- device kernels --------------------------------------------------------
    def _lse_rows(self, outer, inner, out):
        self._touch_K()
        self._ctx.call("otn_lse_rows", self._dc.ptr(), self._ng, vptr(outer), vptr(inner),
                       vptr(out))

    def _lse_cols(self, outer, inner, out):
        self._touch_KT()
        self._ctx.call("otn_lse_cols", *self._dc.col_args(), self._ng,
                       vptr(outer), vptr(inner), vptr(out))

    def refresh(self):
        """Recompute both cached log sums (dual.py:91-102)."""
        if not np.isfinite(self._gamma):
            raise DomainError("gamma must be finite")
        opcount.add(4)
        self._lse_rows(self._u, self._v, self._lr)
        opcount.add(4)
        self._lse_cols(self._v, self._u, self._lc)
        self._cache_valid = True
        self._rowstat = None

    def refresh_row_sums(self):
        self.refresh()
        return self.log_rP

    def _lr_dev(self):
        if not self._cache_valid:
            self.refresh()
        return self._lr

    def _lc_dev(self):
        if not self._cache_valid:
            self.refresh()
        return self._lc

    @property
    def log_rP(self):
        return self._ctx.download(self._lr_dev())

    @property
    def log_cP(self):
        return self._ctx.download(self._lc_dev())

    def set_log_row_sums(self, log_rP):
        self._ctx.upload(self._lr, log_rP)
        self._rowstat = None

    def set_log_col_sums(self, log_cP):
        self._ctx.upload(self._lc, log_cP)

    def mark_cache_valid(self):
        self._cache_valid = True

    def row_sums(self):
        return np.exp(self.log_rP)

    def col_sums(self):
        return np.exp(self.log_cP)

    # -- derived quantities (device reductions) ---------------------------------
    def _row_stats(self):
        """(||exp(log_rP) - r||_1, sum r^2/exp(log_rP), flags); g = exp(log_rP) - r
        is left in self._g.  Cached until log_rP or r changes."""
        if self._rowstat is None:
            lr = self._lr_dev()
            out = (ctypes.c_double * 2)()
            fl = ctypes.c_int(0)
            # g = exp(lr) - r and the row statistics in one pass
            self._ctx.call("otn_row_stats", vptr(lr), vptr(self._r), vptr(self._g), out,
                           ctypes.byref(fl))
            self._rowstat = (float(out[0]), float(out[1]), int(fl.value))
        return self._rowstat

    def _row_grad_norm(self):
        return self._row_stats()[0]

    def _chi_sq(self):
        """chi_sq_div(r, row_sums()) (core.py:42-52) with its domain checks."""
        _, s, fl = self._row_stats()
        if fl & 1:
            raise DomainError("chi_sq_div requires strictly positive reference x")
        if fl & 2:
            raise DomainError("chi_sq_div requires nonnegative y")
        return float(s - 1.0)

    def gradient(self):
        """(grad_u, grad_v) = (r(P) - r, c(P) - c) as host arrays (dual.py:142-144)."""
        return self.row_sums() - self.r, self.col_sums() - self.c

    def grad_norm_l1(self):
        """||r(P) - r||_1 + ||c(P) - c||_1 on the device (dual.py:146-148)."""
        out = (ctypes.c_double * 2)()
        self._ctx.call("otn_reduce", _lib.RED_GRAD_L1, vptr(self._lr_dev()), vptr(self._r),
                       vptr(self._lc_dev()), vptr(self._c), out, None)
        return float(out[0] + out[1])

    def _grad_norm_l1_deferred(self):
        """grad_norm_l1 without waiting for it: the reduction is enqueued and its
        result read back stream-ordered into a page-locked slot; value() waits
        for the stream only if it has not passed the copy yet."""
        t = torch()
        slots = getattr(self, "_gn_slots", None)
        if slots is None or self._gn_next == slots.shape[0]:
            slots = self._gn_slots = t.empty((64, 2), dtype=t.float64, pin_memory=True)
            self._gn_next = 0
        host = slots[self._gn_next]
        self._gn_next += 1
        self._ctx.call("otn_reduce_async", _lib.RED_GRAD_L1, vptr(self._lr_dev()), vptr(self._r),
                       vptr(self._lc_dev()), vptr(self._c), ctypes.c_void_p(host.data_ptr()))
        return DeferredScalar(host, t.cuda.current_stream(self._ctx.device))

    def dual_value(self):
        """sum(P) - 1 - <u, r> - <v, c> (dual.py:150-153)."""
        k = self._ctx
        out = (ctypes.c_double * 2)()
        k.call("otn_reduce", _lib.RED_SUM_EXP, vptr(self._lr_dev()), None, None, None, out, None)
        mass = float(out[0])
        k.call("otn_reduce", _lib.RED_DOT, vptr(self._u), vptr(self._r), None, None, out, None)
        ur = float(out[0])
        k.call("otn_reduce", _lib.RED_DOT, vptr(self._v), vptr(self._c), None, None, out, None)
        vc = float(out[0])
        return mass - 1.0 - ur - vc

    # -- plan --------------------------------------------------------------------
    def _materialize(self, reuse_buffer=False, icP=None, rP=None, mu=None, check=True):
        """Device plan (P n x ld, segment mask); optional fused Jacobi diagonal (K4 + K5)."""
        opcount.add(4)
        self._touch_K()
        k = self._ctx
        if reuse_buffer:
            if self._plan_buf is None:
                self._plan_buf = (k.mat(), k.seg_mask())
            P, mask = self._plan_buf
        else:
            P, mask = k.mat(), k.seg_mask()
        flag = ctypes.c_int(0)
        rc = k.call("otn_materialize", self._dc.ptr(), self._ng, vptr(self._u), vptr(self._v),
                    vptr(P), vptr(icP), vptr(rP), vptr(mu),
                    ctypes.byref(flag) if check else None, vptr(mask))
        if rc == _lib.OTN_ST_PLAN_OVERFLOW:
            _lib.raise_for_status(rc, "materialize_plan")
        return P, mask

    def materialize_plan(self, reuse_buffer=False):
        """Linear-domain plan (dual.py:155-169); host array for host problems."""
        P, _ = self._materialize(reuse_buffer=reuse_buffer)
        if is_tensor(self.problem.C):
            return P[:, : self.n]
        return P[:, : self.n].cpu().numpy()

    def _trial(self, d_u, d_v, alpha, out):
        """Trial log column sums at (u + alpha d_u, v + alpha d_v) and the plan
        mass (dual.py:171-175 + projector.py:122-126); returns the mass."""
        opcount.add(4)
        self._touch_KT()
        mass = ctypes.c_double(0.0)
        self._ctx.call("otn_trial_cols", *self._dc.col_args(), self._ng,
                       vptr(self._u), vptr(d_u), vptr(self._v), vptr(d_v), float(alpha),
                       vptr(out), ctypes.byref(mass))
        return float(mass.value)

    def _trial_buf(self):
        return self._trial_vec

    def _tally_trial(self):
        """Op tally of one _trial call (its pass ran inside otn_newton_step)."""
        opcount.add(4)
        self._touch_KT()

    def _newton_step(self, sys, eta, rho0, zero_init, max_cg_iters, d_u, d_v, armijo_c1,
                     slope_floor):
        """Newton direction + first trial + (if accepted) accept path in one
        synchronization (otn_newton_step); see projector.project."""
        from .newton import _newton_step_device
        # host work the driver queued for the next GPU-bound wait (mdot: the
        # next stage's candidate targets), run while the GPU solves this step
        prework = self.__dict__.pop("_prework", None)
        res, mass, rowstat = _newton_step_device(self, sys, self._g, eta, rho0, zero_init,
                                                 max_cg_iters, d_u, d_v, armijo_c1, slope_floor,
                                                 prework=prework)
        if rowstat is not None:
            # the device ran _accept(1.0, d_u, d_v) + refresh_rows_only + _row_stats
            self._cache_valid = True
            self._rowstat = rowstat
        return res, mass, rowstat is not None

    def _tally_refresh_rows(self):
        opcount.add(4)                              # refresh_rows_only (dual.py:203-208)

    def trial_log_col_sums(self, d_u, d_v, alpha):
        k = self._ctx
        du = d_u if is_tensor(d_u) else k.vec(d_u)
        dv = d_v if is_tensor(d_v) else k.vec(d_v)
        out = k.vec()
        self._trial(du, dv, alpha, out)
        return k.download(out)

    # -- exact scaling updates (dual.py:179-208) --------------------------------
    def rebalance_columns(self):
        """v = log c - LSE_cols(u); log c(P) := log c; refresh rows (dual.py:179-184)."""
        opcount.add(4)
        self._touch_KT()
        self._ctx.call("otn_rebalance_cols", *self._dc.col_args(), self._ng,
                       vptr(self._log_c), vptr(self._u), vptr(self._v))
        self._invalidate()
        self._ctx.copy(self._lc, self._log_c)
        self.refresh_rows_only()

    def scale_rows_to_target(self):
        """u += log r - log r(P); log r(P) := log r; column cache (dual.py:186-194)."""
        lr = self._lr_dev()
        self._ctx.call("otn_vec", _lib.VEC_ADD_SUB, 0.0, vptr(self._u), vptr(self._log_r),
                       vptr(lr), None, vptr(self._u))
        self._invalidate()
        self._ctx.copy(self._lr, self._log_r)
        opcount.add(4)
        self._lse_cols(self._v, self._u, self._lc)
        self._cache_valid = True

    def scale_cols_to_target(self):
        """v += log c - log c(P); log c(P) := log c; refresh rows (dual.py:196-201)."""
        lc = self._lc_dev()
        self._ctx.call("otn_vec", _lib.VEC_ADD_SUB, 0.0, vptr(self._v), vptr(self._log_c),
                       vptr(lc), None, vptr(self._v))
        self._invalidate()
        self._ctx.copy(self._lc, self._log_c)
        self.refresh_rows_only()

    def refresh_rows_only(self):
        """log r(P) = LSE_rows, column cache assumed current (dual.py:203-208)."""
        opcount.add(4)
        self._lse_rows(self._u, self._v, self._lr)
        self._rowstat = None
        self._cache_valid = True

    # -- stacked potentials (dual.py:212-219) ------------------------------------
    @property
    def z(self):
        return np.concatenate([self.u, self.v])

    def set_z(self, z):
        n = self.n
        if is_tensor(z):
            self._u[:n].copy_(z[:n])
            self._v[:n].copy_(z[n:])
            self._invalidate()
        else:
            self.u = np.asarray(z[:n], dtype=np.float64)
            self.v = np.asarray(z[n:], dtype=np.float64)

    # -- hooks used by project() / mdot() (shared with the point-cloud state) ---
    def _row_scaling_update(self):
        """u = (u + log r) - log r(P)  (projector.py:146, dual.py:189)."""
        self._ctx.call("otn_vec", _lib.VEC_ADD_SUB, 0.0, vptr(self._u), vptr(self._log_r),
                       vptr(self._lr_dev()), None, vptr(self._u))
        self._invalidate()

    def _accept(self, alpha, d_u, d_v):
        """u += alpha d_u; v = (v + alpha d_v) + (log c - trial); log c(P) = log c
        (projector.py:234-236)."""
        self._ctx.call("otn_accept", float(alpha), vptr(self._u), vptr(d_u), vptr(self._v),
                       vptr(d_v), vptr(self._log_c), vptr(self._trial_vec), vptr(self._lc))
        self._invalidate()

    def _system(self):
        from .newton import DiscountedSystem
        return DiscountedSystem.from_state(self, check_flags=False)   # the Newton launch checks

    def _dir_bufs(self):
        bufs = getattr(self, "_dirbufs", None)
        if bufs is None:
            bufs = (self._ctx.vec(), self._ctx.vec())
            self._dirbufs = bufs
        return bufs

    def _download_rows(self, buf):
        return self._ctx.download(buf)

    def _snapshot(self):
        """Device copy of (u, v) for the annealing driver's extrapolation.  The
        driver holds at most the previous and the current snapshot, so two
        buffer pairs alternate (stream-ordered copies, no allocation)."""
        k = self._ctx
        pairs = getattr(self, "_snap_bufs", None)
        if pairs is None:
            pairs = self._snap_bufs = ((k.vec(), k.vec()), (k.vec(), k.vec()))
            self._snap_next = 0
        u, v = pairs[self._snap_next]
        self._snap_next ^= 1
        k.copy(u, self._u)
        k.copy(v, self._v)
        return u, v

    def _extrapolate(self, step, z_cur, z_prev):
        """(u, v) = z + step * (z - z_prev)  (driver.py:170-175)."""
        k = self._ctx
        k.call("otn_vec", _lib.VEC_EXTRAP, float(step), vptr(z_cur[0]), vptr(z_prev[0]), None,
               None, vptr(self._u))
        k.call("otn_vec", _lib.VEC_EXTRAP, float(step), vptr(z_cur[1]), vptr(z_prev[1]), None,
               None, vptr(self._v))
        self._invalidate()

    def _finalize(self, problem):
        """Fresh plan, rounding onto U(r, c), primal <P, C> (driver.py:306-310).
        Returns (P in the problem's array type, primal cost)."""
        from ._device import TELEMETRY
        from .driver import _round_device
        k = self._ctx
        P, _ = self._materialize(reuse_buffer=True)
        primal = _round_device(k, P, self._dc.C, k.vec(problem.r), k.vec(problem.c))
        opcount.add(1)          # <P, C>  (driver.py:309)
        if is_tensor(problem.C):
            # the returned plan leaves the state: a later from_state /
            # materialize_plan(reuse_buffer=True) on final_state gets a new
            # buffer instead of overwriting Solution.P (the reference returns
            # a fresh array from round_plan, driver.py:178-208)
            self._plan_buf = None
            return P[:, : problem.n], primal
        # D2H through page-locked memory (DMA at full PCIe/C2C rate; a pageable
        # copy of the 134 MB plan is ~25x slower); torch caches the pinned block
        t = torch()
        host = t.empty((problem.n, problem.n), dtype=t.float64, pin_memory=True)
        host.copy_(P[:, : problem.n])
        TELEMETRY.d2h += host.numel() * 8
        return host.numpy(), primal
