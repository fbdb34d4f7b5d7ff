"""CPU oracle for the truncated-Newton EOT hot path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The B200 package (``paper_2504_02067_b200``)
never imports anything from ``oracle/`` and fails loudly when its CUDA library
is missing.

It is a from-scratch numpy restatement of the reference solver
(``otnewton`` 0.1.0, ``/root/reference/pkg/src/otnewton``).  Every function
names the reference lines it restates.  The restatement keeps the reference's
floating-point operand order (same numpy reductions, same BLAS dgemv calls,
same 256-row tiling of the dense kernels) so that its results are
*bit-identical* to the reference on the same inputs.

Parity pin: ``tests/test_oracle_pin.py`` checks this module against golden
vectors produced by the reference itself (``tests/golden/make_golden.py``,
run in the build container where ``/root/reference`` is importable) and
against the reference's own known-answer values (closed-form n=2 fixture,
Jacobi-exact direction, eps_rule / error-bound constants, ...).
"""

from __future__ import annotations

import math
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# constants (reference: newton.py:31-40, projector.py:23-37, driver.py:27-34,
# _kernels.py:16-19)
# ---------------------------------------------------------------------------
TILE_ROWS = 256            # _kernels.py:16  (BLOCK)
EXP_OVERFLOW = 700.0       # _kernels.py:19  (LOG_OVERFLOW)
RHO_FLOOR_GAP = 1e-12      # newton.py:32    (RHO_CAP)
RHO_DIVISOR = 4.0          # newton.py:34    (RHO_DECAY)
CG_SHARE = 0.25            # newton.py:36    (CG_TOL_FRACTION)
REFRESH_EVERY = 50         # newton.py:38    (TRUE_RESIDUAL_REFRESH)
C1 = 0.01                  # projector.py:24 (ARMIJO_C1)
SLOPE_FLOOR = 1e-13        # projector.py:28 (ARMIJO_SLOPE_FLOOR)
ETA_CAP = 0.99             # projector.py:31 (ETA_MAX)
CHI_POW = 0.4              # projector.py:33 (CHI_EXPONENT)
ALPHA_MIN = 2.0 ** -30     # projector.py:34 (MIN_ALPHA)
W_ROW, W_COL = 0.45, 0.05  # driver.py:27-28
Q_UP, Q_DOWN = 0.95, 0.8   # driver.py:29-30
Q_HI, Q_LO = 2.0, 2.0 ** (1.0 / 16.0)  # driver.py:31-34


class OracleFailure(Exception):
    """Any solver failure; ``kind`` names the reference exception class."""

    def __init__(self, kind, msg, best=None, diag=None):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind
        self.best = best
        self.diag = dict(diag or {})


# Primitive call counter (bench.py's CPU-baseline kernel mix; not in the reference).
CALLS = {}


def _hit(name):
    CALLS[name] = CALLS.get(name, 0) + 1


# ---------------------------------------------------------------------------
# operation tally (restates opcount.py:36-66; categories at the same sites)
# ---------------------------------------------------------------------------
class Tally:
    def __init__(self):
        self.counts = {}
        self.stack = []

    def bump(self, k):
        key = self.stack[-1] if self.stack else "other"
        self.counts[key] = self.counts.get(key, 0) + k

    def total(self):
        return sum(self.counts.values())

    class _Scope:
        def __init__(self, tally, name):
            self.tally, self.name = tally, name

        def __enter__(self):
            self.tally.stack.append(self.name)

        def __exit__(self, *exc):
            self.tally.stack.pop()

    def under(self, name):
        return Tally._Scope(self, name)


# ---------------------------------------------------------------------------
# dense kernels (restate _kernels.py:22-74 and newton.py:43-56)
# ---------------------------------------------------------------------------
# Host threads for the 256-row slabs of the dense kernels.  Every slab is an
# independent computation (its own max, exps, pairwise sums / dgemv), so the
# result is bit-identical for any thread count; only bench.py's CPU baseline
# raises it (set_threads).
THREADS = 1
_POOL = None
_LOCAL = threading.local()


def set_threads(k):
    """Run the slabs of the dense kernels on ``k`` host threads (numpy releases
    the GIL inside its ufunc loops and OpenBLAS calls)."""
    global THREADS, _POOL
    k = max(1, int(k))
    if k != THREADS:
        if _POOL is not None:
            _POOL.shutdown(wait=True)
        _POOL = ThreadPoolExecutor(max_workers=k) if k > 1 else None
        THREADS = k


def _slabs(rows, fn):
    spans = [(a, min(a + TILE_ROWS, rows)) for a in range(0, rows, TILE_ROWS)]
    if _POOL is None or len(spans) == 1:
        for a, b in spans:
            fn(a, b)
    else:
        for f in [_POOL.submit(fn, a, b) for a, b in spans]:
            f.result()


def _scratch(rows, cols):
    buf = getattr(_LOCAL, "buf", None)
    if buf is None or buf.shape[0] < rows or buf.shape[1] != cols:
        buf = _LOCAL.buf = np.empty((rows, cols))
    return buf[:rows]


def tiled_row_lse(K, outer, inner):
    """outer + LSE_j(K_ij + inner_j), all -inf rows -> -inf.  (_kernels.py:22-42)

    Per-row shift by the row max, numpy pairwise sum of the shifted exps over
    the whole row; tiled in 256-row slabs exactly like the reference.
    """
    _hit("lse")
    rows = K.shape[0]
    res = np.empty(rows)

    def slab(a, b):
        t = _scratch(b - a, K.shape[1])
        np.add(K[a:b], inner[None, :], out=t)
        mx = t.max(axis=1)
        ok = np.isfinite(mx)
        sh = np.where(ok, mx, 0.0)
        np.subtract(t, sh[:, None], out=t)
        np.exp(t, out=t)
        with np.errstate(divide="ignore"):
            val = sh + np.log(t.sum(axis=1))
        res[a:b] = np.where(ok, val, -np.inf)
    _slabs(rows, slab)
    return outer + res


def tiled_plan(K, u, v, out=None):
    """exp((K + v) + u) with the >700 overflow rejection.  (_kernels.py:45-61)"""
    _hit("plan")
    rows, cols = K.shape
    out = np.empty((rows, cols)) if out is None else out
    over = []

    def slab(a, b):
        t = out[a:b]
        np.add(K[a:b], v[None, :], out=t)
        np.add(t, u[a:b, None], out=t)
        m = t.max()
        if m > EXP_OVERFLOW:
            over.append((a, m))
            return
        with np.errstate(under="ignore"):
            np.exp(t, out=t)
    _slabs(rows, slab)
    if over:
        raise OracleFailure("PlanOverflowError", f"log-plan entry {min(over)[1]:.3g}")
    return out


def tiled_square_mv(P, w):
    """(P*P) @ w, one dgemv per 256-row slab.  (_kernels.py:64-74)"""
    _hit("sqmv")
    rows = P.shape[0]
    res = np.empty(rows)

    def slab(a, b):
        t = _scratch(b - a, P.shape[1])
        np.multiply(P[a:b], P[a:b], out=t)
        res[a:b] = t @ w
    _slabs(rows, slab)
    return res


def mv(P, x, tally):
    """P @ x (BLAS dgemv-N).  (newton.py:43-48)"""
    _hit("mv")
    tally.bump(1)
    return P @ x


def rmv(P, x, tally):
    """P.T @ x (BLAS dgemv-T).  (newton.py:51-56)"""
    _hit("rmv")
    tally.bump(1)
    return P.T @ x


# ---------------------------------------------------------------------------
# small numerics (restate core.py:42-72)
# ---------------------------------------------------------------------------
def entropy(p):
    pos = p[p > 0.0]
    return float(-np.sum(pos * np.log(pos)))


def chi2(y, x):
    if np.any(x <= 0.0) or np.any(y < 0.0):
        raise OracleFailure("DomainError", "chi-square needs x > 0, y >= 0")
    return float(np.sum(y * y / x) - 1.0)


# ---------------------------------------------------------------------------
# dual state (restates dual.py:22-219)
# ---------------------------------------------------------------------------
class Dual:
    """u, v, gamma, targets; lazily cached log row/col sums with invalidation."""

    def __init__(self, C, gamma, u, v, r, c, tally):
        self.C = C
        self.tally = tally
        self._gamma = float(gamma)
        self._u = np.array(u, dtype=np.float64)
        self._v = np.array(v, dtype=np.float64)
        self.r, self.c = r, c
        self._K = self._KT = None
        self._sym = None
        self._lr = self._lc = None
        self.valid = False
        self._plan = None

    # assignments invalidate the caches (dual.py:48-54)
    @property
    def u(self):
        return self._u

    @u.setter
    def u(self, val):
        self._u, self.valid = val, False

    @property
    def v(self):
        return self._v

    @v.setter
    def v(self, val):
        self._v, self.valid = val, False

    @property
    def gamma(self):
        return self._gamma

    @gamma.setter
    def gamma(self, g):
        self._gamma, self.valid = float(g), False
        self._K = self._KT = None

    def K(self):  # dual.py:71-75
        if self._K is None:
            self.tally.bump(1)
            self._K = -self._gamma * self.C
        return self._K

    def KT(self):  # dual.py:77-89
        if self._KT is None:
            if self._sym is None:
                self._sym = bool((self.C == self.C.T).all())
            if self._sym:
                self._KT = self.K()
            else:
                K = self.K()
                self.tally.bump(1)
                self._KT = np.ascontiguousarray(K.T)
        return self._KT

    def _full_refresh(self):  # dual.py:91-102
        self.tally.bump(4)
        lr = tiled_row_lse(self.K(), self._u, self._v)
        self.tally.bump(4)
        lc = tiled_row_lse(self.KT(), self._v, self._u)
        self._lr, self._lc, self.valid = lr, lc, True

    @property
    def log_r(self):
        if not self.valid:
            self._full_refresh()
        return self._lr

    @property
    def log_c(self):
        if not self.valid:
            self._full_refresh()
        return self._lc

    def rows_now(self):
        return np.exp(self.log_r)

    def cols_now(self):
        return np.exp(self.log_c)

    def gnorm(self):  # dual.py:142-148
        gu = self.rows_now() - self.r
        gv = self.cols_now() - self.c
        return float(np.abs(gu).sum() + np.abs(gv).sum())

    def dual_value(self):  # dual.py:150-153
        mass = float(np.exp(self.log_r).sum())
        return mass - 1.0 - float(self._u @ self.r) - float(self._v @ self.c)

    def plan(self, reuse=False):  # dual.py:155-169
        self.tally.bump(4)
        buf = None
        if reuse:
            if self._plan is None:
                self._plan = np.empty_like(self.C)
            buf = self._plan
        return tiled_plan(self.K(), self._u, self._v, out=buf)

    def trial_log_c(self, du, dv, a):  # dual.py:171-175
        self.tally.bump(4)
        return tiled_row_lse(self.KT(), self._v + a * dv, self._u + a * du)

    def refresh_rows(self):  # dual.py:203-208
        self.tally.bump(4)
        self._lr = tiled_row_lse(self.K(), self._u, self._v)
        self.valid = True

    def balance_cols(self):  # dual.py:179-184
        self.tally.bump(4)
        self.v = np.log(self.c) - tiled_row_lse(self.KT(), 0.0, self._u)
        self._lc = np.log(self.c)
        self.refresh_rows()

    def balance_rows_exit(self):  # dual.py:186-194
        lr_target = np.log(self.r)
        self.u = self._u + lr_target - self.log_r
        self._lr = lr_target
        self.tally.bump(4)
        self._lc = tiled_row_lse(self.KT(), self._v, self._u)
        self.valid = True

    def z(self):
        return np.concatenate([self._u, self._v])

    def set_z(self, z):
        n = self._u.shape[0]
        self.u = np.asarray(z[:n], dtype=np.float64).copy()
        self.v = np.asarray(z[n:], dtype=np.float64).copy()


# ---------------------------------------------------------------------------
# discounted Newton system and its solvers (restate newton.py:69-217)
# ---------------------------------------------------------------------------
class System:
    def __init__(self, P, rP, cP, tally):
        self.P, self.rP, self.cP, self.tally = P, rP, cP, tally
        if np.any(rP <= 0.0) or np.any(cP <= 0.0):
            raise OracleFailure("ConditioningError", "nonpositive plan sums")
        self._mu = None

    @classmethod
    def of(cls, st):  # newton.py:81-90
        return cls(st.plan(reuse=True), st.rows_now(), st.cols_now(), st.tally)

    def pc(self, d):  # newton.py:96-98
        return rmv(self.P, d, self.tally) / self.cP

    def F(self, rho, d):  # newton.py:100-105
        out = self.rP * d
        if rho != 0.0:
            out -= rho * mv(self.P, rmv(self.P, d, self.tally) / self.cP, self.tally)
        return out

    def mu(self):  # newton.py:107-112
        if self._mu is None:
            self.tally.bump(2)
            self._mu = tiled_square_mv(self.P, 1.0 / self.cP) / self.rP
        return self._mu


def cg(sysm, rho, b, tol, x0=None, cap=None):
    """Jacobi-PCG on F(rho) x = b with the L1 recurrence-residual stop.

    Restates newton.py:123-172.  Returns (x, iterations).
    """
    if not 0.0 <= rho < 1.0:
        raise OracleFailure("ConditioningError", f"rho {rho}")
    if tol <= 0.0:
        raise OracleFailure("ConditioningError", "tol must be positive")
    n = b.shape[0]
    cap = 10 * n if cap is None else cap
    M = sysm.rP * (1.0 - rho * sysm.mu())
    if np.any(M <= 0.0):
        raise OracleFailure("ConditioningError", "nonpositive preconditioner")
    if x0 is None:
        x = np.zeros(n)
        r = b.copy()
    else:
        x = np.array(x0, dtype=np.float64, copy=True)
        r = b - sysm.F(rho, x)
    if np.abs(r).sum() <= tol:
        return x, 0
    z = r / M
    p = z.copy()
    rz = float(r @ z)
    for k in range(1, cap + 1):
        q = sysm.F(rho, p)
        pq = float(p @ q)
        if pq <= 0.0:
            raise OracleFailure("ConditioningError", f"curvature {pq:.3g}")
        a = rz / pq
        x += a * p
        r -= a * q
        if k % REFRESH_EVERY == 0:
            r = b - sysm.F(rho, x)
        if np.abs(r).sum() <= tol:
            return x, k
        z = r / M
        rz2 = float(r @ z)
        p = z + (rz2 / rz) * p
        rz = rz2
    raise OracleFailure("NonconvergenceError", "CG budget", best=x,
                        diag={"rho": rho, "residual_l1": float(np.abs(r).sum())})


@dataclass
class Direction:
    d_u: np.ndarray
    rho_final: float
    cg_iters: int
    resid: float


def newton_direction(g, sysm, eta, rho0=0.0, zero_init=False, cap=None):
    """rho-annealed discounted solves until the forcing test holds.

    Restates newton.py:175-210.
    """
    if eta <= 0.0:
        raise OracleFailure("ConditioningError", "eta must be positive")
    if not 0.0 <= rho0 < 1.0:
        raise OracleFailure("ConditioningError", "rho0 out of range")
    gn = float(np.abs(g).sum())
    if gn == 0.0:
        return Direction(np.zeros(g.shape[0]), rho0, 0, 0.0)
    d = -g / sysm.rP
    rho, used, total = rho0, rho0, 0
    tol = CG_SHARE * eta * gn
    while True:
        res = sysm.F(1.0, d) + g
        rn = float(np.abs(res).sum())
        if rn <= eta * gn:
            return Direction(d, used, total, rn)
        if 1.0 - rho < RHO_FLOOR_GAP:
            raise OracleFailure("StagnationError", f"rho {rho}")
        d, it = cg(sysm, rho, -g, tol, x0=None if zero_init else d, cap=cap)
        total += it
        used = rho
        rho = 1.0 - (1.0 - rho) / RHO_DIVISOR


def rho_restart(rho_old):  # newton.py:213-217
    return max(0.0, 1.0 - (1.0 - rho_old) * RHO_DIVISOR)


# ---------------------------------------------------------------------------
# projection (restates projector.py:89-260)
# ---------------------------------------------------------------------------
@dataclass
class Step:
    eta: float
    grad_before: float
    grad_after: float
    alpha: float
    delta: float
    rho_final: float
    cg_iters: int
    backtracks: int
    terminal: bool
    exited_after: bool = False


@dataclass
class Proj:
    newton_steps: int = 0
    cg_iters: int = 0
    sinkhorn_steps: int = 0
    backtracks: int = 0
    delta_min: float = math.inf
    delta_min_all: float = math.inf
    grad_norm_final: float = math.nan
    rho_final: float = 0.0
    steps: list = field(default_factory=list)


def chi_balance(st, r, c, eps_chi, budget=10 ** 6):  # projector.py:129-149
    st.r, st.c = r, c
    lr = np.log(r)
    n_sweeps = 0
    with st.tally.under("chi_sinkhorn"):
        while chi2(r, st.rows_now()) > eps_chi:
            if n_sweeps >= budget:
                raise OracleFailure("NonconvergenceError", "chi budget")
            st.u = st.u + lr - st.log_r
            st.balance_cols()
            n_sweeps += 1
    return n_sweeps


def project(st, r, c, eps_d, rho0=0.0, newton_budget=200, chi_budget=10 ** 6,
            adaptive_rho0=True, zero_init=False, cg_cap=None):
    """Alg. 4: entry column balance, Newton steps with mass-form Armijo, exit
    row scaling.  Restates projector.py:152-260."""
    if not 0.0 < eps_d < 1.0:
        raise OracleFailure("DomainError", "eps_d")
    if np.min(r) <= 0.0 or np.min(c) <= 0.0:
        raise OracleFailure("DomainError", "marginals must be positive")
    tl = st.tally
    st.r, st.c = r, c
    out = Proj()
    lc = np.log(c)
    eps_chi = eps_d ** CHI_POW
    rho_next = rho0 if adaptive_rho0 else 0.0
    with tl.under("mirror_descent"):
        st.balance_cols()
    while True:
        g = st.rows_now() - r
        gn = float(np.abs(g).sum())
        if gn <= eps_d:
            break
        if out.newton_steps >= newton_budget:
            raise OracleFailure("NonconvergenceError", "newton budget",
                                diag={"gamma": st.gamma, "eps_d": eps_d, "grad_norm": gn})
        out.sinkhorn_steps += chi_balance(st, r, c, eps_chi, budget=chi_budget)
        g = st.rows_now() - r
        gn = float(np.abs(g).sum())
        if gn == 0.0:
            break
        quad, term = gn, 0.8 * eps_d / gn
        eta, terminal = min(max(quad, term), ETA_CAP), term > quad
        with tl.under("newton_solve"):
            sysm = System.of(st)
            res = newton_direction(g, sysm, eta, rho0=rho_next, zero_init=zero_init,
                                   cap=cg_cap)
            du = res.d_u
            dv = -sysm.pc(du)
        out.rho_final = res.rho_final
        rho_next = rho_restart(res.rho_final) if adaptive_rho0 else 0.0
        slope = float(-(g @ du))
        if slope <= 0.0:
            with tl.under("chi_sinkhorn"):
                st.u = st.u + np.log(r) - st.log_r
                st.balance_cols()
            out.sinkhorn_steps += 1
            continue
        a = 1.0
        with tl.under("newton_solve"):
            trial = st.trial_log_c(du, dv, a)
        nb = 0
        while True:
            with np.errstate(over="ignore"):
                mass = float(np.exp(trial).sum())
            if not (slope > SLOPE_FLOOR and mass - 1.0 > (1.0 - C1) * a * slope):
                break
            a *= 0.5
            if a < ALPHA_MIN:
                raise OracleFailure("LineSearchError", "alpha floor",
                                    diag={"gamma": st.gamma, "grad_norm": gn,
                                          "slope": slope, "eta": eta})
            with tl.under("line_search"):
                trial = st.trial_log_c(du, dv, a)
            nb += 1
        st.u = st.u + a * du
        st.v = st.v + a * dv + (lc - trial)
        st._lc = lc
        with tl.under("newton_solve"):
            st.refresh_rows()
        g_after = float(np.abs(st.rows_now() - r).sum())
        delta = (gn - g_after) / ((1.0 - eta) * gn)
        out.steps.append(Step(eta, gn, g_after, a, delta, res.rho_final, res.cg_iters,
                              nb, terminal))
        out.newton_steps += 1
        out.cg_iters += res.cg_iters
        out.backtracks += nb
    with tl.under("mirror_descent"):
        st.balance_rows_exit()
    out.grad_norm_final = st.gnorm()
    if out.steps:
        out.steps[-1].exited_after = True
        out.delta_min_all = min(s.delta for s in out.steps)
        kept = [s.delta for s in out.steps if not (s.terminal and s.exited_after)]
        out.delta_min = min(kept) if kept else math.inf
    return out


# ---------------------------------------------------------------------------
# annealing driver (restates driver.py:128-343)
# ---------------------------------------------------------------------------
def eps_rule(gamma, p, r, c):  # driver.py:128-132
    return min(entropy(r), entropy(c)) / gamma ** p


def smooth(r, c, eps, w_r=W_ROW, w_c=W_COL):  # driver.py:135-153
    n = r.shape[0]
    return ((1.0 - w_r * eps) * r + (w_r * eps / n),
            (1.0 - w_c * eps) * c + (w_c * eps / len(c)))


def next_q(q, dmin):  # driver.py:156-167
    if dmin > Q_UP:
        return min(Q_HI, q * q)
    if dmin < Q_DOWN:
        return max(Q_LO, math.sqrt(q))
    return q


def extrapolate(z, zp, g_next, g, g_prev):  # driver.py:170-175
    step = (g_next - g) / (g - g_prev)
    return z + step * (z - zp)


def round_to_polytope(P, r, c, tally):  # driver.py:178-208
    _hit("round")
    if P.min() < 0.0:
        raise OracleFailure("DomainError", "negative plan")
    if not P.sum() > 0.0:
        raise OracleFailure("DegenerateInputError", "zero mass")
    tally.bump(2)
    rP = P.sum(axis=1)
    with np.errstate(divide="ignore", invalid="ignore"):
        rs = np.where(rP > 0.0, np.minimum(1.0, r / rP), 1.0)
    P = P * rs[:, None]
    tally.bump(2)
    cP = P.sum(axis=0)
    with np.errstate(divide="ignore", invalid="ignore"):
        cs = np.where(cP > 0.0, np.minimum(1.0, c / cP), 1.0)
    P = P * cs[None, :]
    tally.bump(1)
    er = r - P.sum(axis=1)
    ec = c - P.sum(axis=0)
    deficit = er.sum()
    if deficit > 0.0:
        tally.bump(1)
        P = P + np.outer(er, ec) / deficit
    return P


@dataclass
class Run:
    P: np.ndarray
    primal: float
    bound: float
    stages: list          # (t, gamma, eps_d, q_next, Proj)
    state: Dual
    ops: dict
    dual_value: float


def mdot(C, r, c, gamma_i, gamma_f, p=1.5, q_init=2.0, adaptive_q=True,
         adaptive_rho0=True, zero_init=False, newton_budget=200, w_r=W_ROW, w_c=W_COL,
         projector="newton", sinkhorn_budget=10 ** 6):
    """MDOT annealing with the truncated-Newton projector (Alg. 1).

    Restates driver.py:226-343; ``projector="sinkhorn"`` is the baseline branch
    (driver.py:218-223,277-279: log-domain Sinkhorn to eps_d/2, rho0 untouched,
    delta_min = +inf so the schedule grows q).
    """
    tally = Tally()
    g, g_prev, q = min(gamma_i, gamma_f), 0.0, float(q_init)
    t = 1
    st = None
    z_prev = None
    rho_next = 0.0
    stages = []
    while True:
        done = g == gamma_f
        eps = eps_rule(g, p, r, c)
        if eps >= 1.0:
            raise OracleFailure("DomainError", "eps_d >= 1")
        rs, cs = smooth(r, c, eps, w_r, w_c)
        if t == 1:
            st = Dual(C, g, np.log(rs), np.log(cs), rs, cs, tally)
            z_prev = st.z()
        else:
            st.gamma = g
            st.r, st.c = rs, cs
        if projector == "newton":
            pr = project(st, rs, cs, eps / 2.0, rho0=rho_next, newton_budget=newton_budget,
                         adaptive_rho0=adaptive_rho0, zero_init=zero_init)
            rho_next = rho_restart(pr.rho_final) if adaptive_rho0 else 0.0
        else:
            pr = Proj()
            pr.sinkhorn_steps = sinkhorn_sweeps(st, rs, cs, eps / 2.0, budget=sinkhorn_budget)
            pr.grad_norm_final = st.gnorm()
        if adaptive_q:
            q = next_q(q, pr.delta_min)
        g_next = min(q * g, gamma_f)
        z = st.z()
        z_new = extrapolate(z, z_prev, g_next, g, g_prev)
        stages.append((t, g, eps, q, pr))
        if done:
            break
        z_prev = z
        g_prev = g
        g = g_next
        st.set_z(z_new)
        t += 1
    with tally.under("mirror_descent"):
        P = st.plan()
        P = round_to_polytope(P, r, c, tally)
        tally.bump(1)
        primal = float(np.vdot(P, C))
    ops = dict(tally.counts)
    ops["total"] = tally.total()
    bound = 2.0 * min(entropy(r), entropy(c)) / gamma_f
    return Run(P, primal, bound, stages, st, ops, st.dual_value())


def sinkhorn_sweeps(st, r, c, eps_d, budget=10 ** 6):
    """Log-domain Sinkhorn until the full gradient norm is <= eps_d.

    Restates oracles.py:243-265 (the §8(f) rank-2 baseline projector).
    """
    st.r, st.c = r, c
    n = 0
    with st.tally.under("sinkhorn"):
        while st.gnorm() > eps_d:
            if n >= budget:
                raise OracleFailure("NonconvergenceError", "sinkhorn budget")
            st.balance_rows_exit()
            lc = np.log(st.c)
            st.v = st.v + lc - st.log_c
            st._lc = lc
            st.refresh_rows()
            n += 1
    return n
