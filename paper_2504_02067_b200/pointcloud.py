"""On-the-fly point-cloud solver: D4 (n = 65536) / D5 (n = 2^20), SURVEY §8(d)-(e).

No n x n array exists anywhere: every O(n^2) pass recomputes
``C_ij = (sum_k (x_ik - y_jk)^2) / C_max`` and the plan entry from the point
coordinates in the C-ABI pair kernel (``otn_pc_pass``), bit-identical to the
host-materialized cost of ``PointCloudProblem.materialize_cost`` and with the
stored path's exponent rounding ((K + v) + u, ``_kernels.py:52-53``).

Each pass is milliseconds to seconds of FP64 work, so the CG / Newton loops run
on the host (``newton.py:123-210`` restated over device vectors) — a host
round trip is noise next to a pass — which also lets the solve be **row
sharded** across GPUs: rank g owns rows [g n/G, (g+1) n/G) of X (all of Y is
replicated, 24n bytes).  Row-direction work (row LSE, P w, the Jacobi
diagonal, CG vector algebra) is local; every column-direction product (column
LSE, P^T x) yields per-rank partials combined by ONE allreduce per product:
P^T x partials are summed; the column LSE is formed against a known shift
(the previous column LSE, SURVEY §7 hard part 4) so its partial sums need one
SUM allreduce too, with the MAX-then-SUM combine as the fallback when a sum
leaves [2^-700, 2^700].  CG dots / norms are reduced into a device buffer and
allreduced there, one host read per CG scalar step (``Comm``).  On one GPU
``Comm`` is the identity.

The state class mirrors the private hooks ``project()`` and ``mdot()`` use on
``DualState``, so the projector and driver are shared with the stored path.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib, opcount
from ._device import TELEMETRY, Context, torch, vptr
from .errors import (
    ConditioningError,
    DegenerateInputError,
    DomainError,
    PlanOverflowError,
)

RHO_CAP = 1e-12
RHO_DECAY = 4.0
CG_TOL_FRACTION = 0.25
TRUE_RESIDUAL_REFRESH = 50


class Comm:
    """Collectives of a row-sharded solve (torch.distributed: NCCL between
    GPUs; gloo in the CPU tests and the GPU process-group test, where CUDA
    tensors are staged through the host).

    ``world == 1`` (no process group) makes every method the identity.
    ``stats`` counts the collectives (vector / scalar allreduces, bytes)."""

    def __init__(self, group=None):
        self.group = group
        try:
            import torch.distributed as dist
            self.dist = dist if dist.is_available() and dist.is_initialized() else None
        except Exception:
            self.dist = None
        self.world = self.dist.get_world_size(group) if self.dist else 1
        self.rank = self.dist.get_rank(group) if self.dist else 0
        self.backend = str(self.dist.get_backend(group)) if self.dist else None
        self.stats = {"vector_allreduces": 0, "scalar_allreduces": 0, "bytes": 0}

    @classmethod
    def local(cls):
        """A one-rank communicator even inside a process group (the 1-GPU
        reference solve of a multi-rank job)."""
        c = cls.__new__(cls)
        c.group, c.dist, c.world, c.rank, c.backend = None, None, 1, 0, None
        c.stats = {"vector_allreduces": 0, "scalar_allreduces": 0, "bytes": 0}
        return c

    def shard(self, n):
        lo = (self.rank * n) // self.world
        hi = ((self.rank + 1) * n) // self.world
        return lo, hi

    def barrier(self):
        if self.world > 1:
            self.dist.barrier(group=self.group)

    def _allreduce(self, t, op, kind):
        if self.world == 1:
            return t
        self.stats[kind] += 1
        self.stats["bytes"] += t.numel() * t.element_size()
        if self.backend == "gloo" and t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h, op=op, group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, op=op, group=self.group)
        return t

    def sum_(self, t, kind="vector_allreduces"):
        return self._allreduce(t, self.dist.ReduceOp.SUM if self.dist else None, kind)

    def max_(self, t):
        return self._allreduce(t, self.dist.ReduceOp.MAX if self.dist else None,
                               "vector_allreduces")

    def sum_scalars(self, vals, device):
        if self.world == 1:
            return [float(v) for v in vals]
        t = torch().tensor(list(vals), dtype=torch().float64, device=device)
        self.sum_(t, "scalar_allreduces")
        return [float(v) for v in t.tolist()]

    def max_scalars(self, vals, device):
        if self.world == 1:
            return [float(v) for v in vals]
        t = torch().tensor(list(vals), dtype=torch().float64, device=device)
        self._allreduce(t, self.dist.ReduceOp.MAX, "scalar_allreduces")
        return [float(v) for v in t.tolist()]


class CudaBackend:
    """The C-ABI pair / vector / reduction kernels on one CUDA device."""

    def __init__(self, device):
        self.device = device
        self.ctx = Context.get(32, device)        # stream + scalar plumbing only

    def pass_(self, op, A, na, B, nb, d, cmax, ng, order, colpot, colpot_d, alpha, rowpot, vec,
              outer, outer_d, mode, out, out2):
        self.ctx.call("otn_pc_pass", int(op), vptr(A), int(na), int(na), vptr(B), int(nb),
                      int(nb), int(d), float(cmax), float(ng), int(order), vptr(colpot),
                      vptr(colpot_d), float(alpha), vptr(rowpot), vptr(vec), vptr(outer),
                      vptr(outer_d), int(mode), vptr(out), vptr(out2))

    def vec(self, n, op, out, a, b=None, c=None, d=None, s=0.0):
        self.ctx.call("otn_vec_n", int(n), int(op), float(s), vptr(a), vptr(b), vptr(c), vptr(d),
                      vptr(out))

    def reduce(self, n, op, a, b=None, c=None, d=None):
        out = (ctypes.c_double * 2)()
        fl = ctypes.c_int(0)
        self.ctx.call("otn_reduce_n", int(n), int(op), vptr(a), vptr(b), vptr(c), vptr(d), out,
                      ctypes.byref(fl))
        TELEMETRY.d2h += 20                     # two sums and the flag word
        return float(out[0]), float(out[1]), int(fl.value)

    def reduce_dev(self, n, op, dst, a, b=None, c=None, d=None):
        """The two sums into device memory dst[0:2] (stream-ordered, no sync)."""
        self.ctx.call("otn_reduce_dev", int(n), int(op), vptr(a), vptr(b), vptr(c), vptr(d),
                      vptr(dst))

    def tensor(self, arr):
        TELEMETRY.h2d += arr.nbytes
        return torch().from_numpy(arr.copy()).to(self.device)


class PointCloudCost:
    """Device-resident point sets of a (possibly row-sharded) point-cloud problem.

    ``backend`` executes the O(n^2) passes and vector kernels (the CUDA C-ABI;
    tests inject a CPU double to exercise the sharding logic under gloo)."""

    def __init__(self, problem, device, comm=None, backend=None):
        self.problem = problem
        self.comm = comm or Comm()
        self.device = device
        self.be = backend or CudaBackend(device)
        self.n = problem.n
        self.d = problem.dim
        if not 1 <= self.d <= 4:
            raise DomainError("on-the-fly cost supports point dimension 1..4")
        self.row0, self.row1 = self.comm.shard(self.n)
        self.rows = self.row1 - self.row0
        X = np.ascontiguousarray(problem.X[self.row0:self.row1].T)   # SoA: d x rows
        Y = np.ascontiguousarray(problem.Y.T)                        # SoA: d x n
        self.Xt = self.be.tensor(X)
        self.Yt = self.be.tensor(Y)
        self.symmetric = bool(np.array_equal(problem.X, problem.Y))
        self._scal_buf = None
        self._colL = None          # last column LSE (sharded runs: the next call's shift)
        if problem.cmax is not None:
            self.cmax = float(problem.cmax)
        else:
            self.cmax = self._exact_cmax()
        if not self.cmax > 0.0:
            raise DegenerateInputError("point sets have zero diameter")

    def _exact_cmax(self):
        """max_ij D_ij by one O(n^2) pass (no exp) + a MAX allreduce."""
        t = torch()
        per_row = t.empty(self.rows, dtype=t.float64, device=self.device)
        self.pass_(_lib.PC_MAXD, rows_first=True, cmax=0.0, out=per_row)
        local = self.reduce(self.rows, _lib.RED_MAX, per_row)[0]
        return self.comm.max_scalars([local], self.device)[0]

    # ---- thin wrappers over the backend ----------------------------------------
    def pass_(self, op, rows_first, out, ng=0.0, order=0, colpot=None, colpot_d=None, alpha=0.0,
              rowpot=None, vec=None, outer=None, outer_d=None, mode=0, out2=None, cmax=None):
        """rows_first: A = own X rows, B = all Y (row pass); else A = Y, B = own X."""
        if rows_first:
            A, na, B, nb = self.Xt, self.rows, self.Yt, self.n
        else:
            A, na, B, nb = self.Yt, self.n, self.Xt, self.rows
        self.be.pass_(op, A, na, B, nb, self.d, self.cmax if cmax is None else cmax, ng, order,
                      colpot, colpot_d, alpha, rowpot, vec, outer, outer_d, mode, out, out2)

    def vec(self, n, op, out, a, b=None, c=None, d=None, s=0.0):
        self.be.vec(n, op, out, a, b, c, d, s)

    def reduce(self, n, op, a, b=None, c=None, d=None):
        return self.be.reduce(n, op, a, b, c, d)

    def rsum(self, *items):
        """Sum-reductions over ALL rows: each item (n, op, a, b, ...) is reduced
        over this shard; on several ranks the shard sums go into one device
        buffer, ONE allreduce combines them and one host read returns them.
        Returns a list of (s0, s1) pairs."""
        if self.comm.world == 1:
            return [self.be.reduce(*it)[:2] for it in items]
        t = torch()
        buf = self._scal_buf
        if buf is None or buf.numel() < 2 * len(items):
            buf = self._scal_buf = t.zeros(max(8, 2 * len(items)), dtype=t.float64,
                                           device=self.device)
        for k, it in enumerate(items):
            n, op, *vecs = it
            vecs = list(vecs) + [None] * (4 - len(vecs))
            self.be.reduce_dev(n, op, buf[2 * k: 2 * k + 2], *vecs)
        view = buf[: 2 * len(items)]
        self.comm.sum_(view, "scalar_allreduces")
        vals = view.tolist()
        TELEMETRY.d2h += 16 * len(items)
        return [(vals[2 * k], vals[2 * k + 1]) for k in range(len(items))]

    def zeros(self, n):
        t = torch()
        return t.zeros(n, dtype=t.float64, device=self.device)

    def upload(self, values):
        return self.be.tensor(np.ascontiguousarray(values, dtype=np.float64))

    # ---- column-direction log-sum-exp (all rows, across shards) ----------------
    def lse_cols(self, ng, inner, inner_d, alpha, outer, outer_d, mode, out):
        """out_j = outer_j (+ alpha outer_d_j) +/- LSE_i(ng C_ij + inner_i (+ alpha inner_d_i))."""
        if self.comm.world == 1:
            self.pass_(_lib.PC_LSE, rows_first=False, out=out, ng=ng, colpot=inner,
                       colpot_d=inner_d, alpha=alpha, outer=outer, outer_d=outer_d, mode=mode)
            return
        n = self.n
        zero = self.zeros(n)
        L = self.zeros(n)
        done = False
        self.comm.stats["column_products"] = self.comm.stats.get("column_products", 0) + 1
        if self._colL is not None:
            # ONE allreduce: shard sums of exp(e_ij - L_prev_j), L = L_prev + log(sum)
            s = self.zeros(n)
            self.pass_(_lib.PC_LSE_SHIFT, rows_first=False, out=s, ng=ng, colpot=inner,
                       colpot_d=inner_d, alpha=alpha, outer=self._colL)
            self.comm.sum_(s)
            # every rank holds the same s: the same verdict everywhere
            if self.reduce(n, _lib.RED_OUTSIDE, s)[0] == 0.0:
                self.vec(n, _lib.VEC_LSE_FIN, L, zero, self._colL, s)
                done = True
            self.comm.stats["lse_shift_fallbacks"] = (
                self.comm.stats.get("lse_shift_fallbacks", 0) + (0 if done else 1))
        if not done:
            # exact combine: MAX of the shard maxima, then SUM of the rescaled sums
            m = self.zeros(n)
            s = self.zeros(n)
            self.pass_(_lib.PC_LSE_PART, rows_first=False, out=m, out2=s, ng=ng, colpot=inner,
                       colpot_d=inner_d, alpha=alpha)
            M = m.clone()
            self.comm.max_(M)
            self.vec(n, _lib.VEC_RESCALE, s, s, m, M)         # s * exp(m - M)
            self.comm.sum_(s)
            self.vec(n, _lib.VEC_LSE_FIN, L, zero, M, s)
        self._colL = L
        base = outer
        if outer_d is not None:
            base = self.zeros(n)
            self.vec(n, _lib.VEC_AXPY, base, outer, outer_d, s=alpha)
        if base is None:
            base = zero
        self.vec(n, _lib.VEC_ADD if mode == 0 else _lib.VEC_SUB, out, base, L)


class PointCloudState:
    """Dual state of a point-cloud problem; row vectors are this rank's shard.

    Implements the hooks ``project()`` / ``mdot()`` call on ``DualState``."""

    def __init__(self, cost, gamma, u, v, r, c):
        if not np.isfinite(gamma) or gamma <= 0.0:
            raise DomainError(f"gamma must be positive and finite, got {gamma}")
        self._pc = cost
        self.problem = cost.problem
        lo, hi = cost.row0, cost.row1
        self._gamma = float(gamma)
        self._u = cost.upload(np.asarray(u, dtype=np.float64)[lo:hi])
        self._v = cost.upload(np.asarray(v, dtype=np.float64))
        nr, n = cost.rows, cost.n
        self._lr = cost.zeros(nr)
        self._lc = cost.zeros(n)
        self._g = cost.zeros(nr)
        self._trial_vec = cost.zeros(n)
        self._cache_valid = False
        self._rowstat = None
        self._K_formed = False
        self._KT_formed = False
        self.set_targets(r, c)

    # -- attributes ---------------------------------------------------------------
    @property
    def n(self):
        return self._pc.n

    @property
    def gamma(self):
        return self._gamma

    @gamma.setter
    def gamma(self, value):
        self._gamma = float(value)
        self._invalidate()
        self._K_formed = self._KT_formed = False

    @property
    def _ng(self):
        return -self._gamma

    def _invalidate(self):
        self._cache_valid = False
        self._rowstat = None

    @property
    def u(self):
        """This rank's rows of u (the whole vector on one GPU)."""
        return self._u.cpu().numpy().copy()

    @property
    def v(self):
        return self._v.cpu().numpy().copy()

    def set_targets(self, r, c, _logs=None):
        self.r = np.asarray(r, dtype=np.float64)
        self.c = np.asarray(c, dtype=np.float64)
        lo, hi = self._pc.row0, self._pc.row1
        with np.errstate(divide="ignore", invalid="ignore"):
            self._r = self._pc.upload(self.r[lo:hi])
            self._log_r = self._pc.upload(np.log(self.r[lo:hi]))
            self._c = self._pc.upload(self.c)
            self._log_c = self._pc.upload(np.log(self.c))
        self._rowstat = None

    def _touch_K(self):
        if not self._K_formed:
            opcount.add(1)
            self._K_formed = True

    def _touch_KT(self):
        if not self._KT_formed:
            self._touch_K()
            if not self._pc.symmetric:
                opcount.add(1)
            self._KT_formed = True

    # -- log-domain reductions ------------------------------------------------------
    def _lse_rows_into(self, out):
        self._touch_K()
        self._pc.pass_(_lib.PC_LSE, rows_first=True, out=out, ng=self._ng, colpot=self._v,
                       outer=self._u)

    def refresh(self):
        opcount.add(4)
        self._lse_rows_into(self._lr)
        opcount.add(4)
        self._touch_KT()
        self._pc.lse_cols(self._ng, self._u, None, 0.0, self._v, None, 0, self._lc)
        self._cache_valid = True
        self._rowstat = None

    def _lr_dev(self):
        if not self._cache_valid:
            self.refresh()
        return self._lr

    def _lc_dev(self):
        if not self._cache_valid:
            self.refresh()
        return self._lc

    def refresh_rows_only(self):
        opcount.add(4)
        self._lse_rows_into(self._lr)
        self._rowstat = None
        self._cache_valid = True

    def rebalance_columns(self):
        """v = log c - LSE_cols(u); log c(P) := log c; refresh rows (dual.py:179-184)."""
        opcount.add(4)
        self._touch_KT()
        self._pc.lse_cols(self._ng, self._u, None, 0.0, self._log_c, None, 1, self._v)
        self._invalidate()
        self._lc.copy_(self._log_c)
        self.refresh_rows_only()

    def scale_rows_to_target(self):
        """u += log r - log r(P); column cache from the new u (dual.py:186-194)."""
        lr = self._lr_dev()
        self._pc.vec(self._pc.rows, _lib.VEC_ADD_SUB, self._u, self._u, self._log_r, lr)
        self._invalidate()
        self._lr.copy_(self._log_r)
        opcount.add(4)
        self._touch_KT()
        self._pc.lse_cols(self._ng, self._u, None, 0.0, self._v, None, 0, self._lc)
        self._cache_valid = True

    def scale_cols_to_target(self):
        lc = self._lc_dev()
        self._pc.vec(self.n, _lib.VEC_ADD_SUB, self._v, self._v, self._log_c, lc)
        self._invalidate()
        self._lc.copy_(self._log_c)
        self.refresh_rows_only()

    # -- reductions -------------------------------------------------------------------
    def _row_stats(self):
        if self._rowstat is None:
            pc = self._pc
            lr = self._lr_dev()
            pc.vec(pc.rows, _lib.VEC_GRAD, self._g, lr, self._r)
            s0, s1, fl = pc.reduce(pc.rows, _lib.RED_ROW_STATS, lr, self._r)
            if pc.comm.world > 1:                         # one allreduce: sums + flag counts
                s0, s1, f1, f2 = pc.comm.sum_scalars([s0, s1, fl & 1, (fl >> 1) & 1],
                                                     pc.device)
                fl = (1 if f1 > 0 else 0) | (2 if f2 > 0 else 0)
            self._rowstat = (s0, s1, fl)
        return self._rowstat

    def _row_grad_norm(self):
        return self._row_stats()[0]

    def _chi_sq(self):
        _, s, fl = self._row_stats()
        if fl & 1:
            raise DomainError("chi_sq_div requires strictly positive reference x")
        if fl & 2:
            raise DomainError("chi_sq_div requires nonnegative y")
        return float(s - 1.0)

    def grad_norm_l1(self):
        pc = self._pc
        gu = pc.rsum((pc.rows, _lib.RED_GRAD_L1, self._lr_dev(), self._r, self._lc_dev(),
                      self._c))[0][0]
        gv = pc.reduce(self.n, _lib.RED_GRAD_L1, self._lc_dev(), self._c, self._lc_dev(),
                       self._c)[0]
        return float(gu + gv)

    def dual_value(self):
        pc = self._pc
        (mass, _), (ur, _) = pc.rsum((pc.rows, _lib.RED_SUM_EXP, self._lr_dev()),
                                     (pc.rows, _lib.RED_DOT, self._u, self._r))
        vc = pc.reduce(self.n, _lib.RED_DOT, self._v, self._c)[0]
        return mass - 1.0 - ur - vc

    # -- projector hooks ----------------------------------------------------------------
    def _trial_buf(self):
        return self._trial_vec

    def _trial(self, d_u, d_v, alpha, out):
        """Trial column sums at (u + alpha d_u, v + alpha d_v) and the plan mass."""
        opcount.add(4)
        self._touch_KT()
        self._pc.lse_cols(self._ng, self._u, d_u, float(alpha), self._v, d_v, 0, out)
        return self._pc.reduce(self.n, _lib.RED_SUM_EXP, out)[0]

    def _row_scaling_update(self):
        pc = self._pc
        pc.vec(pc.rows, _lib.VEC_ADD_SUB, self._u, self._u, self._log_r, self._lr_dev())
        self._invalidate()

    def _accept(self, alpha, d_u, d_v):
        pc = self._pc
        pc.vec(pc.rows, _lib.VEC_AXPY, self._u, self._u, d_u, s=float(alpha))
        pc.vec(self.n, _lib.VEC_STEP_V, self._v, self._v, d_v, self._log_c, self._trial_vec,
               s=float(alpha))
        self._invalidate()
        self._lc.copy_(self._log_c)

    def _system(self):
        return PointCloudSystem(self)

    def _dir_bufs(self):
        bufs = getattr(self, "_dirbufs", None)
        if bufs is None:
            bufs = (self._pc.zeros(self._pc.rows), self._pc.zeros(self.n))
            self._dirbufs = bufs
        return bufs

    def _download_rows(self, buf):
        return buf.cpu().numpy().copy()

    # -- driver hooks --------------------------------------------------------------------
    def _snapshot(self):
        return self._u.clone(), self._v.clone()

    def _extrapolate(self, step, z_cur, z_prev):
        pc = self._pc
        pc.vec(pc.rows, _lib.VEC_EXTRAP, self._u, z_cur[0], z_prev[0], s=float(step))
        pc.vec(self.n, _lib.VEC_EXTRAP, self._v, z_cur[1], z_prev[1], s=float(step))
        self._invalidate()

    def _finalize(self, problem):
        """Streaming rounding onto U(r, c) and the primal cost.

        Restates driver.py:178-208 + 306-310 without materializing P: the
        row / column scales, the residual marginals and <P_rounded, C> come from
        O(n^2) passes that recompute the plan.  The rounded plan itself is
        returned in factored form (``Solution.P`` is None):
            P_ij = rs_i P_ij cs_j + err_r_i err_c_j / deficit.
        """
        pc, t = self._pc, torch()
        nr, n = pc.rows, self.n
        lo, hi = pc.row0, pc.row1
        self._touch_K()
        opcount.add(4)                                  # materialize (dual.py:163)
        ones = pc.upload(np.ones(n))
        rsum = pc.zeros(nr)
        pc.pass_(_lib.PC_DOT, rows_first=True, out=rsum, ng=self._ng, colpot=self._v,
                 rowpot=self._u, vec=ones)
        total = pc.comm.sum_scalars([pc.reduce(nr, _lib.RED_DOT, rsum, ones)[0]], pc.device)[0]
        if not total > 0.0:
            raise DegenerateInputError("round_plan needs positive total mass")
        r_loc = pc.upload(problem.r[lo:hi])
        c_all = pc.upload(problem.c)
        rs = pc.zeros(nr)
        pc.vec(nr, _lib.VEC_ROUND_SCALE, rs, r_loc, rsum)             # driver.py:193
        opcount.add(2)
        csum = pc.zeros(n)
        pc.pass_(_lib.PC_DOT, rows_first=False, out=csum, ng=self._ng, order=1,
                 rowpot=self._v, colpot=self._u, vec=rs)
        pc.comm.sum_(csum)
        cs = pc.zeros(n)
        pc.vec(n, _lib.VEC_ROUND_SCALE, cs, c_all, csum)              # driver.py:198
        opcount.add(2)
        rsum2 = pc.zeros(nr)
        pc.pass_(_lib.PC_DOT, rows_first=True, out=rsum2, ng=self._ng, colpot=self._v,
                 rowpot=self._u, vec=cs)
        err_r = pc.zeros(nr)
        pc.vec(nr, _lib.VEC_SUB_MUL, err_r, r_loc, rs, rsum2)          # driver.py:201
        err_c = pc.zeros(n)
        pc.vec(n, _lib.VEC_SUB_MUL, err_c, c_all, cs, csum)            # driver.py:202
        opcount.add(1)
        deficit = pc.comm.sum_scalars([pc.reduce(nr, _lib.RED_DOT, err_r,
                                                 pc.upload(np.ones(nr)))[0]], pc.device)[0]
        # <P, C> = sum_i rs_i sum_j P_ij C_ij cs_j (+ rank-one term)
        tcost = pc.zeros(nr)
        pc.pass_(_lib.PC_DOTC, rows_first=True, out=tcost, ng=self._ng, colpot=self._v,
                 rowpot=self._u, vec=cs)
        primal = pc.reduce(nr, _lib.RED_DOT, rs, tcost)[0]
        if deficit > 0.0:
            opcount.add(1)                              # rank-one repair (driver.py:206)
            t2 = pc.zeros(nr)
            pc.pass_(_lib.PC_CDOT, rows_first=True, out=t2, vec=err_c)
            primal = primal + pc.reduce(nr, _lib.RED_DOT, err_r, t2)[0] / deficit
        primal = pc.comm.sum_scalars([primal], pc.device)[0]
        opcount.add(1)                                  # <P, C> (driver.py:309)
        self.rounding = dict(row_scale=rs, col_scale=cs, err_r=err_r, err_c=err_c,
                             deficit=deficit)
        return None, float(primal)


class _Result:
    """Outcome record with the fields of otn_solve_result (newton.py:59-66 + slope)."""

    def __init__(self):
        self.status = _lib.OTN_OK
        self.pcg_calls = 0
        self.cg_iters = 0
        self.hvps = 0
        self.rho_final = 0.0
        self.resid_l1 = 0.0
        self.slope = 0.0
        self.diag_rho = 0.0
        self.diag_resid = 0.0


class PointCloudSystem:
    """F(rho) = D(rP)(I - rho P_rc) with the plan recomputed on the fly."""

    def __init__(self, state):
        pc = self._pc = state._pc
        self.state = state
        nr, n = pc.rows, pc.n
        self.n = n
        state._touch_K()
        opcount.add(4)                                  # DiscountedSystem.from_state materializes
        self._u, self._v, self._ng = state._u, state._v, state._ng
        self._rP = pc.zeros(nr)
        self._cP = pc.zeros(n)
        self._icP = pc.zeros(n)
        pc.vec(nr, _lib.VEC_EXP, self._rP, state._lr_dev())
        pc.vec(n, _lib.VEC_EXP, self._cP, state._lc_dev())
        pc.vec(n, _lib.VEC_DIV, self._icP, pc.upload(np.ones(n)), self._cP)
        # Jacobi diagonal + the materialize overflow check in one pass
        sq = pc.zeros(nr)
        emax = pc.zeros(nr)
        pc.pass_(_lib.PC_DIAG, rows_first=True, out=sq, out2=emax, ng=self._ng, colpot=self._v,
                 rowpot=self._u, vec=self._icP)
        top = pc.comm.max_scalars([pc.reduce(nr, _lib.RED_MAX, emax)[0]], pc.device)[0]
        if top > 700.0:
            raise PlanOverflowError(f"log-plan entry {top:.3g} would overflow exp(); "
                                    "warm start is broken")
        bad = pc.reduce(nr, _lib.RED_NONPOS, self._rP)[0] + pc.reduce(n, _lib.RED_NONPOS,
                                                                         self._cP)[0]
        if pc.comm.sum_scalars([bad], pc.device)[0] > 0:
            raise ConditioningError("plan row/column sums must be strictly positive")
        self._mu = pc.zeros(nr)
        pc.vec(nr, _lib.VEC_DIV, self._mu, sq, self._rP)
        self._mu_counted = False
        self._w = pc.zeros(n)
        self._s = pc.zeros(nr)

    def _dot(self, a, b):
        pc = self._pc
        return pc.rsum((pc.rows, _lib.RED_DOT, a, b))[0][0]

    def _rmatvec(self, x, out):
        """out = P^T x, summed over all shards (newton.py:51-56)."""
        pc = self._pc
        pc.pass_(_lib.PC_DOT, rows_first=False, out=out, ng=self._ng, order=1, rowpot=self._v,
                 colpot=self._u, vec=x)
        if pc.comm.world > 1:
            pc.comm.stats["column_products"] = pc.comm.stats.get("column_products", 0) + 1
        pc.comm.sum_(out)

    def _hvp(self, rho, x, out, res):
        """out = rP*x - rho*P((P^T x)/cP)  (newton.py:100-105)."""
        pc = self._pc
        if rho != 0.0:
            res.hvps += 1
            opcount.add(2)
            self._rmatvec(x, self._w)
            pc.vec(self.n, _lib.VEC_DIV, self._w, self._w, self._cP)
            pc.pass_(_lib.PC_DOT, rows_first=True, out=self._s, ng=self._ng, colpot=self._v,
                     rowpot=self._u, vec=self._w)
            pc.vec(pc.rows, _lib.VEC_MUL_SUB, out, self._rP, x, self._s, s=float(rho))
        else:
            pc.vec(pc.rows, _lib.VEC_MUL, out, self._rP, x)

    def _pcg(self, rho, b, tol, x, has_x0, max_iters, res):
        """Jacobi-PCG (newton.py:123-172) over device vectors; returns (status, iters, resid)."""
        pc = self._pc
        nr = pc.rows
        if not self._mu_counted:
            opcount.add(2)
            self._mu_counted = True
        M = pc.zeros(nr)
        pc.vec(nr, _lib.VEC_PRECOND, M, self._rP, self._mu, s=float(rho))
        if pc.rsum((nr, _lib.RED_NONPOS, M))[0][0] > 0:
            return _lib.OTN_ST_PRECOND, 0, 0.0
        r = pc.zeros(nr)
        q = pc.zeros(nr)
        if has_x0:
            self._hvp(rho, x, q, res)
            pc.vec(nr, _lib.VEC_SUB, r, b, q)
        else:
            x.zero_()
            r.copy_(b)
        z = pc.zeros(nr)
        pc.vec(nr, _lib.VEC_DIV, z, r, M)
        norm, rz = pc.rsum((nr, _lib.RED_L1_DOT, r, z))[0]
        if norm <= tol:
            return _lib.OTN_OK, 0, norm
        p = z.clone()
        for k in range(1, max_iters + 1):
            self._hvp(rho, p, q, res)
            pq = self._dot(p, q)
            if pq <= 0.0:
                return _lib.OTN_ST_BREAKDOWN, k, pq
            alpha = rz / pq
            pc.vec(nr, _lib.VEC_AXPY, x, x, p, s=alpha)
            pc.vec(nr, _lib.VEC_AXPY, r, r, q, s=-alpha)
            if k % TRUE_RESIDUAL_REFRESH == 0:
                self._hvp(rho, x, q, res)
                pc.vec(nr, _lib.VEC_SUB, r, b, q)
            pc.vec(nr, _lib.VEC_DIV, z, r, M)
            norm, rz_new = pc.rsum((nr, _lib.RED_L1_DOT, r, z))[0]
            if norm <= tol:
                return _lib.OTN_OK, k, norm
            pc.vec(nr, _lib.VEC_AXPY, p, z, p, s=rz_new / rz)
            rz = rz_new
        return _lib.OTN_ST_NONCONVERGENCE, max_iters, norm

    def _newton_dir(self, grad_u, eta, rho0, zero_init, max_cg_iters, d_u, d_v):
        """newton_solve (newton.py:175-210) + d_v and slope (projector.py:201-205)."""
        pc = self._pc
        nr = pc.rows
        res = _Result()
        if max_cg_iters is None:
            max_cg_iters = 10 * self.n
        gn = pc.rsum((nr, _lib.RED_L1, grad_u))[0][0]
        res.rho_final = rho0
        if gn == 0.0:
            d_u.zero_()
        else:
            pc.vec(nr, _lib.VEC_NEG_DIV, d_u, grad_u, self._rP)
            b = pc.zeros(nr)
            pc.vec(nr, _lib.VEC_SUB, b, b, grad_u)      # b = 0 - g = -g (exact)
            rho, used, total = rho0, rho0, 0
            tol = CG_TOL_FRACTION * eta * gn
            target = eta * gn
            q = pc.zeros(nr)
            while True:
                self._hvp(1.0, d_u, q, res)
                rn = pc.rsum((nr, _lib.RED_L1_ADD, q, grad_u))[0][0]
                if rn <= target:
                    res.resid_l1 = rn
                    break
                if 1.0 - rho < RHO_CAP:
                    res.status = _lib.OTN_ST_STAGNATION
                    res.resid_l1 = rn
                    res.diag_rho = rho
                    break
                res.pcg_calls += 1
                st, it, resid = self._pcg(rho, b, tol, d_u, not zero_init, max_cg_iters, res)
                total += it
                if st != _lib.OTN_OK:
                    res.status = st
                    res.diag_rho = rho
                    res.diag_resid = resid
                    break
                used = rho
                rho = 1.0 - (1.0 - rho) / RHO_DECAY
            res.cg_iters = total
            res.rho_final = used
        opcount.add(1)                                  # d_v = -apply_pc(d_u)
        if res.status == _lib.OTN_OK:
            self._rmatvec(d_u, self._w)
            pc.vec(self.n, _lib.VEC_NEG_DIV, d_v, self._w, self._cP)
            res.slope = -self._dot(grad_u, d_u)
        return res
