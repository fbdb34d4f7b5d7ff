"""The reference-side binding of INTEGRATION.md §2, executable.

A maintainer of ``otnewton`` who keeps the reference's Python driver and only
moves its O(n^2) operators to a B200 adds this file as ``otnewton/_b200.py``
and rebinds the operator seam:

    from otnewton import _b200
    seam = _b200.Seam("/path/to/libotn_b200.so")
    otnewton._kernels.log_plan_row_sums = seam.log_plan_row_sums    # _kernels.py:22-42
    otnewton._kernels.materialize_plan = seam.materialize_plan      # _kernels.py:45-61
    otnewton._kernels.square_matvec = seam.square_matvec            # _kernels.py:64-74
    otnewton.newton._matvec = seam.matvec                           # newton.py:43-48
    otnewton.newton._rmatvec = seam.rmatvec                         # newton.py:51-56

Each function keeps the seam's contract -- host numpy arrays in, a fresh host
array out (``out=`` honoured by ``materialize_plan``), PlanOverflowError when a
log-plan entry exceeds 700 -- and runs one C-ABI call of ``libotn_b200.so``
on device copies of its operands.  The binding is self-contained (its own
ctypes declarations, taken from include/otn_b200.h); tests/test_gpu_seam_binding.py
runs a complete solve through it (on the oracle's restatement of the same
seam, since /root/reference does not travel to the GPU box).

Operands are copied host -> device on every call (the seam has no notion of
device residency); that is the price of keeping the reference's driver.  The
package's own ``mdot`` keeps everything resident instead.
"""

from __future__ import annotations

import ctypes

import numpy as np

_P = ctypes.c_void_p
_D = ctypes.c_double
_I = ctypes.c_int
_I64 = ctypes.c_int64

_SIGS = {
    "otn_abi_version": ([], _I),
    "otn_last_error": ([], ctypes.c_char_p),
    "otn_create": ([ctypes.POINTER(_P), _I, _I64, _I64, _P], _I),
    "otn_destroy": ([_P], _I),
    "otn_lse_rows": ([_P, _P, _D, _P, _P, _P], _I),
    "otn_materialize": ([_P, _P, _D, _P, _P, _P, _P, _P, _P, ctypes.POINTER(_I), _P], _I),
    "otn_square_matvec": ([_P, _P, _P, _P], _I),
    "otn_matvec": ([_P, _P, _P, _P, _P], _I),
    "otn_rmatvec": ([_P, _P, _P, _P, _P], _I),
}
OTN_ST_PLAN_OVERFLOW = 10                # include/otn_b200.h


class Seam:
    """The five seam operators on one CUDA device (one library context per n)."""

    def __init__(self, lib_path, device=0, overflow_error=RuntimeError):
        import torch
        self.torch = torch
        self.lib = ctypes.CDLL(lib_path)
        for name, (args, res) in _SIGS.items():
            fn = getattr(self.lib, name)
            fn.argtypes, fn.restype = args, res
        self.device = torch.device("cuda", device)
        self.overflow_error = overflow_error     # the reference's PlanOverflowError
        self.ctxs = {}

    # -- plumbing ------------------------------------------------------------
    def _check(self, rc, what):
        if rc not in (0, OTN_ST_PLAN_OVERFLOW):
            raise RuntimeError(f"{what}: {self.lib.otn_last_error().decode()}")
        return rc

    def _ctx(self, n):
        h = self.ctxs.get(n)
        if h is None:
            h = _P()
            stream = self.torch.cuda.current_stream(self.device).cuda_stream
            self._check(self.lib.otn_create(ctypes.byref(h), self.device.index, n,
                                            (n + 31) // 32 * 32, _P(stream)), "otn_create")
            self.ctxs[n] = h
        return h

    def _mat(self, A):
        """n x n host array -> device (n, ld) float64, zero padding columns."""
        n = A.shape[0]
        ld = (n + 31) // 32 * 32
        D = self.torch.zeros((n, ld), dtype=self.torch.float64, device=self.device)
        D[:, :n].copy_(self.torch.from_numpy(np.ascontiguousarray(A, dtype=np.float64)))
        return D

    def _vec(self, x, n):
        ld = (n + 31) // 32 * 32
        d = self.torch.zeros(ld, dtype=self.torch.float64, device=self.device)
        d[:n].copy_(self.torch.from_numpy(np.array(
            np.broadcast_to(np.asarray(x, dtype=np.float64), (n,)))))
        return d

    @staticmethod
    def _p(t):
        return None if t is None else _P(t.data_ptr())

    def _host(self, d, n):
        self.torch.cuda.synchronize(self.device)
        return d[:n].cpu().numpy().copy()

    # -- the seam (_kernels.py:22-74, newton.py:43-56) -------------------------
    # (every device operand is bound to a local until the call has completed:
    # a temporary tensor freed while its kernel is in flight would hand its
    # memory to the next allocation)
    def log_plan_row_sums(self, K, u, v):
        """u + LSE_j(K_ij + v_j); all -inf rows -> -inf (u may be a scalar)."""
        n = K.shape[0]
        Kd, vd = self._mat(K), self._vec(v, n)
        outer = None if np.isscalar(u) and u == 0.0 else self._vec(u, n)
        out = self._vec(0.0, n)
        self._check(self.lib.otn_lse_rows(self._ctx(n), self._p(Kd), 1.0, self._p(outer),
                                          self._p(vd), self._p(out)), "otn_lse_rows")
        return self._host(out, n)

    def materialize_plan(self, K, u, v, out=None):
        """exp((K + v) + u); raises the overflow error past a log entry of 700."""
        n = K.shape[0]
        P = self._mat(np.zeros((n, n)))
        Kd, ud, vd = self._mat(K), self._vec(u, n), self._vec(v, n)
        flag = _I(0)
        rc = self.lib.otn_materialize(self._ctx(n), self._p(Kd), 1.0, self._p(ud), self._p(vd),
                                      self._p(P), None, None, None, ctypes.byref(flag), None)
        if self._check(rc, "otn_materialize") == OTN_ST_PLAN_OVERFLOW or flag.value:
            raise self.overflow_error("log-plan entry would overflow exp(); warm start is broken")
        self.torch.cuda.synchronize(self.device)
        host = P[:, :n].cpu().numpy()
        if out is None:
            return host.copy()
        out[...] = host
        return out

    def square_matvec(self, P, w):
        """(P * P) @ w."""
        n = P.shape[0]
        Pd, wd, out = self._mat(P), self._vec(w, n), self._vec(0.0, n)
        self._check(self.lib.otn_square_matvec(self._ctx(n), self._p(Pd), self._p(wd),
                                               self._p(out)), "otn_square_matvec")
        return self._host(out, n)

    def matvec(self, P, x):
        """P @ x."""
        n = P.shape[0]
        Pd, xd, out = self._mat(P), self._vec(x, n), self._vec(0.0, n)
        self._check(self.lib.otn_matvec(self._ctx(n), self._p(Pd), None, self._p(xd),
                                        self._p(out)), "otn_matvec")
        return self._host(out, n)

    def rmatvec(self, P, x):
        """P.T @ x."""
        n = P.shape[0]
        Pd, xd, out = self._mat(P), self._vec(x, n), self._vec(0.0, n)
        self._check(self.lib.otn_rmatvec(self._ctx(n), self._p(Pd), None, self._p(xd),
                                         self._p(out)), "otn_rmatvec")
        return self._host(out, n)
