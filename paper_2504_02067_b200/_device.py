"""Device plumbing: contexts, padded device buffers, the device-resident cost.

PyTorch is used only for device memory, streams and host<->device copies; all
arithmetic on the solver path runs in the C-ABI library (``_lib``).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import DeviceError

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda(device=None):
    t = torch()
    if not t.cuda.is_available():
        raise DeviceError("a CUDA device is required: this package has no CPU fallback")
    if device is None:
        device = t.device("cuda", t.cuda.current_device())
    device = t.device(device)
    if device.type != "cuda":
        raise DeviceError(f"expected a CUDA device, got {device}")
    if device.index is None:
        device = t.device("cuda", t.cuda.current_device())
    return device


def round_up(n, k=32):
    return (n + k - 1) // k * k


def vptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


# Kernel launches issued by each C-ABI entry point (for the bench's
# gpu_launches claim).  otn_lse_cols / otn_rebalance_cols / otn_trial_cols launch
# one kernel for symmetric costs (or a materialized transpose) and two
# otherwise; trial adds the mass reduce.  Every persistent-solver entry point
# launches k_partition then k_coop.
LAUNCHES = {
    "otn_lse_rows": 1, "otn_lse_cols": 2, "otn_rebalance_cols": 2, "otn_trial_cols": 3,
    "otn_materialize": 1, "otn_plan_mask": 1, "otn_system_prep": 1, "otn_square_matvec": 1,
    "otn_matvec": 2, "otn_rmatvec": 2, "otn_apply_F": 2, "otn_apply_pc": 2, "otn_pcg": 2,
    "otn_newton": 2, "otn_probe": 2,
    # newton (2) + gate + trial (1 | 2) + mass + gate + accept (u, v, lc) + row LSE
    # + row stats with the gradient
    "otn_newton_step": 9, "otn_newton_step_wait": 0,
    "otn_vec": 1, "otn_reduce": 1, "otn_row_stats": 1, "otn_accept": 1, "otn_reduce_async": 1, "otn_round_plan": 10, "otn_pc_pass": 1,
    "otn_vec_n": 1, "otn_reduce_n": 1, "otn_reduce_dev": 1, "otn_zero": 0,
    "otn_is_symmetric": 1, "otn_transpose": 1, "otn_pixel_cost": 3,
}


class Telemetry:
    """Host-side counters for the bench: kernel launches, host<->device bytes,
    and (when enabled) CUDA-event timing of the persistent solver launches."""

    def __init__(self):
        self.reset()
        self.time_coop = False

    def reset(self):
        self.launches = 0
        self.calls = {}
        self.h2d = 0
        self.d2h = 0
        self.coop = []        # (device ms, hvps, d_v formed, n, plan mode, nnz, span entries,
                              #  cg iterations) per timed k_coop launch

    def count(self, name, sym=False):
        k = LAUNCHES.get(name, 0)
        if sym and name in ("otn_lse_cols", "otn_rebalance_cols", "otn_trial_cols",
                            "otn_newton_step"):
            k -= 1
        self.launches += k
        self.calls[name] = self.calls.get(name, 0) + 1


TELEMETRY = Telemetry()
_SYM_CALLS = ("otn_lse_cols", "otn_rebalance_cols", "otn_trial_cols")
_SYM_ARG = {name: 1 for name in _SYM_CALLS}
_SYM_ARG["otn_newton_step"] = 14


def is_tensor(x):
    return type(x).__module__.startswith("torch") and hasattr(x, "data_ptr")


class Context:
    """One C-ABI context (device workspace) per (device, n)."""

    _cache = {}

    def __init__(self, n, device):
        self.lib = _lib.load()
        self.n = int(n)
        self.ld = round_up(self.n, 32)
        self.device = device
        t = torch()
        with t.cuda.device(device):
            stream = t.cuda.current_stream(device).cuda_stream
            h = ctypes.c_void_p()
            rc = self.lib.otn_create(ctypes.byref(h), device.index, self.n, self.ld,
                                     ctypes.c_void_p(stream))
            _lib.check(rc, "otn_create")
        self.h = h
        self._stream = stream
        self._fns = {}
        info = (ctypes.c_int64 * 4)()
        _lib.check(self.lib.otn_info(self.h, info), "otn_info")
        self.coop_blocks = int(info[2])
        self.workspace_bytes = int(info[3])
        cfg = (ctypes.c_int64 * 4)()
        _lib.check(self.lib.otn_config(self.h, cfg), "otn_config")
        self.config = {"sms": int(cfg[0]), "lse_bulk_ctas": int(cfg[1]),
                       "lse_slabs": int(cfg[2]), "config_error": int(cfg[3])}

    @classmethod
    def get(cls, n, device):
        key = (device.index, int(n))
        ctx = cls._cache.get(key)
        if ctx is None:
            ctx = cls(n, device)
            cls._cache[key] = ctx
        ctx.sync_stream()
        return ctx

    def sync_stream(self):
        s = torch().cuda.current_stream(self.device).cuda_stream
        if s != self._stream:
            _lib.check(self.lib.otn_set_stream(self.h, ctypes.c_void_p(s)), "otn_set_stream")
            self._stream = s

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.otn_destroy(self.h)
        except Exception:
            pass

    def coop_timing(self):
        """Match the library's launch timing to TELEMETRY.time_coop; returns it."""
        on = bool(TELEMETRY.time_coop)
        if getattr(self, "_timing", False) != on:
            _lib.check(self.lib.otn_set_timing(self.h, int(on)), "otn_set_timing")
            self._timing = on
        return on

    def coop_ms(self):
        """Device time of the last persistent-solver launch (timing on)."""
        ms = ctypes.c_float(0.0)
        _lib.check(self.lib.otn_coop_ms(self.h, ctypes.byref(ms)), "otn_coop_ms")
        return float(ms.value)

    # ---- buffers ---------------------------------------------------------
    def zeros(self, shape, dtype=None):
        """A zeroed device buffer: torch allocates (caching allocator), the
        library zeroes it stream-ordered (a memset, no framework kernel)."""
        t = torch()
        buf = t.empty(shape, dtype=dtype or t.float64, device=self.device)
        self.call("otn_zero", vptr(buf), buf.numel() * buf.element_size())
        return buf

    def vec(self, init=None):
        """Padded device vector (ld entries, zeros beyond n); returns the buffer."""
        buf = self.zeros(self.ld)
        if init is not None:
            self.upload(buf, init)
        return buf

    def upload_async(self, buf, values, slot):
        """H2D copy of a host vector through a reusable page-locked staging
        buffer (per `slot`) as one stream-ordered C-ABI copy: no host stall.
        The staging buffer is reused only after its previous copy completed."""
        t = torch()
        pool = self.__dict__.setdefault("_staging", {})
        ent = pool.get(slot)
        if ent is None:
            ent = (t.empty(self.n, dtype=t.float64, pin_memory=True), t.cuda.Event())
            pool[slot] = ent
        host, ev = ent
        ev.synchronize()
        host.numpy()[:] = np.asarray(values, dtype=np.float64)
        self.call("otn_upload", vptr(buf), ctypes.c_void_p(host.data_ptr()), self.n)
        ev.record(t.cuda.current_stream(self.device))
        TELEMETRY.h2d += host.numel() * 8
        return buf

    def upload_rows_async(self, block, rows, slot):
        """block[i, :n] = rows[i] for a contiguous (k, ld) device block, as ONE
        stream-ordered copy from page-locked staging (padding copied as 0)."""
        t = torch()
        pool = self.__dict__.setdefault("_staging", {})
        key = (slot, block.shape[0])
        ent = pool.get(key)
        if ent is None:
            ent = (t.zeros(block.shape, dtype=t.float64, pin_memory=True), t.cuda.Event())
            pool[key] = ent
        host, ev = ent
        ev.synchronize()
        h = host.numpy()
        for i, v in enumerate(rows):
            h[i, : self.n] = v
        self.call("otn_upload", vptr(block), ctypes.c_void_p(host.data_ptr()), block.numel())
        ev.record(t.cuda.current_stream(self.device))
        TELEMETRY.h2d += host.numel() * 8
        return block

    def copy(self, dst, src):
        """dst[:ld] = src[:ld] on the ctx stream (one C-ABI call)."""
        self.call("otn_copy", vptr(dst), vptr(src), self.ld)

    def upload(self, buf, values):
        t = torch()
        if is_tensor(values):
            buf[: self.n].copy_(values.reshape(-1)[: self.n].to(dtype=t.float64), non_blocking=True)
        else:
            arr = np.array(np.broadcast_to(np.asarray(values, dtype=np.float64), (self.n,)))
            buf[: self.n].copy_(t.from_numpy(arr), non_blocking=False)
            TELEMETRY.h2d += arr.nbytes
        return buf

    def download(self, buf):
        out = buf[: self.n].detach().cpu().numpy().copy()
        TELEMETRY.d2h += out.nbytes
        return out

    def mat(self):
        return self.zeros((self.n, self.ld))

    def seg_mask(self):
        """Plan segment-occupancy mask (OTN_MASK_WORDS(ld) uint64 words per row)."""
        return self.zeros((self.n, (self.ld + 4095) // 4096 + 1), dtype=torch().int64)

    # ---- thin call helpers -----------------------------------------------
    def call(self, name, *args):
        # the host issues ~450 calls per n = 4096 solve, many while the GPU
        # waits on it: one cached lookup per call
        ent = self._fns.get(name)
        if ent is None:
            ent = self._fns[name] = (getattr(self.lib, name), LAUNCHES.get(name, 0),
                                     _SYM_ARG.get(name))
        fn, k, si = ent
        if si is not None and args[si]:
            k -= 1                       # a symmetric cost: the column pass is one kernel
        T = TELEMETRY
        T.launches += k
        T.calls[name] = T.calls.get(name, 0) + 1
        rc = fn(self.h, *args)
        return _lib.check(rc, name) if rc else rc


class DeviceCost:
    """Device-resident cost matrix with leading dimension ld (multiple of 32).

    For a problem whose C is already a CUDA tensor the prepared cost (the
    symmetry verdict, an asymmetric cost's transpose) is kept on the Problem
    and reused by later solves while the tensor is unchanged (same storage,
    same torch version counter); a host C is uploaded by every solve."""

    @classmethod
    def of(cls, problem, device):
        C = problem.C
        if not (is_tensor(C) and C.is_cuda and C.device == device):
            return cls(problem, device)
        key = (C.data_ptr(), tuple(C.shape), tuple(C.stride()), C._version)
        cached = problem.__dict__.get("_otn_device_cost")
        if cached is not None and cached[0] == key:
            return cached[1]
        dc = cls(problem, device)
        problem.__dict__["_otn_device_cost"] = (key, dc)
        return dc

    def __init__(self, problem, device):
        t = torch()
        self.n = problem.n
        self.ctx = Context.get(self.n, device)
        ld = self.ctx.ld
        C = problem.C
        if is_tensor(C):
            if not C.is_cuda:
                C = C.to(device)
            padded = getattr(C, "_otn_padded", None)
            if (padded is not None and padded.device == C.device and padded.data_ptr() == C.data_ptr()
                    and tuple(padded.shape) == (self.n, ld)):
                self.C = padded                  # built in the solver's layout (pixel_cost_device)
            elif ld == self.n and C.is_contiguous():
                self.C = C
            else:
                self.C = self.ctx.zeros((self.n, ld))
                self.C[:, : self.n].copy_(C)
        else:
            host = t.from_numpy(np.ascontiguousarray(C, dtype=np.float64))
            TELEMETRY.h2d += host.numel() * 8
            if ld == self.n:
                self.C = host.to(device, non_blocking=False)
            else:
                self.C = self.ctx.zeros((self.n, ld))
                self.C[:, : self.n].copy_(host)
        self._symmetric = None

    @property
    def symmetric(self):
        """(C == C.T).all(), evaluated once (dual.py:80-88), by the library's
        tiled comparison kernel."""
        if self._symmetric is None:
            flag = ctypes.c_int(0)
            self.ctx.call("otn_is_symmetric", vptr(self.C), ctypes.byref(flag))
            self._symmetric = bool(flag.value)
        return self._symmetric

    def ptr(self):
        return vptr(self.C)

    def col_args(self):
        """(matrix, symmetric flag) for a column-direction pass.  An asymmetric
        cost gets its transpose materialized once on first use (the reference
        forms K^T likewise, dual.py:77-89) so column log-sum-exps run as
        coalesced row passes; a symmetric one is its own transpose."""
        if self.symmetric:
            return vptr(self.C), 1
        if getattr(self, "CT", None) is None:
            self.CT = self.ctx.zeros((self.n, self.ctx.ld))
            self.ctx.call("otn_transpose", vptr(self.CT), vptr(self.C))
        return vptr(self.CT), 1
