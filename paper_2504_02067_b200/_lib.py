"""ctypes binding of the in-tree C-ABI library ``libotn_b200.so``.

The library is the only compute path: there is no CPU fallback.  If it is
missing or cannot be loaded, every solver entry point raises ``DeviceError``.
The signatures below are exactly those declared in ``include/otn_b200.h``.
"""

from __future__ import annotations

import ctypes
import os

from .errors import (
    ConditioningError,
    DeviceError,
    DomainError,
    NonconvergenceError,
    PlanOverflowError,
    StagnationError,
)

LIB_NAME = "libotn_b200.so"
# OTN_LIB_AB: alternate build of the same library, for side-by-side kernel timing (tools/)
LIB_PATH = os.environ.get("OTN_LIB_AB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                         LIB_NAME)

OTN_OK = 0
OTN_ERR_CUDA = 1
OTN_ERR_ARG = 2
OTN_ST_PLAN_OVERFLOW = 10
OTN_ST_NONPOSITIVE_SUMS = 11
OTN_ST_BREAKDOWN = 12
OTN_ST_PRECOND = 13
OTN_ST_NONCONVERGENCE = 14
OTN_ST_STAGNATION = 15
OTN_ST_DOMAIN = 16

(VEC_ADD_SUB, VEC_AXPY, VEC_STEP_V, VEC_EXTRAP, VEC_EXP, VEC_GRAD, VEC_MUL_SUB, VEC_DIV,
 VEC_SUB, VEC_ADD, VEC_PRECOND, VEC_NEG_DIV, VEC_RESCALE, VEC_LSE_FIN, VEC_LSE_FIN_SUB,
 VEC_ROUND_SCALE, VEC_SUB_MUL, VEC_MUL, VEC_COPY) = range(19)
(RED_ROW_STATS, RED_GRAD_L1, RED_SUM_EXP, RED_DOT, RED_L1, RED_L1_ADD, RED_NONPOS,
 RED_MAX, RED_L1_DOT, RED_OUTSIDE) = range(10)
PC_LSE, PC_DOT, PC_DIAG, PC_MAXD, PC_LSE_PART, PC_DOTC, PC_CDOT, PC_LSE_SHIFT = range(8)


ABI_VERSION = 2                 # include/otn_b200.h OTN_ABI_VERSION


class SolveResult(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int32),
        ("pcg_calls", ctypes.c_int32),
        ("cg_iters", ctypes.c_int64),
        ("hvps", ctypes.c_int64),
        ("rho_final", ctypes.c_double),
        ("resid_l1", ctypes.c_double),
        ("slope", ctypes.c_double),
        ("diag_rho", ctypes.c_double),
        ("diag_resid", ctypes.c_double),
        ("plan_mode", ctypes.c_int32),
        ("plan_rows_max", ctypes.c_int32),
        ("plan_nnz", ctypes.c_int64),
        ("plan_span", ctypes.c_int64),
    ]


_P = ctypes.c_void_p
_D = ctypes.c_double
_I = ctypes.c_int
_I64 = ctypes.c_int64
_DP = ctypes.POINTER(ctypes.c_double)
_IP = ctypes.POINTER(ctypes.c_int)

# name -> argtypes (restype is int unless noted)
SIGNATURES = {
    "otn_abi_version": [],
    "otn_last_error": [],
    "otn_create": [ctypes.POINTER(_P), _I, _I64, _I64, _P],
    "otn_destroy": [_P],
    "otn_set_stream": [_P, _P],
    "otn_info": [_P, ctypes.POINTER(_I64)],
    "otn_config": [_P, ctypes.POINTER(_I64)],
    "otn_read_flags": [_P, _IP],
    "otn_set_timing": [_P, _I],
    "otn_coop_ms": [_P, ctypes.POINTER(ctypes.c_float)],
    "otn_copy": [_P, _P, _P, _I64],
    "otn_upload": [_P, _P, _P, _I64],
    "otn_lse_rows": [_P, _P, _D, _P, _P, _P],
    "otn_lse_cols": [_P, _P, _I, _D, _P, _P, _P],
    "otn_rebalance_cols": [_P, _P, _I, _D, _P, _P, _P],
    "otn_trial_cols": [_P, _P, _I, _D, _P, _P, _P, _P, _D, _P, _DP],
    "otn_materialize": [_P, _P, _D, _P, _P, _P, _P, _P, _P, _IP, _P],
    "otn_plan_mask": [_P, _P, _P],
    "otn_system_prep": [_P, _P, _P, _P, _P, _P, _IP],
    "otn_square_matvec": [_P, _P, _P, _P],
    "otn_matvec": [_P, _P, _P, _P, _P],
    "otn_rmatvec": [_P, _P, _P, _P, _P],
    "otn_apply_F": [_P, _P, _P, _P, _P, _D, _P, _P],
    "otn_apply_pc": [_P, _P, _P, _P, _P, _P],
    "otn_pcg": [_P, _P, _P, _P, _P, _P, _D, _P, _D, _P, _I, _I64, ctypes.POINTER(SolveResult)],
    "otn_newton": [_P, _P, _P, _P, _P, _P, _P, _D, _D, _I, _I64, _P, _P,
                   ctypes.POINTER(SolveResult)],
    "otn_newton_step": [_P, _P, _P, _P, _P, _P, _P, _D, _D, _I, _I64, _P, _P, _P, _P, _I, _D, _P, _P,
                        _P, _P, _P, _P, _P, _P, _D, _D, ctypes.POINTER(SolveResult), _DP, _IP],
    "otn_newton_step_wait": [_P, ctypes.POINTER(SolveResult), _DP, _IP],
    "otn_probe": [_P, _P, _P, _P, _P, _P, _P, _I, _I64],
    "otn_coop_layout": [_P],
    "otn_pc_pass": [_P, _I, _P, _I64, _I64, _P, _I64, _I64, _I, _D, _D, _I, _P, _P, _D, _P, _P,
                    _P, _P, _I, _P, _P],
    "otn_vec_n": [_P, _I64, _I, _D, _P, _P, _P, _P, _P],
    "otn_reduce_n": [_P, _I64, _I, _P, _P, _P, _P, _DP, _IP],
    "otn_reduce_dev": [_P, _I64, _I, _P, _P, _P, _P, _P],
    "otn_zero": [_P, _P, _I64],
    "otn_is_symmetric": [_P, _P, _IP],
    "otn_transpose": [_P, _P, _P],
    "otn_pixel_cost": [_P, _P, _P, _I64, _P, _DP],
    "otn_vec": [_P, _I, _D, _P, _P, _P, _P, _P],
    "otn_reduce": [_P, _I, _P, _P, _P, _P, _DP, _IP],
    "otn_row_stats": [_P, _P, _P, _P, _DP, _IP],
    "otn_accept": [_P, _D, _P, _P, _P, _P, _P, _P, _P],
    "otn_reduce_async": [_P, _I, _P, _P, _P, _P, _P],
    "otn_round_plan": [_P, _P, _P, _P, _P, _DP, _IP],
}

_lib = None
_load_error = None


def load():
    """Load (once) and return the ctypes library; raise DeviceError if absent."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if _load_error is not None:
        raise DeviceError(_load_error)
    if not os.path.exists(LIB_PATH):
        _load_error = (f"{LIB_PATH} not found: build it with `make -C "
                       f"paper_2504_02067_b200/csrc` (or __graft_entry__.build()); "
                       "there is no CPU fallback")
        raise DeviceError(_load_error)
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        _load_error = f"cannot load {LIB_PATH}: {exc}"
        raise DeviceError(_load_error) from exc
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = ctypes.c_char_p if name == "otn_last_error" else ctypes.c_int
    if lib.otn_abi_version() != ABI_VERSION:
        _load_error = (f"{LIB_PATH} has ABI {lib.otn_abi_version()}, this package needs "
                       f"{ABI_VERSION}: rebuild it (make -C paper_2504_02067_b200/csrc)")
        raise DeviceError(_load_error)
    _lib = lib
    return lib


def exported_symbols():
    return list(SIGNATURES)


def last_error():
    return load().otn_last_error().decode(errors="replace")


def check(rc, what):
    """Map a non-solver return code onto DeviceError; pass solver codes through."""
    if rc in (OTN_ERR_CUDA, OTN_ERR_ARG):
        raise DeviceError(f"{what}: {last_error()}")
    return rc


def raise_for_status(rc, what, best=None, diagnostics=None, message=None):
    """Raise the reference's exception class for a solver status code."""
    if rc == OTN_OK:
        return
    check(rc, what)
    if rc == OTN_ST_PLAN_OVERFLOW:
        raise PlanOverflowError(message or "log-plan entry would overflow exp(); warm start is broken")
    if rc == OTN_ST_NONPOSITIVE_SUMS:
        raise ConditioningError("plan row/column sums must be strictly positive")
    if rc == OTN_ST_PRECOND:
        raise ConditioningError("preconditioner has a nonpositive diagonal entry")
    if rc == OTN_ST_BREAKDOWN:
        raise ConditioningError(message or "CG breakdown: nonpositive curvature along search direction")
    if rc == OTN_ST_NONCONVERGENCE:
        raise NonconvergenceError(message or "CG did not reach its tolerance", best=best,
                                  diagnostics=diagnostics)
    if rc == OTN_ST_STAGNATION:
        raise StagnationError(message or "discount annealing stagnated")
    if rc == OTN_ST_DOMAIN:
        raise DomainError(message or "domain error")
    raise DeviceError(f"{what}: unknown status {rc}")
