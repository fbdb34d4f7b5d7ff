"""CPU test double for the point-cloud kernels (tests only).

Implements the same pass / vector / reduction operations as the C-ABI on torch
CPU tensors so the ROW-SHARDED host logic (pointcloud.Comm, column-LSE
combines, scalar allreduces) can run under gloo with several processes on a
machine without GPUs.  It is never used by the package itself.
"""

import numpy as np
import torch

from paper_2504_02067_b200 import _lib

F64 = torch.float64


class CpuPairBackend:
    def tensor(self, arr):
        return torch.from_numpy(np.array(arr, dtype=np.float64))

    def pass_(self, op, A, na, B, nb, d, cmax, ng, order, colpot, colpot_d, alpha, rowpot, vec,
              outer, outer_d, mode, out, out2):
        a = A.view(d, na)
        b = B.view(d, nb)
        D = None
        for k in range(d):
            diff = a[k][:, None] - b[k][None, :]
            sq = diff * diff
            D = sq if D is None else D + sq
        C = D / cmax if cmax > 0.0 else D
        if op == _lib.PC_MAXD:
            out[:na] = C.max(dim=1).values
            return
        if op == _lib.PC_CDOT:
            out[:na] = C @ vec[:nb]
            return
        cp = torch.zeros(nb, dtype=F64) if colpot is None else colpot[:nb].clone()
        if colpot_d is not None:
            cp = cp + alpha * colpot_d[:nb]
        rp = None if rowpot is None else rowpot[:na]
        kc = ng * C
        if op == _lib.PC_LSE_SHIFT:
            e = kc + cp[None, :]
            if rp is not None:
                e = e + rp[:, None]
            out[:na] = torch.exp(e - outer[:na][:, None]).sum(dim=1)
            return
        if op in (_lib.PC_LSE, _lib.PC_LSE_PART):
            e = kc + cp[None, :]
            if rp is not None:
                e = e + rp[:, None]
            m = e.max(dim=1).values
            s = torch.exp(e - m[:, None]).sum(dim=1)
            if op == _lib.PC_LSE_PART:
                out[:na] = m
                out2[:na] = s
                return
            lse = torch.where(torch.isfinite(m), m + torch.log(s), torch.full_like(m, -np.inf))
            o = torch.zeros(na, dtype=F64) if outer is None else outer[:na].clone()
            if outer_d is not None:
                o = o + alpha * outer_d[:na]
            out[:na] = o + lse if mode == 0 else o - lse
            return
        rpp = torch.zeros(na, dtype=F64) if rp is None else rp
        e = (kc + cp[None, :]) + rpp[:, None] if order == 0 else (kc + rpp[:, None]) + cp[None, :]
        P = torch.exp(e)
        if op == _lib.PC_DOT:
            out[:na] = P @ vec[:nb]
        elif op == _lib.PC_DOTC:
            out[:na] = (P * C) @ vec[:nb]
        elif op == _lib.PC_DIAG:
            out[:na] = (P * P) @ vec[:nb]
            if out2 is not None:
                out2[:na] = e.max(dim=1).values
        else:
            raise ValueError(op)

    def vec(self, n, op, out, a, b=None, c=None, d=None, s=0.0):
        A = a[:n]
        B = b[:n] if b is not None else None
        Cv = c[:n] if c is not None else None
        Dv = d[:n] if d is not None else None
        L = _lib

        def lse(m, ss):
            return torch.where(torch.isfinite(m), m + torch.log(ss), torch.full_like(m, -np.inf))
        res = {
            L.VEC_ADD_SUB: lambda: (A + B) - Cv,
            L.VEC_AXPY: lambda: A + s * B,
            L.VEC_STEP_V: lambda: (A + s * B) + (Cv - Dv),
            L.VEC_EXTRAP: lambda: A + s * (A - B),
            L.VEC_EXP: lambda: torch.exp(A),
            L.VEC_GRAD: lambda: torch.exp(A) - B,
            L.VEC_MUL_SUB: lambda: A * B - s * Cv,
            L.VEC_DIV: lambda: A / B,
            L.VEC_SUB: lambda: A - B,
            L.VEC_ADD: lambda: A + B,
            L.VEC_PRECOND: lambda: A * (1.0 - s * B),
            L.VEC_NEG_DIV: lambda: (-A) / B,
            L.VEC_RESCALE: lambda: A * torch.exp(B - Cv),
            L.VEC_LSE_FIN: lambda: A + lse(B, Cv),
            L.VEC_LSE_FIN_SUB: lambda: A - lse(B, Cv),
            L.VEC_ROUND_SCALE: lambda: torch.where(B > 0, torch.clamp(A / B, max=1.0),
                                                   torch.ones_like(A)),
            L.VEC_SUB_MUL: lambda: A - B * Cv,
            L.VEC_MUL: lambda: A * B,
        }[op]()
        out[:n] = res

    def reduce(self, n, op, a, b=None, c=None, d=None):
        A = a[:n]
        L = _lib
        if op == L.RED_ROW_STATS:
            x, y = torch.exp(A), b[:n]
            fl = (1 if bool((x <= 0).any()) else 0) | (2 if bool((y < 0).any()) else 0)
            return float((x - y).abs().sum()), float((y * y / x).sum()), fl
        if op == L.RED_GRAD_L1:
            return (float((torch.exp(A) - b[:n]).abs().sum()),
                    float((torch.exp(c[:n]) - d[:n]).abs().sum()), 0)
        if op == L.RED_SUM_EXP:
            return float(torch.exp(A).sum()), 0.0, 0
        if op == L.RED_DOT:
            return float(A @ b[:n]), 0.0, 0
        if op == L.RED_L1:
            return float(A.abs().sum()), 0.0, 0
        if op == L.RED_L1_ADD:
            return float((A + b[:n]).abs().sum()), 0.0, 0
        if op == L.RED_NONPOS:
            return float((A <= 0).sum()), 0.0, 0
        if op == L.RED_MAX:
            return float(A.max()) if n else -np.inf, 0.0, 0
        if op == L.RED_L1_DOT:
            return float(A.abs().sum()), float(A @ b[:n]), 0
        if op == L.RED_OUTSIDE:
            ok = (A >= 2.0 ** -700) & (A <= 2.0 ** 700)
            return float((~ok).sum()), 0.0, 0
        raise ValueError(op)

    def reduce_dev(self, n, op, dst, a, b=None, c=None, d=None):
        s0, s1, _ = self.reduce(n, op, a, b, c, d)
        dst[0] = s0
        dst[1] = s1
