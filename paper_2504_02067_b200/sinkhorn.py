"""Log-domain Sinkhorn projector on the same device kernels.

Mirrors ``oracles.py:243-265`` ``sinkhorn_project`` — the paper's baseline and
the ``MdotOptions(projector="sinkhorn")`` branch of the driver
(``driver.py:218-223,277-279``).  Each sweep is one exact row scaling (one
column LSE) plus one exact column scaling (one row LSE); the stopping test is
the full L1 gradient norm, reduced on the device.
"""

from __future__ import annotations

import numpy as np

from . import opcount
from .errors import DomainError, NonconvergenceError


def sinkhorn_project(state, r, c, eps_d, sweep_budget=10 ** 6):
    """Sinkhorn sweeps until ||grad||_1 <= eps_d; returns ``(state, sweeps)``."""
    if np.min(r) <= 0.0 or np.min(c) <= 0.0:
        raise DomainError("sinkhorn_project requires strictly positive marginals")
    state.set_targets(r, c)
    steps = 0
    with opcount.category("sinkhorn"):
        while state.grad_norm_l1() > eps_d:
            if steps >= sweep_budget:
                raise NonconvergenceError(
                    f"Sinkhorn still at gradient norm {state.grad_norm_l1():.3g} "
                    f"> {eps_d:.3g} after {steps} sweeps",
                    diagnostics={"gamma": state.gamma, "eps_d": eps_d})
            state.scale_rows_to_target()
            state.scale_cols_to_target()
            steps += 1
    return state, steps
