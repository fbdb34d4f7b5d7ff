"""Check the executable seam binding (integration/otnewton_b200.py) operator
by operator against numpy on random inputs (diagnostic)."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "integration")
from otnewton_b200 import Seam  # noqa: E402

from paper_2504_02067_b200 import _lib  # noqa: E402

s = Seam(_lib.LIB_PATH)
rng = np.random.default_rng(0)
for n in (64, 70, 256):
    K = -rng.random((n, n)) * 5
    u = rng.standard_normal(n)
    v = rng.standard_normal(n)
    t = K + v[None, :]
    m = t.max(1)
    want = u + m + np.log(np.exp(t - m[:, None]).sum(1))
    got = s.log_plan_row_sums(K, u, v)
    print(n, "lse", np.abs(got - want).max(), got[:3], want[:3])
    Pr = np.exp((K + v[None, :]) + u[:, None])
    P = s.materialize_plan(K, u, v)
    print(n, "plan", np.abs(P - Pr).max() / Pr.max())
    w = rng.random(n)
    print(n, "sq", np.abs(s.square_matvec(Pr, w) - (Pr * Pr) @ w).max() / np.abs((Pr * Pr) @ w).max())
    print(n, "mv", np.abs(s.matvec(Pr, w) - Pr @ w).max() / np.abs(Pr @ w).max())
    print(n, "rmv", np.abs(s.rmatvec(Pr, w) - Pr.T @ w).max() / np.abs(Pr.T @ w).max())
