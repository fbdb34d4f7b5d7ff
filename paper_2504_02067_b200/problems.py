"""Problem inputs: dense-cost problems, point-cloud problems, seeded generators.

``Problem`` keeps the reference input contract (``problems.py:31-65``): a dense
n-by-n cost with entries in [0, 1] plus two simplex marginals.  ``C`` may be a
host numpy array (the reference's type) or a device-resident ``torch`` CUDA
float64 tensor (the bench's HBM-resident input); either way ``r`` and ``c``
live on the host.

``PointCloudProblem`` is the large-n input the reference does not have
(SURVEY §8(b)): the cost ``C_ij = ||x_i - y_j||^2 / C_max`` is never stored and
is recomputed tile by tile on the GPU.  ``materialize_cost()`` builds the same
matrix on the host with the identical operand order, so the on-the-fly kernels
are bit-exact against a stored-C run at small n.

Generators reproduce the reference's seeded streams bit for bit
(``problems.py:87-144``, ``cli.py:88-98``); the point-cloud generators are
this package's synthetic D1/D3/D4/D5 workloads.
"""

from __future__ import annotations

import csv
import ctypes
from dataclasses import dataclass, fields

import numpy as np

from .errors import DimensionError, DomainError, ParseError

SIMPLEX_TOL = 1e-12          # problems.py:18
PARSE_SIMPLEX_TOL = 1e-9     # problems.py:21
COL_SEED_OFFSET = 1          # cli.py:32

TRACE_HEADER = [
    "t", "gamma", "eps_d", "newton_steps", "cg_iters", "sinkhorn_steps",
    "linesearch_backtracks", "grad_norm_l1", "rho_final", "delta_min", "q",
    "ops_n2", "wall_ms",
]


def _is_device_tensor(x):
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _check_marginals(n, r, c):
    if r.shape != (n,) or c.shape != (n,):
        raise DimensionError(f"marginal lengths {r.shape}, {c.shape} do not match n={n}")
    for name, m in (("r", r), ("c", c)):
        if np.any(m < 0.0):
            raise DomainError(f"marginal {name} has negative entries")
        if abs(m.sum() - 1.0) > SIMPLEX_TOL:
            raise DomainError(f"marginal {name} sums to {m.sum():.17g}, not 1")


@dataclass
class Problem:
    """Dense cost plus row/column marginals on the simplex (problems.py:31-65)."""

    C: object
    r: np.ndarray
    c: np.ndarray
    label: str = ""

    def __post_init__(self):
        if not _is_device_tensor(self.C):
            self.C = np.ascontiguousarray(self.C, dtype=np.float64)
        self.r = np.ascontiguousarray(self.r, dtype=np.float64)
        self.c = np.ascontiguousarray(self.c, dtype=np.float64)
        self.validate()

    @property
    def n(self):
        return int(self.C.shape[0])

    @property
    def on_device(self):
        return _is_device_tensor(self.C)

    def validate(self):
        C = self.C
        if C.ndim != 2 or C.shape[0] != C.shape[1]:
            raise DimensionError(f"cost matrix must be square, got {tuple(C.shape)}")
        n = int(C.shape[0])
        if _is_device_tensor(C):
            import torch
            if C.dtype != torch.float64:
                raise DomainError("device cost must be float64")
            if not bool(torch.isfinite(C).all()):
                raise DomainError("cost matrix must be finite")
            if float(C.min()) < 0.0 or float(C.max()) > 1.0:
                raise DomainError("cost entries must lie in [0, 1]")
        else:
            if not np.all(np.isfinite(C)):
                raise DomainError("cost matrix must be finite")
            if C.min() < 0.0 or C.max() > 1.0:
                raise DomainError("cost entries must lie in [0, 1]")
        _check_marginals(n, self.r, self.c)


@dataclass
class PointCloudProblem:
    """Squared-Euclidean OT between point sets, cost recomputed on the fly.

    ``C_ij = (sum_k (x_ik - y_jk)^2) / C_max`` with the coordinate sum taken
    left to right and ``C_max`` the exact maximum over all pairs.
    """

    X: np.ndarray
    Y: np.ndarray
    r: np.ndarray
    c: np.ndarray
    label: str = ""
    cmax: float | None = None

    def __post_init__(self):
        self.X = np.ascontiguousarray(self.X, dtype=np.float64)
        self.Y = np.ascontiguousarray(self.Y, dtype=np.float64)
        self.r = np.ascontiguousarray(self.r, dtype=np.float64)
        self.c = np.ascontiguousarray(self.c, dtype=np.float64)
        if self.X.ndim != 2 or self.X.shape != self.Y.shape:
            raise DimensionError(f"point sets must be n-by-d, got {self.X.shape}, {self.Y.shape}")
        if not (np.all(np.isfinite(self.X)) and np.all(np.isfinite(self.Y))):
            raise DomainError("points must be finite")
        _check_marginals(self.X.shape[0], self.r, self.c)

    @property
    def n(self):
        return int(self.X.shape[0])

    @property
    def dim(self):
        return int(self.X.shape[1])

    on_device = False

    def raw_cost_rows(self, lo, hi):
        """Unnormalized squared distances for rows [lo, hi), fixed operand order."""
        acc = None
        for k in range(self.dim):
            d = self.X[lo:hi, k][:, None] - self.Y[None, :, k]
            sq = d * d
            acc = sq if acc is None else acc + sq
        return acc

    def materialize_cost(self):
        """Host dense C with the on-the-fly kernels' exact operand order (small n)."""
        D = self.raw_cost_rows(0, self.n)
        m = self.cmax if self.cmax is not None else D.max()
        if m > 0.0:
            D /= m
        return D


@dataclass
class TraceRow:
    """Per-outer-iteration telemetry row (problems.py:68-84)."""

    t: int
    gamma: float
    eps_d: float
    newton_steps: int
    cg_iters: int
    sinkhorn_steps: int
    linesearch_backtracks: int
    grad_norm_l1: float
    rho_final: float
    delta_min: float
    q: float
    ops_n2: int
    wall_ms: float


# ---------------------------------------------------------------------------
# generators
# ---------------------------------------------------------------------------
def grid_points_cost(n, metric, side=None):
    """Normalized L1 / squared-L2 cost between the first n pixels of a grid.

    Same layout and values as problems.py:87-111 (row-major pixels, integer
    distances, one division by the maximum).
    """
    if n < 1:
        raise DimensionError("need at least one grid point")
    side = int(np.ceil(np.sqrt(n))) if side is None else side
    row, col = np.divmod(np.arange(n), side)
    dr = (row[:, None] - row[None, :]).astype(np.float64)
    dc = (col[:, None] - col[None, :]).astype(np.float64)
    metric = metric.lower()
    if metric == "l1":
        C = np.abs(dr) + np.abs(dc)
    elif metric == "l2sq":
        C = dr * dr + dc * dc
    else:
        raise DomainError(f"unknown metric {metric!r}; use 'l1' or 'l2sq'")
    top = C.max()
    if top > 0.0:
        C /= top
    return C


def gen_grid_cost(side, metric):
    """Cost over a side-by-side pixel grid, n = side^2 (problems.py:114-118)."""
    if side < 1:
        raise DimensionError("grid side must be >= 1")
    return grid_points_cost(side * side, metric, side=side)


def gen_marginal(n, kind, seed):
    """Seeded simplex vector; same PCG64 stream as problems.py:121-144."""
    if n < 1:
        raise DimensionError("marginal length must be >= 1")
    kind = kind.lower()
    if kind == "uniform":
        return np.full(n, 1.0 / n)
    rng = np.random.default_rng(seed)
    if kind == "smooth-random":
        walk = np.cumsum(rng.standard_normal(n)) * 0.25
        w = np.exp(walk - walk.max())
    elif kind == "spiky-random":
        w = np.maximum(rng.exponential(scale=1.0, size=n), 1e-12)
    else:
        raise DomainError(f"unknown marginal kind {kind!r}")
    return w / w.sum()


def grid_problem(side, metric, seed, marginal="smooth-random"):
    """The CLI's grid generator (cli.py:88-98): c uses seed + 1."""
    n = side * side
    return Problem(C=gen_grid_cost(side, metric),
                   r=gen_marginal(n, marginal, seed),
                   c=gen_marginal(n, marginal, seed + COL_SEED_OFFSET),
                   label=f"grid-{metric}-s{side}-{marginal}-seed{seed}")


def uniform_points(n, dim, seed):
    """X, Y ~ U[0,1)^dim from one PCG64 stream (X first)."""
    rng = np.random.default_rng(seed)
    return rng.random((n, dim)), rng.random((n, dim))


def pixel_points(n, dim, seed):
    """MNIST-shaped 8-bit point sets: integer intensities 0..255 as float64.

    Integer coordinates keep every squared distance an exact integer below
    2^53, so the setup GEMM is exact regardless of BLAS summation order and
    the cost matrix is bit-reproducible on any host.
    """
    rng = np.random.default_rng(seed)
    X = rng.integers(0, 256, size=(n, dim)).astype(np.float64)
    Y = rng.integers(0, 256, size=(n, dim)).astype(np.float64)
    return X, Y


def points_problem(n, dim, seed, kind="uniform"):
    X, Y = (uniform_points if kind == "uniform" else pixel_points)(n, dim, seed)
    r = np.full(n, 1.0 / n)
    return PointCloudProblem(X=X, Y=Y, r=r, c=r.copy(), label=f"points{dim}-{kind}-n{n}-seed{seed}")


def pixel_cost_device(X, Y, device=None):
    """The 8-bit point-set cost built on the GPU (K10, problems.py:87-111's
    setup GEMM): ``max(|x|^2 + |y|^2 - 2 X Y^T, 0) / max`` from integer
    intensities 0..255 (host arrays or CUDA tensors, n x d float64), computed
    with exact u8 x u8 -> s32 tensor-core products, so the result equals the
    host evaluation bit for bit (``otn_pixel_cost``).  Returns the n x n
    float64 CUDA tensor (a view of the solver's ld-padded layout, reused by
    the solver without a copy)."""
    import torch

    from ._device import Context, vptr
    device = torch.device(device or "cuda")
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())

    def dev(a):
        t = a if torch.is_tensor(a) else torch.from_numpy(np.ascontiguousarray(a, np.float64))
        return t.to(device=device, dtype=torch.float64).contiguous()
    Xd, Yd = dev(X), dev(Y)
    if Xd.ndim != 2 or Xd.shape != Yd.shape:
        raise DimensionError(f"point sets must be n-by-d, got {tuple(Xd.shape)}, {tuple(Yd.shape)}")
    n, d = int(Xd.shape[0]), int(Xd.shape[1])
    ctx = Context.get(n, device)
    buf = ctx.zeros((n, ctx.ld))
    cmax = ctypes.c_double(0.0)
    ctx.call("otn_pixel_cost", vptr(Xd), vptr(Yd), d, vptr(buf), ctypes.byref(cmax))
    if not cmax.value > 0.0:
        raise DomainError("pixel cost: all point pairs coincide (zero maximum)")
    C = buf[:, :n]
    C._otn_padded = buf                  # the solver's layout (DeviceCost uses it as is)
    return C


def dense_points_problem(n, dim, seed, kind="uniform", device=None):
    """Stored-cost Problem from a point cloud (D1: dim 2, D3: dim 784 pixels).

    device (pixel sets only): build C on that GPU (pixel_cost_device) instead
    of on the host; the two are bit-identical."""
    pc = points_problem(n, dim, seed, kind)
    if device is not None:
        if kind != "pixel":
            raise DomainError("device cost construction is for 8-bit pixel sets")
        return Problem(C=pixel_cost_device(pc.X, pc.Y, device), r=pc.r, c=pc.c, label=pc.label)
    if dim <= 8:
        C = pc.materialize_cost()
    else:
        sx = (pc.X * pc.X).sum(axis=1)
        sy = (pc.Y * pc.Y).sum(axis=1)
        C = sx[:, None] + sy[None, :] - 2.0 * (pc.X @ pc.Y.T)   # exact integers
        np.maximum(C, 0.0, out=C)
        C /= C.max()
    return Problem(C=C, r=pc.r, c=pc.c, label=pc.label)


def workload(spec, device=None):
    """Problem from a compact spec string (used by tests, bench and fixtures).

    ``grid:<side>:<l1|l2sq>:<seed>``  |  ``pts:<n>:<dim>:<seed>`` (uniform,
    stored C)  |  ``pix:<n>:<dim>:<seed>`` (8-bit points, stored C)  |
    ``otf:<n>:<dim>:<seed>`` (uniform points, on-the-fly PointCloudProblem).
    device: build a ``pix`` cost on that GPU (pixel_cost_device).
    """
    kind, *rest = spec.split(":")
    if kind not in ("grid", "pts", "pix", "otf") or len(rest) != 3:
        raise DomainError(f"unknown workload spec {spec!r}")
    try:
        if kind == "grid":
            side, metric, seed = int(rest[0]), rest[1], int(rest[2])
            return grid_problem(side, metric, seed)
        n, dim, seed = int(rest[0]), int(rest[1]), int(rest[2])
    except ValueError as exc:
        raise DomainError(f"bad workload spec {spec!r}: {exc}") from exc
    if kind == "pts":
        return dense_points_problem(n, dim, seed, "uniform")
    if kind == "pix":
        return dense_points_problem(n, dim, seed, "pixel", device=device)
    if kind == "otf":
        return points_problem(n, dim, seed, "uniform")
    raise DomainError(f"unknown workload spec {spec!r}")


# ---------------------------------------------------------------------------
# file formats (problems.py:151-231)
# ---------------------------------------------------------------------------
def _fmt(x):
    return format(float(x), ".17g")


def save_problem(problem, path):
    """Plain-text ``OTP`` format, 17 significant digits (problems.py:151-158)."""
    C = problem.C
    if _is_device_tensor(C):
        C = C.cpu().numpy()
    out = [f"OTP {problem.n}", " ".join(map(_fmt, problem.r)), " ".join(map(_fmt, problem.c))]
    out.extend(" ".join(map(_fmt, row)) for row in C)
    with open(path, "w") as fh:
        fh.write("\n".join(out) + "\n")


def _floats(text, n, lineno, what):
    parts = text.split()
    if len(parts) != n:
        raise ParseError(f"line {lineno}: expected {n} values for {what}, got {len(parts)}")
    try:
        return np.array([float(t) for t in parts])
    except ValueError as exc:
        raise ParseError(f"line {lineno}: bad float in {what}: {exc}") from exc


def load_problem(path):
    """Inverse of save_problem, renormalizing within 1e-9 (problems.py:170-206)."""
    with open(path) as fh:
        lines = [ln.rstrip("\n") for ln in fh if ln.strip() != ""]
    if not lines:
        raise ParseError("line 1: empty problem file")
    head = lines[0].split()
    if len(head) != 2 or head[0] != "OTP":
        raise ParseError(f"line 1: expected header 'OTP n', got {lines[0]!r}")
    try:
        n = int(head[1])
    except ValueError as exc:
        raise ParseError(f"line 1: bad dimension {head[1]!r}") from exc
    if n < 1:
        raise ParseError("line 1: dimension must be >= 1")
    if len(lines) != 3 + n:
        raise ParseError(f"line {len(lines)}: expected {3 + n} lines for n={n}, got {len(lines)}")
    r = _floats(lines[1], n, 2, "row marginal")
    c = _floats(lines[2], n, 3, "column marginal")
    C = np.vstack([_floats(lines[3 + i], n, 4 + i, f"cost row {i}") for i in range(n)])
    for lineno, name, m in ((2, "row marginal", r), (3, "column marginal", c)):
        s = m.sum()
        if abs(s - 1.0) > PARSE_SIMPLEX_TOL:
            raise ParseError(f"line {lineno}: {name} sums to {s:.17g}, outside tolerance")
        if abs(s - 1.0) > SIMPLEX_TOL:
            m /= s
    return Problem(C=C, r=r, c=c, label=str(path))


def write_trace(rows, path):
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(TRACE_HEADER)
        for row in rows:
            w.writerow([getattr(row, k) for k in TRACE_HEADER])


def read_trace(path):
    kinds = {f.name: f.type for f in fields(TraceRow)}
    rows = []
    with open(path, newline="") as fh:
        rd = csv.DictReader(fh)
        if rd.fieldnames != TRACE_HEADER:
            raise ParseError(f"line 1: unexpected trace header {rd.fieldnames}")
        for rec in rd:
            rows.append(TraceRow(**{k: (int(rec[k]) if kinds[k] == "int" else float(rec[k]))
                                    for k in TRACE_HEADER}))
    return rows
