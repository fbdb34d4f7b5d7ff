"""K10 on the tensor cores: the 8-bit point-set cost (problems.py:87-111's
setup GEMM for the 784-d pixel sets of BASELINE's D3) built on the GPU with
exact u8 x u8 -> s32 MMAs equals the host's float64 evaluation bit for bit,
so a solve on it is the solve on the host-built cost."""

import numpy as np
import pytest

from conftest import load_traj
from paper_2504_02067_b200 import mdot, problems
from paper_2504_02067_b200.errors import DomainError

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,d,seed", [(256, 784, 0), (1000, 784, 3), (300, 100, 1),
                                      (4096, 784, 0), (33, 7, 2)])
def test_device_cost_is_bitwise_the_host_cost(n, d, seed):
    import torch
    host = problems.dense_points_problem(n, d, seed, "pixel") if d > 8 else None
    X, Y = problems.pixel_points(n, d, seed)
    if host is None:                                  # d <= 8: the same GEMM formula on the host
        sx, sy = (X * X).sum(axis=1), (Y * Y).sum(axis=1)
        C = np.maximum(sx[:, None] + sy[None, :] - 2.0 * (X @ Y.T), 0.0)
        want = C / C.max()
    else:
        want = host.C
    got = problems.pixel_cost_device(X, Y, "cuda")
    assert got.shape == (n, n)
    g = got.cpu().numpy()
    assert np.array_equal(g, want), float(np.abs(g - want).max())
    pad = got._otn_padded
    assert pad.shape[1] % 32 == 0
    assert float(pad[:, n:].abs().max().item() if pad.shape[1] > n else 0.0) == 0.0
    # device tensors as input give the same bits
    g2 = problems.pixel_cost_device(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda())
    assert torch.equal(g2, got)


def test_rejects_non_pixel_input():
    X, Y = problems.pixel_points(64, 50, 0)
    X[3, 7] = 12.5
    with pytest.raises(Exception, match="integer in"):
        problems.pixel_cost_device(X, Y)
    X[3, 7] = 256.0
    with pytest.raises(Exception, match="integer in"):
        problems.pixel_cost_device(X, Y)
    with pytest.raises(DomainError):
        problems.pixel_cost_device(np.zeros((8, 4)), np.zeros((8, 4)))


def test_solve_on_device_built_cost_matches_reference_trajectory():
    """pix256_784_s0 golden (the reference's own trajectory) through the
    device-built cost: the strict gate's discrete trajectory and potentials."""
    meta, arr = load_traj("pix256_784_s0")
    prob = problems.workload(meta["spec"], device="cuda")
    assert prob.on_device
    sol = mdot(prob, meta["gamma_i"], meta["gamma_f"])
    assert [it.stats.cg_iters for it in sol.iterations] == [s["cg_iters"] for s in meta["stages"]]
    du = np.abs(sol.final_state.u - arr["u"]).max() / np.abs(arr["u"]).max()
    assert du <= max(1e-10, 100 * meta["self_spread"]["du"])
    assert sol.primal_cost == pytest.approx(meta["primal"], rel=1e-9)
