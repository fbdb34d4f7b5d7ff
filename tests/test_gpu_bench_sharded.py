"""bench.py's multi-rank path (N > 1: the row-sharded on-the-fly solve) end
to end on this one-GPU box: two ranks launched by torch.distributed.run, both
on cuda:0 with the gloo backend (BENCH_DIST_BACKEND=gloo, BENCH_DEVICE=0; a
real run uses one rank per GPU on NCCL).  Checks the JSON line's contract
fields and that the sharded solve reaches the same precision as one rank."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_sharded_d4():
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo", BENCH_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "1",
           "--d4-n", "8192"]
    out = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["scaling"] == "strong"
    assert rec["config"]["parallelism"] == "rows2" and rec["config"]["n"] == 8192
    assert rec["value"] > 0 and rec["e2e"]["value"] > 0
    solve, one = rec["solve"], rec["extras"]["d4_1gpu"]
    assert solve["gpus"] == 2 and one["gpus"] == 1
    assert solve["stages"] == one["stages"] and solve["cg"] == one["cg"]
    assert solve["primal"] == pytest.approx(one["primal"], rel=1e-9)
    assert solve["true_marginal_err"] == pytest.approx(one["true_marginal_err"], rel=1e-6)
    col = solve["collectives"]
    # one allreduce per column-direction product (+ the first column LSE and
    # the rounding's column sums)
    fb = col.get("lse_shift_fallbacks", 0)
    assert col["vector_allreduces"] == col["column_products"] + 2 + 2 * fb
    assert "d2_replicas" in rec["extras"]
