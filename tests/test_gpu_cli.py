"""CLI end to end on the GPU (reference tests/test_cli.py:39-139)."""
import json

import pytest

from paper_2504_02067_b200.cli import main
from paper_2504_02067_b200.problems import read_trace

pytestmark = pytest.mark.gpu


def _fixture(tmp_path):
    path = tmp_path / "sym.otp"
    path.write_text("OTP 2\n0.5 0.5\n0.5 0.5\n0 1\n1 0\n")
    return path


def test_solve_within_bound(tmp_path, capsys):
    rep, tr = tmp_path / "report.json", tmp_path / "trace.csv"
    assert main(["solve", "--problem", str(_fixture(tmp_path)), "--gamma-init", "32",
                 "--gamma-final", str(2.0 ** 14), "--report", str(rep), "--trace", str(tr)]) == 0
    report = json.loads(rep.read_text())
    assert report["primal_cost_rounded"] <= report["error_bound"]   # exact optimum is 0
    assert read_trace(tr)[0].t == 1
    assert json.loads(capsys.readouterr().out)["n"] == 2


def test_single_temperature_sinkhorn(tmp_path):
    assert main(["solve", "--problem", str(_fixture(tmp_path)), "--solver", "mdot-sinkhorn",
                 "--gamma-init", "64", "--gamma-final", "64"]) == 0


def test_sweep_outputs(tmp_path):
    cfg = {"problems": [{"kind": "grid", "metric": "l1", "side": 2, "seed": 1},
                        {"kind": "grid", "metric": "l1", "side": 2, "seed": 2},
                        {"kind": "grid", "metric": "l2sq", "side": 2, "seed": 3}],
           "settings": [{"name": "adaptive", "gamma_i": 16, "gamma_f": 1024, "q_init": 2.0,
                         "adaptive_q": True},
                        {"name": "fixed-sqrt2", "gamma_i": 16, "gamma_f": 1024,
                         "q_init": 1.41421356, "adaptive_q": False}],
           "seeds": [0], "output_dir": str(tmp_path / "out")}
    (tmp_path / "bench.json").write_text(json.dumps(cfg))
    assert main(["bench", "--config", str(tmp_path / "bench.json")]) == 0
    out = tmp_path / "out"
    assert len(list(out.glob("*.json"))) == 6
    assert len(list(out.glob("*.csv"))) == 7               # 6 traces + summary.csv
    summary = (out / "summary.csv").read_text().strip().split("\n")
    assert summary[0].startswith("setting,label,runs,failures") and len(summary) == 7
    assert all(line.endswith("exact") for line in summary[1:])
    for line in summary[1:]:                               # rounded cost >= the optimum
        cols = dict(zip(summary[0].split(","), line.split(",")))
        assert float(cols["gap_med"]) >= -1e-9


def test_summary_ops_median_is_an_order_statistic(tmp_path):
    cfg = {"problems": [{"kind": "grid", "metric": "l1", "side": 2, "seed": 5}],
           "settings": [{"name": "s", "gamma_i": 16, "gamma_f": 256}], "seeds": [0, 1, 2],
           "output_dir": str(tmp_path / "out")}
    (tmp_path / "bench.json").write_text(json.dumps(cfg))
    assert main(["bench", "--config", str(tmp_path / "bench.json")]) == 0
    out = tmp_path / "out"
    ops = sorted(json.loads(p.read_text())["ops"]["total"] for p in out.glob("*.json"))
    head, row = (out / "summary.csv").read_text().strip().split("\n")
    assert float(dict(zip(head.split(","), row.split(",")))["ops_med"]) == ops[1]
