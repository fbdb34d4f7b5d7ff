"""CLI host logic (no GPU): problem generation, argument defaults and
overrides, config round trip, exit codes, sweep summary statistics, and the
exact small-problem optimum used for gaps (reference tests/test_cli.py,
tests/test_oracles.py:44-56)."""
import json

import numpy as np
import pytest

from paper_2504_02067_b200.cli import BenchConfig, _exact_cost, _summary_rows, build_parser, main
from paper_2504_02067_b200.problems import load_problem


def test_gen_writes_valid_problem(tmp_path, capsys):
    out = tmp_path / "p.otp"
    assert main(["gen", "--kind", "grid", "--metric", "l1", "--side", "8", "--marginal",
                 "smooth-random", "--seed", "1", "--out", str(out)]) == 0
    assert load_problem(out).n == 64
    assert "n=64" in capsys.readouterr().out


def test_gen_degenerate_side_one(tmp_path):
    out = tmp_path / "p1.otp"
    assert main(["gen", "--side", "1", "--out", str(out)]) == 0
    assert load_problem(out).n == 1


def test_gen_byte_identical(tmp_path):
    args = ["gen", "--side", "4", "--marginal", "spiky-random", "--seed", "9"]
    main(args + ["--out", str(tmp_path / "a.otp")])
    main(args + ["--out", str(tmp_path / "b.otp")])
    assert (tmp_path / "a.otp").read_bytes() == (tmp_path / "b.otp").read_bytes()


def test_missing_inputs_are_io_errors(tmp_path):
    assert main(["solve", "--problem", str(tmp_path / "nope.otp")]) == 3
    assert main(["bench", "--config", str(tmp_path / "nope.json")]) == 3
    assert not list(tmp_path.iterdir())


def test_defaults_match_the_benchmark_setup():
    a = build_parser().parse_args(["solve", "--problem", "x.otp"])
    assert (a.gamma_init, a.gamma_final, a.p, a.q_init, a.adaptive_q) == (
        2.0 ** 5, 2.0 ** 18, 1.5, 2.0, True)


def test_bench_config_round_trip_and_flags():
    cfg = BenchConfig.from_dict({"problems": [{"kind": "grid", "side": 4}],
                                 "settings": [{"name": "a", "gamma_f": 1024.0, "q_init": 1.5}],
                                 "seeds": [3, 4], "repeats": 2, "output_dir": "x"})
    assert BenchConfig.from_dict(json.loads(json.dumps(cfg.to_dict()))) == cfg
    flat = BenchConfig.from_dict({"problems": [], "gamma_f": 4096.0})
    assert flat.settings[0].name == "default" and flat.settings[0].gamma_f == 4096.0
    a = build_parser().parse_args(["bench", "--config", "c.json", "--gamma-final", "256",
                                   "--seeds", "5,6", "--no-adaptive-q"])
    assert (a.gamma_f, a.seeds, a.adaptive_q) == (256.0, "5,6", False)


def test_summary_medians_are_order_statistics():
    runs = [{"setting": "s", "label": "L", "ok": True, "wall_ms": w, "ops_total": o,
             "ops": {"newton_solve": o - 1}, "gap": g, "gap_basis": "exact"}
            for w, o, g in ((3.0, 30, 1e-3), (1.0, 10, 3e-3), (2.0, 20, 2e-3))]
    runs.append({"setting": "s", "label": "L", "ok": False, "error": "x"})
    head, row = _summary_rows(runs)
    cols = dict(zip(head.split(","), row.split(",")))
    assert cols["runs"] == "4" and cols["failures"] == "1"
    assert float(cols["wall_ms_med"]) == 2.0 and float(cols["ops_med"]) == 20.0
    assert float(cols["ops_newton_solve_med"]) == 19.0
    assert cols["gap_basis"] == "exact"


def test_exact_cost_known_answers():
    C = np.array([[0.0, 1.0], [1.0, 0.0]])
    assert _exact_cost(C, np.array([0.5, 0.5]), np.array([0.5, 0.5])) == pytest.approx(0.0, abs=1e-12)
    assert _exact_cost(C, np.array([0.7, 0.3]), np.array([0.4, 0.6])) == pytest.approx(0.3, rel=1e-9)
    rng = np.random.default_rng(12345)            # test_oracles.py:49-56 frozen fixture
    C = rng.random((3, 3))
    r = rng.dirichlet(np.ones(3))
    c = rng.dirichlet(np.ones(3))
    assert _exact_cost(C, r, c) == pytest.approx(0.49308641326299063, rel=1e-9)
