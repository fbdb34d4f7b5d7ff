"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports
every symbol include/otn_b200.h declares; input generators reproduce the
reference's inputs (sha256 of the golden fixtures); host-side schedule logic
matches the reference's known values.  No compute call needs a GPU here."""

import ctypes
import hashlib
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_traj, traj_names
from paper_2504_02067_b200 import _lib, driver, problems, projector
from paper_2504_02067_b200.errors import DeviceError, DomainError

HEADER = os.path.join(ROOT, "include", "otn_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(otn_\w+)\s*\(", text, re.M)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.exported_symbols())


def test_library_loads_and_exports_every_symbol():
    assert os.path.exists(_lib.LIB_PATH), "build the library first (make -C paper_2504_02067_b200/csrc)"
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert _lib.load().otn_abi_version() == _lib.ABI_VERSION == 2


def test_no_cpu_fallback_without_device():
    """Without a GPU every solver entry point fails loudly (no silent CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2504_02067_b200 as ot
    prob = problems.workload("grid:4:l1:0")
    with pytest.raises(DeviceError):
        ot.mdot(prob, 16.0, 64.0)
    with pytest.raises(DeviceError):
        ot.DualState(prob, 4.0)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.mark.parametrize("name", [n for n in traj_names() if not n.startswith("D3")])
def test_generators_reproduce_reference_inputs(name):
    meta, _ = load_traj(name)
    p = problems.workload(meta["spec"])
    assert sha(p.C) == meta["sha_C"]
    assert sha(p.r) == meta["sha_r"]
    assert sha(p.c) == meta["sha_c"]


def test_schedule_rules_match_reference_values():
    u = np.full(4096, 1.0 / 4096)
    assert driver.eps_rule(2.0 ** 5, 1.5, u, u) == pytest.approx(0.045949, rel=1e-4)
    assert driver.error_bound(2.0 ** 18, u, u) == pytest.approx(6.3459e-5, rel=1e-4)
    r, _ = driver.smooth_marginals(np.array([1.0, 0.0]), np.array([0.5, 0.5]), 0.1)
    np.testing.assert_allclose(r, [0.9775, 0.0225], rtol=1e-14)
    assert driver.adjust_schedule(2.0, 0.97) == 2.0
    assert driver.adjust_schedule(1.2, float("inf")) == pytest.approx(1.44)
    assert driver.adjust_schedule(1.3, 0.85) == 1.3
    np.testing.assert_allclose(driver.extrapolate(np.array([1.0]), np.array([0.0]), 8.0, 4.0, 2.0),
                               [3.0])
    with pytest.raises(DomainError):
        driver.extrapolate(np.zeros(2), np.zeros(2), 8.0, 4.0, 4.0)
    with pytest.raises(DomainError):
        driver.smooth_marginals(r, r, 0.1, w_r=0.3, w_c=0.3)


def test_projector_scalar_rules():
    assert projector.eta_rule(0.1, 1e-3) == pytest.approx(0.1)
    assert projector.eta_rule(0.002, 1e-3) == pytest.approx(0.4)
    assert projector.eta_rule(2.0, 1e-3) == pytest.approx(0.99)
    assert projector.delta_ratio(0.1, 0.01, 0.1) == pytest.approx(1.0)
    assert projector.armijo_accept(1.0, 1.005, np.array([-0.01]), np.array([1.0]))
    assert not projector.armijo_accept(1.0, 1.0101, np.array([-0.01]), np.array([1.0]))
    with pytest.raises(DomainError):
        projector.delta_ratio(0.1, 0.0, 1.0)


def test_otp_round_trip(tmp_path):
    p = problems.workload("grid:4:l2sq:3")
    path = tmp_path / "p.otp"
    problems.save_problem(p, path)
    q = problems.load_problem(path)
    np.testing.assert_array_equal(q.C, p.C)
    np.testing.assert_array_equal(q.r, p.r)


def test_point_cloud_cost_matches_stored_cost():
    pc = problems.points_problem(64, 3, 0)
    dense = problems.dense_points_problem(64, 3, 0)
    np.testing.assert_array_equal(pc.materialize_cost(), dense.C)


def test_seam_binding_declares_header_symbols():
    """integration/otnewton_b200.py (the executable INTEGRATION.md §2 binding)
    declares only entry points of include/otn_b200.h, with the same argument
    counts as the package's own binding."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "otnewton_b200", os.path.join(ROOT, "integration", "otnewton_b200.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    declared = set(declared_symbols())
    for name, (args, _) in mod._SIGS.items():
        assert name in declared, name
        assert len(args) == len(_lib.SIGNATURES[name]), name
