"""Shared fixtures.  Tests marked ``gpu`` need a B200 (run with ``-m gpu``);
everything else runs on CPU (``-m "not gpu"``)."""

import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_traj(name):
    """Golden reference trajectory (tests/golden/make_golden.py)."""
    z = np.load(os.path.join(GOLDEN, f"traj_{name}.npz"), allow_pickle=False)
    meta = json.loads(str(z["meta"]))
    arrays = {k: z[k] for k in z.files if k != "meta"}
    return meta, arrays


def traj_names():
    return sorted(os.path.basename(p)[5:-4] for p in glob.glob(os.path.join(GOLDEN, "traj_*.npz")))


def load_kernels():
    z = np.load(os.path.join(GOLDEN, "kernels.npz"))
    return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def kernels_golden():
    return load_kernels()
