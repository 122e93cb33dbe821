"""Test configuration.

`-m "not gpu"` (CPU, this container): oracle vs golden vectors and the reference,
host logic, C-ABI loading/exports, multi-process (gloo) sharding logic.
`-m gpu` (a B200): parity of every CUDA kernel against the oracle, through the
C-ABI and through the reference's own HostKernel API (drop-in tests).
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np

    d = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(d, "golden.json")) as f:
        meta = json.load(f)
    arrays = dict(np.load(os.path.join(d, "golden.npz")))
    return meta, arrays


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a visible CUDA device")
    return torch.device("cuda:0")


@pytest.fixture
def option():
    """Sets libtir_b200 planner switches (tir_b200_set_option) for one test and
    restores them afterwards."""
    import paper_2207_04296_b200 as tb

    saved = {}

    def set_(name, value):
        if name not in saved:
            saved[name] = tb.get_option(name)
        tb.set_option(name, value)

    yield set_
    for k, v in saved.items():
        tb.set_option(k, v)
