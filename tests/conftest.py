"""Shared fixtures.  ``-m gpu`` tests need a CUDA device (B200); the rest run on CPU."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden0():
    return dict(np.load(os.path.join(GOLDEN, "cfg0.npz")))


@pytest.fixture(scope="session")
def golden1():
    return dict(np.load(os.path.join(GOLDEN, "cfg1.npz")))


@pytest.fixture(scope="session")
def scan0():
    from paper_2003_12726_b200.synth import make_scan
    return make_scan(0)


@pytest.fixture(scope="session")
def scan1():
    from paper_2003_12726_b200.synth import make_scan
    return make_scan(1)
