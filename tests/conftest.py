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


@pytest.fixture(scope="session")
def golden_reg():
    return dict(np.load(os.path.join(GOLDEN, "reg0.npz")))


def default_schedule_dicts(n):
    """recon.default_schedule(n) as the oracle's schedule dicts (recon.py:451-468)."""
    sig = [5.0, 3.0] + [1.0] * max(0, n - 2)
    return [dict(half_ss=4 if i == 0 else 2, half_fs=4 if i == 0 else 2, subpixel_grid=None,
                 quadratic_refinement=True, sigma=sig[i], integrate=True,
                 update_translations=i >= 1, t_half_ss=2, t_half_fs=2, t_subpixel_grid=None)
            for i in range(n)]
