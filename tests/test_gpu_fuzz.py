"""Randomised parity sweep (tools/fuzz_parity.py): small scans with random
detector sizes, scan rasters, pixel-map laws, masks, bad frames, ROIs, frame
weights and search windows (fast-path, one-row and generic kernels, sub-pixel
grids), each through make_reference -> update_pixel_map -> update_translations
-> calc_error against the CPU oracle at the BASELINE bars.  The 600-case run
is recorded in profiles/fuzz_r02.txt; the suite keeps a fixed subset."""

from __future__ import annotations

import os
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import fuzz_loop  # noqa: E402
import fuzz_parity  # noqa: E402


@pytest.mark.parametrize("block", range(6))
def test_random_cases_vs_oracle(block):
    for seed in range(8 * block, 8 * block + 8):
        fuzz_parity.one(seed)          # raises on the first bar that fails


@pytest.mark.parametrize("block", range(4))
def test_hard_random_cases_vs_oracle(block):
    """Seeds >= 1000: dead whitefield blocks, the reference formed on a smaller
    rectangle than the one searched (invalid cells, samples off the grid, exact
    ties), 15x15 / 17x17 / 1x17 / 17x1 windows."""
    for seed in range(1000 + 8 * block, 1000 + 8 * block + 8):
        fuzz_parity.one(seed)


@pytest.mark.parametrize("block", range(3))
def test_random_main_loops_vs_oracle(block):
    """tools/fuzz_loop.py: run_main_loop over random schedules against the
    oracle's loop, half of the cases also over two shares of the device."""
    for seed in range(6 * block, 6 * block + 6):
        fuzz_loop.one(seed)
