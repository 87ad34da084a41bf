"""Host-side grid rule of make_reference (engine.DeviceScan.host_bbox) against
the oracle's bbox (recon.py:126-132), including extrema on non-work pixels
and non-finite inputs (no GPU needed: the method only reads host arrays)."""
import numpy as np
import pytest

from oracle import pxst_oracle as orc
from paper_2003_12726_b200 import engine
from paper_2003_12726_b200.synth import make_scan


class _Scan:   # the two attributes host_bbox reads
    def __init__(self, s):
        self._work_host = s.m.mask & (s.w.w > 0)
        self.good_idx = np.flatnonzero(s.scan.good_frames)


def _oracle(s, u, di, dj):
    good, rows, cols, *_ = orc.work_set(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask, None)
    return orc.object_bbox(u[0][rows, cols], u[1][rows, cols], di[good], dj[good])


@pytest.mark.parametrize("cfg", [0, 1])
def test_host_bbox_matches_oracle(cfg):
    s = make_scan(cfg)
    d = _Scan(s)
    assert engine.DeviceScan.host_bbox(d, s.u0.u, s.t0.di, s.t0.dj) == \
        _oracle(s, s.u0.u, s.t0.di, s.t0.dj)


def test_host_bbox_extrema_off_the_work_set():
    s = make_scan(0)
    d = _Scan(s)
    u = s.u0.u.copy()
    off = np.flatnonzero(~d._work_host.ravel())
    u[0].ravel()[off[0]] = -1e6          # global extrema on pixels outside the work set
    u[1].ravel()[off[-1]] = 1e6
    di = s.t0.di.copy()
    bad = np.flatnonzero(~np.asarray(s.scan.good_frames, bool))
    if bad.size:
        di[bad[0]] = 1e6                 # and on a frame outside the good set
    assert engine.DeviceScan.host_bbox(d, u, di, s.t0.dj) == _oracle(s, u, di, s.t0.dj)


def test_host_bbox_non_finite_defers_to_device():
    s = make_scan(0)
    d = _Scan(s)
    u = s.u0.u.copy()
    u[0][d._work_host] = np.nan
    assert engine.DeviceScan.host_bbox(d, u, s.t0.di, s.t0.dj) is None
