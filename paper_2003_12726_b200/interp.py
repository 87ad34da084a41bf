"""Drop-in of ``pxst.interp`` (interp.py:21-135) backed by the GPU primitives.

``gather`` (masked bilinear read) and ``scatter_accumulate`` (bilinear
splat) run the same device code the hot-path kernels inline
(``pxst_gather`` / ``pxst_splat``); ``normalize`` is the elementwise
ratio.  Arrays in and out are float64 numpy, as in the reference.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .engine import DeviceRef, to_device


@dataclass
class WeightedAccumulator:
    """Value and weight planes (interp.py:21-30)."""

    values: np.ndarray
    weights: np.ndarray

    @classmethod
    def zeros(cls, shape) -> "WeightedAccumulator":
        return cls(np.zeros(shape, dtype=np.float64), np.zeros(shape, dtype=np.float64))


def _dev():
    _native.lib()
    return torch.device("cuda", torch.cuda.current_device())


def gather(f: np.ndarray, m: np.ndarray, x, y):
    """Masked bilinear read of ``f`` at ``(x, y)`` (interp.py:53-85).

    Values are computed in float32 on the device (the hot path's
    precision) and returned as float64.
    """
    dev = _dev()
    f = np.asarray(f)
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    x, y = np.broadcast_arrays(x, y)
    shape = x.shape
    ref = DeviceRef.from_host(f, np.asarray(m).astype(np.float64), (0, 0), dev)
    xd = to_device(x.ravel(), np.float64, dev)
    yd = to_device(y.ravel(), np.float64, dev)
    n = xd.numel()
    vals = torch.empty(n, dtype=torch.float64, device=dev)
    ok = torch.empty(n, dtype=torch.uint8, device=dev)
    lib = _native.lib()
    c_ref = ref.struct()
    _native.check(lib.pxst_gather(ctypes.byref(c_ref), xd.data_ptr(), yd.data_ptr(), n,
                                  vals.data_ptr(), ok.data_ptr(), _native.stream_ptr()))
    return vals.cpu().numpy().reshape(shape), ok.cpu().numpy().astype(bool).reshape(shape)


def scatter_accumulate(acc: WeightedAccumulator, x, y, value, weight=1.0) -> int:
    """Bilinear scatter of ``value*weight`` into ``acc`` (interp.py:88-123).

    Accumulates in float64 on the device; returns the number of dropped
    (out-of-grid) points.
    """
    dev = _dev()
    x = np.atleast_1d(np.asarray(x, dtype=np.float64)).ravel()
    y = np.atleast_1d(np.asarray(y, dtype=np.float64)).ravel()
    value = np.broadcast_to(np.asarray(value, dtype=np.float64), x.shape).ravel()
    weight = np.broadcast_to(np.asarray(weight, dtype=np.float64), x.shape).ravel()
    os_, of = acc.values.shape
    av = to_device(acc.values, np.float64, dev)
    aw = to_device(acc.weights, np.float64, dev)
    xd, yd = to_device(x, np.float64, dev), to_device(y, np.float64, dev)
    vd, wd = to_device(value, np.float64, dev), to_device(weight, np.float64, dev)
    dropped = ctypes.c_int64(0)
    lib = _native.lib()
    _native.check(lib.pxst_splat(av.data_ptr(), aw.data_ptr(), os_, of, xd.data_ptr(),
                                 yd.data_ptr(), vd.data_ptr(), wd.data_ptr(), x.size,
                                 ctypes.byref(dropped), _native.stream_ptr()))
    acc.values[...] = av.cpu().numpy()
    acc.weights[...] = aw.cpu().numpy()
    return int(dropped.value)


def normalize(acc: WeightedAccumulator):
    """``values / weights`` where ``weights > 0`` (interp.py:126-135)."""
    valid = acc.weights > 0
    out = np.zeros_like(acc.values)
    np.divide(acc.values, acc.weights, out=out, where=valid)
    return out, valid
