"""ctypes binding of ``libpxst_b200.so`` (the C ABI in ``include/pxst_b200.h``).

This is the only door to the GPU kernels.  There is no CPU fallback: if the
library is missing or no CUDA device is present, :func:`lib` raises.
Status codes map to exceptions as the reference's errors do: PXST_EINVAL ->
``ValueError`` (bad window, empty work set, ...), everything else ->
``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_char_p, c_double, c_int, c_int64, c_uint8, c_uint64, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PXST_LIB", os.path.join(HERE, "libpxst_b200.so"))
ABI_VERSION = 2

PXST_OK, PXST_EINVAL, PXST_ECUDA, PXST_ENOMEM = 0, 1, 2, 3


class PxstScan(ctypes.Structure):
    _fields_ = [("frames", c_void_p), ("n_frames", c_int64), ("ss", c_int64), ("fs", c_int64),
                ("good", c_void_p), ("n_good", c_int64), ("w64", c_void_p), ("w32", c_void_p),
                ("work", c_void_p), ("roi", c_int64 * 4)]


class PxstStats(ctypes.Structure):
    _fields_ = [("var_pm", c_void_p), ("sigma2", c_void_p), ("frame_norm", c_void_p),
                ("scalars", c_void_p)]


class PxstRef(ctypes.Structure):
    _fields_ = [("fm", c_void_p), ("valid", c_void_p), ("os", c_int64), ("of", c_int64),
                ("n0", c_int64), ("m0", c_int64), ("fm64", c_void_p)]


class PxstAccum(ctypes.Structure):
    _fields_ = [("num", c_void_p), ("den", c_void_p), ("num_fine", c_void_p),
                ("den_fine", c_void_p), ("touched", c_void_p), ("quanta", c_void_p)]


class PxstCgInfo(ctypes.Structure):
    _fields_ = [("iterations", c_int64), ("residual", c_double), ("converged", c_int)]


_SIGS = {
    "pxst_abi_version": (c_int, []),
    "pxst_last_error": (c_char_p, []),
    "pxst_launch_count": (c_int64, []),
    "pxst_release_pool": (c_int, []),
    "pxst_stack_stats": (c_int, [POINTER(PxstScan), c_void_p, POINTER(PxstStats), c_void_p]),
    "pxst_stack_stats_parts": (c_int, [POINTER(PxstScan), c_void_p, POINTER(PxstStats), c_int,
                                       c_void_p]),
    "pxst_bbox": (c_int, [POINTER(PxstScan), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pxst_bbox_grid": (c_int, [POINTER(PxstScan), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                               c_void_p]),
    "pxst_accum_zero": (c_int, [POINTER(PxstAccum), c_int64, c_void_p]),
    "pxst_add_i64": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "pxst_add_f64": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "pxst_or_u8": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "pxst_stack_absmax": (c_int, [POINTER(PxstScan), c_void_p, c_void_p]),
    "pxst_object_quanta": (c_int, [POINTER(PxstScan), c_void_p, c_void_p, c_void_p]),
    "pxst_plane_quanta": (c_int, [POINTER(PxstScan), c_void_p, POINTER(PxstStats),
                                  POINTER(PxstRef), c_void_p, c_void_p]),
    "pxst_object_splat": (c_int, [POINTER(PxstScan), c_void_p, c_void_p, c_void_p, c_int64,
                                  c_int64, c_int64, c_int64, c_int64, c_int64,
                                  POINTER(PxstAccum), c_void_p, c_void_p]),
    "pxst_object_finish_peers": (c_int, [POINTER(PxstAccum), c_int, c_int64, c_int64, c_void_p,
                                         c_void_p, c_void_p, c_void_p, c_void_p]),
    "pxst_object_finish": (c_int, [POINTER(PxstAccum), c_int64, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p]),
    "pxst_object_map": (c_int, [POINTER(PxstScan), c_void_p, c_void_p, c_void_p, c_int64,
                                c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_void_p]),
    "pxst_pixel_map_search": (c_int, [POINTER(PxstScan), POINTER(PxstStats), POINTER(PxstRef),
                                      c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_double,
                                      c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pxst_pixel_map_search_ex": (c_int, [POINTER(PxstScan), POINTER(PxstStats),
                                         POINTER(PxstRef), c_void_p, c_void_p, c_void_p, c_int64,
                                         c_int64, c_double, c_int, c_void_p, c_void_p, c_void_p,
                                         c_void_p, c_void_p, c_void_p]),
    "pxst_tile_spans": (c_int, [POINTER(PxstScan), c_void_p, c_void_p, c_void_p]),
    "pxst_translation_search": (c_int, [POINTER(PxstScan), POINTER(PxstStats), POINTER(PxstRef),
                                        c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                                        c_double, c_int64, c_int64, c_void_p, c_void_p,
                                        c_void_p, c_void_p]),
    "pxst_translation_search_ex": (c_int, [POINTER(PxstScan), POINTER(PxstStats),
                                           POINTER(PxstRef), c_void_p, c_void_p, c_void_p,
                                           c_int64, c_int64, c_double, c_int64, c_int64,
                                           c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pxst_tile_spans3": (c_int, [POINTER(PxstScan), c_void_p, c_void_p, c_void_p]),
    "pxst_error_maps": (c_int, [POINTER(PxstScan), POINTER(PxstStats), POINTER(PxstRef),
                                c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_void_p, c_void_p]),
    "pxst_error_maps_splat": (c_int, [POINTER(PxstScan), POINTER(PxstStats), POINTER(PxstRef),
                                      c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_int64, POINTER(PxstAccum),
                                      c_void_p]),
    "pxst_masked_moments": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "pxst_stack_to_f32": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_void_p]),
    "pxst_grid_rule": (c_int, [c_void_p, c_void_p, c_void_p]),
    "pxst_error_partials": (c_int, [POINTER(PxstScan), POINTER(PxstStats), POINTER(PxstRef),
                                    c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                    POINTER(PxstAccum), c_void_p]),
    "pxst_gather": (c_int, [POINTER(PxstRef), c_void_p, c_void_p, c_int64, c_void_p, c_void_p,
                            c_void_p]),
    "pxst_splat": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                           c_void_p, c_int64, POINTER(c_int64), c_void_p]),
    "pxst_smooth_displacement": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_double,
                                         c_void_p]),
    "pxst_integrate_gradient": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_double,
                                        c_int64, c_int, c_void_p, POINTER(PxstCgInfo),
                                        c_void_p]),
    "pxst_project_irrotational": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_double,
                                          c_int64, c_int, POINTER(PxstCgInfo), c_void_p]),
    "pxst_split_weights": (c_int, [c_uint64, c_int64, c_int64, c_int64, c_int, c_void_p,
                                   c_void_p]),
    "pxst_split_counts": (c_int, [c_uint64, c_void_p, c_int64, c_int64, c_int64, c_void_p,
                                  c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load and type the shared library (no CUDA device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"libpxst_b200.so not found at {path}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'`")
        cdll = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(cdll, name)
            fn.restype = res
            fn.argtypes = args
        if cdll.pxst_abi_version() != ABI_VERSION:
            raise RuntimeError("libpxst_b200.so ABI version mismatch; rebuild it")
        _lib = cdll
        return cdll


def lib() -> ctypes.CDLL:
    """The library, with a CUDA device required (no CPU fallback exists)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2003_12726_b200 needs a CUDA (B200) device; none is visible")
    return load_library()


def check(rc: int) -> None:
    if rc == PXST_OK:
        return
    msg = (_lib.pxst_last_error() or b"").decode(errors="replace")
    if rc == PXST_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"pxst CUDA error ({rc}): {msg}")


_RAW_STREAM = None


def stream_ptr(stream=None) -> int:
    """cudaStream_t of `stream` (default: torch's current stream on the current
    device) as an integer.  The default goes through torch's raw-stream getter
    when it has one: torch.cuda.current_stream() builds a Stream object and
    resolves the device index in Python, ~15 us a call and ~16 calls per
    iteration of the drop-in API."""
    global _RAW_STREAM
    import torch
    if stream is not None:
        return int(stream.cuda_stream)
    if _RAW_STREAM is None:
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        dev = getattr(torch._C, "_cuda_getDevice", None)
        _RAW_STREAM = (raw, dev) if raw is not None and dev is not None else False
    if _RAW_STREAM:
        return int(_RAW_STREAM[0](_RAW_STREAM[1]()))
    return int(torch.cuda.current_stream().cuda_stream)


def launch_count() -> int:
    return int(load_library().pxst_launch_count())
