"""B200-native PXST (ptychographic X-ray speckle tracking) hot path.

A from-scratch sm_100a implementation of the reconstruction hot path of
arXiv 2003.12726 behind the reference's own Python API (``pxst.recon``):
``make_reference`` / ``make_object_map``, ``update_pixel_map``,
``update_translations``, ``calc_error`` and ``run_main_loop``, with the same
dataclasses and float64 arrays in and out.  Kernels live in
``libpxst_b200.so`` (C ABI: ``include/pxst_b200.h``); torch provides device
buffers, streams and ``torch.distributed`` only.
"""

from . import analysis, data_model, geometry, integration
from .data_model import (
    ErrorMetrics,
    Geometry,
    PixelMap,
    PixelMask,
    PixelTranslations,
    ReferenceImage,
    Roi,
    ScanData,
    Whitefield,
)
from .engine import clear_cache
from .multigpu import Devices
from .recon import (
    IterationSettings,
    LoopResult,
    SearchWindow,
    UpdateOptions,
    calc_error,
    default_schedule,
    make_object_map,
    make_reference,
    quadratic_subpixel_refine,
    run_main_loop,
    update_pixel_map,
    update_translations,
)

__version__ = "0.1.0"
