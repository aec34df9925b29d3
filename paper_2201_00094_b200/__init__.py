"""B200-native wavelet order-independent transparency (arXiv 2201.00094), hot path only.

Drop-in for the reference ``woit`` package's wavelet compositor: the Python
entry points mirror ``woit.pipeline`` / ``woit.wavelet`` / ``woit.packing`` and
run hand-written sm_100a CUDA kernels from ``libwoit.so`` (C ABI in
include/woit.h). Importing the package does not need a GPU; calling a kernel
without ``libwoit.so`` raises (there is no CPU fallback).
"""

from . import _lib  # noqa: F401
from .synth import WORKLOADS, SynthFrame, generate  # noqa: F401
from .wavelet import (TouchCounter, build_into, cells_raw_batch, interp_absorbance_batch,  # noqa: F401
                      total_absorbance_batch, bin_by_pixel, normalize_depth_array)
from .frame import FrameFragments  # noqa: F401
from .pipeline import (METHODS, Camera, FrameBuffers, RayGrid, RenderConfig, Workspace,  # noqa: F401
                       camera_rays, eval_bounds, render_band, render_frame, step1_depth_bounds,
                       resolve_blur, step2_build, step2_build_atomic, step3_accumulate, step4_composite,
                       pixel_ids, render_baseline)
from .packing import pack_rgb9e5, unpack_rgb9e5, roundtrip_coeff_array, bytes_per_pixel  # noqa: F401

__version__ = "0.1.0"
from .scene import PRESET_NAMES, Scene, cast_frame, preset  # noqa: F401,E402
