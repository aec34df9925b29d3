"""ctypes binding of libwoit.so (include/woit.h).

The library is the only compute path: if it is missing or cannot be loaded the
import fails loudly — there is no CPU or PyTorch fallback.
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
# WOIT_LIB selects an alternative build (tuning variants, tools/variants.py)
LIB_PATH = os.environ.get("WOIT_LIB") or os.path.join(_HERE, "libwoit.so")

ABI_VERSION = 3

OK = 0
EINVAL = -1
EWORKSPACE = -2
ECUDA = -3
ERANK = -4
ETAPS = -5

REFRACTION = 0x01
CHROMATIC_ABERRATION = 0x02
CUBE_TRANSMISSION = 0x04
NORMALIZE = 0x08
PACKED_STORAGE = 0x10
LITERAL_SPECTRAL_T = 0x20
CUBE_BACKFACE_ONLY = 0x40
DIFFUSION = 0x80
METHOD_ABUFFER, METHOD_WBOIT, METHOD_MLAB4 = 1, 2, 3

BUILD_BINNED = 0
BUILD_ATOMIC = 1

SYNTH_IDS = {"plane4": 0, "smoke": 1, "particles": 2, "ragged": 3}

_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_sz = C.c_size_t


class Frags(C.Structure):
    _fields_ = [("width", _i32), ("height", _i32), ("npix", _i64), ("nfrag", _i64),
                ("pixel_base", _i64), ("frag_base", _i64), ("offsets", _vp), ("depth", _vp),
                ("alpha", _vp), ("trans", _vp), ("radiance", _vp), ("normal", _vp), ("ior", _vp),
                ("backface", _vp), ("opaque_depth", _vp), ("opaque_color", _vp)]


class Params(C.Structure):
    _fields_ = [("rank", _i32), ("flags", _i32), ("aberration_taps", _i32), ("diffusion_radius", _i32),
                ("refraction_scale", C.c_double), ("cam_forward", C.c_double * 3),
                ("cam_right", C.c_double * 3), ("cam_up", C.c_double * 3),
                ("tan_half", C.c_double), ("aspect", C.c_double), ("diffusion", C.c_double)]


class Bufs(C.Structure):
    _fields_ = [("near", _vp), ("far", _vp), ("coeffs", _vp), ("accum", _vp), ("weight", _vp),
                ("refraction_offset", _vp), ("output", _vp), ("vhat", _vp),
                ("full_opaque_image", _vp), ("diffusion", _vp), ("blurred_image", _vp), ("coeff_words", _vp)]


_d3 = C.c_double * 3
_d2 = C.c_double * 2


class Prim(C.Structure):
    """woit_prim_t"""
    _fields_ = [("kind", _i32), ("count", _i32), ("profile", _i32), ("flags", _i32), ("d", C.c_double),
                ("center", _d3), ("radius", C.c_double), ("particle_radius", C.c_double), ("extent", _d2),
                ("pcenter", _d2), ("alpha", C.c_double), ("ior", C.c_double), ("trans", _d3), ("radiance", _d3),
                ("sigma", _d3), ("color", _d3), ("checker", _d3), ("near", C.c_double), ("far", C.c_double),
                ("cell", C.c_double), ("positions", _vp), ("radiance_scale", _vp), ("box", _vp)]


class SceneC(C.Structure):
    """woit_scene_t"""
    _fields_ = [("nprims", _i32), ("bg_cell", _i32), ("bg_has_checker", _i32), ("reserved", _i32), ("prims", _vp),
                ("origin", _d3), ("forward", _d3), ("right", _d3), ("up", _d3), ("tan_half", C.c_double),
                ("aspect", C.c_double), ("bg_color", _d3), ("bg_checker", _d3)]


PRIM_PLANE, PRIM_SPHERE, PRIM_FOG, PRIM_PARTICLES, PRIM_BACKDROP = 0, 1, 2, 3, 4

_SIGS = {
    "woit_abi_version": (C.c_int, []),
    "woit_status_string": (C.c_char_p, [C.c_int]),
    "woit_frame_workspace_bytes": (_sz, [_i64, _i64]),
    "woit_render_band": (C.c_int, [C.POINTER(Frags), C.POINTER(Params), C.POINTER(Bufs), _vp, _sz, _vp]),
    "woit_step1_depth_bounds": (C.c_int, [C.POINTER(Frags), C.POINTER(Bufs), _vp, _sz, _vp]),
    "woit_step2_build": (C.c_int, [C.POINTER(Frags), C.POINTER(Params), C.POINTER(Bufs), _vp, _sz, _vp]),
    "woit_step3_accumulate": (C.c_int, [C.POINTER(Frags), C.POINTER(Params), C.POINTER(Bufs), _vp, _sz,
                                        _vp]),
    "woit_step4_composite": (C.c_int, [C.POINTER(Frags), C.POINTER(Params), C.POINTER(Bufs), _vp]),
    "woit_fragment_indices": (C.c_int, [C.POINTER(Frags), _vp, _vp, C.c_int, _vp, _vp, _vp, _vp]),
    "woit_blur_workspace_bytes": (_sz, [_i32, _i32]),
    "woit_build_atomic_workspace_bytes": (_sz, [_i64]),
    "woit_baseline_workspace_bytes": (_sz, [C.c_int, _i64, _i64]),
    "woit_cast_workspace_bytes": (_sz, [_i64]),
    "woit_cast_offsets": (C.c_int, [C.POINTER(SceneC), _i32, _i32, _vp, _vp, _sz, _vp]),
    "woit_cast_fill": (C.c_int, [C.POINTER(SceneC), _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                 _vp]),
    "woit_render_baseline": (C.c_int, [C.POINTER(Frags), C.c_int, C.c_int, _vp, _vp, _vp, _sz, _vp]),
    "woit_build_atomic": (C.c_int, [C.POINTER(Frags), _vp, C.POINTER(Params), C.POINTER(Bufs), _vp, _sz, _vp]),
    "woit_resolve_blur": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _vp, _sz, _vp]),
    "woit_build_into_workspace_bytes": (_sz, [_i64, _i64]),
    "woit_build_into": (C.c_int, [_vp, _i64, _vp, _vp, _vp, _i64, C.c_int, C.c_int, _vp, _sz, _vp]),
    "woit_interp_absorbance": (C.c_int, [_vp, _i64, _vp, _vp, _i64, C.c_int, _vp, _vp]),
    "woit_cells_raw": (C.c_int, [_vp, _i64, _vp, _vp, _i64, C.c_int, _vp, _vp]),
    "woit_total_absorbance": (C.c_int, [_vp, _i64, C.c_int, _vp, _vp]),
    "woit_bin_workspace_bytes": (_sz, [_i64, _i64]),
    "woit_bin_by_pixel": (C.c_int, [_vp, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
    "woit_bin_frame_workspace_bytes": (_sz, [_i64, _i64]),
    "woit_bin_frame": (C.c_int, [_vp, C.POINTER(Frags), C.POINTER(Frags), _vp, _vp, _vp, _sz, _vp]),
    "woit_pack_rgb9e5": (C.c_int, [_vp, _i64, _vp, _vp]),
    "woit_unpack_rgb9e5": (C.c_int, [_vp, _i64, _vp, _vp]),
    "woit_synth_workspace_bytes": (_sz, [_i64]),
    "woit_synth_offsets": (C.c_int, [C.c_int, _i32, _i32, C.c_uint32, _i32, _i32, _i32, _vp, _vp, _sz,
                                     _vp]),
    "woit_synth_fill": (C.c_int, [C.c_int, _i32, _i32, C.c_uint32, _i32, _i32, _i32, _vp, _vp, _vp, _vp,
                                  _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
}

EXPORTED = tuple(_SIGS)

_lib: Optional[C.CDLL] = None


def load() -> C.CDLL:
    """Load libwoit.so once; raise ImportError (no fallback) if it is unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2201_00094_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.woit_abi_version() != ABI_VERSION:
        raise ImportError(f"libwoit ABI {lib.woit_abi_version()} != expected {ABI_VERSION}")
    _lib = lib
    return lib


def check(status: int, what: str) -> None:
    if status == OK:
        return
    msg = f"{what}: {load().woit_status_string(status).decode()} (status {status})"
    if status in (EINVAL, ERANK, ETAPS, EWORKSPACE):
        raise ValueError(msg)
    raise RuntimeError(msg)
