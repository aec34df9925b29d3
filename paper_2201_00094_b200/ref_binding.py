"""The reference-side binding: the reference package's own hot-path entry points,
re-implemented over libwoit, with the reference's signatures, argument types
(numpy float64 arrays in the reference's ``FrameFragments`` / ``FrameBuffers`` /
``RayGrid`` / ``RenderConfig`` / ``TouchCounter`` / ``Scene``) and results.

This is what a maintainer of ``woit`` adds to route its wavelet compositor to a
B200: ``install()`` re-binds

    woit.pipeline.step1_depth_bounds   pipeline.py:131-134
    woit.pipeline.step2_build          pipeline.py:148-155
    woit.pipeline.step3_accumulate     pipeline.py:170-217
    woit.pipeline.step4_composite      pipeline.py:284-308
    woit.pipeline._wavelet_band        pipeline.py:321-330
    woit.pipeline.render_frame         pipeline.py:333-375
    woit.wavelet.build_into / cells_raw_batch / interp_absorbance_batch /
        total_absorbance_batch         wavelet.py:272-337

to the functions below. Each uploads the reference's arrays (fp32 SoA, the
device layout of include/woit.h), runs the CUDA path through the C ABI and
writes the results back into the caller's arrays in place (the reference's
steps mutate ``FrameBuffers`` and return None). Bands keep their pixel_base, so
``render_frame(workers=k)`` is bit-identical for every k, as the reference's
``test_workers_do_not_change_output`` requires.

Nothing here is imported by the product path; the reference package itself must
be importable (``baseline/_ref``, tools/install_ref.sh) for ``install()``.
"""

from __future__ import annotations

import dataclasses
from typing import Dict, Optional

import numpy as np
import torch

from . import pipeline as P
from . import wavelet as Wv
from .frame import FrameFragments

# calls routed through this binding (the conformance suite checks they happened)
CALLS: Dict[str, int] = {}

_CFG_FIELDS = ("method", "rank", "width", "height", "refraction", "chromatic_aberration", "cube_transmission",
               "normalize", "packed_storage", "aberration_taps", "refraction_scale", "workers",
               "literal_spectral_t", "cube_backface_only", "wboit_weight")


def _count(name: str) -> None:
    CALLS[name] = CALLS.get(name, 0) + 1


def _dev() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


def config(cfg) -> P.RenderConfig:
    """The reference's RenderConfig -> ours (same fields, same validation)."""
    kw = {k: getattr(cfg, k) for k in _CFG_FIELDS if hasattr(cfg, k)}
    if "wboit_weight" in kw:
        kw["wboit_weight"] = tuple(float(x) for x in kw["wboit_weight"])
    return P.RenderConfig(**kw)


def frame_to_device(frame, pixel_base: int = 0) -> FrameFragments:
    """A reference FrameFragments (f64 numpy, CSR by pixel) -> the device stream."""
    return FrameFragments.from_numpy(frame.width, frame.height, frame.offsets, frame.depth, frame.alpha,
                                     frame.trans, frame.radiance, frame.normal, frame.ior, frame.backface,
                                     frame.opaque_depth, frame.opaque_color, device=_dev(),
                                     pixel_base=int(pixel_base))


def slice_frame(frame, p0: int, p1: int):
    """The reference's ``_slice_frame`` (pipeline.py:311-318) on its own types:
    pixels [p0, p1) with rebased pixel ids and offsets."""
    lo, hi = int(frame.offsets[p0]), int(frame.offsets[p1])
    return type(frame)(frame.width, frame.height, frame.pixel[lo:hi] - p0, frame.depth[lo:hi],
                       frame.alpha[lo:hi], frame.trans[lo:hi], frame.radiance[lo:hi], frame.normal[lo:hi],
                       frame.ior[lo:hi], frame.backface[lo:hi], frame.offsets[p0:p1 + 1] - lo,
                       frame.opaque_depth[p0:p1], frame.opaque_color[p0:p1])


def rays_camera(rays) -> P.RayGrid:
    """The reference's RayGrid -> ours (the camera frame the kernels read; the
    per-pixel directions are recomputed on the device in the same f64 order)."""
    t = lambda v: tuple(float(x) for x in np.asarray(v, dtype=np.float64))
    return P.RayGrid(t(rays.origin), t(rays.forward), t(rays.right), t(rays.up), int(rays.width),
                     int(rays.height), float(rays.tan_half), float(rays.aspect))


_BUF_FIELDS = ("near", "far", "coeffs", "accum", "accum_weight", "refraction_offset", "opaque_depth",
               "opaque_color", "output")


def bufs_to_device(bufs, vhat_n: int = 0) -> P.FrameBuffers:
    f32 = lambda a: torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float32))).to(_dev())
    d = {k: f32(getattr(bufs, k)) for k in _BUF_FIELDS}
    return P.FrameBuffers(int(bufs.width), int(bufs.height), int(bufs.rank), d["near"], d["far"], d["coeffs"],
                          d["accum"], d["accum_weight"], d["refraction_offset"], d["opaque_depth"],
                          d["opaque_color"], d["output"], None,
                          torch.zeros(d["near"].numel(), dtype=torch.float32, device=_dev()))


def _write_back(bufs, g: P.FrameBuffers, names) -> None:
    for k in names:
        getattr(bufs, k)[...] = getattr(g, k).double().cpu().numpy()


def _full_image(img) -> Optional[torch.Tensor]:
    if img is None:
        return None
    return torch.from_numpy(np.ascontiguousarray(np.asarray(img, dtype=np.float32))).to(_dev())


# ---------------------------------------------------------------------------
# woit.pipeline


def step1_depth_bounds(frame, bufs) -> None:
    _count("step1_depth_bounds")
    g = bufs_to_device(bufs)
    P.step1_depth_bounds(frame_to_device(frame), g)
    _write_back(bufs, g, ("near", "far"))


def step2_build(frame, bufs, cfg, counter=None) -> None:
    _count("step2_build")
    g = bufs_to_device(bufs)
    P.step2_build(frame_to_device(frame), g, config(cfg), counter)
    _write_back(bufs, g, ("coeffs",))


def step3_accumulate(rays, frame, bufs, cfg, counter=None, pixel_base: int = 0) -> None:
    _count("step3_accumulate")
    g = bufs_to_device(bufs)
    P.step3_accumulate(rays_camera(rays), frame_to_device(frame, pixel_base), g, config(cfg), counter,
                       pixel_base=pixel_base)
    _write_back(bufs, g, ("accum", "accum_weight", "refraction_offset"))


def step4_composite(bufs, cfg, counter=None, pixel_base: int = 0, full_opaque_image=None) -> None:
    _count("step4_composite")
    g = bufs_to_device(bufs)
    P.step4_composite(g, config(cfg), counter, pixel_base=pixel_base,
                      full_opaque_image=_full_image(full_opaque_image))
    _write_back(bufs, g, ("output",))


def _wavelet_band(rays, frame, cfg, full_img, p0: int, p1: int, counter):
    """pipeline.py:321-330: all four passes of one band, fused in one kernel."""
    _count("_wavelet_band")
    from woit.pipeline import FrameBuffers  # the reference's type, returned to its caller

    band = slice_frame(frame, p0, p1) if (p0, p1) != (0, frame.npix) else frame
    g = P.render_band(frame_to_device(band, p0), config(cfg), rays_camera(rays),
                      full_opaque_image=_full_image(full_img), counter=counter)
    bufs = FrameBuffers.allocate(band, cfg.rank)
    _write_back(bufs, g, ("near", "far", "coeffs", "accum", "accum_weight", "refraction_offset", "output"))
    return bufs


def scene_from_reference(scene):
    """A reference Scene -> this package's (same primitives, materials, seed), for
    casting on the device."""
    from . import scene as S

    def conv(v):
        if dataclasses.is_dataclass(v) and type(v).__name__ == "Spectrum3":
            return (float(v.r), float(v.g), float(v.b))
        if dataclasses.is_dataclass(v) and not isinstance(v, type):
            cls = P.Camera if type(v).__name__ == "Camera" else getattr(S, type(v).__name__, None)
            if cls is None:
                raise ValueError(f"no device caster for {type(v).__name__}")
            kw = {f.name: conv(getattr(v, f.name)) for f in dataclasses.fields(v)}
            if type(v).__name__ == "ParticleCloud":
                kw["positions"] = kw["radiance_scale"] = None  # re-seeded identically by Scene
            return cls(**kw)
        if isinstance(v, tuple):
            return tuple(conv(x) for x in v)
        return v

    return conv(scene)


def render_frame(scene, cfg, counter=None, frame=None) -> np.ndarray:
    """pipeline.py:333-375: (H, W, 3) float64. Without ``frame`` the scene is cast on
    the device (our cast_frame, CSR identical to the reference's); the comparison
    methods run as the float64 per-pixel GPU kernels."""
    _count("render_frame")
    gcfg = config(cfg)
    if frame is None:
        from .scene import cast_frame

        dframe = cast_frame(scene_from_reference(scene), gcfg.width, gcfg.height, device=_dev())
    else:
        dframe = frame_to_device(frame)
    img = P.render_frame(getattr(scene, "camera", None), gcfg, counter=counter, frame=dframe)
    torch.cuda.synchronize()
    return img.double().cpu().numpy()


# ---------------------------------------------------------------------------
# woit.wavelet (float64 kernels, bit-exact to the reference)


def build_into(coeffs, pix, z, a, rank, counter=None):
    _count("build_into")
    return Wv.build_into(coeffs, pix, z, a, rank, counter)


def cells_raw_batch(coeffs, pix, cells, rank, counter=None):
    _count("cells_raw_batch")
    return Wv.cells_raw_batch(coeffs, pix, cells, rank, counter)


def interp_absorbance_batch(coeffs, pix, z, rank, counter=None):
    _count("interp_absorbance_batch")
    return Wv.interp_absorbance_batch(coeffs, pix, z, rank, counter)


def total_absorbance_batch(coeffs, rank, counter=None):
    _count("total_absorbance_batch")
    return Wv.total_absorbance_batch(coeffs, rank, counter)


_PIPELINE = ("step1_depth_bounds", "step2_build", "step3_accumulate", "step4_composite", "_wavelet_band",
             "render_frame")
_WAVELET = ("build_into", "cells_raw_batch", "interp_absorbance_batch", "total_absorbance_batch")


def install() -> None:
    """Re-bind the reference's hot-path entry points to this module (before the
    caller imports names from woit.pipeline / woit.wavelet)."""
    import woit.pipeline as rp
    import woit.wavelet as rw

    g = globals()
    for name in _PIPELINE:
        setattr(rp, name, g[name])
    for name in _WAVELET:
        setattr(rw, name, g[name])

