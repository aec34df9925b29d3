"""Drop-in mirror of the reference's wavelet frame path (pipeline.py), on B200.

Same names, arguments and error behaviour as ``woit.pipeline``:
``RenderConfig`` (pipeline.py:45-73), ``FrameBuffers`` (:76-107), ``eval_bounds``
(:110-128), ``step1_depth_bounds`` .. ``step4_composite`` (:131-308) and
``render_frame`` (:333-375). Buffers are torch CUDA tensors (fp32), every pass is
a hand-written sm_100a kernel in libwoit.so reached through its C ABI, and
``render_frame`` runs all four passes fused in one kernel that reads each
fragment from HBM once.

Differences from the reference, all deliberate:
* fp32 storage (the reference is float64); z and every index derived from it
  are still computed in f64 / fixed point and are bit-identical;
* without ``frame=``, ``render_frame`` casts the scene on the GPU
  (``scene.cast_frame``, the reference's scene.py:463-630);
* the comparison methods (``method="abuffer" | "wboit" | "mlab4"``,
  baselines.py:135-220) run as float64 per-pixel kernels (``render_baseline``);
  they need ``frame=`` like the wavelet path;
* ``diffusion`` / ``diffusion_radius`` (default off) add the north star's
  "resolve and blur" pass, which the reference does not have (SURVEY.md §8 row
  GAP): an in-repo definition, documented in include/woit.h (WOIT_DIFFUSION) and
  DESIGN.md, parity unpinned. With diffusion == 0 nothing changes.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Optional, Tuple

import torch

from . import _lib
from .frame import FrameFragments, ptr
from .wavelet import TouchCounter

METHODS = ("wavelet", "abuffer", "wboit", "mlab4")
DEFAULT_WBOIT_WEIGHT = (10.0, 0.01, 3000.0)  # baselines.py:21 (gain, clamp lo, clamp hi)
_WORLD_UP = (0.0, 1.0, 0.0)   # scene.py:43
_ALT_UP = (1.0, 0.0, 0.0)     # scene.py:44


@dataclass(frozen=True)
class RenderConfig:
    method: str = "wavelet"
    rank: int = 3
    width: int = 256
    height: int = 256
    refraction: bool = False
    chromatic_aberration: bool = False
    cube_transmission: bool = False
    normalize: bool = True
    packed_storage: bool = False
    aberration_taps: int = 5
    refraction_scale: float = 40.0
    workers: int = 1
    literal_spectral_t: bool = False
    cube_backface_only: bool = False
    wboit_weight: Tuple[float, float, float] = DEFAULT_WBOIT_WEIGHT
    diffusion: float = 0.0        # in-repo "resolve and blur" strength (0 = off)
    diffusion_radius: int = 4     # Gaussian taps each side, sigma = radius / 2

    def __post_init__(self):
        if self.method not in METHODS:
            raise ValueError(f"unknown method {self.method!r}; valid: {', '.join(METHODS)}")
        if not (0 <= self.rank <= 6):
            raise ValueError(f"rank must lie in [0, 6], got {self.rank}")
        if self.aberration_taps < 3 or self.aberration_taps % 2 == 0:
            raise ValueError("aberration taps must be odd and >= 3")
        if self.width < 1 or self.height < 1:
            raise ValueError("frame must be at least 1x1")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if not (math.isfinite(self.diffusion) and self.diffusion >= 0.0):
            raise ValueError("diffusion must be finite and >= 0")
        if not (1 <= self.diffusion_radius <= 64):
            raise ValueError("diffusion_radius must lie in [1, 64]")

    @property
    def flags(self) -> int:
        f = 0
        f |= _lib.REFRACTION if self.refraction else 0
        f |= _lib.CHROMATIC_ABERRATION if self.chromatic_aberration else 0
        f |= _lib.CUBE_TRANSMISSION if self.cube_transmission else 0
        f |= _lib.NORMALIZE if self.normalize else 0
        f |= _lib.PACKED_STORAGE if self.packed_storage else 0
        f |= _lib.LITERAL_SPECTRAL_T if self.literal_spectral_t else 0
        f |= _lib.CUBE_BACKFACE_ONLY if self.cube_backface_only else 0
        f |= _lib.DIFFUSION if self.diffusion > 0.0 else 0
        return f


@dataclass(frozen=True)
class Camera:
    """scene.py:135-150."""

    position: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    forward: Tuple[float, float, float] = (0.0, 0.0, 1.0)
    fov_deg: float = 60.0

    def basis(self):
        f = _normalize(self.forward)
        up0 = _WORLD_UP if abs(_dot(f, _WORLD_UP)) <= 0.999 else _ALT_UP
        right = _normalize(_cross(up0, f))
        up = _cross(f, right)
        return f, right, up


@dataclass(frozen=True)
class RayGrid:
    """Camera frame of ``camera_rays`` (scene.py:184-212) without the per-pixel
    direction array: kernels recompute each pixel's direction in f64."""

    origin: Tuple[float, float, float]
    forward: Tuple[float, float, float]
    right: Tuple[float, float, float]
    up: Tuple[float, float, float]
    width: int
    height: int
    tan_half: float
    aspect: float


def _dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def _cross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def _normalize(v):
    n = math.sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2])
    return (v[0] / n, v[1] / n, v[2] / n)


def camera_rays(camera: Camera, width: int, height: int) -> RayGrid:
    f, right, up = camera.basis()
    tan_half = math.tan(math.radians(camera.fov_deg) * 0.5)
    return RayGrid(tuple(float(c) for c in camera.position), f, right, up, width, height, tan_half,
                   width / height)


@dataclass
class FrameBuffers:
    """Per-pixel working state on the device (pipeline.py:76-107), fp32."""

    width: int
    height: int
    rank: int
    near: torch.Tensor
    far: torch.Tensor
    coeffs: torch.Tensor
    accum: torch.Tensor
    accum_weight: torch.Tensor
    refraction_offset: torch.Tensor
    opaque_depth: torch.Tensor
    opaque_color: torch.Tensor
    output: torch.Tensor
    vhat: Optional[torch.Tensor] = None  # per-fragment transmittance (filled by step3 / render)
    diffusion: Optional[torch.Tensor] = None  # per-pixel coverage D_p (WOIT_DIFFUSION)
    # packed storage (cfg.packed_storage): [P][S] E5B9G9R9 words (packing.py:46-77), int32
    # tensor holding the uint32 bit patterns -- the paper's 4 S bytes per pixel
    coeff_words: Optional[torch.Tensor] = None

    @classmethod
    def allocate(cls, frame: FrameFragments, rank: int, vhat: bool = False,
                 packed: bool = False) -> "FrameBuffers":
        P, dev = frame.npix, frame.device
        z = lambda *s: torch.zeros(*s, dtype=torch.float32, device=dev)
        return cls(frame.width, frame.height, rank,
                   torch.full((P,), math.inf, dtype=torch.float32, device=dev),
                   torch.full((P,), -math.inf, dtype=torch.float32, device=dev),
                   z(P, 1 << (rank + 1), 3), z(P, 3), z(P, 3), z(P, 2),
                   frame.opaque_depth.clone(), frame.opaque_color.clone(), z(P, 3),
                   z(frame.nfrag, 3) if vhat else None, z(P),
                   torch.zeros(P, 1 << (rank + 1), dtype=torch.int32, device=dev) if packed else None)

    def image(self) -> torch.Tensor:
        return self.output.reshape(-1, self.width, 3)

    def c_struct(self, full_opaque_image: Optional[torch.Tensor] = None,
                 blurred_image: Optional[torch.Tensor] = None) -> _lib.Bufs:
        b = _lib.Bufs()
        b.near, b.far, b.coeffs = ptr(self.near), ptr(self.far), ptr(self.coeffs)
        b.accum, b.weight = ptr(self.accum), ptr(self.accum_weight)
        b.refraction_offset, b.output = ptr(self.refraction_offset), ptr(self.output)
        b.vhat = ptr(self.vhat)
        if full_opaque_image is not None:
            full_opaque_image = full_opaque_image.to(torch.float32).contiguous()
            self._img_keepalive = full_opaque_image
        b.full_opaque_image = ptr(full_opaque_image)
        b.diffusion = ptr(self.diffusion)
        if blurred_image is not None:
            blurred_image = blurred_image.to(torch.float32).contiguous()
            self._blur_keepalive = blurred_image
        b.blurred_image = ptr(blurred_image)
        b.coeff_words = ptr(self.coeff_words)
        return b


def _params(cfg: RenderConfig, rank: int, rays: Optional[RayGrid] = None) -> _lib.Params:
    if rays is None:
        rays = camera_rays(Camera(), cfg.width, cfg.height)
    p = _lib.Params()
    p.rank, p.flags, p.aberration_taps = rank, cfg.flags, cfg.aberration_taps
    p.refraction_scale = float(cfg.refraction_scale)
    for i in range(3):
        p.cam_forward[i] = float(rays.forward[i])
        p.cam_right[i] = float(rays.right[i])
        p.cam_up[i] = float(rays.up[i])
    p.tan_half, p.aspect = float(rays.tan_half), float(rays.aspect)
    p.diffusion, p.diffusion_radius = float(cfg.diffusion), int(cfg.diffusion_radius)
    return p


class Workspace:
    """Device scratch for the frame kernels, grown on demand and reused.

    A workspace holds per-launch state (the window-claim counter and the
    long-pixel list, include/woit.h): give each stream / host thread that may
    launch concurrently its own. Without one, every call takes fresh scratch from
    torch's stream-ordered caching allocator, which is safe under any concurrency.
    """

    def __init__(self):
        self.buf: Optional[torch.Tensor] = None

    def get(self, nbytes: int, device) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != torch.device(device):
            self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        return self.buf


def _scratch(nbytes: int, device, ws: Optional[Workspace]) -> torch.Tensor:
    if ws is not None:
        return ws.get(nbytes, device)
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _frame_ws(frame: FrameFragments, ws: Optional[Workspace]):
    lib = _lib.load()
    n = lib.woit_frame_workspace_bytes(frame.npix, frame.nfrag)
    t = _scratch(n, frame.device, ws)
    return t, t.numel()


def _check_frame(frame: FrameFragments, bufs: FrameBuffers) -> None:
    if bufs.near.numel() != frame.npix:
        raise ValueError(f"buffers hold {bufs.near.numel()} pixels, frame has {frame.npix}")


def eval_bounds(near: torch.Tensor, far: torch.Tensor, rank: int):
    """Padded mapping bounds (pipeline.py:110-128), f64 on the tensors' device."""
    near = near.double()
    far = far.double()
    cells = 1 << (rank + 1)
    covered = near <= far
    rng = torch.where(covered, far - near, torch.zeros_like(near))
    if cells > 2:
        margin = rng / (cells - 2)
        return torch.where(covered, near - margin, near), torch.where(covered, far + margin, far)
    return near, torch.where(covered, far + rng, far)


def step1_depth_bounds(frame: FrameFragments, bufs: FrameBuffers, ws: Optional[Workspace] = None) -> None:
    """Tight min/max transparent depth per pixel (pipeline.py:131-134)."""
    _check_frame(frame, bufs)
    lib = _lib.load()
    f, b = frame.c_struct(), bufs.c_struct()
    w, wn = _frame_ws(frame, ws)
    _lib.check(lib.woit_step1_depth_bounds(f, b, ptr(w), wn, _stream()), "step1_depth_bounds")


def step2_build(frame: FrameFragments, bufs: FrameBuffers, cfg: RenderConfig,
                counter: Optional[TouchCounter] = None, ws: Optional[Workspace] = None) -> None:
    """Closed-form Haar projection of every fragment (pipeline.py:148-155)."""
    _check_frame(frame, bufs)
    lib = _lib.load()
    f, b = frame.c_struct(), bufs.c_struct()
    w, wn = _frame_ws(frame, ws)
    _lib.check(lib.woit_step2_build(f, _params(cfg, bufs.rank), b, ptr(w), wn, _stream()), "step2_build")
    if counter is not None:
        counter.record_insert(frame.nfrag, frame.nfrag * (bufs.rank + 2))


def pixel_ids(frame: FrameFragments) -> torch.Tensor:
    """int32 pixel id per fragment (the reference's FrameFragments.pixel, scene.py:369)."""
    run = frame.offsets[1:] - frame.offsets[:-1]
    return torch.repeat_interleave(torch.arange(frame.npix, device=frame.device, dtype=torch.int32), run)


def step2_build_atomic(frame: FrameFragments, bufs: FrameBuffers, cfg: RenderConfig,
                       pix: Optional[torch.Tensor] = None, ws: Optional[Workspace] = None) -> None:
    """step2_build through the north star's alternative: fp32 red.global atomics of the
    closed-form projection from an unbinned stream (``pix`` = pixel id per fragment).

    Kept for the measured comparison against the CSR tile build;
    not bit-reproducible run to run. ``bufs.coeffs`` is accumulated into.
    """
    _check_frame(frame, bufs)
    if cfg.packed_storage:
        raise ValueError("the atomic build has no packed storage")
    lib = _lib.load()
    if pix is None:
        pix = pixel_ids(frame)
    if pix.dtype != torch.int32 or pix.numel() < frame.nfrag:
        raise ValueError("pix must be int32 with one id per fragment")
    n = lib.woit_build_atomic_workspace_bytes(frame.npix)
    t = _scratch(n, frame.device, ws)
    f, b = frame.c_struct(), bufs.c_struct()
    _lib.check(lib.woit_build_atomic(f, ptr(pix), _params(cfg, bufs.rank), b, ptr(t), t.numel(), _stream()),
               "step2_build_atomic")


def step3_accumulate(rays, frame: FrameFragments, bufs: FrameBuffers, cfg: RenderConfig,
                     counter: Optional[TouchCounter] = None, pixel_base: int = 0,
                     ws: Optional[Workspace] = None) -> None:
    """Visibility-weighted accumulation and refraction offsets (pipeline.py:170-217).

    ``rays`` is a ``RayGrid`` (this module's or the reference's) or None for the
    default camera. Writes ``bufs.vhat`` when it is allocated.
    """
    _check_frame(frame, bufs)
    lib = _lib.load()
    if pixel_base and frame.pixel_base != pixel_base:
        frame = FrameFragments(**{**frame.__dict__, "pixel_base": pixel_base})
    f, b = frame.c_struct(), bufs.c_struct()
    w, wn = _frame_ws(frame, ws)
    _lib.check(lib.woit_step3_accumulate(f, _params(cfg, bufs.rank, rays), b, ptr(w), wn, _stream()),
               "step3_accumulate")
    if counter is not None and frame.nfrag:
        counter.record_eval(2 * frame.nfrag, 2 * frame.nfrag * (bufs.rank + 2))


def resolve_blur(image: torch.Tensor, radius: int, ws: Optional[Workspace] = None) -> torch.Tensor:
    """K_resolve: separable edge-clamped Gaussian blur of an (H, W, 3) fp32 image.

    The in-repo diffusion definition (include/woit.h, WOIT_DIFFUSION); the
    reference has no such pass (SURVEY.md §8 row GAP), so its parity is unpinned.
    """
    if image.dim() != 3 or image.shape[-1] != 3:
        raise ValueError("image must be (H, W, 3)")
    if not (1 <= radius <= 64):
        raise ValueError("diffusion_radius must lie in [1, 64]")
    lib = _lib.load()
    img = image.to(torch.float32).contiguous()
    H, W = int(img.shape[0]), int(img.shape[1])
    out = torch.empty_like(img)
    n = lib.woit_blur_workspace_bytes(W, H)
    t = _scratch(n, img.device, ws)
    _lib.check(lib.woit_resolve_blur(ptr(img), W, H, int(radius), ptr(out), ptr(t), t.numel(), _stream()),
               "resolve_blur")
    return out



def _background_image(bufs_or_frame, full_opaque_image: Optional[torch.Tensor]) -> torch.Tensor:
    """The image the background is read from: the full frame, else the band itself."""
    if full_opaque_image is not None:
        return full_opaque_image
    return bufs_or_frame.opaque_color.reshape(-1, bufs_or_frame.width, 3)


def step4_composite(bufs: FrameBuffers, cfg: RenderConfig, counter: Optional[TouchCounter] = None,
                    pixel_base: int = 0, full_opaque_image: Optional[torch.Tensor] = None,
                    blurred_image: Optional[torch.Tensor] = None) -> None:
    """Blend over the (refracted / aberrated) background (pipeline.py:284-308).

    With ``cfg.diffusion > 0`` the background is lerped towards ``blurred_image``
    (computed here by ``resolve_blur`` when not given) by min(1, diffusion * D_p).
    """
    lib = _lib.load()
    P = bufs.near.numel()
    f = _lib.Frags()
    f.width, f.height = bufs.width, bufs.height
    f.npix, f.pixel_base = P, pixel_base
    f.opaque_color = ptr(bufs.opaque_color)
    if cfg.diffusion > 0.0 and blurred_image is None:
        blurred_image = resolve_blur(_background_image(bufs, full_opaque_image), cfg.diffusion_radius)
    b = bufs.c_struct(full_opaque_image, blurred_image)
    _lib.check(lib.woit_step4_composite(f, _params(cfg, bufs.rank), b, _stream()), "step4_composite")
    if counter is not None:
        counter.record_eval(P, P * (bufs.rank + 2))


def render_band(frame: FrameFragments, cfg: RenderConfig, rays: Optional[RayGrid] = None,
                bufs: Optional[FrameBuffers] = None, full_opaque_image: Optional[torch.Tensor] = None,
                vhat: bool = False, counter: Optional[TouchCounter] = None,
                ws: Optional[Workspace] = None, blurred_image: Optional[torch.Tensor] = None) -> FrameBuffers:
    """All four passes fused in one kernel (pipeline.py:321-330, _wavelet_band).

    With ``cfg.diffusion > 0`` the K_resolve blur of the background image runs
    first (``resolve_blur``; pass ``blurred_image`` to reuse one across bands).
    """
    lib = _lib.load()
    if bufs is None:
        bufs = FrameBuffers.allocate(frame, cfg.rank, vhat=vhat, packed=cfg.packed_storage)
    _check_frame(frame, bufs)
    if cfg.diffusion > 0.0 and blurred_image is None:
        blurred_image = resolve_blur(_background_image(frame, full_opaque_image), cfg.diffusion_radius)
    f, b = frame.c_struct(), bufs.c_struct(full_opaque_image, blurred_image)
    w, wn = _frame_ws(frame, ws)
    _lib.check(lib.woit_render_band(f, _params(cfg, bufs.rank, rays), b, ptr(w), wn, _stream()),
               "render_band")
    if counter is not None:
        counter.record_insert(frame.nfrag, frame.nfrag * (cfg.rank + 2))
        if frame.nfrag:
            counter.record_eval(2 * frame.nfrag, 2 * frame.nfrag * (cfg.rank + 2))
        counter.record_eval(frame.npix, frame.npix * (cfg.rank + 2))
    return bufs


def render_frame(scene, cfg: RenderConfig, counter: Optional[TouchCounter] = None,
                 frame: Optional[FrameFragments] = None) -> torch.Tensor:
    """Render the frame; returns linear (H, W, 3) fp32 on the device (pipeline.py:333-375).

    ``scene`` supplies the camera (any object with a ``camera`` attribute, or a
    Camera, or None for the default). ``workers > 1`` renders that many row bands
    one after another; the result is bit-identical to one band.
    """
    if frame is None:
        # cast on the device (scene.py:463-630 -> paper_2201_00094_b200.scene.cast_frame)
        from .scene import Scene, cast_frame

        if not isinstance(scene, Scene):
            raise ValueError("render_frame without frame= needs a Scene to cast")
        frame = cast_frame(scene, cfg.width, cfg.height)
    if frame.npix != cfg.width * cfg.height:
        raise ValueError("frame size does not match the config")
    if cfg.method != "wavelet":
        return render_baseline(frame, cfg).reshape(cfg.height, cfg.width, 3)
    cam = getattr(scene, "camera", scene) if scene is not None else None
    rays = camera_rays(cam if isinstance(cam, Camera) else _as_camera(cam), cfg.width, cfg.height)
    full_img = frame.opaque_color.reshape(cfg.height, cfg.width, 3)
    blurred = resolve_blur(full_img, cfg.diffusion_radius) if cfg.diffusion > 0.0 else None
    if cfg.workers == 1 or cfg.height < 2 * cfg.workers:
        bufs = render_band(frame, cfg, rays, full_opaque_image=full_img, counter=counter, blurred_image=blurred)
        return bufs.output.reshape(cfg.height, cfg.width, 3)
    rows = [int(r) for r in torch.linspace(0, cfg.height, cfg.workers + 1).to(torch.int64)]
    out = torch.empty(frame.npix, 3, dtype=torch.float32, device=frame.device)
    for r0, r1 in zip(rows[:-1], rows[1:]):
        if r0 >= r1:
            continue
        p0, p1 = r0 * cfg.width, r1 * cfg.width
        band = frame.band(p0, p1)
        bufs = render_band(band, cfg, rays, full_opaque_image=full_img, counter=counter, blurred_image=blurred)
        out[p0:p1] = bufs.output
    return out.reshape(cfg.height, cfg.width, 3)


_METHOD_IDS = {"abuffer": _lib.METHOD_ABUFFER, "wboit": _lib.METHOD_WBOIT, "mlab4": _lib.METHOD_MLAB4}


def render_baseline(frame: FrameFragments, cfg: RenderConfig, ws: Optional[Workspace] = None) -> torch.Tensor:
    """The reference's comparison methods over a frame (pipeline.py:341-354 ->
    baselines.abuffer_frame / wboit_frame / mlab_frame): (npix, 3) fp32 over the
    opaque colour, computed per pixel in float64."""
    if cfg.method not in _METHOD_IDS:
        raise ValueError(f"{cfg.method!r} is not a comparison method")
    lib = _lib.load()
    method = _METHOD_IDS[cfg.method]
    out = torch.empty(frame.npix, 3, dtype=torch.float32, device=frame.device)
    n = lib.woit_baseline_workspace_bytes(method, frame.npix, frame.nfrag)
    t = _scratch(n, frame.device, ws)
    wb = (C.c_double * 3)(*[float(x) for x in cfg.wboit_weight])
    flags = _lib.CUBE_TRANSMISSION if cfg.cube_transmission else 0
    _lib.check(lib.woit_render_baseline(frame.c_struct(), method, flags, C.cast(wb, C.c_void_p), ptr(out),
                                        ptr(t), t.numel(), _stream()), "render_baseline")
    return out


def _as_camera(cam) -> Camera:
    if cam is None:
        return Camera()
    return Camera(tuple(cam.position), tuple(cam.forward), float(cam.fov_deg))
