"""Analytic scenes and the on-device fragment producer.

Mirrors the reference's scene description (scene.py:44-190: Material, Plane,
Sphere, FogSlab, ParticleCloud, OpaqueBackdrop, Background, Scene and the
presets, scene.py:630-760) and replaces its vectorised caster ``cast_frame``
(scene.py:463-630) with ``woit_cast_offsets`` / ``woit_cast_fill``: one CUDA
thread per pixel casts the primary ray in float64 and writes the CSR stream in
cast_frame's row order straight into HBM, so real presets run at 4K/8K without
a host round trip. The scene itself (a few primitives; particle positions drawn
with numpy's generator exactly as the reference seeds them) is set up on the
host -- it is not on the hot path.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, replace
from typing import Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from .frame import FrameFragments, ptr
from .pipeline import Camera, _stream

RAY_EPS = 1e-9  # scene.py:41
Spectrum = Tuple[float, float, float]


def gray(v: float) -> Spectrum:
    return (v, v, v)


@dataclass(frozen=True)
class Material:
    alpha: float = 1.0
    transmission: Spectrum = gray(1.0)
    radiance: Spectrum = gray(0.0)
    ior: float = 1.0


@dataclass(frozen=True)
class Plane:
    """Camera-facing plane (a pane when ``extent`` is set) at forward distance d."""

    d: float
    material: Material
    extent: Optional[Tuple[float, float]] = None
    center: Tuple[float, float] = (0.0, 0.0)


@dataclass(frozen=True)
class Sphere:
    center: Tuple[float, float, float]
    radius: float
    material: Material


@dataclass(frozen=True)
class FogSlab:
    near: float
    far: float
    sigma: Spectrum
    slices: int = 32
    color: Spectrum = gray(0.0)

    def __post_init__(self):
        if self.slices < 1:
            raise ValueError("fog slab needs at least one slice")
        if any(s < 0.0 for s in self.sigma):
            raise ValueError("fog extinction must be nonnegative")


@dataclass(frozen=True)
class ParticleCloud:
    """Seeded camera-facing discs uniform in a sphere (scene.py:93-122)."""

    center: Tuple[float, float, float]
    radius: float
    count: int
    particle_radius: float
    material: Material
    profile: str = "gauss"
    seed_offset: int = 0
    positions: Optional[np.ndarray] = None
    radiance_scale: Optional[np.ndarray] = None

    def __post_init__(self):
        if self.profile not in ("gauss", "mask"):
            raise ValueError(f"unknown particle profile {self.profile!r}")

    def seeded(self, scene_seed: int) -> "ParticleCloud":
        # the reference's draws, in its order: directions, radii, radiance scales
        rng = np.random.default_rng((scene_seed + self.seed_offset) & 0xFFFFFFFFFFFFFFFF)
        dirs = rng.normal(size=(self.count, 3))
        dirs /= np.sqrt((dirs * dirs).sum(axis=1))[:, None]
        rad = self.radius * np.cbrt(rng.uniform(0.0, 1.0, self.count))
        pos = np.asarray(self.center, dtype=np.float64) + dirs * rad[:, None]
        scale = rng.uniform(0.7, 1.3, self.count)
        return replace(self, positions=pos, radiance_scale=scale)


@dataclass(frozen=True)
class OpaqueBackdrop:
    d: float
    color: Spectrum
    checker: Optional[Spectrum] = None
    cell: float = 0.5


@dataclass(frozen=True)
class Background:
    color: Spectrum = (0.05, 0.06, 0.08)
    checker: Optional[Spectrum] = None
    cell: int = 16


@dataclass(frozen=True)
class Scene:
    camera: Camera
    primitives: Tuple[object, ...]
    background: Background = Background()
    rng_seed: int = 0

    def __post_init__(self):
        prims = tuple(p.seeded(self.rng_seed) if isinstance(p, ParticleCloud) else p for p in self.primitives)
        object.__setattr__(self, "primitives", prims)


# ---------------------------------------------------------------------------
# presets (scene.py:632-760): the same primitives, materials and seeds


def _single_plane() -> Scene:
    return Scene(Camera(), (Plane(1.0, Material(0.25, gray(0.0), (0.18, 0.18, 0.20))),
                            OpaqueBackdrop(2.0, (0.85, 0.45, 0.12))))


def _wine_bottle() -> Scene:
    glass = Material(1.0, (0.96, 0.97, 0.96), (0.040, 0.040, 0.045), 1.5)
    wine = Material(1.0, (0.74, 0.25, 0.34), (0.020, 0.005, 0.008), 1.12)
    return Scene(Camera(), (Sphere((0.0, 0.0, 1.5), 0.5, glass), Sphere((0.0, 0.0, 1.5), 0.35, wine),
                            OpaqueBackdrop(3.0, (0.85, 0.80, 0.72), (0.25, 0.22, 0.20), 0.35)))


def _car_fog() -> Scene:
    window = Material(0.95, (0.30, 0.34, 0.38), (0.050, 0.060, 0.070), 1.5)
    window2 = Material(0.95, (0.35, 0.38, 0.40), (0.030, 0.035, 0.040), 1.5)
    return Scene(Camera(), (FogSlab(0.5, 4.0, (0.35, 0.40, 0.45), 32, (0.55, 0.60, 0.68)),
                            Plane(2.0, window, (1.1, 0.65), (0.0, 0.0)),
                            Plane(2.6, window2, (1.1, 0.65), (0.15, 0.0)),
                            OpaqueBackdrop(4.5, (0.10, 0.09, 0.08))))


def _smoke_fire() -> Scene:
    smoke = Material(0.40, (0.30, 0.30, 0.33), (0.38, 0.40, 0.44))
    fire = Material(0.50, (0.05, 0.03, 0.02), (1.30, 0.45, 0.10))
    return Scene(Camera(), (ParticleCloud((-0.35, 0.05, 2.3), 0.65, 130, 0.085, smoke, "gauss", 1),
                            ParticleCloud((0.45, -0.12, 1.6), 0.42, 90, 0.070, fire, "gauss", 2),
                            OpaqueBackdrop(3.2, (0.90, 0.50, 0.14))), rng_seed=7)


def _glass_stack() -> Scene:
    tints = ((0.93, 0.95, 0.97), (0.96, 0.93, 0.91), (0.94, 0.96, 0.93), (0.95, 0.94, 0.96),
             (0.94, 0.95, 0.96), (0.70, 0.74, 0.68), (0.93, 0.94, 0.92), (0.66, 0.72, 0.76))
    highlights = (0.045, 0.035, 0.050, 0.040, 0.080, 0.010, 0.080, 0.010)
    panes = []
    for i in range(8):
        h = highlights[i]
        m = Material(1.0, tints[i], (1.00 * h, 0.95 * h, 0.88 * h), 1.5)
        panes.append(Plane(1.0 + 0.25 * i, m, (1.25 - 0.07 * i, 0.95 - 0.05 * i), (0.12 if i % 2 else -0.06, 0.0)))
    prims = [panes[i] for i in (0, 1, 3, 5, 7, 2, 4, 6)]  # scrambled submission order
    prims.append(OpaqueBackdrop(3.5, (0.82, 0.74, 0.62), (0.28, 0.24, 0.20), 0.45))
    return Scene(Camera(), tuple(prims))


def _leaves() -> Scene:
    leaf = Material(0.92, (0.06, 0.12, 0.04), (0.10, 0.35, 0.07))
    return Scene(Camera(), (ParticleCloud((0.0, 0.0, 1.5), 0.55, 48, 0.16, leaf, "mask", 3),
                            OpaqueBackdrop(3.0, (0.55, 0.68, 0.88), (0.42, 0.50, 0.62), 0.6)), rng_seed=11)


_PRESETS = {"single-plane": _single_plane, "wine-bottle": _wine_bottle, "car-fog": _car_fog,
            "smoke-fire": _smoke_fire, "glass-stack": _glass_stack, "leaves": _leaves}
PRESET_NAMES = tuple(sorted(_PRESETS))


def preset(name: str) -> Scene:
    try:
        return _PRESETS[name]()
    except KeyError:
        raise ValueError(f"unknown preset {name!r}; valid presets: {', '.join(PRESET_NAMES)}") from None


# ---------------------------------------------------------------------------
# scene description files (the grammar of scene.py:1-26, parse_scene :783-850)


def _floats(text: str, n: int) -> Tuple[float, ...]:
    parts = text.split(",")
    if len(parts) != n:
        raise ValueError(f"expected {n} comma-separated numbers, got {text!r}")
    return tuple(float(p) for p in parts)


def _material(kv) -> Material:
    return Material(float(kv.pop("alpha", 1.0)), _floats(kv.pop("transmission", "1,1,1"), 3),
                    _floats(kv.pop("radiance", "0,0,0"), 3), float(kv.pop("ior", 1.0)))


def parse_scene(text: str) -> Scene:
    camera, background, seed, prims = Camera(), Background(), 0, []
    for line_no, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        head, *rest = line.split()
        if head == "seed":
            if len(rest) != 1:
                raise ValueError(f"line {line_no}: seed takes one integer")
            seed = int(rest[0])
            continue
        kv = {}
        for tok in rest:
            if "=" not in tok:
                raise ValueError(f"line {line_no}: expected key=value, got {tok!r}")
            k, v = tok.split("=", 1)
            kv[k] = v
        try:
            if head == "camera":
                camera = Camera(_floats(kv.pop("pos", "0,0,0"), 3), _floats(kv.pop("forward", "0,0,1"), 3),
                                float(kv.pop("fov", 60.0)))
            elif head == "background":
                checker = kv.pop("checker", None)
                background = Background(_floats(kv.pop("color", "0.05,0.06,0.08"), 3),
                                        _floats(checker, 3) if checker else None, int(kv.pop("cell", 16)))
            elif head == "plane":
                d = float(kv.pop("d"))
                extent = kv.pop("extent", None)
                center = kv.pop("center", "0,0")
                prims.append(Plane(d, _material(kv), _floats(extent, 2) if extent else None, _floats(center, 2)))
            elif head == "sphere":
                center = _floats(kv.pop("center"), 3)
                radius = float(kv.pop("radius"))
                prims.append(Sphere(center, radius, _material(kv)))
            elif head == "fog_slab":
                prims.append(FogSlab(float(kv.pop("near")), float(kv.pop("far")), _floats(kv.pop("sigma"), 3),
                                     int(kv.pop("slices", 32)), _floats(kv.pop("color", "0,0,0"), 3)))
            elif head == "particle_cloud":
                center = _floats(kv.pop("center"), 3)
                radius = float(kv.pop("radius"))
                count = int(kv.pop("count"))
                pr = float(kv.pop("particle_radius"))
                profile = kv.pop("profile", "gauss")
                seed_offset = int(kv.pop("seed_offset", 0))
                prims.append(ParticleCloud(center, radius, count, pr, _material(kv), profile, seed_offset))
            elif head == "opaque_backdrop":
                checker = kv.pop("checker", None)
                prims.append(OpaqueBackdrop(float(kv.pop("d")), _floats(kv.pop("color"), 3),
                                            _floats(checker, 3) if checker else None, float(kv.pop("cell", 0.5))))
            else:
                raise ValueError(f"unknown primitive {head!r}")
        except KeyError as exc:
            raise ValueError(f"line {line_no}: {head} is missing required key {exc}") from None
        if kv:
            raise ValueError(f"line {line_no}: unknown keys for {head}: {', '.join(sorted(kv))}")
    return Scene(camera, tuple(prims), background, seed)


def load_scene(path) -> Scene:
    with open(path, "r", encoding="utf-8") as fh:
        return parse_scene(fh.read())


def resolve_scene(name_or_path: str) -> Scene:
    """Preset name, or path to a scene description file."""
    import os

    return load_scene(name_or_path) if os.path.exists(name_or_path) else preset(name_or_path)


# ---------------------------------------------------------------------------
# device scene + caster


def _camera_frame(cam: Camera, width: int, height: int):
    f, right, up = (np.asarray(v, dtype=np.float64) for v in cam.basis())
    tan_half = math.tan(math.radians(cam.fov_deg) * 0.5)
    return np.asarray(cam.position, dtype=np.float64), f, right, up, tan_half, width / height


def particle_boxes(cloud: ParticleCloud, cam: Camera, width: int, height: int) -> np.ndarray:
    """cast_frame's conservative per-particle screen box (scene.py:580-600) with the
    reference's arithmetic; x0 > x1 marks a culled particle (behind the near limit
    or off screen)."""
    o, f, right, up, tan_half, aspect = _camera_frame(cam, width, height)
    box = np.empty((cloud.count, 4), dtype=np.int32)
    for i in range(cloud.count):
        p = cloud.positions[i]
        rel = p - o
        zf = float(rel @ f)
        zmin = zf - cloud.particle_radius
        box[i] = (1, 0, 1, 0)
        if zmin <= RAY_EPS:
            continue
        sx = float(rel @ right) / (zf * tan_half * aspect)
        sy = float(rel @ up) / (zf * tan_half)
        cx = (sx + 1.0) * 0.5 * width - 0.5
        cy = (1.0 - sy) * 0.5 * height - 0.5
        tx = tan_half * aspect
        ty = tan_half
        rx = cloud.particle_radius * (1.0 + abs(sx) * tx) / (zmin * tx) * (width * 0.5) * 1.05 + 2.0
        ry = cloud.particle_radius * (1.0 + abs(sy) * ty) / (zmin * ty) * (height * 0.5) * 1.05 + 2.0
        x0, x1 = max(0, int(cx - rx)), min(width - 1, int(cx + rx) + 1)
        y0, y1 = max(0, int(cy - ry)), min(height - 1, int(cy + ry) + 1)
        if x0 > x1 or y0 > y1:
            continue
        box[i] = (x0, x1, y0, y1)
    return box


class DeviceScene:
    """A Scene packed as woit_scene_t / woit_prim_t with device-resident arrays."""

    def __init__(self, scene: Scene, width: int, height: int, device=None):
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.keep = []
        prims = (_lib.Prim * max(1, len(scene.primitives)))()
        for i, pr in enumerate(scene.primitives):
            q = prims[i]
            m = getattr(pr, "material", None)
            if m is not None:
                q.alpha, q.ior = float(m.alpha), float(m.ior)
                q.trans[:] = [float(x) for x in m.transmission]
                q.radiance[:] = [float(x) for x in m.radiance]
            if isinstance(pr, Plane):
                q.kind, q.d = _lib.PRIM_PLANE, float(pr.d)
                if pr.extent is not None:
                    q.flags |= 1
                    q.extent[:] = [float(x) for x in pr.extent]
                    q.pcenter[:] = [float(x) for x in pr.center]
            elif isinstance(pr, Sphere):
                q.kind, q.radius = _lib.PRIM_SPHERE, float(pr.radius)
                q.center[:] = [float(x) for x in pr.center]
            elif isinstance(pr, FogSlab):
                q.kind, q.count, q.near, q.far = _lib.PRIM_FOG, int(pr.slices), float(pr.near), float(pr.far)
                q.sigma[:] = [float(x) for x in pr.sigma]
                q.color[:] = [float(x) for x in pr.color]
            elif isinstance(pr, ParticleCloud):
                q.kind, q.count, q.profile = _lib.PRIM_PARTICLES, int(pr.count), 0 if pr.profile == "gauss" else 1
                q.particle_radius = float(pr.particle_radius)
                q.center[:] = [float(x) for x in pr.center]
                pos = torch.as_tensor(np.ascontiguousarray(pr.positions, dtype=np.float64), device=dev)
                sc = torch.as_tensor(np.ascontiguousarray(pr.radiance_scale, dtype=np.float64), device=dev)
                box = torch.as_tensor(particle_boxes(pr, scene.camera, width, height), device=dev)
                self.keep += [pos, sc, box]
                q.positions, q.radiance_scale, q.box = ptr(pos), ptr(sc), ptr(box)
            elif isinstance(pr, OpaqueBackdrop):
                q.kind, q.d, q.cell = _lib.PRIM_BACKDROP, float(pr.d), float(pr.cell)
                q.color[:] = [float(x) for x in pr.color]
                if pr.checker is not None:
                    q.flags |= 2
                    q.checker[:] = [float(x) for x in pr.checker]
            else:
                raise TypeError(f"unknown primitive {type(pr).__name__}")
        raw = torch.frombuffer(bytearray(bytes(prims)), dtype=torch.uint8).to(dev)
        self.keep.append(raw)
        s = _lib.SceneC()
        s.nprims = len(scene.primitives)
        s.prims = ptr(raw)
        o, f, right, up, tan_half, aspect = _camera_frame(scene.camera, width, height)
        s.origin[:], s.forward[:], s.right[:], s.up[:] = list(o), list(f), list(right), list(up)
        s.tan_half, s.aspect = tan_half, aspect
        bg = scene.background
        s.bg_color[:] = [float(x) for x in bg.color]
        if bg.checker is not None:
            s.bg_has_checker, s.bg_cell = 1, int(bg.cell)
            s.bg_checker[:] = [float(x) for x in bg.checker]
        self.c = s
        self.device = dev


def cast_frame(scene: Scene, width: int, height: int, device=None) -> FrameFragments:
    """Fragments of every pixel, in HBM (scene.py:463-630 cast_frame, on the GPU)."""
    if width < 1 or height < 1:
        raise ValueError("frame must be at least 1x1")
    lib = _lib.load()
    ds = DeviceScene(scene, width, height, device)
    dev = ds.device
    npix = width * height
    with torch.cuda.device(dev):
        offsets = torch.empty(npix + 1, dtype=torch.int64, device=dev)
        ws = torch.empty(lib.woit_cast_workspace_bytes(npix), dtype=torch.uint8, device=dev)
        _lib.check(lib.woit_cast_offsets(ds.c, width, height, ptr(offsets), ptr(ws), ws.numel(), _stream()),
                   "woit_cast_offsets")
        n = int(offsets[-1].item())
        f = lambda *s: torch.empty(*s, dtype=torch.float32, device=dev)
        depth, alpha, ior = f(n), f(n), f(n)
        trans, rad, normal = f(n, 3), f(n, 3), f(n, 3)
        bf = torch.empty(n, dtype=torch.uint8, device=dev)
        od, oc = f(npix), f(npix, 3)
        _lib.check(lib.woit_cast_fill(ds.c, width, height, ptr(offsets), ptr(depth), ptr(alpha), ptr(trans), ptr(rad),
                                      ptr(normal), ptr(ior), ptr(bf), ptr(od), ptr(oc), _stream()), "woit_cast_fill")
        torch.cuda.current_stream(dev).synchronize()  # the scene's host structs go out of scope
    return FrameFragments(width, height, offsets, depth, alpha, trans, rad, normal, ior, bf, od, oc, 0, 0)
