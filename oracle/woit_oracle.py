"""CPU oracle for the wavelet OIT hot path — TEST INFRASTRUCTURE ONLY.

This module is a float64 numpy restatement of the reference ``woit`` package's
four-pass wavelet compositor (``/root/reference/pkg/src/woit``) and is used as
the *checker*: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
The product path (``paper_2201_00094_b200``) never imports, links or falls back
to anything here.

Parity pinning: ``tests/golden/make_golden.py`` runs the *reference itself*
(imported from /root/reference in the build container) on the same inputs and
commits the outputs as fixtures; ``tests/test_oracle.py`` checks this module
against those fixtures (<= 1e-12) and against the reference tests' own
hand-derived known-answer values.

Every function cites the reference lines it restates. Arithmetic order follows
the reference where it matters for bit-exact indices (z, slot and cell ids).
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np

TRANSMITTANCE_FLOOR = 1e-6      # core.py:23
EPS_Z = 2.0 ** -24              # wavelet.py:32
NORM_EPS = 1e-6                 # pipeline.py:41
DIR_EPS = 1e-9                  # pipeline.py:42
WORLD_UP = (0.0, 1.0, 0.0)      # scene.py:43
ALT_UP = (1.0, 0.0, 0.0)        # scene.py:44


# ---------------------------------------------------------------------------
# inputs


@dataclass
class OFrame:
    """CSR-by-pixel fragment stream in float64 (scene.py:367-392 field set)."""

    width: int
    height: int
    pixel: np.ndarray
    depth: np.ndarray
    alpha: np.ndarray
    trans: np.ndarray
    radiance: np.ndarray
    normal: np.ndarray
    ior: np.ndarray
    backface: np.ndarray
    offsets: np.ndarray
    opaque_depth: np.ndarray
    opaque_color: np.ndarray

    @property
    def npix(self) -> int:
        return self.offsets.size - 1

    @classmethod
    def from_arrays(cls, width, height, offsets, depth, alpha, trans, radiance,
                    normal=None, ior=None, backface=None, opaque_depth=None,
                    opaque_color=None) -> "OFrame":
        """Upcast an fp32 SoA stream (the device layout) to the oracle's f64."""
        offsets = np.asarray(offsets, dtype=np.int64)
        npix = offsets.size - 1
        n = int(offsets[-1])
        f64 = lambda a: np.asarray(a, dtype=np.float64)
        if normal is None:
            normal = np.tile([0.0, 0.0, -1.0], (n, 1))
        if ior is None:
            ior = np.ones(n)
        if backface is None:
            backface = np.zeros(n, dtype=bool)
        if opaque_depth is None:
            opaque_depth = np.full(npix, np.inf)
        if opaque_color is None:
            opaque_color = np.zeros((npix, 3))
        pixel = np.repeat(np.arange(npix, dtype=np.int64), np.diff(offsets))
        return cls(width, height, pixel, f64(depth), f64(alpha), f64(trans).reshape(n, 3),
                   f64(radiance).reshape(n, 3), f64(normal).reshape(n, 3), f64(ior),
                   np.asarray(backface).astype(bool), offsets, f64(opaque_depth),
                   f64(opaque_color).reshape(npix, 3))

    @classmethod
    def from_synth(cls, sf) -> "OFrame":
        return cls.from_arrays(sf.width, sf.rows, sf.offsets, sf.depth, sf.alpha, sf.trans,
                               sf.radiance, sf.normal, sf.ior, sf.backface, sf.opaque_depth,
                               sf.opaque_color)

    def net_transmittance(self, cube: bool = False, cube_backface_only: bool = False) -> np.ndarray:
        """t = 1 - alpha (1 - T'), T' = T^3 on cubed refractive fragments (scene.py:394-402)."""
        T = self.trans
        if cube:
            sel = self.ior > 1.0
            if cube_backface_only:
                sel = sel & self.backface
            T = np.where(sel[:, None], T * T * T, T)
        return 1.0 - self.alpha[:, None] * (1.0 - T)

    def band(self, p0: int, p1: int) -> "OFrame":
        """Contiguous pixel band with rebased ids/offsets (pipeline.py:311-318)."""
        lo, hi = int(self.offsets[p0]), int(self.offsets[p1])
        return OFrame(self.width, self.height, self.pixel[lo:hi] - p0, self.depth[lo:hi],
                      self.alpha[lo:hi], self.trans[lo:hi], self.radiance[lo:hi],
                      self.normal[lo:hi], self.ior[lo:hi], self.backface[lo:hi],
                      self.offsets[p0:p1 + 1] - lo, self.opaque_depth[p0:p1],
                      self.opaque_color[p0:p1])


@dataclass(frozen=True)
class OConfig:
    """Wavelet-method subset of RenderConfig (pipeline.py:45-73)."""

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
    diffusion: float = 0.0        # in-repo diffusion (no reference twin; see blur_image)
    diffusion_radius: int = 4


@dataclass(frozen=True)
class OCamera:
    """Camera of scene.py:135-150; the default looks down +z."""

    position: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    forward: Tuple[float, float, float] = (0.0, 0.0, 1.0)
    fov_deg: float = 60.0


# ---------------------------------------------------------------------------
# camera (scene.py:141-150, 199-212)


def camera_basis(cam: OCamera):
    f = np.asarray(cam.forward, dtype=np.float64)
    f = f / np.sqrt((f * f).sum())
    up0 = np.asarray(WORLD_UP if abs(float(f @ np.asarray(WORLD_UP))) <= 0.999 else ALT_UP,
                     dtype=np.float64)
    right = np.cross(up0, f)
    right = right / np.sqrt((right * right).sum())
    up = np.cross(f, right)
    return f, right, up


def ray_dirs(cam: OCamera, width: int, height: int) -> np.ndarray:
    """Unit primary ray direction per pixel, row-major (scene.py:199-212)."""
    f, right, up = camera_basis(cam)
    tan_half = math.tan(math.radians(cam.fov_deg) * 0.5)
    aspect = width / height
    u = (2.0 * (np.arange(width, dtype=np.float64) + 0.5) / width - 1.0) * tan_half * aspect
    v = (1.0 - 2.0 * (np.arange(height, dtype=np.float64) + 0.5) / height) * tan_half
    d = (f[None, None, :] + u[None, :, None] * right[None, None, :]
         + v[:, None, None] * up[None, None, :]).reshape(-1, 3)
    d /= np.sqrt((d * d).sum(axis=1))[:, None]
    return d


# ---------------------------------------------------------------------------
# Haar math (wavelet.py)


def eval_bounds(near: np.ndarray, far: np.ndarray, rank: int):
    """Padded mapping bounds: one cell of margin each side (pipeline.py:110-128)."""
    cells = 1 << (rank + 1)
    covered = near <= far
    rng = np.where(covered, far - near, 0.0)
    if cells > 2:
        margin = rng / (cells - 2)
        return np.where(covered, near - margin, near), np.where(covered, far + margin, far)
    return near, np.where(covered, far + rng, far)


def normalize_depth_array(x, near, far):
    """z in [0, 1 - 2^-24] over padded bounds (wavelet.py:130-135)."""
    rng = far - near
    pad = np.maximum(1e-4 * rng, 1e-6)
    return np.clip((x - (near - pad)) / (rng + 2.0 * pad), 0.0, 1.0 - EPS_Z)


def slot_indices(z: np.ndarray, rank: int) -> np.ndarray:
    """k_n = min(floor(2^n z), 2^n - 1) per level, shape (n, rank+1) (wavelet.py:281)."""
    out = np.empty((z.size, rank + 1), dtype=np.int64)
    for n in range(rank + 1):
        s = 1 << n
        out[:, n] = np.minimum((s * z).astype(np.int64), s - 1)
    return out


def cell_indices(z: np.ndarray, rank: int):
    """(c0, c1, t) of the interpolated evaluation (wavelet.py:309-315)."""
    M = 1 << (rank + 1)
    u = z * M - 0.5
    c0 = np.floor(u).astype(np.int64)
    t = np.where((c0 < 0) | (c0 >= M - 1), 0.0, u - c0)
    c0 = np.clip(c0, 0, M - 1)
    return c0, np.minimum(c0 + 1, M - 1), t


def build_into(coeffs, pix, z, a, rank) -> None:
    """Closed-form scatter of absorbance steps (wavelet.py:272-287)."""
    if z.size == 0:
        return
    np.add.at(coeffs, (pix, 0), a * (1.0 - z)[:, None])
    for n in range(rank + 1):
        s = 1 << n
        k = np.minimum((s * z).astype(np.int64), s - 1)
        u = s * z - k
        psi = 2.0 ** (-0.5 * n) * np.minimum(u, 1.0 - u)
        np.add.at(coeffs, (pix, s + k), -(a * psi[:, None]))


def cells_raw_batch(coeffs, pix, cells, rank):
    """Staircase value at a cell centre (wavelet.py:290-303)."""
    val = coeffs[pix, 0, :].copy()
    for n in range(rank + 1):
        m = rank + 1 - n
        sign = 1.0 - 2.0 * ((cells >> (m - 1)) & 1)
        val += 2.0 ** (0.5 * n) * sign[:, None] * coeffs[pix, (1 << n) + (cells >> m), :]
    return val


def interp_absorbance_batch(coeffs, pix, z, rank):
    """Lerp between adjacent cell centres, clamped >= 0 (wavelet.py:306-319)."""
    c0, c1, t = cell_indices(z, rank)
    left = cells_raw_batch(coeffs, pix, c0, rank)
    right = cells_raw_batch(coeffs, pix, c1, rank)
    return np.maximum((1.0 - t)[:, None] * left + t[:, None] * right, 0.0)


def total_absorbance_batch(coeffs, rank):
    """A(z -> 1) per pixel (wavelet.py:322-337)."""
    val = coeffs[:, 0, :].copy()
    for n in range(rank + 1):
        val -= 2.0 ** (0.5 * n) * coeffs[:, (1 << (n + 1)) - 1, :]
    return np.maximum(val, 0.0)


# ---------------------------------------------------------------------------
# E5B9G9R9 packing (packing.py:46-111)

_MANT = 9
_BIAS = 15
_MMAX = (1 << _MANT) - 1
MAX_PACKED = float(_MMAX) / (1 << _MANT) * 2.0 ** (31 - _BIAS)


def pack_rgb9e5(v) -> np.ndarray:
    v = np.asarray(v, dtype=np.float64)
    if np.any(np.isnan(v)):
        raise ValueError("cannot pack NaN")
    v = np.clip(v, 0.0, MAX_PACKED)
    mx = v.max(axis=-1)
    with np.errstate(divide="ignore"):
        fl = np.floor(np.log2(mx, where=mx > 0.0, out=np.full_like(mx, -np.inf)))
    e = np.maximum(np.maximum(-_BIAS - 1.0, fl) + 1.0 + _BIAS, 0.0)
    scale = np.exp2(e - _BIAS - _MANT)
    bump = np.floor(mx / scale + 0.5) >= (1 << _MANT)
    e = e + bump
    scale = np.where(bump, 2.0 * scale, scale)
    m = np.minimum(np.floor(v / scale[..., None] + 0.5).astype(np.uint32), _MMAX)
    return (m[..., 0] | (m[..., 1] << 9) | (m[..., 2] << 18)
            | (e.astype(np.uint32) << 27)).astype(np.uint32)


def unpack_rgb9e5(w) -> np.ndarray:
    w = np.asarray(w, dtype=np.uint64)
    scale = np.exp2(((w >> 27) & 31).astype(np.float64) - _BIAS - _MANT)
    out = np.stack([(w & _MMAX), ((w >> 9) & _MMAX), ((w >> 18) & _MMAX)], axis=-1)
    return out.astype(np.float64) * scale[..., None]


def roundtrip_coeffs(coeffs) -> np.ndarray:
    """Packed storage: |c| quantised, slot 0 positive, others negative (packing.py:107-111)."""
    out = unpack_rgb9e5(pack_rgb9e5(np.abs(coeffs)))
    out[:, 1:, :] *= -1.0
    return out


# ---------------------------------------------------------------------------
# the four passes (pipeline.py:76-308)


@dataclass
class OBuffers:
    """Per-pixel state, as FrameBuffers.allocate (pipeline.py:93-104)."""

    width: int
    height: int
    rank: int
    near: np.ndarray
    far: np.ndarray
    coeffs: np.ndarray
    accum: np.ndarray
    accum_weight: np.ndarray
    refraction_offset: np.ndarray
    opaque_depth: np.ndarray
    opaque_color: np.ndarray
    output: np.ndarray
    vhat: Optional[np.ndarray] = field(default=None)
    diffusion: Optional[np.ndarray] = field(default=None)

    @classmethod
    def allocate(cls, frame: OFrame, rank: int) -> "OBuffers":
        P = frame.npix
        return cls(frame.width, frame.height, rank, np.full(P, np.inf), np.full(P, -np.inf),
                   np.zeros((P, 1 << (rank + 1), 3)), np.zeros((P, 3)), np.zeros((P, 3)),
                   np.zeros((P, 2)), frame.opaque_depth.copy(), frame.opaque_color.copy(),
                   np.zeros((P, 3)), None, np.zeros(P))


def fragment_z(frame: OFrame, bufs: OBuffers) -> np.ndarray:
    """pipeline.py:137-140."""
    ne, fe = eval_bounds(bufs.near, bufs.far, bufs.rank)
    return normalize_depth_array(frame.depth, ne[frame.pixel], fe[frame.pixel])


def fragment_absorbance(frame: OFrame, cfg: OConfig) -> np.ndarray:
    """-ln(max(1e-6, t)) per channel (pipeline.py:143-145)."""
    t = frame.net_transmittance(cfg.cube_transmission, cfg.cube_backface_only)
    return -np.log(np.maximum(TRANSMITTANCE_FLOOR, t))


def step1_depth_bounds(frame: OFrame, bufs: OBuffers) -> None:
    """pipeline.py:131-134."""
    np.minimum.at(bufs.near, frame.pixel, frame.depth)
    np.maximum.at(bufs.far, frame.pixel, frame.depth)


def step2_build(frame: OFrame, bufs: OBuffers, cfg: OConfig) -> None:
    """pipeline.py:148-155."""
    build_into(bufs.coeffs, frame.pixel, fragment_z(frame, bufs),
               fragment_absorbance(frame, cfg), bufs.rank)
    if cfg.packed_storage:
        bufs.coeffs = roundtrip_coeffs(bufs.coeffs)


def step3_accumulate(dirs: np.ndarray, forward, right, up, frame: OFrame, bufs: OBuffers,
                     cfg: OConfig, pixel_base: int = 0) -> None:
    """Visibility-weighted accumulation + refraction offsets (pipeline.py:170-217).

    Also records the per-fragment transmittance v̂ in ``bufs.vhat``.
    """
    if frame.pixel.size == 0:
        bufs.vhat = np.zeros((0, 3))
        return
    z = fragment_z(frame, bufs)
    vhat = np.exp(-interp_absorbance_batch(bufs.coeffs, frame.pixel, z, bufs.rank))
    bufs.vhat = vhat
    np.add.at(bufs.accum, frame.pixel, frame.radiance * frame.alpha[:, None] * vhat)
    opac = 1.0 - frame.net_transmittance(cfg.cube_transmission, cfg.cube_backface_only)
    np.add.at(bufs.accum_weight, frame.pixel, opac * vhat)
    if cfg.diffusion > 0.0:
        # in-repo diffusion coverage D_p = sum alpha * mean(v̂) (include/woit.h WOIT_DIFFUSION)
        np.add.at(bufs.diffusion, frame.pixel, frame.alpha * vhat.sum(axis=1) / 3.0)
    if not cfg.refraction:
        return
    sel = np.nonzero(frame.ior > 1.0)[0]
    if sel.size == 0:
        return
    pix = frame.pixel[sel]
    d = dirs[pixel_base + pix]
    n = frame.normal[sel]
    ci = -(d * n).sum(axis=1)
    eta = 1.0 / frame.ior[sel]
    s2 = eta * eta * (1.0 - ci * ci)
    t_opq = bufs.opaque_depth[pix]
    ok = (ci > DIR_EPS) & (s2 <= 1.0) & np.isfinite(t_opq)
    tdir = eta[:, None] * d + (eta * ci - np.sqrt(np.clip(1.0 - s2, 0.0, None)))[:, None] * n
    tdir_f = tdir @ forward
    dir_f = d @ forward
    ok &= tdir_f > DIR_EPS
    s = np.where(ok, (t_opq * dir_f - frame.depth[sel] * dir_f) / np.where(ok, tdir_f, 1.0), 0.0)
    dw = (frame.depth[sel, None] * d + s[:, None] * tdir) - t_opq[:, None] * d
    off = np.stack([dw @ right, -(dw @ up)], axis=1) * (cfg.refraction_scale * (bufs.width / 512.0))
    off = np.where((ok & np.isfinite(off).all(axis=1))[:, None], off, 0.0)
    np.add.at(bufs.refraction_offset, pix, off)


def smoothstep(e0, e1, x):
    """pipeline.py:220-223."""
    u = min(1.0, max(0.0, (x - e0) / (e1 - e0)))
    return u * u * (3.0 - 2.0 * u)


def spectral_weight(i: int, k: int, literal_t: bool = False) -> np.ndarray:
    """(w_r, w_g, w_b) of aberration tap i of k (pipeline.py:226-239)."""
    if not (0 <= i < k):
        raise ValueError(f"tap index {i} out of range for k={k}")
    t = 0.5 + 2.0 * i / (k - 1) if literal_t else i / (k - 1)
    wr = smoothstep(0.5, 1.0 / 3.0, t)
    wb = smoothstep(0.5, 2.0 / 3.0, t)
    return np.array([wr, 1.0 - wr - wb, wb])


def bilinear_sample(img, x, y):
    """Edge-clamped bilinear lookup (pipeline.py:242-255)."""
    h, w = img.shape[:2]
    x = np.clip(x, 0.0, w - 1.0)
    y = np.clip(y, 0.0, h - 1.0)
    x0 = np.floor(x).astype(np.int64)
    y0 = np.floor(y).astype(np.int64)
    x1 = np.minimum(x0 + 1, w - 1)
    y1 = np.minimum(y0 + 1, h - 1)
    tx = (x - x0)[..., None]
    ty = (y - y0)[..., None]
    top = img[y0, x0] * (1.0 - tx) + img[y0, x1] * tx
    bot = img[y1, x0] * (1.0 - tx) + img[y1, x1] * tx
    return top * (1.0 - ty) + bot * ty


def chromatic_gather(img, px, py, offset, k, literal_t=False):
    """k-tap spectrally weighted gather along the offset (pipeline.py:258-281)."""
    num = np.zeros(px.shape + (3,))
    den = np.zeros(3)
    for i in range(k):
        w = spectral_weight(i, k, literal_t)
        fac = 2.0 * i / (k - 1)
        num += w * bilinear_sample(img, px + offset[..., 0] * fac, py + offset[..., 1] * fac)
        den += w
    center = bilinear_sample(img, px + offset[..., 0], py + offset[..., 1])
    safe = den > 0.0
    return np.where(safe, num / np.where(safe, den, 1.0), center)


def gaussian_taps(radius: int) -> np.ndarray:
    """In-repo diffusion blur weights (no reference twin): exp(-i^2 / (2 sigma^2)),
    sigma = radius / 2, i = -radius..radius, normalised to sum 1 (include/woit.h)."""
    sigma = 0.5 * radius
    i = np.arange(-radius, radius + 1, dtype=np.float64)
    g = np.exp(-(i * i) / (2.0 * sigma * sigma))
    return g / g.sum()


def blur_image(img, radius: int) -> np.ndarray:
    """K_resolve twin: separable edge-clamped Gaussian, rows then columns, f64."""
    img = np.asarray(img, dtype=np.float64)
    H, W = img.shape[:2]
    g = gaussian_taps(radius)
    xs = np.arange(W)
    ys = np.arange(H)
    tmp = np.zeros_like(img)
    for k, w in zip(range(-radius, radius + 1), g):
        tmp += w * img[:, np.clip(xs + k, 0, W - 1)]
    out = np.zeros_like(img)
    for k, w in zip(range(-radius, radius + 1), g):
        out += w * tmp[np.clip(ys + k, 0, H - 1)]
    return out


def _background(img, bufs: OBuffers, cfg: OConfig, px, py, own):
    """Background sample (pipeline.py:290-303) of ``img``; ``own`` = the pixels' own colours."""
    if cfg.chromatic_aberration:
        return chromatic_gather(img, px, py, bufs.refraction_offset, cfg.aberration_taps,
                                cfg.literal_spectral_t)
    if cfg.refraction:
        return bilinear_sample(img, px + bufs.refraction_offset[:, 0],
                               py + bufs.refraction_offset[:, 1])
    return own


def step4_composite(bufs: OBuffers, cfg: OConfig, pixel_base: int = 0, full_img=None,
                    blurred_img=None) -> None:
    """Blend over the (refracted / aberrated) background (pipeline.py:284-308).

    With ``cfg.diffusion > 0`` (in-repo, no reference twin) the background is
    lerped towards the same sample of the blurred image by min(1, diffusion * D_p).
    """
    v_total = np.exp(-total_absorbance_batch(bufs.coeffs, bufs.rank))
    img = bufs.opaque_color.reshape(-1, bufs.width, 3) if full_img is None else full_img
    gp = pixel_base + np.arange(bufs.near.size)
    px = (gp % bufs.width).astype(np.float64)
    py = (gp // bufs.width).astype(np.float64)
    bg = _background(img, bufs, cfg, px, py, bufs.opaque_color)
    if cfg.diffusion > 0.0:
        if blurred_img is None:
            blurred_img = blur_image(img, cfg.diffusion_radius)
        base = full_img is not None
        own = blurred_img.reshape(-1, 3)[gp if base else np.arange(bufs.near.size)]
        bb = _background(blurred_img, bufs, cfg, px, py, own)
        w = np.minimum(1.0, cfg.diffusion * bufs.diffusion)[:, None]
        bg = bg + w * (bb - bg)
    if cfg.normalize:
        bufs.output[:] = bufs.accum / np.maximum(NORM_EPS, bufs.accum_weight) * (1.0 - v_total) \
            + bg * v_total
    else:
        bufs.output[:] = bufs.accum + bg * v_total


# ---------------------------------------------------------------------------
# comparison methods (RenderConfig.method != "wavelet"; baselines.py:135-220),
# per-pixel Python loops: test-size inputs only

WBOIT_WEIGHT = (10.0, 0.01, 3000.0)  # baselines.py:21
WEIGHT_EPS = 1e-5                    # baselines.py:22


def abuffer_frame(frame: OFrame, background, cube: bool = False) -> np.ndarray:
    """Exact compositing in (depth, arrival) order, front to back (baselines.py:135-148)."""
    t = frame.net_transmittance(cube)
    c = frame.radiance * frame.alpha[:, None]
    out = np.empty((frame.npix, 3))
    for p in range(frame.npix):
        s, e = int(frame.offsets[p]), int(frame.offsets[p + 1])
        acc, vis = np.zeros(3), np.ones(3)
        for i in s + np.argsort(frame.depth[s:e], kind="stable"):
            acc = acc + c[i] * vis
            vis = vis * t[i]
        out[p] = acc + background[p] * vis
    return out


def wboit_frame(frame: OFrame, background, cube: bool = False, weight=WBOIT_WEIGHT) -> np.ndarray:
    """Weighted blended OIT over the pixel's depth bounds (baselines.py:151-167)."""
    gain, lo, hi = weight
    t = frame.net_transmittance(cube)
    out = np.empty((frame.npix, 3))
    for p in range(frame.npix):
        s, e = int(frame.offsets[p]), int(frame.offsets[p + 1])
        d = frame.depth[s:e]
        near, far = (d.min(), d.max()) if e > s else (np.inf, -np.inf)
        rng = far - near
        acc, wsum, rev = np.zeros(3), 0.0, np.ones(3)
        for i in range(s, e):
            z = (frame.depth[i] - near) / rng if rng > 0.0 else 0.5
            z = min(max(z, 0.0), 1.0)
            w = min(max(gain / (WEIGHT_EPS + z * z + np.power(z, 6)), lo), hi)
            acc = acc + (w * frame.alpha[i]) * frame.radiance[i]
            wsum = wsum + w * frame.alpha[i]
            rev = rev * t[i]
        avg = acc / max(1e-6, wsum)
        out[p] = avg * (1.0 - rev) + background[p] * rev
    return out


def mlab_frame(frame: OFrame, background, k: int = 4, cube: bool = False) -> np.ndarray:
    """k-node multi-layer alpha blending in arrival order (baselines.py:74-96, 170-220):
    a node goes after every node at depth <= its own; k + 1 nodes merge the last two
    (c = c1 + t1 c2, t = t1 t2); then front to back."""
    if k < 2:
        raise ValueError("mlab needs at least 2 slots")
    t = frame.net_transmittance(cube)
    c = frame.radiance * frame.alpha[:, None]
    out = np.empty((frame.npix, 3))
    for p in range(frame.npix):
        nodes = []  # (depth, colour, transmittance)
        for i in range(int(frame.offsets[p]), int(frame.offsets[p + 1])):
            pos = sum(1 for n in nodes if n[0] <= frame.depth[i])
            nodes.insert(pos, (frame.depth[i], c[i], t[i]))
            if len(nodes) > k:
                d1, c1, t1 = nodes[k - 1]
                _, c2, t2 = nodes[k]
                nodes[k - 1:] = [(d1, c1 + t1 * c2, t1 * t2)]
        acc, vis = np.zeros(3), np.ones(3)
        for _, cn, tn in nodes:
            acc = acc + cn * vis
            vis = vis * tn
        out[p] = acc + background[p] * vis
    return out


def render_band(frame: OFrame, cfg: OConfig, cam: OCamera, full_img, p0: int, p1: int,
                dirs=None, blurred_img=None) -> OBuffers:
    """One row band through the four passes (pipeline.py:321-330)."""
    band = frame if (p0, p1) == (0, frame.npix) else frame.band(p0, p1)
    if dirs is None and cfg.refraction:
        dirs = ray_dirs(cam, frame.width, frame.height)
    f, r, u = camera_basis(cam)
    bufs = OBuffers.allocate(band, cfg.rank)
    step1_depth_bounds(band, bufs)
    step2_build(band, bufs, cfg)
    step3_accumulate(dirs, f, r, u, band, bufs, cfg, pixel_base=p0)
    step4_composite(bufs, cfg, pixel_base=p0, full_img=full_img, blurred_img=blurred_img)
    return bufs


def render_frame(frame: OFrame, cfg: OConfig, cam: OCamera = OCamera(),
                 workers: Optional[int] = None) -> OBuffers:
    """Whole frame, row bands on a thread pool like pipeline.py:356-375.

    Returns the concatenated per-pixel buffers (coeffs, accum, ..., output)
    plus ``vhat`` so parity tests can compare every output of the path.
    """
    W, H = frame.width, frame.height
    workers = cfg.workers if workers is None else workers
    full_img = frame.opaque_color.reshape(H, W, 3)
    dirs = ray_dirs(cam, W, H) if cfg.refraction else None
    blurred = blur_image(full_img, cfg.diffusion_radius) if cfg.diffusion > 0.0 else None
    if workers == 1 or H < 2 * workers:
        return render_band(frame, cfg, cam, full_img, 0, frame.npix, dirs, blurred)
    rows = np.linspace(0, H, workers + 1).astype(int)
    spans = [(rows[i] * W, rows[i + 1] * W) for i in range(workers) if rows[i] < rows[i + 1]]
    with ThreadPoolExecutor(max_workers=len(spans)) as pool:
        parts = list(pool.map(lambda s: render_band(frame, cfg, cam, full_img, s[0], s[1], dirs,
                                                    blurred), spans))
    cat = lambda name: np.concatenate([getattr(b, name) for b in parts], axis=0)
    out = OBuffers(W, H, cfg.rank, cat("near"), cat("far"), cat("coeffs"), cat("accum"),
                   cat("accum_weight"), cat("refraction_offset"), cat("opaque_depth"),
                   cat("opaque_color"), cat("output"))
    out.vhat = cat("vhat")
    out.diffusion = cat("diffusion")
    return out


def default_workers() -> int:
    return max(1, os.cpu_count() or 1)
