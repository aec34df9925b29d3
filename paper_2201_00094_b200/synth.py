"""Synthetic fragment streams, bit-identical on the host (numpy) and the device.

The reference renders analytic scenes through ``cast_frame`` (scene.py:463-570);
that producer is out of scope for this build, so the
benchmark and parity workloads are generated from a counter-based hash:

    u(seed, pixel, layer, field) = (mix(...) >> 8) * 2**-24        (exact fp32)

Every derived quantity is a fixed sequence of fp32 multiplies/adds/divides
(no FMA contraction, no transcendental library call), so the numpy twin in
this file and the CUDA generator in ``csrc/synth.cu`` produce the same bits.
The device generator is what the benchmark uses (the stream must already be
resident in HBM, SURVEY.md §7 "Capacity"); this twin feeds the CPU oracle and
the reference arm of ``bench.py`` with the identical workload.

Workloads:

* ``plane4``    config 1: 64x64, the single-plane preset's pane (scene.py:636-642)
                plus 4 uniform random layers per pixel.
* ``smoke``     config 2: 1080p, 32 stratified layers per pixel, gaussian alpha.
* ``particles`` configs 4/5: 128 or 256 layers per pixel, depth-varying alpha.
* ``ragged``    parity-only: per-pixel run length drawn from [0, max_run].

All streams are CSR by pixel (``offsets`` of length P+1), the reference's own
contract (scene.py:367-374).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

WORKLOADS = ("plane4", "smoke", "particles", "ragged")
WORKLOAD_IDS = {name: i for i, name in enumerate(WORKLOADS)}

# field ids fed to the hash (layer, field) -> independent uniforms
_F_DEPTH, _F_ALPHA, _F_T0, _F_T1, _F_T2, _F_L0, _F_L1, _F_L2 = range(8)
_PIXEL_LAYER = 0xFFFF  # per-pixel quantities use this pseudo layer
_P_NEAR, _P_SPAN, _P_RUN = 0, 1, 2

_U = np.uint32
_F = np.float32
_INV24 = _F(2.0 ** -24)


def _mix32(x: np.ndarray) -> np.ndarray:
    """lowbias32 avalanche (uint32 wrap-around arithmetic)."""
    x = x ^ (x >> _U(16))
    x = x * _U(0x7FEB352D)
    x = x ^ (x >> _U(15))
    x = x * _U(0x846CA68B)
    x = x ^ (x >> _U(16))
    return x


def hash_u32(seed: int, pixel: np.ndarray, layer: np.ndarray, field: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        s = _mix32(np.asarray([(seed ^ 0x9E3779B9) & 0xFFFFFFFF], dtype=_U))[0]
        h = _mix32(pixel.astype(_U) ^ s)
        key = (layer.astype(_U) << _U(4)) | _U(field)
        h = _mix32(h + key * _U(0x85EBCA6B))
    return h


def uniform(seed: int, pixel: np.ndarray, layer: np.ndarray, field: int) -> np.ndarray:
    """U[0,1) in fp32 with 24 random bits, exact."""
    return (hash_u32(seed, pixel, layer, field) >> _U(8)).astype(_F) * _INV24


# exp(y) Taylor coefficients 1/k!, k = 0..7, rounded to fp32
_EXP_C = [_F(1.0 / f) for f in (1, 1, 2, 6, 24, 120, 720, 5040)]


def gauss_profile(r: np.ndarray) -> np.ndarray:
    """exp(-4 r^2) for r in [0,1) as a fixed fp32 op sequence.

    exp(x) = exp(x/8)^8 with exp(x/8) from a degree-7 Horner polynomial;
    |error| < 2e-7. Only products and sums, so the device twin matches bitwise.
    """
    x = (r * r) * _F(-4.0)
    y = x * _F(0.125)
    p = np.full_like(y, _EXP_C[7])
    for c in _EXP_C[6::-1]:
        p = p * y + c
    p = p * p
    p = p * p
    p = p * p
    return p


@dataclass
class SynthFrame:
    """Host copy of a CSR fragment stream in the device layout (fp32 SoA)."""

    width: int
    height: int
    row0: int            # first global row of this band
    rows: int            # rows in this band
    offsets: np.ndarray  # int64 (P+1,), band-local
    depth: np.ndarray    # f32 (n,)
    alpha: np.ndarray    # f32 (n,)
    trans: np.ndarray    # f32 (n,3)
    radiance: np.ndarray  # f32 (n,3)
    normal: np.ndarray   # f32 (n,3)
    ior: np.ndarray      # f32 (n,)
    backface: np.ndarray  # u8 (n,)
    opaque_depth: np.ndarray  # f32 (P,)  (inf = no opaque hit)
    opaque_color: np.ndarray  # f32 (P,3)

    @property
    def npix(self) -> int:
        return self.offsets.size - 1

    @property
    def nfrag(self) -> int:
        return int(self.offsets[-1])

    def pixel_ids(self) -> np.ndarray:
        """Band-local pixel id per fragment (the reference's ``pixel`` array)."""
        return np.repeat(np.arange(self.npix, dtype=np.int64), np.diff(self.offsets))


def run_lengths(workload: str, width: int, height: int, seed: int, layers: int,
                row0: int = 0, rows: Optional[int] = None) -> np.ndarray:
    """Fragments per pixel of the band [row0, row0+rows)."""
    rows = height - row0 if rows is None else rows
    npix = rows * width
    if workload == "plane4":
        return np.full(npix, 5, dtype=np.int64)
    if workload in ("smoke", "particles"):
        return np.full(npix, layers, dtype=np.int64)
    if workload == "ragged":
        gp = np.arange(row0 * width, (row0 + rows) * width, dtype=np.int64)
        u = uniform(seed, gp, np.full(npix, _PIXEL_LAYER), _P_RUN)
        # ~1/8 of the pixels are empty; the rest draw uniformly from [1, layers]
        run = (u * _F(layers + 1)).astype(np.int64)
        return np.minimum(run, layers)
    raise ValueError(f"unknown workload {workload!r}; valid: {', '.join(WORKLOADS)}")


def _checker(width: int, gp: np.ndarray) -> np.ndarray:
    px = gp % width
    py = gp // width
    odd = ((px >> 4) + (py >> 4)) & 1
    light = np.array([0.85, 0.80, 0.72], dtype=_F)
    dark = np.array([0.25, 0.22, 0.20], dtype=_F)
    return np.where(odd[:, None] == 1, dark[None, :], light[None, :]).astype(_F)


def generate(workload: str, width: int, height: int, seed: int = 1, layers: int = 32,
             row0: int = 0, rows: Optional[int] = None) -> SynthFrame:
    """numpy twin of the device generator (``woit_synth_fill``)."""
    rows = height - row0 if rows is None else rows
    if not (0 <= row0 and rows >= 0 and row0 + rows <= height):
        raise ValueError("band outside the frame")
    npix = rows * width
    run = run_lengths(workload, width, height, seed, layers, row0, rows)
    offsets = np.zeros(npix + 1, dtype=np.int64)
    np.cumsum(run, out=offsets[1:])
    n = int(offsets[-1])
    gp0 = row0 * width
    lp = np.repeat(np.arange(npix, dtype=np.int64), run)   # band-local pixel
    gp = lp + gp0                                           # global pixel id
    j = (np.arange(n, dtype=np.int64) - offsets[lp])        # layer within pixel
    u = lambda f: uniform(seed, gp, j, f)

    depth = np.empty(n, _F)
    alpha = np.empty(n, _F)
    trans = np.empty((n, 3), _F)
    rad = np.empty((n, 3), _F)
    normal = np.zeros((n, 3), _F)
    normal[:, 2] = _F(-1.0)
    ior = np.ones(n, _F)
    backface = np.zeros(n, np.uint8)
    gpix = np.arange(gp0, gp0 + npix, dtype=np.int64)
    opaque_depth = np.full(npix, np.inf, _F)
    opaque_color = _checker(width, gpix)

    if workload == "plane4":
        first = j == 0
        depth[:] = u(_F_DEPTH) * _F(1.7) + _F(0.25)
        alpha[:] = u(_F_ALPHA)
        for c in range(3):
            trans[:, c] = u(_F_T0 + c)
            rad[:, c] = u(_F_L0 + c)
        depth[first] = _F(1.0)
        alpha[first] = _F(0.25)
        trans[first] = _F(0.0)
        rad[first] = np.array([0.18, 0.18, 0.20], dtype=_F)
        opaque_depth[:] = _F(2.0)
        opaque_color[:] = np.array([0.85, 0.45, 0.12], dtype=_F)
    elif workload == "smoke":
        pl = np.full(n, _PIXEL_LAYER)
        near = uniform(seed, gp, pl, _P_NEAR) * _F(0.5) + _F(0.5)
        span = uniform(seed, gp, pl, _P_SPAN) * _F(2.0) + _F(1.0)
        inv = _F(1.0 / layers) if (layers & (layers - 1)) == 0 else None
        frac = j.astype(_F) + u(_F_DEPTH)
        frac = frac * inv if inv is not None else frac / _F(layers)
        depth[:] = frac * span + near
        alpha[:] = _F(0.4) * gauss_profile(u(_F_ALPHA))
        tg = u(_F_T0) * _F(0.3) + _F(0.2)
        lg = u(_F_L0) * _F(0.15) + _F(0.3)
        trans[:] = tg[:, None]
        rad[:] = lg[:, None]
    elif workload in ("particles", "ragged"):
        depth[:] = u(_F_DEPTH) * _F(2.2) + _F(1.0)
        fade = _F(1.0) - ((depth - _F(1.0)) / _F(2.2)) * _F(0.5)
        alpha[:] = (_F(0.5) * gauss_profile(u(_F_ALPHA))) * fade
        for c in range(3):
            trans[:, c] = u(_F_T0 + c) * _F(0.31) + _F(0.02)
            rad[:, c] = u(_F_L0 + c) * _F(1.3)
    else:  # pragma: no cover - run_lengths already validated
        raise AssertionError(workload)

    return SynthFrame(width, height, row0, rows, offsets, depth, alpha, trans, rad,
                      normal, ior, backface, opaque_depth, opaque_color)
