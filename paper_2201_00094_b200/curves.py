"""Visibility curves along one pixel's ray (the reference's curves.py:1-111, for the CLI's
``graph`` command and the curve columns of ``compare``).

Every curve is sampled on the normalized grid z_i = (i + 1/2) / samples that the
wavelet evaluation uses, mapped to world depth through the pixel's padded bounds
(eval_bounds, then normalize_depth's 1e-4 pad: curves.py:83-87). The wavelet curve
comes from the GPU kernels -- the pixel's coefficients by ``build_into`` (bit-exact
to the reference's batch build) and exp(-A) at the grid by
``interp_absorbance_batch`` -- and the truth, A-buffer, WBOIT and MLAB-4 curves from
the pixel's stream on the device (one pixel: a few hundred fragments at most).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Dict, Iterable

import numpy as np
import torch

from .frame import FrameFragments
from .pipeline import eval_bounds
from .wavelet import build_into, interp_absorbance_batch, normalize_depth_array

# per-channel reductions of an RGB visibility (curves.py:22-27)
CHANNELS = {
    "luminance": (0.2126, 0.7152, 0.0722),
    "r": (1.0, 0.0, 0.0),
    "g": (0.0, 1.0, 0.0),
    "b": (0.0, 0.0, 1.0),
}
CURVE_METHODS = ("wavelet", "abuffer", "wboit", "mlab4")
TRANSMITTANCE_FLOOR = 1e-6  # -ln(max(floor, T)) (core.py)
MLAB_SLOTS = 4


@dataclass
class RayCurves:
    """One ray's sampled visibility: the grid, its world depths, truth, per method."""

    z: np.ndarray
    x: np.ndarray
    truth: np.ndarray
    methods: Dict[str, np.ndarray]
    empty: bool = False


def _weights(channel: str) -> torch.Tensor:
    if channel not in CHANNELS:
        raise ValueError(f"unknown channel {channel!r}; valid: {', '.join(CHANNELS)}")
    return torch.tensor(CHANNELS[channel], dtype=torch.float64, device="cuda")


def pixel_stream(frame: FrameFragments, px: int, py: int) -> FrameFragments:
    """Pixel (px, py) of a cast frame as a one-pixel stream (its CSR run, arrival order)."""
    if not (0 <= px < frame.width and 0 <= py < frame.height):
        raise ValueError(f"pixel {px},{py} outside the {frame.width}x{frame.height} grid")
    p = py * frame.width + px
    return frame.band(p, p + 1)


def _mlab_trans_nodes(depth: np.ndarray, net: np.ndarray, k: int):
    """The transmittance and depth of MLAB's k blending nodes (baselines.py:74-96): each
    fragment is inserted after the nodes of depth <= its own; past k nodes the two
    farthest merge, the merged node keeping the nearer depth and the product of the
    transmittances."""
    nodes = []  # [depth, trans(3)] in depth order
    for d, t in zip(depth.tolist(), net):
        pos = len(nodes)
        while pos > 0 and nodes[pos - 1][0] > d:
            pos -= 1
        nodes.insert(pos, [d, t.copy()])
        if len(nodes) > k:
            far = nodes.pop()
            nodes[-1][1] = nodes[-1][1] * far[1]
    return nodes


def extract_curves(stream: FrameFragments, methods: Iterable[str], rank: int, samples: int = 512,
                   channel: str = "luminance", cube_transmission: bool = False) -> RayCurves:
    """Truth and each requested method's visibility along the ray (curves.py:66-111)."""
    names = list(methods)
    for m in names:
        if m not in CURVE_METHODS:
            raise ValueError(f"unknown method {m!r}; valid: {', '.join(CURVE_METHODS)}")
    w = _weights(channel)
    z = (torch.arange(samples, dtype=torch.float64, device="cuda") + 0.5) / samples
    n = stream.nfrag
    if n == 0:
        ones = np.ones(samples)
        zh = z.cpu().numpy()
        return RayCurves(zh, zh.copy(), ones, {m: ones.copy() for m in names}, empty=True)
    depth = stream.depth.double()
    net = stream.net_transmittance(cube_transmission)  # (n, 3) f64
    a = -torch.log(torch.clamp(net, min=TRANSMITTANCE_FLOOR))
    dmin, dmax = depth.min(), depth.max()
    near_e, far_e = eval_bounds(dmin.reshape(1), dmax.reshape(1), rank)
    pad = torch.clamp(1e-4 * (far_e - near_e), min=1e-6)
    near_p, far_p = near_e - pad, far_e + pad
    x = near_p + z * (far_p - near_p)
    # truth: product of the transmittances of the fragments strictly in front of x
    # (left-continuous steps), in depth order
    order = torch.sort(depth, stable=True).indices
    sd = depth[order]
    cum = torch.cumprod(net[order], dim=0)
    cnt = torch.searchsorted(sd, x, right=False)
    vis = torch.where((cnt > 0)[:, None], cum[(cnt - 1).clamp(min=0)], torch.ones_like(cum[:1]))
    truth = vis @ w
    out: Dict[str, torch.Tensor] = {}
    for m in names:
        if m == "wavelet":
            S = 2 << rank
            coeffs = torch.zeros(1, S, 3, dtype=torch.float64, device="cuda")
            zf = normalize_depth_array(depth, near_e, far_e)
            pix = torch.zeros(n, dtype=torch.int64, device="cuda")
            build_into(coeffs, pix, zf, a, rank)
            A = interp_absorbance_batch(coeffs, torch.zeros(samples, dtype=torch.int64, device="cuda"), z, rank)
            out[m] = torch.exp(-A) @ w
        elif m == "abuffer":
            out[m] = truth.clone()
        elif m == "wboit":
            reveal = torch.prod(net, dim=0)
            a_tot = -torch.log(torch.clamp(reveal, min=TRANSMITTANCE_FLOOR))
            rng = dmax - dmin
            zr = torch.clamp((x - dmin) / rng, 0.0, 1.0) if float(rng) > 0.0 else (x >= dmin).double()
            out[m] = torch.exp(-zr[:, None] * a_tot[None, :]) @ w
        else:  # mlab4
            nodes = _mlab_trans_nodes(depth.cpu().numpy(), net.cpu().numpy(), MLAB_SLOTS)
            xh = x.cpu().numpy()
            v = np.ones((samples, 3))
            for d, t in nodes:
                v[xh > d] *= t
            out[m] = torch.from_numpy(v).to(w.device) @ w
    h = lambda t: t.detach().cpu().numpy()
    return RayCurves(h(z), h(x), h(truth), {m: h(v) for m, v in out.items()})


def curve_errors(rc: RayCurves, method: str):
    """L1 (mean), L2 (root mean square) and L-infinity distance of a method's curve
    from the truth (the reference compare's curve columns, cli.py:171-174)."""
    d = np.abs(rc.methods[method] - rc.truth)
    return float(d.mean()), float(math.sqrt(float((d * d).mean()))), float(d.max())
