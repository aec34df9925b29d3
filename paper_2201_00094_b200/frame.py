"""Device-resident fragment stream: the reference's ``FrameFragments`` (scene.py:367-428)
in HBM as fp32 SoA, CSR-indexed by pixel.

Field names, shapes and the CSR contract are the reference's; dtypes are fp32
(depth, alpha, trans, radiance, normal, ior, opaque_*), int64 offsets and uint8
backface. ``pixel`` is not stored: every kernel derives a fragment's pixel from
``offsets`` (saving 8 B/fragment of HBM traffic); the property materialises it
on demand for callers that want the reference's array.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .synth import SynthFrame, WORKLOADS


def _dev(device) -> torch.device:
    d = torch.device(device if device is not None else "cuda")
    if d.type != "cuda":
        raise ValueError("FrameFragments live in CUDA memory (no CPU path)")
    return d


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


@dataclass
class FrameFragments:
    width: int
    height: int
    offsets: torch.Tensor       # int64 (P+1,)
    depth: torch.Tensor         # f32 (n,)
    alpha: torch.Tensor         # f32 (n,)
    trans: torch.Tensor         # f32 (n,3)
    radiance: torch.Tensor      # f32 (n,3)
    normal: torch.Tensor        # f32 (n,3)
    ior: torch.Tensor           # f32 (n,)
    backface: torch.Tensor      # u8 (n,)
    opaque_depth: torch.Tensor  # f32 (P,)
    opaque_color: torch.Tensor  # f32 (P,3)
    pixel_base: int = 0         # global id of this band's first pixel
    frag_base: int = 0          # global id of fragment index 0 of this band

    @property
    def npix(self) -> int:
        return self.offsets.numel() - 1

    @property
    def nfrag(self) -> int:
        return self.depth.numel()

    @property
    def device(self) -> torch.device:
        return self.depth.device

    @property
    def pixel(self) -> torch.Tensor:
        """Band-local pixel id per fragment (the reference's ``pixel`` array)."""
        counts = self.offsets[1:] - self.offsets[:-1]
        return torch.repeat_interleave(torch.arange(self.npix, device=self.device), counts)

    # -- construction -------------------------------------------------------------

    @classmethod
    def from_numpy(cls, width, height, offsets, depth, alpha, trans, radiance, normal=None, ior=None,
                   backface=None, opaque_depth=None, opaque_color=None, device=None,
                   pixel_base: int = 0, frag_base: int = 0) -> "FrameFragments":
        """Upload a host CSR stream (any float dtype; stored as fp32)."""
        dev = _dev(device)
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        npix = offsets.size - 1
        n = int(offsets[-1])
        if int(offsets[0]) != 0 or np.any(np.diff(offsets) < 0):
            raise ValueError("offsets must start at 0 and be non-decreasing (CSR by pixel)")
        f32 = lambda a, shape: torch.from_numpy(
            np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(shape))).to(dev)
        if normal is None:
            normal = np.tile(np.array([0.0, 0.0, -1.0], np.float32), (n, 1))
        if ior is None:
            ior = np.ones(n, np.float32)
        if backface is None:
            backface = np.zeros(n, np.uint8)
        if opaque_depth is None:
            opaque_depth = np.full(npix, np.inf, np.float32)
        if opaque_color is None:
            opaque_color = np.zeros((npix, 3), np.float32)
        return cls(width, height, torch.from_numpy(offsets).to(dev), f32(depth, (n,)), f32(alpha, (n,)),
                   f32(trans, (n, 3)), f32(radiance, (n, 3)), f32(normal, (n, 3)), f32(ior, (n,)),
                   torch.from_numpy(np.ascontiguousarray(np.asarray(backface).astype(np.uint8))).to(dev),
                   f32(opaque_depth, (npix,)), f32(opaque_color, (npix, 3)), pixel_base, frag_base)

    @classmethod
    def from_reference(cls, frame, device=None) -> "FrameFragments":
        """From a reference ``woit.scene.FrameFragments`` (f64 numpy arrays)."""
        return cls.from_numpy(frame.width, frame.height, frame.offsets, frame.depth, frame.alpha,
                              frame.trans, frame.radiance, frame.normal, frame.ior, frame.backface,
                              frame.opaque_depth, frame.opaque_color, device=device)

    @classmethod
    def from_synth(cls, sf: SynthFrame, device=None) -> "FrameFragments":
        base = sf.row0 * sf.width
        return cls.from_numpy(sf.width, sf.height, sf.offsets, sf.depth, sf.alpha, sf.trans, sf.radiance,
                              sf.normal, sf.ior, sf.backface, sf.opaque_depth, sf.opaque_color,
                              device=device, pixel_base=base)

    @classmethod
    def synthetic(cls, workload: str, width: int, height: int, seed: int = 1, layers: int = 32,
                  row0: int = 0, rows: Optional[int] = None, device=None,
                  frag_base: Optional[int] = None) -> "FrameFragments":
        """Generate a synthetic stream directly in HBM (bit-identical to ``synth.generate``)."""
        if workload not in WORKLOADS:
            raise ValueError(f"unknown workload {workload!r}; valid: {', '.join(WORKLOADS)}")
        dev = _dev(device)
        lib = _lib.load()
        rows = height - row0 if rows is None else rows
        npix = rows * width
        wid = _lib.SYNTH_IDS[workload]
        with torch.cuda.device(dev):
            offsets = torch.empty(npix + 1, dtype=torch.int64, device=dev)
            ws = torch.empty(lib.woit_synth_workspace_bytes(npix), dtype=torch.uint8, device=dev)
            _lib.check(lib.woit_synth_offsets(wid, width, height, seed, layers, row0, rows,
                                              ptr(offsets), ptr(ws), ws.numel(), _stream()),
                       "woit_synth_offsets")
            n = int(offsets[-1].item())
            f = lambda *s: torch.empty(*s, dtype=torch.float32, device=dev)
            depth, alpha, ior = f(n), f(n), f(n)
            trans, rad, normal = f(n, 3), f(n, 3), f(n, 3)
            bf = torch.empty(n, dtype=torch.uint8, device=dev)
            od, oc = f(npix), f(npix, 3)
            _lib.check(lib.woit_synth_fill(wid, width, height, seed, layers, row0, rows, ptr(offsets),
                                           ptr(depth), ptr(alpha), ptr(trans), ptr(rad), ptr(normal),
                                           ptr(ior), ptr(bf), ptr(od), ptr(oc), _stream()),
                       "woit_synth_fill")
        if frag_base is None:
            frag_base = _band_frag_base(workload, width, height, seed, layers, row0)
        return cls(width, height, offsets, depth, alpha, trans, rad, normal, ior, bf, od, oc,
                   row0 * width, frag_base)

    @classmethod
    def from_unbinned(cls, width: int, height: int, pix: torch.Tensor, depth: torch.Tensor, alpha: torch.Tensor,
                      trans: torch.Tensor, radiance: torch.Tensor, normal: Optional[torch.Tensor] = None,
                      ior: Optional[torch.Tensor] = None, backface: Optional[torch.Tensor] = None,
                      opaque_depth: Optional[torch.Tensor] = None, opaque_color: Optional[torch.Tensor] = None,
                      npix: Optional[int] = None, pixel_base: int = 0, return_perm: bool = False):
        """CSR stream from an unbinned one (the producer's arrival order, a pixel id per
        fragment): ``woit_bin_frame`` -- a stable sort by pixel whose last pass scatters
        every fragment's fields into its CSR slot (scene.py:559-566: offsets =
        cumsum(bincount), each pixel's fragments in arrival order). Device tensors in,
        device tensors out; with ``return_perm`` also argsort(pix, kind="stable")."""
        dev = depth.device
        lib = _lib.load()
        n = depth.numel()
        P = width * height if npix is None else npix
        if pix.dtype != torch.int32 or pix.numel() != n or pix.device != dev:
            raise ValueError("pix must be an int32 device tensor with one pixel id per fragment")
        f32 = lambda t, *shape: t.to(dev, torch.float32).contiguous().reshape(*shape)
        ins = dict(depth=f32(depth, n), alpha=f32(alpha, n), trans=f32(trans, n, 3), radiance=f32(radiance, n, 3))
        if normal is not None:
            ins["normal"] = f32(normal, n, 3)
        if ior is not None:
            ins["ior"] = f32(ior, n)
        if backface is not None:
            ins["backface"] = backface.to(dev, torch.uint8).contiguous()
        outs = {k: torch.empty_like(v) for k, v in ins.items()}
        # absent refraction fields are not moved: their CSR arrays are the constants
        # the frame kernels take for "none" (normal (0, 0, -1), ior 1, front face)
        if normal is None:
            outs["normal"] = torch.tensor([0.0, 0.0, -1.0], device=dev).repeat(n, 1)
        if ior is None:
            outs["ior"] = torch.ones(n, device=dev)
        if backface is None:
            outs["backface"] = torch.zeros(n, dtype=torch.uint8, device=dev)
        offsets = torch.empty(P + 1, dtype=torch.int64, device=dev)
        perm = torch.empty(max(n, 1), dtype=torch.int64, device=dev) if return_perm else None
        fi, fo = _lib.Frags(), _lib.Frags()
        for f, d in ((fi, ins), (fo, outs)):
            f.width, f.height, f.npix, f.nfrag = width, height, P, n
            for k in ins:
                setattr(f, k, ptr(d[k]))
        wsn = lib.woit_bin_frame_workspace_bytes(n, P)
        ws = torch.empty(max(wsn, 1), dtype=torch.uint8, device=dev)
        with torch.cuda.device(dev):
            _lib.check(lib.woit_bin_frame(ptr(pix), fi, fo, ptr(offsets), ptr(perm), ptr(ws), wsn, _stream()),
                       "woit_bin_frame")
        od = opaque_depth if opaque_depth is not None else torch.full((P,), float("inf"), device=dev)
        oc = opaque_color if opaque_color is not None else torch.zeros(P, 3, device=dev)
        frame = cls(width, height, offsets, outs["depth"], outs["alpha"], outs["trans"], outs["radiance"],
                    outs["normal"], outs["ior"], outs["backface"], f32(od, P), f32(oc, P, 3), pixel_base, 0)
        return (frame, perm[:n]) if return_perm else frame

    # -- views --------------------------------------------------------------------

    def band(self, p0: int, p1: int) -> "FrameFragments":
        """Pixel band [p0, p1) with rebased offsets (pipeline.py:311-318); arrays are views."""
        lo = int(self.offsets[p0].item())
        hi = int(self.offsets[p1].item())
        return FrameFragments(self.width, self.height, self.offsets[p0:p1 + 1] - lo, self.depth[lo:hi],
                              self.alpha[lo:hi], self.trans[lo:hi], self.radiance[lo:hi],
                              self.normal[lo:hi], self.ior[lo:hi], self.backface[lo:hi],
                              self.opaque_depth[p0:p1], self.opaque_color[p0:p1],
                              self.pixel_base + p0, self.frag_base + lo)

    def to_synth(self) -> SynthFrame:
        """Host copy in the generator's layout (for the CPU oracle)."""
        h = lambda t: t.detach().cpu().numpy()
        rows = self.npix // self.width
        return SynthFrame(self.width, self.height, self.pixel_base // self.width, rows, h(self.offsets),
                          h(self.depth), h(self.alpha), h(self.trans), h(self.radiance), h(self.normal),
                          h(self.ior), h(self.backface), h(self.opaque_depth), h(self.opaque_color))

    def c_struct(self) -> _lib.Frags:
        f = _lib.Frags()
        f.width, f.height = self.width, self.height
        f.npix, f.nfrag = self.npix, self.nfrag
        f.pixel_base, f.frag_base = self.pixel_base, self.frag_base
        f.offsets = ptr(self.offsets)
        for name in ("depth", "alpha", "trans", "radiance", "normal", "ior", "backface", "opaque_depth",
                     "opaque_color"):
            t = getattr(self, name)
            if not t.is_contiguous():
                raise ValueError(f"{name} must be contiguous")
            setattr(f, name, ptr(t))
        return f

    def net_transmittance(self, cube_transmission: bool = False,
                          cube_backface_only: bool = False) -> torch.Tensor:
        """scene.py:394-402 on device (convenience; the kernels fuse this)."""
        T = self.trans.double()
        if cube_transmission:
            sel = self.ior > 1.0
            if cube_backface_only:
                sel = sel & (self.backface != 0)
            T = torch.where(sel[:, None], T * T * T, T)
        return 1.0 - self.alpha.double()[:, None] * (1.0 - T)


def _band_frag_base(workload: str, width: int, height: int, seed: int, layers: int, row0: int) -> int:
    """Global id of the first fragment of the band starting at row0."""
    if row0 == 0:
        return 0
    from .synth import run_lengths
    return int(run_lengths(workload, width, height, seed, layers, 0, row0).sum())
