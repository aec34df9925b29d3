"""Batch Haar kernels of the reference (wavelet.py:48-71, 130-135, 272-337) on B200.

Same names and arguments as ``woit.wavelet``. Inputs may be numpy arrays (the
reference's calling convention; results come back as numpy) or CUDA tensors.
Everything is float64 like the reference: with ``mode="binned"`` (default) the
build performs its f64 additions in exactly np.add.at's order, so coefficients
are bit-identical to the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

EPS_Z = 2.0 ** -24


@dataclass
class TouchCounter:
    """Coefficient slots touched per insert / reconstruction (wavelet.py:48-71).

    The kernels' access pattern is fixed (N+2 slots per insert, N+2 per cell
    reconstruction), so the counts are recorded analytically per launch.
    """

    inserts: int = 0
    insert_touches: int = 0
    evals: int = 0
    eval_touches: int = 0

    def record_insert(self, events: int, touched: int) -> None:
        self.inserts += events
        self.insert_touches += touched

    def record_eval(self, events: int, touched: int) -> None:
        self.evals += events
        self.eval_touches += touched

    @property
    def per_insert(self) -> float:
        return self.insert_touches / self.inserts if self.inserts else 0.0

    @property
    def per_eval(self) -> float:
        return self.eval_touches / self.evals if self.evals else 0.0


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _to_dev(x, dtype, device):
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x), dtype=None)).to(device=device, dtype=dtype)


def _device_of(*xs):
    for x in xs:
        if isinstance(x, torch.Tensor) and x.is_cuda:
            return x.device
    return torch.device("cuda")


def normalize_depth_array(x, near, far):
    """wavelet.py:130-135 (f64, device or numpy)."""
    if not isinstance(x, torch.Tensor):
        rng = far - near
        pad = np.maximum(1e-4 * rng, 1e-6)
        return np.clip((x - (near - pad)) / (rng + 2.0 * pad), 0.0, 1.0 - EPS_Z)
    rng = far - near
    pad = torch.clamp(1e-4 * rng, min=1e-6)
    return torch.clamp((x - (near - pad)) / (rng + 2.0 * pad), 0.0, 1.0 - EPS_Z)


def build_into(coeffs, pix, z, a, rank: int, counter: TouchCounter | None = None,
               mode: str = "binned") -> None:
    """Scatter-add interfaces (pixel, z, absorbance) into ``coeffs`` in place (wavelet.py:272-287)."""
    lib = _lib.load()
    n = int(np.asarray(z.shape)[0]) if len(z.shape) else 0
    if n == 0:
        return
    dev = _device_of(coeffs, pix, z, a)
    c = _to_dev(coeffs, torch.float64, dev)
    P = c.shape[0]
    pix_t = _to_dev(pix, torch.int64, dev)
    z_t = _to_dev(z, torch.float64, dev)
    a_t = _to_dev(a, torch.float64, dev).reshape(n, 3)
    m = {"binned": _lib.BUILD_BINNED, "atomic": _lib.BUILD_ATOMIC}[mode]
    wsn = lib.woit_build_into_workspace_bytes(n, P)
    ws = torch.empty(wsn, dtype=torch.uint8, device=dev)
    _lib.check(lib.woit_build_into(c.data_ptr(), P, pix_t.data_ptr(), z_t.data_ptr(), a_t.data_ptr(), n, rank,
                                   m, ws.data_ptr(), wsn, _stream()), "build_into")
    if isinstance(coeffs, torch.Tensor):
        if c.data_ptr() != coeffs.data_ptr():
            coeffs.copy_(c)
    else:
        coeffs[...] = c.cpu().numpy()
    if counter is not None:
        counter.record_insert(n, n * (rank + 2))


def _ret(like, t: torch.Tensor):
    return t if isinstance(like, torch.Tensor) else t.cpu().numpy()


def cells_raw_batch(coeffs, pix, cells, rank: int, counter: TouchCounter | None = None):
    """Staircase values at per-query cell indices (wavelet.py:290-303)."""
    lib = _lib.load()
    dev = _device_of(coeffs, pix, cells)
    c = _to_dev(coeffs, torch.float64, dev)
    p = _to_dev(pix, torch.int64, dev)
    ce = _to_dev(cells, torch.int64, dev)
    n = p.numel()
    out = torch.empty(n, 3, dtype=torch.float64, device=dev)
    _lib.check(lib.woit_cells_raw(c.data_ptr(), c.shape[0], p.data_ptr(), ce.data_ptr(), n, rank,
                                  out.data_ptr(), _stream()), "cells_raw_batch")
    if counter is not None:
        counter.record_eval(n, n * (rank + 2))
    return _ret(coeffs, out)


def interp_absorbance_batch(coeffs, pix, z, rank: int, counter: TouchCounter | None = None):
    """Interpolated absorbance, clamped >= 0 (wavelet.py:306-319)."""
    lib = _lib.load()
    dev = _device_of(coeffs, pix, z)
    c = _to_dev(coeffs, torch.float64, dev)
    p = _to_dev(pix, torch.int64, dev)
    zt = _to_dev(z, torch.float64, dev)
    n = p.numel()
    out = torch.empty(n, 3, dtype=torch.float64, device=dev)
    _lib.check(lib.woit_interp_absorbance(c.data_ptr(), c.shape[0], p.data_ptr(), zt.data_ptr(), n, rank,
                                          out.data_ptr(), _stream()), "interp_absorbance_batch")
    if counter is not None:
        counter.record_eval(2 * n, 2 * n * (rank + 2))
    return _ret(coeffs, out)


def total_absorbance_batch(coeffs, rank: int, counter: TouchCounter | None = None):
    """Absorbance at z -> 1 per pixel (wavelet.py:322-337)."""
    lib = _lib.load()
    dev = _device_of(coeffs)
    c = _to_dev(coeffs, torch.float64, dev)
    P = c.shape[0]
    out = torch.empty(P, 3, dtype=torch.float64, device=dev)
    _lib.check(lib.woit_total_absorbance(c.data_ptr(), P, rank, out.data_ptr(), _stream()),
               "total_absorbance_batch")
    if counter is not None:
        counter.record_eval(P, P * (rank + 2))
    return _ret(coeffs, out)


def bin_by_pixel(pix, npix: int):
    """Stable CSR binning of an unbinned stream: (offsets, perm) as CUDA tensors."""
    lib = _lib.load()
    dev = _device_of(pix)
    p = _to_dev(pix, torch.int64, dev)
    n = p.numel()
    offsets = torch.empty(npix + 1, dtype=torch.int64, device=dev)
    perm = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    wsn = lib.woit_bin_workspace_bytes(n, npix)
    ws = torch.empty(max(wsn, 1), dtype=torch.uint8, device=dev)
    _lib.check(lib.woit_bin_by_pixel(p.data_ptr(), n, npix, offsets.data_ptr(), perm.data_ptr(),
                                     ws.data_ptr(), wsn, _stream()), "bin_by_pixel")
    return offsets, perm[:n]
