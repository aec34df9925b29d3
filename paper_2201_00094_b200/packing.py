"""E5B9G9R9 shared-exponent coefficient storage (packing.py:1-111 of the reference) on B200.

Word layout (bit 0 = LSB): red 0-8, green 9-17, blue 18-26, exponent 27-31
(bias 15); value = mantissa * 2^(exponent - 24). Slot 0 is stored positive,
every wavelet slot as a magnitude that unpacks negative (packing.py:1-21).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

MANTISSA_BITS = 9
EXPONENT_BITS = 5
EXPONENT_BIAS = 15
MAX_VALUE = 511.0 / 512.0 * 2.0 ** 16
BYTES_PER_WORD = 4


def bytes_per_pixel(rank: int) -> int:
    return BYTES_PER_WORD * (1 << (rank + 1))


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def pack_rgb9e5(values):
    """Non-negative triples (..., 3) -> uint32 words (packing.py:46-77)."""
    lib = _lib.load()
    host = not isinstance(values, torch.Tensor)
    v = torch.as_tensor(np.asarray(values, dtype=np.float64) if host else values,
                        dtype=torch.float64, device="cuda" if host else values.device)
    if v.shape[-1:] != (3,):
        raise ValueError(f"expected triples on the last axis, got shape {tuple(v.shape)}")
    if bool(torch.isnan(v).any()):
        raise ValueError("cannot pack NaN")
    shape = v.shape[:-1]
    flat = v.reshape(-1, 3).contiguous()
    words = torch.empty(flat.shape[0], dtype=torch.int32, device=flat.device)
    _lib.check(lib.woit_pack_rgb9e5(flat.data_ptr(), flat.shape[0], words.data_ptr(), _stream()), "pack")
    words = words.reshape(shape)
    if host:
        w = words.cpu().numpy().view(np.uint32)
        return w[()] if w.ndim == 0 else w
    return words


def unpack_rgb9e5(words):
    """uint32 words -> float64 triples (packing.py:80-88)."""
    lib = _lib.load()
    host = not isinstance(words, torch.Tensor)
    if host:
        w = np.array(words, dtype=np.uint32, order="C", copy=True).view(np.int32)
        wt = torch.from_numpy(w).cuda()
    else:
        wt = words.to(torch.int32)
    shape = wt.shape
    flat = wt.reshape(-1).contiguous()
    out = torch.empty(flat.numel(), 3, dtype=torch.float64, device=flat.device)
    _lib.check(lib.woit_unpack_rgb9e5(flat.data_ptr(), flat.numel(), out.data_ptr(), _stream()), "unpack")
    out = out.reshape(*shape, 3)
    return out.cpu().numpy() if host else out


def roundtrip_coeff_array(coeffs):
    """Packed storage of a (pixels, slots, 3) array (packing.py:107-111)."""
    host = not isinstance(coeffs, torch.Tensor)
    c = torch.as_tensor(coeffs, dtype=torch.float64, device="cuda" if host else coeffs.device)
    out = unpack_rgb9e5(pack_rgb9e5(c.abs()))
    out[:, 1:, :] = -out[:, 1:, :]
    return out.cpu().numpy() if host else out
