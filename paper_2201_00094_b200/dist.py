"""Row-band sharding of a frame across GPUs (one process per GPU) and the image gather.

Pixels are independent through all four passes, so rank r
renders a contiguous band of rows — the reference's own split for its worker
threads, ``np.linspace(0, H, workers + 1).astype(int)`` (pipeline.py:362-364) —
and the only collective is one gather of the fp32 image bands
(``all_gather_into_tensor`` over NCCL on GPUs; gloo works for CPU tests).
``frag_base`` / ``pixel_base`` carry the band's global offsets into the kernels,
so a sharded render is bit-identical to a single-GPU one.
"""

from __future__ import annotations

from typing import List, Tuple

import numpy as np
import torch


def band_rows(height: int, world: int) -> List[Tuple[int, int]]:
    """(row0, rows) per rank, pipeline.py:362-364's split."""
    edges = np.linspace(0, height, world + 1).astype(int)
    return [(int(edges[i]), int(edges[i + 1] - edges[i])) for i in range(world)]


def my_band(height: int, world: int, rank: int) -> Tuple[int, int]:
    return band_rows(height, world)[rank]


def gather_image(band_out: torch.Tensor, height: int, width: int, world: int, group=None) -> torch.Tensor:
    """All ranks' (rows*width, 3) fp32 bands -> the (height, width, 3) image on every rank.

    Bands of unequal height (H not divisible by the world size) are padded to the
    largest band for the collective and trimmed afterwards.
    """
    import torch.distributed as dist

    bands = band_rows(height, world)
    maxrows = max(r for _, r in bands)
    chunk = maxrows * width
    send = band_out.new_zeros(chunk, 3)
    send[: band_out.shape[0]] = band_out
    if band_out.is_cuda and dist.get_backend(group) == "gloo":
        # gloo gathers host tensors (used by the tests that run ranks on one GPU)
        host = [torch.empty(chunk, 3, dtype=send.dtype) for _ in range(world)]
        dist.all_gather(host, send.cpu(), group=group)
        recv = torch.cat(host, 0).to(band_out.device)
    else:
        recv = band_out.new_empty(world * chunk, 3)
        dist.all_gather_into_tensor(recv, send, group=group)
    parts = [recv[i * chunk: i * chunk + rows * width] for i, (_, rows) in enumerate(bands)]
    return torch.cat(parts, 0).reshape(height, width, 3)


def render_sharded(workload: str, cfg, seed: int = 1, layers: int = 32, group=None, device=None,
                   full_opaque_image: torch.Tensor = None):
    """Generate this rank's band of a synthetic frame in HBM, render it fused, gather the image.

    Refraction / aberration gathers read the opaque image at arbitrary offsets, so
    for those flags every rank must hold the full (replicated) opaque image.
    """
    import torch.distributed as dist

    from .frame import FrameFragments
    from .pipeline import render_band

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    row0, rows = my_band(cfg.height, world, rank)
    frame = FrameFragments.synthetic(workload, cfg.width, cfg.height, seed=seed, layers=layers, row0=row0,
                                     rows=rows, device=device)
    bufs = render_band(frame, cfg, full_opaque_image=full_opaque_image)
    return gather_image(bufs.output, cfg.height, cfg.width, world, group), frame, bufs
