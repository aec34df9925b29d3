"""CPU, world_size 2 over gloo: row-band split and the image gather used by the
multi-GPU path (the kernels themselves are covered by the GPU tests)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2201_00094_b200 import dist as D


def test_band_rows_match_reference_split():
    """pipeline.py:362-364: np.linspace(0, H, workers + 1).astype(int)."""
    for H, N in ((1080, 8), (23, 3), (7, 2), (4320, 8), (5, 4)):
        edges = np.linspace(0, H, N + 1).astype(int)
        bands = D.band_rows(H, N)
        assert [b[0] for b in bands] == list(edges[:-1])
        assert sum(r for _, r in bands) == H


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, H, W, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    row0, rows = D.my_band(H, world, rank)
    # band values encode the global pixel id so the gather order is checkable
    gp = torch.arange(row0 * W, (row0 + rows) * W, dtype=torch.float32)
    band = torch.stack([gp, gp * 2, gp * 3], 1)
    img = D.gather_image(band, H, W, world)
    q.put((rank, img.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("H,W", [(6, 5), (7, 3)])
def test_gather_image_world2(H, W):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, W, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gp = np.arange(H * W, dtype=np.float32)
    want = np.stack([gp, gp * 2, gp * 3], 1).reshape(H, W, 3)
    for _, img in out:
        np.testing.assert_array_equal(img, want)
