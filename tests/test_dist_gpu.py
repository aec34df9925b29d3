"""The multi-GPU path end to end on the one GPU this environment has: two ranks
(world_size 2, gloo -- NCCL refuses two ranks on one device) each render their
row band with the CUDA kernels on cuda:0 and gather the image. The kernels of
the two ranks never wait on each other (only the CPU-side gather does), so this
is the N-GPU code path, not a stand-in for N GPUs' timing.

* ``dist.render_sharded`` (generation of the band in HBM, fused render, gather)
  is bitwise equal to one-GPU ``render_band`` of the whole frame
  (test_pipeline.py:361-365's workers check, across processes);
* ``bench.py --gpus 2`` (re-launched under torchrun) runs its world > 1 code and
  reports the config-4 strong-scaling sub-record with the gathered image bitwise
  equal to the 1-GPU render.
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, workload, w, hgt, layers, q):
    import torch.distributed as dist

    import paper_2201_00094_b200 as W
    from paper_2201_00094_b200 import dist as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = W.RenderConfig(rank=3, width=w, height=hgt)
    img, frame, bufs = D.render_sharded(workload, cfg, seed=5, layers=layers, device="cuda:0")
    torch.cuda.synchronize()
    q.put((rank, img.cpu().numpy(), frame.pixel_base))
    dist.destroy_process_group()


@pytest.mark.parametrize("workload,w,hgt,layers", [("ragged", 48, 30, 40), ("particles", 40, 16, 128),
                                                   ("smoke", 33, 7, 32)])
def test_render_sharded_two_ranks_bitwise(workload, w, hgt, layers):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2201_00094_b200 as W

    frame = W.FrameFragments.synthetic(workload, w, hgt, seed=5, layers=layers, device="cuda:0")
    want = W.render_band(frame, W.RenderConfig(rank=3, width=w, height=hgt)).output
    want = want.reshape(hgt, w, 3).cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, workload, w, hgt, layers, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, img, base in outs:
        assert np.array_equal(img, want), f"rank {rank}"
    assert sorted(b for _, _, b in outs) == [0, (hgt // 2) * w]


def test_bench_world2_strong_scaling_record():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    env = dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", "0"))
    env.pop("WORLD_SIZE", None)
    # LOCAL_RANK 1 must map to the same device: both ranks see cuda:0 only via
    # WOIT_BENCH_ONE_DEVICE (bench.py maps every local rank to device 0 with it)
    env["WOIT_BENCH_ONE_DEVICE"] = "1"
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--backend", "gloo",
                          "--tiny", "--steps", "3", "--warmup", "3", "--c4-steps", "3", "--no-cpu", "--no-e2e"],
                         capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["config"]["height"] == 2 * (1080 // 8)
    c4 = line["config4_strong"]
    assert c4["n_gpus"] == 2 and c4["gathered_image_bitwise_equal_1gpu"] is True
    assert c4["fragments"] == (3840 // 8) * (2160 // 8) * 128
