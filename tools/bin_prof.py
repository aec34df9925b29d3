"""Per-kernel view of woit_bin_frame at config 2 (1080p x 32, layer-major arrival, core
fields): run under ncu for the launch list.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \\
        python tools/bin_prof.py [--random]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2201_00094_b200 as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--random", action="store_true")
ap.add_argument("--iters", type=int, default=2)
a = ap.parse_args()
frame = W.FrameFragments.synthetic("smoke", 1920, 1080, seed=1, layers=32)
n, P = frame.nfrag, frame.npix
run = frame.offsets[1:] - frame.offsets[:-1]
L = int(run.max())
if a.random:
    od = torch.randperm(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(5))
else:
    lm = frame.offsets[:-1][None, :] + torch.arange(L, device="cuda")[:, None]
    od = lm[torch.arange(L, device="cuda")[:, None] < run[None, :]].contiguous()
pix = W.pixel_ids(frame)[od].to(torch.int32).contiguous()
ins = [frame.depth[od], frame.alpha[od], frame.trans[od], frame.radiance[od]]
for _ in range(a.iters):
    fb = W.FrameFragments.from_unbinned(1920, 1080, pix, *ins)
torch.cuda.synchronize()
print("ok", bool(torch.equal(fb.offsets, frame.offsets)))
