"""Run the fused frame kernel a few times on a BASELINE config (for ncu / nsys captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2201_00094_b200 as W  # noqa: E402
from paper_2201_00094_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="smoke")
ap.add_argument("--width", type=int, default=1920)
ap.add_argument("--height", type=int, default=1080)
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--rank", type=int, default=3)
ap.add_argument("--iters", type=int, default=3)
args = ap.parse_args()

frame = W.FrameFragments.synthetic(args.workload, args.width, args.height, seed=1, layers=args.layers)
cfg = W.RenderConfig(rank=args.rank, width=args.width, height=args.height)
lib = _lib.load()
P, n = frame.npix, frame.nfrag
coeffs = torch.empty(P, 2 << args.rank, 3, device="cuda")
vhat = torch.empty(n, 3, device="cuda")
out = torch.empty(P, 3, device="cuda")
wsn = lib.woit_frame_workspace_bytes(P, n)
ws = torch.empty(wsn, dtype=torch.uint8, device="cuda")
bs = _lib.Bufs()
bs.coeffs, bs.vhat, bs.output = coeffs.data_ptr(), vhat.data_ptr(), out.data_ptr()
fs, ps = frame.c_struct(), W.pipeline._params(cfg, args.rank)
st = torch.cuda.current_stream().cuda_stream
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.iters)]
for i in range(args.iters):
    ev[2 * i].record()
    _lib.check(lib.woit_render_band(fs, ps, bs, ws.data_ptr(), wsn, st), "render")
    ev[2 * i + 1].record()
torch.cuda.synchronize()
print("ms per frame:", [round(ev[2 * i].elapsed_time(ev[2 * i + 1]), 3) for i in range(args.iters)])
