"""Where config 3's frame time goes: the full frame against the same pixels with no
fragments (every window empty) and against the same stream with the optional features
off. CUDA events, median of 3 batches of --iters launches, inputs resident.

    python tools/c3_split.py [--iters 20]
"""
import argparse
import dataclasses
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_00094_b200 as W  # noqa: E402
import config3  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--only", choices=("full", "plain", "refraction", "empty"), default=None,
                    help="time one case only (e.g. under ncu with --iters 1)")
    args = ap.parse_args()
    sf, cam = config3.load()
    Wd, H = sf.width, sf.height
    frame = W.FrameFragments.from_synth(sf)
    rays = W.camera_rays(W.Camera(**cam), Wd, H)
    full = frame.opaque_color.reshape(H, Wd, 3)
    st = torch.cuda.current_stream()
    ws = W.Workspace()

    def timed(fn, batches=3):
        if args.iters <= 1:  # one launch (profiling)
            fn()
            torch.cuda.synchronize()
            return 0.0
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(batches):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(args.iters):
                fn()
            b.record(st)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / args.iters)
        return float(np.median(ts))

    def run(fr, **kw):
        cfg = W.RenderConfig(width=Wd, height=H, rank=3, **kw)
        bufs = W.FrameBuffers.allocate(fr, cfg.rank, vhat=True)
        return timed(lambda: W.render_band(fr, cfg, rays, bufs=bufs, full_opaque_image=full, ws=ws))

    flags = dict(refraction=True, chromatic_aberration=True, cube_transmission=True, aberration_taps=5)
    off = frame.offsets
    counts = (off[1:] - off[:-1]).view(-1, 32) if frame.npix % 32 == 0 else None
    res = {"fragments": frame.nfrag, "pixels": frame.npix}
    if counts is not None:
        res["windows"] = int(counts.shape[0])
        res["nonempty_windows"] = int((counts.sum(1) > 0).sum())
        res["nonempty_pixels"] = int((off[1:] > off[:-1]).sum())
    if args.only in (None, "full"):
        res["full_ms"] = run(frame, **flags)
    if args.only in (None, "plain"):
        res["plain_flags_ms"] = run(frame)
    if args.only in (None, "refraction"):
        res["refraction_only_ms"] = run(frame, refraction=True)
    ef = dataclasses.replace(frame, offsets=torch.zeros_like(frame.offsets),
                             **{k: getattr(frame, k)[:0].clone() for k in
                                ("depth", "alpha", "trans", "radiance", "normal", "ior", "backface")})
    if args.only in (None, "empty"):
        res["empty_ms"] = run(ef, **flags)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
