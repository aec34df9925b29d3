"""Real presets end to end on one B200: cast the scene on
the device (scene.cast_frame), then render it with the fused wavelet kernel.

    python tools/scenes_bench.py [--width 1920 --height 1080] [--iters 10]

CUDA-event times (median after 3 warm-ups) of the two device passes of the caster
and of the render, per preset, as one JSON object.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_00094_b200 as W  # noqa: E402
from paper_2201_00094_b200 import scene as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--width", type=int, default=1920)
ap.add_argument("--height", type=int, default=1080)
ap.add_argument("--iters", type=int, default=10)
args = ap.parse_args()
st = torch.cuda.current_stream()


def timed(fn):
    ts = []
    for i in range(args.iters + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return float(np.median(ts))


FLAGS = {"wine-bottle": dict(refraction=True, chromatic_aberration=True, cube_transmission=True),
         "glass-stack": dict(refraction=True), "car-fog": {}, "smoke-fire": {}, "leaves": {}, "single-plane": {}}
out = {"width": args.width, "height": args.height}
for name in S.PRESET_NAMES:
    sc = S.preset(name)
    frame = S.cast_frame(sc, args.width, args.height)
    cfg = W.RenderConfig(width=args.width, height=args.height, **FLAGS[name])
    rays = W.camera_rays(sc.camera, args.width, args.height)
    full = frame.opaque_color.reshape(args.height, args.width, 3)
    bufs = W.FrameBuffers.allocate(frame, cfg.rank)
    out[name] = {"fragments": frame.nfrag,
                 "cast_ms": timed(lambda: S.cast_frame(sc, args.width, args.height)),
                 "render_ms": timed(lambda: W.render_band(frame, cfg, rays, bufs=bufs, full_opaque_image=full)),
                 "flags": FLAGS[name]}
print(json.dumps(out))
