"""Measured comparison of the build strategies the north star names (BASELINE.json (1)).

    python tools/build_compare.py [--workload smoke --width 1920 --height 1080 --layers 32]

On one config (default: config 2) it times, with CUDA events on the launching
stream after warm-up (median of --iters):
  tile_build     woit_step2_build: CSR tiles in shared memory (the shipped design,
                 deterministic), bounds from a prior step1
  atomic_build   woit_build_atomic: unbinned stream + pixel ids, fp32 red.global.add
                 of the closed-form projection into coeffs[P][S][3]
  bin_sort       woit_bin_by_pixel on a shuffled (unbinned) stream: stable radix sort
  bin_gather     permuting depth/alpha/T into CSR order (what binning an unbinned
                 stream costs before the tile build)
  fused_frame    woit_render_band: bounds+build+eval+composite in one launch
  bin_frame_{layer_major,random}  woit_bin_frame on an unbinned stream (layer-major
                 arrival, or a random permutation): the hand-written stable sort whose
                 last pass scatters depth/alpha/T/L into CSR order
  unbinned_*_to_rendered  woit_bin_frame + woit_render_band (unbinned stream -> image)
and prints one JSON object. Coefficient agreement between the two builds is
reported as max |diff|.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2201_00094_b200 as W  # noqa: E402
from paper_2201_00094_b200 import _lib  # noqa: E402
from paper_2201_00094_b200.frame import ptr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="smoke")
ap.add_argument("--width", type=int, default=1920)
ap.add_argument("--height", type=int, default=1080)
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--rank", type=int, default=3)
ap.add_argument("--iters", type=int, default=20)
args = ap.parse_args()

lib = _lib.load()
frame = W.FrameFragments.synthetic(args.workload, args.width, args.height, seed=1, layers=args.layers)
cfg = W.RenderConfig(rank=args.rank, width=args.width, height=args.height)
P, n = frame.npix, frame.nfrag
st = torch.cuda.current_stream()


def timed(fn, setup=None):
    ts = []
    for i in range(args.iters + 3):
        if setup:
            setup()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


bufs = W.FrameBuffers.allocate(frame, args.rank)
W.step1_depth_bounds(frame, bufs)
torch.cuda.synchronize()
zero = lambda: bufs.coeffs.zero_()

res = {"config": {"workload": args.workload, "width": args.width, "height": args.height,
                  "layers": args.layers, "rank": args.rank, "nfrag": n, "npix": P}}
res["tile_build_ms"] = timed(lambda: W.step2_build(frame, bufs, cfg), zero)
tile = bufs.coeffs.clone()

pix = W.pixel_ids(frame)
res["atomic_build_ms"] = timed(lambda: W.step2_build_atomic(frame, bufs, cfg, pix), zero)
res["atomic_vs_tile_max_abs"] = float((bufs.coeffs - tile).abs().max())

# an unbinned stream: the same fragments in a random order
g = torch.Generator(device="cuda").manual_seed(7)
order = torch.randperm(n, device="cuda", generator=g)
pix64 = pix.to(torch.int64)[order]
offsets = torch.empty(P + 1, dtype=torch.int64, device="cuda")
perm = torch.empty(n, dtype=torch.int64, device="cuda")
wsn = lib.woit_bin_workspace_bytes(n, P)
ws = torch.empty(max(wsn, 1), dtype=torch.uint8, device="cuda")
res["bin_sort_ms"] = timed(lambda: _lib.check(
    lib.woit_bin_by_pixel(ptr(pix64), n, P, ptr(offsets), ptr(perm), ptr(ws), wsn, st.cuda_stream), "bin"))
res["bin_offsets_equal"] = bool(torch.equal(offsets, frame.offsets))
d_s, a_s, t_s = frame.depth[order], frame.alpha[order], frame.trans[order]
d2, a2, t2 = torch.empty_like(d_s), torch.empty_like(a_s), torch.empty_like(t_s)


def gather():
    torch.index_select(d_s, 0, perm, out=d2)
    torch.index_select(a_s, 0, perm, out=a2)
    torch.index_select(t_s, 0, perm, out=t2)


res["bin_gather_ms"] = timed(gather)
res["binned_total_ms"] = res["bin_sort_ms"] + res["bin_gather_ms"] + res["tile_build_ms"]
pix_shuf = pix[order].contiguous()
fs = W.FrameFragments(**{**frame.__dict__, "depth": d_s, "alpha": a_s, "trans": t_s})
res["atomic_unbinned_build_ms"] = timed(lambda: W.step2_build_atomic(fs, bufs, cfg, pix_shuf), zero)
res["atomic_unbinned_vs_tile_max_abs"] = float((bufs.coeffs - tile).abs().max())

out = W.FrameBuffers.allocate(frame, args.rank)
full = frame.opaque_color.reshape(args.height, args.width, 3)
res["fused_frame_ms"] = timed(lambda: W.render_band(frame, cfg, bufs=out, full_opaque_image=full))

# the hand-written binning (woit_bin_frame): stable radix sort by pixel whose last pass
# scatters the fields into CSR order, then the fused frame on the binned stream. Two
# arrival orders: layer-major (a producer emitting one layer of the whole frame after
# another -- SURVEY.md §8(d)'s unbinned order) and a uniformly random permutation.
run = frame.offsets[1:] - frame.offsets[:-1]
L = int(run.max())
lm = (frame.offsets[:-1][None, :] + torch.arange(L, device="cuda")[:, None])  # [layer][pixel] CSR index
lm = lm[torch.arange(L, device="cuda")[:, None] < run[None, :]].contiguous()  # layer-major arrival order
for tag, od in (("layer_major", lm), ("random", order)):
    pix32 = pix[od].contiguous()
    ins = dict(depth=frame.depth[od], alpha=frame.alpha[od], trans=frame.trans[od], radiance=frame.radiance[od])
    outs = {k: torch.empty_like(v) for k, v in ins.items()}
    fi, fo = _lib.Frags(), _lib.Frags()
    for f, dd in ((fi, ins), (fo, outs)):
        f.width, f.height, f.npix, f.nfrag = args.width, args.height, P, n
        for k, v in dd.items():
            setattr(f, k, ptr(v))
    offs2 = torch.empty(P + 1, dtype=torch.int64, device="cuda")
    wsn2 = lib.woit_bin_frame_workspace_bytes(n, P)
    ws2 = torch.empty(wsn2, dtype=torch.uint8, device="cuda")
    bin_frame = lambda: _lib.check(lib.woit_bin_frame(ptr(pix32), fi, fo, ptr(offs2), None, ptr(ws2), wsn2,
                                                      st.cuda_stream), "bin_frame")
    res[f"bin_frame_{tag}_ms"] = timed(bin_frame)
    res[f"bin_frame_{tag}_offsets_equal"] = bool(torch.equal(offs2, frame.offsets))
    fb = W.FrameFragments(width=args.width, height=args.height, offsets=offs2, depth=outs["depth"],
                          alpha=outs["alpha"], trans=outs["trans"], radiance=outs["radiance"], normal=frame.normal,
                          ior=frame.ior, backface=frame.backface, opaque_depth=frame.opaque_depth,
                          opaque_color=frame.opaque_color)
    out2 = W.FrameBuffers.allocate(frame, args.rank)
    res[f"unbinned_{tag}_to_rendered_ms"] = timed(lambda: (bin_frame(), W.render_band(fb, cfg, bufs=out2,
                                                                                      full_opaque_image=full)))
    res[f"unbinned_{tag}_render_vs_csr_max_abs"] = float((out2.output - out.output).abs().max())
    del ins, outs, ws2
    torch.cuda.empty_cache()
print(json.dumps(res))
