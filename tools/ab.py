"""Same-box A/B timing of libwoit builds (run on the GPU box).

    python tools/ab.py snapshot NAME          # here: build the working tree into variants_lib/libwoit_NAME.so
    python tools/ab.py time [--rounds 3] [--iters 200] [--configs 2,4]   # on the box

Each round times every snapshot on every config in its own process (WOIT_LIB
selects the library), alternating the libraries, with CUDA events around the
render_band launches of a resident synthetic stream (config 2: 1080p x 32 smoke;
config 4: a 540-row quarter of 4K x 128 particles; config 5: a 135-row slice of
the 8K x 256 eighth). Prints the per-round ms and the median per (lib, config).
"""
import glob
import json
import os
import statistics
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VDIR = os.path.join(REPO, "variants_lib")
CFG = {"2": ("smoke", 1920, 1080, 32, 3), "4": ("particles", 3840, 540, 128, 3),
       "5": ("particles", 7680, 135, 256, 3), "5r4": ("particles", 7680, 135, 256, 4),
       "5r2": ("particles", 7680, 135, 256, 2)}


def snapshot(name, defines=()):
    sys.path.insert(0, REPO)
    from paper_2201_00094_b200 import build as B
    os.makedirs(VDIR, exist_ok=True)
    out = os.path.join(VDIR, f"libwoit_{name}.so")
    B.build(defines=tuple(defines) or (f"WOIT_SNAPSHOT_{name}=1",), out=out, force=True)
    print("built", out)


def child(cfg, iters):
    sys.path.insert(0, REPO)
    import torch
    import paper_2201_00094_b200 as W
    from paper_2201_00094_b200 import _lib
    if cfg == "3":  # config 3: the wine-bottle preset cast on the device, refraction + CA + cube
        from paper_2201_00094_b200.scene import cast_frame, preset
        sc = preset("wine-bottle")
        w, h, rank = 1920, 1080, 3
        frame = cast_frame(sc, w, h)
        cfgo = W.RenderConfig(rank=3, width=w, height=h, refraction=True, chromatic_aberration=True,
                              cube_transmission=True)
        rays = W.camera_rays(sc.camera, w, h)
        full = frame.opaque_color.reshape(h, w, 3)
        bufs = W.FrameBuffers.allocate(frame, 3)
        ws = W.Workspace()
        run = lambda: W.render_band(frame, cfgo, rays, bufs=bufs, full_opaque_image=full, ws=ws)
        for _ in range(5):
            run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            run()
        b.record()
        torch.cuda.synchronize()
        print(json.dumps({"ms": a.elapsed_time(b) / iters, "checksum": float(bufs.output.double().sum())}))
        return
    wl, w, h, layers, rank = CFG[cfg]
    frame = W.FrameFragments.synthetic(wl, w, h, seed=1, layers=layers)
    cfgo = W.RenderConfig(rank=rank, width=w, height=h)
    lib = _lib.load()
    P, n = frame.npix, frame.nfrag
    coeffs = torch.empty(P, 2 << rank, 3, device="cuda")
    vhat = torch.empty(n, 3, device="cuda")
    out = torch.empty(P, 3, device="cuda")
    wsn = lib.woit_frame_workspace_bytes(P, n)
    ws = torch.empty(wsn, dtype=torch.uint8, device="cuda")
    bs = _lib.Bufs()
    bs.coeffs, bs.vhat, bs.output = coeffs.data_ptr(), vhat.data_ptr(), out.data_ptr()
    fs, ps = frame.c_struct(), W.pipeline._params(cfgo, rank)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(5):
        _lib.check(lib.woit_render_band(fs, ps, bs, ws.data_ptr(), wsn, st), "render")
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        _lib.check(lib.woit_render_band(fs, ps, bs, ws.data_ptr(), wsn, st), "render")
    b.record()
    torch.cuda.synchronize()
    print(json.dumps({"ms": a.elapsed_time(b) / iters, "checksum": float(out.double().sum())}))


def time_all(rounds, iters, configs):
    libs = sorted(glob.glob(os.path.join(VDIR, "libwoit_*.so")))
    res = {}
    for r in range(rounds):
        order = libs if r % 2 == 0 else libs[::-1]
        for cfg in configs:
            for lib in order:
                name = os.path.basename(lib)[8:-3]
                env = dict(os.environ, WOIT_LIB=lib)
                p = subprocess.run([sys.executable, __file__, "child", cfg, str(iters)], env=env,
                                   capture_output=True, text=True)
                try:
                    d = json.loads(p.stdout.strip().splitlines()[-1])
                except Exception:
                    print(name, cfg, "FAILED", p.stderr[-600:], flush=True)
                    continue
                res.setdefault((name, cfg), []).append(d["ms"])
                print(f"round {r} cfg {cfg} {name}: {d['ms']:.4f} ms  checksum {d['checksum']:.9e}", flush=True)
    print("median:")
    for (name, cfg), v in sorted(res.items(), key=lambda x: (x[0][1], x[0][0])):
        print(f"  cfg {cfg} {name:12s} {statistics.median(v):.4f} ms  {['%.4f' % x for x in v]}")


if __name__ == "__main__":
    if sys.argv[1] == "snapshot":
        snapshot(sys.argv[2], sys.argv[3:])
    elif sys.argv[1] == "child":
        child(sys.argv[2], int(sys.argv[3]))
    else:
        import argparse
        ap = argparse.ArgumentParser()
        ap.add_argument("cmd")
        ap.add_argument("--rounds", type=int, default=3)
        ap.add_argument("--iters", type=int, default=200)
        ap.add_argument("--configs", default="2,4")
        a = ap.parse_args()
        time_all(a.rounds, a.iters, a.configs.split(","))
