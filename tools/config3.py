"""Config 3: the reference's wine-bottle frame at 1920x1080 with
refraction + chromatic aberration (k = 5) + cubed transmission, on one B200.

    python tools/config3.py [--iters 20] [--no-oracle]

Input: data/config3_wine_1080p.npz from tools/make_config3.py (the reference's
own cast_frame output, fp32). Prints one JSON object: the GPU frame time (CUDA
events, inputs resident, median over 3 batches of --iters back-to-back launches, as bench.py times steps) of the general
(GEN) fused kernel, the same with the in-repo diffusion on (K_resolve blur +
frame), roofline numbers with SURVEY.md §8(d)'s config-3 byte count, and the
max |error| of coefficients / v̂ / image against the float64 oracle run on the
same fp32 inputs (all host threads), with the oracle's own wall time.
"""
import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_00094_b200 as W  # noqa: E402
from paper_2201_00094_b200 import synth  # noqa: E402

DATA = os.path.join(REPO, "data", "config3_wine_1080p.npz")


def load():
    """The config-3 stream: data/config3_wine_1080p.npz (the reference's own cast_frame
    output) when present, else the on-device caster's cast of the same preset (its CSR is
    identical to the reference's and its values within one fp32 rounding, tests/test_cast.py)."""
    if os.path.exists(DATA):
        d = np.load(DATA)
        Wd, H = int(d["width"]), int(d["height"])
        sf = synth.SynthFrame(Wd, H, 0, H, d["offsets"], d["depth"], d["alpha"], d["trans"], d["radiance"],
                              d["normal"], d["ior"], d["backface"], d["opaque_depth"], d["opaque_color"])
        cam = dict(position=tuple(d["cam_position"]), forward=tuple(d["cam_forward"]), fov_deg=float(d["cam_fov"]))
        return sf, cam
    from paper_2201_00094_b200 import scene as S

    sc = S.preset("wine-bottle")
    sf = S.cast_frame(sc, 1920, 1080).to_synth()
    c = sc.camera
    return sf, dict(position=tuple(c.position), forward=tuple(c.forward), fov_deg=float(c.fov_deg))


CFG = dict(rank=3, refraction=True, chromatic_aberration=True, cube_transmission=True, aberration_taps=5)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--no-oracle", action="store_true")
    args = ap.parse_args()
    sf, cam = load()
    Wd, H = sf.width, sf.height
    frame = W.FrameFragments.from_synth(sf)
    cfg = W.RenderConfig(width=Wd, height=H, **CFG)
    rays = W.camera_rays(W.Camera(**cam), Wd, H)
    full = frame.opaque_color.reshape(H, Wd, 3)
    bufs = W.FrameBuffers.allocate(frame, cfg.rank, vhat=True)
    st = torch.cuda.current_stream()

    def timed(fn, batches=3):
        """Median over batches of back-to-back launches (CUDA events around each batch
        on the launching stream), as bench.py times its steps."""
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

    ws = W.Workspace()
    ms = timed(lambda: W.render_band(frame, cfg, rays, bufs=bufs, full_opaque_image=full, ws=ws))
    dcfg = W.RenderConfig(width=Wd, height=H, diffusion=0.5, diffusion_radius=4, **CFG)
    dbufs = W.FrameBuffers.allocate(frame, cfg.rank)
    ms_diff = timed(lambda: W.render_band(frame, dcfg, rays, bufs=dbufs, full_opaque_image=full, ws=ws))
    blur_ms = timed(lambda: W.resolve_blur(full, 4))
    P, n = frame.npix, frame.nfrag
    S = 1 << (cfg.rank + 1)
    alg = n * (44 + 16) + P * (32 + 12 * S + 4)  # + normal, ior, opaque depth
    peak = 6451.2
    try:
        peak = float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    res = {"config": "config3: wine-bottle cast_frame 1920x1080, refraction + CA k=5 + cube, rank 3",
           "fragments": n, "pixels": P, "frame_ms": ms, "gfrag_per_s": n / ms / 1e6,
           "algorithmic_bytes": alg, "achieved_gbs": alg / ms / 1e6, "peak_gbs": peak,
           "frac": alg / ms / 1e6 / peak, "with_diffusion_ms": ms_diff, "blur_ms": blur_ms}
    if not args.no_oracle:
        sys.path.insert(0, REPO)
        from oracle import woit_oracle as O

        t0 = time.time()
        ref = O.render_frame(O.OFrame.from_synth(sf), O.OConfig(width=Wd, height=H, workers=O.default_workers(),
                                                                 **CFG), O.OCamera(**cam))
        res["oracle_s"] = time.time() - t0
        res["oracle_threads"] = O.default_workers()
        h = lambda t: t.detach().double().cpu().numpy()
        res["max_err_coeffs"] = float(np.abs(h(bufs.coeffs) - ref.coeffs).max())
        res["max_err_vhat"] = float(np.abs(h(bufs.vhat) - ref.vhat).max())
        res["max_err_image"] = float(np.abs(h(bufs.output) - ref.output).max())
        res["near_far_bit_exact"] = bool(np.array_equal(h(bufs.near), ref.near.astype(np.float32).astype(np.float64))
                                         and np.array_equal(h(bufs.far), ref.far.astype(np.float32).astype(np.float64)))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
