"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container only (it imports /root/reference/pkg/src, which does
not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Each fixture stores the reference's outputs for one input stream, computed by
calling the reference's own functions (``woit.pipeline.FrameBuffers.allocate``,
``step1_depth_bounds`` .. ``step4_composite``, ``woit.wavelet.*_batch``), i.e.
exactly what ``_wavelet_band`` does (pipeline.py:321-330). Synthetic inputs are
regenerated from ``paper_2201_00094_b200.synth`` at test time and pinned here by
a checksum; scene inputs (wine-bottle, glass-stack, ...) come from the
reference's ``cast_frame`` and are stored in full because they are small.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from woit import pipeline as rp  # noqa: E402  (reference)
from woit import wavelet as rw  # noqa: E402
from woit import packing as rpk  # noqa: E402
from woit.scene import FrameFragments, camera_rays, cast_frame, preset, Scene, Camera  # noqa: E402

from paper_2201_00094_b200 import synth  # noqa: E402


def stream_digest(sf) -> str:
    h = hashlib.sha256()
    for a in (sf.offsets, sf.depth, sf.alpha, sf.trans, sf.radiance, sf.normal, sf.ior,
              sf.backface, sf.opaque_depth, sf.opaque_color):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def synth_to_reference(sf) -> FrameFragments:
    f64 = lambda a: np.asarray(a, dtype=np.float64)
    return FrameFragments(sf.width, sf.rows, sf.pixel_ids(), f64(sf.depth), f64(sf.alpha),
                          f64(sf.trans), f64(sf.radiance), f64(sf.normal), f64(sf.ior),
                          sf.backface.astype(bool), sf.offsets.copy(), f64(sf.opaque_depth),
                          f64(sf.opaque_color))


def run_reference(frame: FrameFragments, cfg: rp.RenderConfig, scene_camera=None):
    """All outputs of _wavelet_band for one full-frame band, plus v̂."""
    cam = Camera() if scene_camera is None else scene_camera
    rays = camera_rays(cam, frame.width, frame.height)
    bufs = rp.FrameBuffers.allocate(frame, cfg.rank)
    rp.step1_depth_bounds(frame, bufs)
    rp.step2_build(frame, bufs, cfg)
    if frame.pixel.size:
        z = rp._fragment_z(frame, bufs)
        vhat = np.exp(-rw.interp_absorbance_batch(bufs.coeffs, frame.pixel, z, bufs.rank))
    else:
        z = np.zeros(0)
        vhat = np.zeros((0, 3))
    rp.step3_accumulate(rays, frame, bufs, cfg)
    full = frame.opaque_color.reshape(frame.height, frame.width, 3)
    rp.step4_composite(bufs, cfg, full_opaque_image=full)
    total = rw.total_absorbance_batch(bufs.coeffs, bufs.rank)
    # the whole-frame entry point must agree with the step sequence
    img = rp.render_frame(Scene(cam, ()), cfg, frame=frame)
    assert np.array_equal(img.reshape(-1, 3), bufs.output)
    return dict(near=bufs.near, far=bufs.far, coeffs=bufs.coeffs, accum=bufs.accum,
                weight=bufs.accum_weight, refr=bufs.refraction_offset, output=bufs.output,
                vhat=vhat, z=z, total=total)


def cfg_dict(cfg: rp.RenderConfig) -> dict:
    keys = ("rank", "width", "height", "refraction", "chromatic_aberration", "cube_transmission",
            "normalize", "packed_storage", "aberration_taps", "refraction_scale",
            "literal_spectral_t", "cube_backface_only")
    return {k: getattr(cfg, k) for k in keys}


def save(name: str, **arrays) -> None:
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def synth_case(name, workload, W, H, seed, layers, **cfgkw):
    sf = synth.generate(workload, W, H, seed=seed, layers=layers)
    cfg = rp.RenderConfig(method="wavelet", width=W, height=H, workers=1, **cfgkw)
    out = run_reference(synth_to_reference(sf), cfg)
    meta = dict(kind="synth", workload=workload, width=W, height=H, seed=seed, layers=layers,
                digest=stream_digest(sf), cfg=cfg_dict(cfg))
    save(name, meta=np.array(repr(meta)), **out)


def scene_case(name, preset_name, W, H, shuffle_seed=None, **cfgkw):
    sc = preset(preset_name)
    frame = cast_frame(sc, W, H)
    if shuffle_seed is not None:
        frame = frame.shuffled(shuffle_seed)
    cfg = rp.RenderConfig(method="wavelet", width=W, height=H, workers=1, **cfgkw)
    out = run_reference(frame, cfg, sc.camera)
    cam = sc.camera
    meta = dict(kind="scene", preset=preset_name, width=W, height=H, cfg=cfg_dict(cfg),
                camera=dict(position=cam.position, forward=cam.forward, fov_deg=cam.fov_deg))
    save(name, meta=np.array(repr(meta)), f_offsets=frame.offsets, f_depth=frame.depth,
         f_alpha=frame.alpha, f_trans=frame.trans, f_radiance=frame.radiance,
         f_normal=frame.normal, f_ior=frame.ior, f_backface=frame.backface,
         f_opaque_depth=frame.opaque_depth, f_opaque_color=frame.opaque_color, **out)


def kernel_case():
    """Batch-kernel vectors on an UNBINNED stream (test_wavelet.py:206-257 style)."""
    rng = np.random.default_rng(1234)
    rank = 4
    P, n = 7, 300
    pix = rng.integers(0, P, n)
    z = rng.uniform(0, 1, n)
    a = rng.uniform(0, 1, (n, 3))
    coeffs = np.zeros((P, 1 << (rank + 1), 3))
    c = rw.TouchCounter()
    rw.build_into(coeffs, pix, z, a, rank, c)
    qpix = rng.integers(0, P, 500)
    qz = rng.uniform(0, 1, 500)
    interp = rw.interp_absorbance_batch(coeffs, qpix, qz, rank)
    cells = rng.integers(0, 1 << (rank + 1), 500)
    raw = rw.cells_raw_batch(coeffs, qpix, cells, rank)
    total = rw.total_absorbance_batch(coeffs, rank)
    # E5B9G9R9 words for random + dyadic triples (packing.py:46-88)
    triples = np.concatenate([rng.uniform(0, 2.0 ** 16, (200, 3)),
                              rng.uniform(0, 1e-3, (50, 3)),
                              np.array([[0.5, 0.25, 0.125], [0, 0, 0], [65408, 1, 0],
                                        [1e9, 0, 0], [1e-9, 0, 0]])])
    words = rpk.pack_rgb9e5(triples)
    packed_rt = rpk.roundtrip_coeff_array(coeffs)
    save("kernels", rank=np.array(rank), pix=pix, z=z, a=a, coeffs=coeffs, qpix=qpix, qz=qz,
         interp=interp, cells=cells, raw=raw, total=total, touches=np.array([c.per_insert]),
         triples=triples, words=words, packed_rt=packed_rt)


def baselines_case():
    """The reference's comparison methods (baselines.py:135-220) on fp32-exact inputs:
    synthetic streams, and scene streams rounded to fp32 (so sort order and ties are
    the device's). Reference near/far for WBOIT as pipeline.render_frame computes them."""
    from woit import baselines as rb

    def f32_frame(fr):
        r = lambda a: np.asarray(np.asarray(a, dtype=np.float32), dtype=np.float64)
        return FrameFragments(fr.width, fr.height, fr.pixel, r(fr.depth), r(fr.alpha), r(fr.trans), r(fr.radiance),
                              r(fr.normal), r(fr.ior), fr.backface, fr.offsets, r(fr.opaque_depth),
                              r(fr.opaque_color))

    cases = {
        "ragged": synth_to_reference(synth.generate("ragged", 16, 12, seed=3, layers=40)),
        "particles": synth_to_reference(synth.generate("particles", 8, 6, seed=9, layers=64)),
        "smokefire_shuf": f32_frame(cast_frame(preset("smoke-fire"), 24, 24).shuffled(7)),
        "wine": f32_frame(cast_frame(preset("wine-bottle"), 33, 33)),
    }
    out = {}
    for name, fr in cases.items():
        bg = fr.opaque_color
        near = np.full(fr.npix, np.inf)
        far = np.full(fr.npix, -np.inf)
        np.minimum.at(near, fr.pixel, fr.depth)
        np.maximum.at(far, fr.pixel, fr.depth)
        for cube in (False, True):
            tag = f"{name}_{'cube' if cube else 'plain'}"
            out[f"abuffer_{tag}"] = rb.abuffer_frame(fr, bg, cube)
            out[f"wboit_{tag}"] = rb.wboit_frame(fr, bg, near, far, cube, rb.DEFAULT_WBOIT_WEIGHT)
            out[f"mlab4_{tag}"] = rb.mlab_frame(fr, bg, 4, cube)
        if name in ("smokefire_shuf", "wine"):
            f32 = lambda a: np.asarray(a, dtype=np.float32)
            out[f"in_{name}"] = np.array(repr(dict(width=fr.width, height=fr.height)))
            for k in ("offsets", "depth", "alpha", "trans", "radiance", "normal", "ior", "backface",
                      "opaque_depth", "opaque_color"):
                a = getattr(fr, k)
                out[f"in_{name}_{k}"] = a if k in ("offsets", "backface") else f32(a)
    save("baselines", **out)


def cast_case():
    """The reference caster's CSR output (scene.py:463-630) for every preset at 32x24 and
    for test_scene.py's wide-fov corner-particle scene, plus the seeded particle
    positions (pins the scene description the device caster restates)."""
    from woit.scene import Material, OpaqueBackdrop, ParticleCloud
    from woit.core import Spectrum3

    mat = Material(alpha=0.6, transmission=Spectrum3.gray(0.2), radiance=Spectrum3.gray(0.4))
    wide = Scene(Camera(fov_deg=95.0),
                 (ParticleCloud(center=(-1.9, 0.9, 1.2), radius=0.5, count=60, particle_radius=0.2, material=mat,
                                seed_offset=1),
                  ParticleCloud(center=(2.1, -1.0, 1.4), radius=0.6, count=60, particle_radius=0.25, material=mat,
                                profile="mask", seed_offset=2),
                  OpaqueBackdrop(d=4.0, color=Spectrum3.gray(0.5))), rng_seed=3)
    from woit.scene import PRESET_NAMES
    scenes = [(n, preset(n), 32, 24) for n in PRESET_NAMES] + [("wide-fov", wide, 48, 20)]
    out = {}
    for name, sc, W, H in scenes:
        fr = cast_frame(sc, W, H)
        key = name.replace("-", "_")
        out[f"{key}_size"] = np.array([W, H])
        for k in ("offsets", "depth", "alpha", "trans", "radiance", "normal", "ior", "backface", "opaque_depth",
                  "opaque_color"):
            out[f"{key}_{k}"] = getattr(fr, k)
        for j, pr in enumerate(sc.primitives):
            if isinstance(pr, ParticleCloud):
                out[f"{key}_p{j}_positions"] = pr.positions
                out[f"{key}_p{j}_scale"] = pr.radiance_scale
    save("cast", **out)


def deep_cases():
    """> 160 fragments per pixel (the deep-frame kernel instance, configs 5) at the
    other ranks config 5 sweeps: 8 and 32 coefficients (rank 4: one warp per CTA,
    its own shared-memory layout), plus a 320-fragment rank-2 case (deeper than
    one 256-fragment sub-tile: the long-pixel kernel)."""
    synth_case("particles_256_r2", "particles", 8, 6, 10, 256, rank=2)
    synth_case("particles_256_r4", "particles", 8, 6, 11, 256, rank=4)
    synth_case("particles_192_r4", "particles", 12, 5, 12, 192, rank=4)
    synth_case("particles_320_r2", "particles", 6, 4, 13, 320, rank=2)


def main():
    if "--only-baselines" in sys.argv:
        baselines_case()
        return
    if "--only-cast" in sys.argv:
        cast_case()
        return
    if "--only-deep" in sys.argv:
        deep_cases()
        return
    # config 1 of BASELINE.json: 64x64, the single-plane pane + 4 random layers, rank 3
    synth_case("plane4_64", "plane4", 64, 64, 1, 5, rank=3)
    # ragged CSR (empty pixels, runs up to 40) at every supported rank
    for rank in range(7):
        synth_case(f"ragged_r{rank}", "ragged", 16, 12, 3, 40, rank=rank)
    synth_case("ragged_r3_linear", "ragged", 16, 12, 5, 40, rank=3, normalize=False)
    # deep pixels: the precision regime of configs 4/5
    synth_case("particles_256", "particles", 8, 6, 9, 256, rank=3)
    deep_cases()
    synth_case("smoke_32", "smoke", 40, 24, 2, 32, rank=3)
    # reference scenes through the reference's own caster
    scene_case("wine33_refr_ca_cube", "wine-bottle", 33, 33, rank=3, refraction=True,
               chromatic_aberration=True, cube_transmission=True)
    scene_case("wine65_refr_cube", "wine-bottle", 65, 65, rank=3, refraction=True,
               cube_transmission=True)
    scene_case("wine33_refr_ca7_lit", "wine-bottle", 33, 33, rank=4, refraction=True,
               chromatic_aberration=True, aberration_taps=7, literal_spectral_t=True,
               cube_transmission=True, cube_backface_only=True)
    scene_case("glass48", "glass-stack", 48, 48, rank=3)
    scene_case("glass48_linear", "glass-stack", 48, 48, rank=3, normalize=False)
    scene_case("glass17_refr", "glass-stack", 17, 17, rank=3, refraction=True)
    scene_case("smokefire24", "smoke-fire", 24, 24, rank=3)
    scene_case("smokefire24_shuf7", "smoke-fire", 24, 24, shuffle_seed=7, rank=3)
    scene_case("single5_r0", "single-plane", 5, 5, rank=0)
    scene_case("single5_r3", "single-plane", 5, 5, rank=3)
    scene_case("glass9_packed", "glass-stack", 9, 9, rank=3, packed_storage=True)
    kernel_case()
    baselines_case()
    cast_case()


if __name__ == "__main__":
    main()
