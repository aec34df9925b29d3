"""On-device fragment producer against the reference's own
cast_frame output (tests/golden/cast.npz, make_golden.py --only-cast): the CSR
offsets and backface flags exactly, the float64 geometry rounded once to fp32."""

import os

import numpy as np
import pytest
import torch

from paper_2201_00094_b200 import scene as S
from paper_2201_00094_b200.pipeline import Camera

GOLD = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cast.npz"))


def wide_fov_scene():
    mat = S.Material(0.6, S.gray(0.2), S.gray(0.4))
    return S.Scene(Camera(fov_deg=95.0),
                   (S.ParticleCloud((-1.9, 0.9, 1.2), 0.5, 60, 0.2, mat, seed_offset=1),
                    S.ParticleCloud((2.1, -1.0, 1.4), 0.6, 60, 0.25, mat, "mask", 2),
                    S.OpaqueBackdrop(4.0, S.gray(0.5))), rng_seed=3)


SCENES = [(n, lambda n=n: S.preset(n)) for n in S.PRESET_NAMES] + [("wide-fov", wide_fov_scene)]


@pytest.mark.parametrize("name,make", SCENES)
def test_scene_description_matches_reference(name, make):
    """Particle positions / radiance scales drawn exactly as the reference seeds them."""
    sc = make()
    key = name.replace("-", "_")
    for j, pr in enumerate(sc.primitives):
        if isinstance(pr, S.ParticleCloud):
            np.testing.assert_array_equal(pr.positions, GOLD[f"{key}_p{j}_positions"])
            np.testing.assert_array_equal(pr.radiance_scale, GOLD[f"{key}_p{j}_scale"])


def test_unknown_preset():
    with pytest.raises(ValueError, match="unknown preset"):
        S.preset("nope")


@pytest.mark.gpu
@pytest.mark.parametrize("name,make", SCENES)
def test_device_cast_matches_reference(name, make):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    key = name.replace("-", "_")
    W, H = (int(x) for x in GOLD[f"{key}_size"])
    fr = S.cast_frame(make(), W, H)
    h = lambda t: t.cpu().numpy()
    np.testing.assert_array_equal(h(fr.offsets), GOLD[f"{key}_offsets"])
    np.testing.assert_array_equal(h(fr.backface).astype(bool), GOLD[f"{key}_backface"])
    for k in ("depth", "alpha", "trans", "radiance", "normal", "ior", "opaque_color"):
        ref = GOLD[f"{key}_{k}"]
        got = h(getattr(fr, k)).astype(np.float64).reshape(ref.shape)
        # one fp32 rounding of the f64 geometry (+ exp / sqrt ulps): relative 1e-6
        np.testing.assert_allclose(got, ref, rtol=1e-6, atol=1e-7, err_msg=f"{name}.{k}")
    od = GOLD[f"{key}_opaque_depth"]
    got = h(fr.opaque_depth).astype(np.float64)
    np.testing.assert_array_equal(np.isinf(got), np.isinf(od))
    fin = np.isfinite(od)
    np.testing.assert_allclose(got[fin], od[fin], rtol=1e-6)


@pytest.mark.gpu
def test_render_frame_casts_on_device():
    """render_frame(scene, cfg) without frame=: cast on the GPU, then render -- equal to
    rendering the reference-cast stream of the same scene."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2201_00094_b200 as W

    sc = S.preset("wine-bottle")
    cfg = W.RenderConfig(width=32, height=24, refraction=True, chromatic_aberration=True, cube_transmission=True)
    img = W.render_frame(sc, cfg)
    key = "wine_bottle"
    g = lambda k: GOLD[f"{key}_{k}"]
    frame = W.FrameFragments.from_numpy(32, 24, g("offsets"), g("depth"), g("alpha"), g("trans"), g("radiance"),
                                        g("normal"), g("ior"), g("backface").astype(np.uint8), g("opaque_depth"),
                                        g("opaque_color"))
    ref = W.render_frame(sc, cfg, frame=frame)
    assert (img - ref).abs().max().item() <= 1e-5
