"""Diffusion ("resolve and blur", SURVEY.md §8 row GAP).

The reference has no diffusion pass, so this feature follows
the in-repo definition in include/woit.h (WOIT_DIFFUSION) and its parity is
UNPINNED: the GPU path is checked against the oracle twin (oracle.blur_image,
the D_p accumulation in step3, the lerp in step4), and the oracle twin against
an independent restatement (scipy's correlate1d) and invariants. With diffusion
off, outputs must be bit-identical to the path without the feature.
"""

import dataclasses

import numpy as np
import pytest
import torch

from oracle import woit_oracle as O
from paper_2201_00094_b200 import _lib, synth
from paper_2201_00094_b200.pipeline import RenderConfig
from tests import fixtures

COEF_TOL = 1e-5
VHAT_TOL = 1e-5
IMG_TOL = 1e-4
BLUR_TOL = 2e-6  # fp32 taps and accumulation vs the f64 twin, image values in [0, 1]


# ---------------------------------------------------------------------------
# CPU: the oracle twin and the host-side contract


@pytest.mark.parametrize("r", [1, 2, 4, 9, 64])
def test_gaussian_taps(r):
    g = O.gaussian_taps(r)
    assert g.shape == (2 * r + 1,)
    assert abs(g.sum() - 1.0) < 1e-15
    np.testing.assert_array_equal(g, g[::-1])
    assert np.all(np.diff(g[: r + 1]) > 0)


@pytest.mark.parametrize("shape,r", [((9, 13), 1), ((23, 37), 4), ((16, 5), 7)])
def test_blur_twin_matches_scipy(shape, r):
    from scipy.ndimage import correlate1d

    img = np.random.default_rng(5).random(shape + (3,))
    g = O.gaussian_taps(r)
    ref = correlate1d(correlate1d(img, g, axis=1, mode="nearest"), g, axis=0, mode="nearest")
    np.testing.assert_allclose(O.blur_image(img, r), ref, rtol=0, atol=1e-14)


def test_blur_twin_invariants():
    c = np.full((11, 7, 3), 0.375)
    np.testing.assert_allclose(O.blur_image(c, 5), c, atol=1e-15)
    img = np.random.default_rng(1).random((12, 10, 3))
    b = O.blur_image(img, 3)
    assert b.min() >= img.min() - 1e-15 and b.max() <= img.max() + 1e-15
    # the blur is linear
    img2 = np.random.default_rng(2).random((12, 10, 3))
    np.testing.assert_allclose(O.blur_image(img + 2 * img2, 3), b + 2 * O.blur_image(img2, 3), atol=1e-13)


def _plane4(w=24, h=16):
    sf = synth.generate("plane4", w, h, seed=3)
    return sf, O.OFrame.from_synth(sf)


def test_oracle_diffusion_off_is_identity():
    sf, fr = _plane4()
    a = O.render_frame(fr, O.OConfig(width=24, height=16))
    b = O.render_frame(fr, O.OConfig(width=24, height=16, diffusion=0.0, diffusion_radius=9))
    np.testing.assert_array_equal(a.output, b.output)


def test_oracle_diffusion_only_moves_the_background_term():
    sf, fr = _plane4()
    cfg = O.OConfig(width=24, height=16, diffusion=0.7, diffusion_radius=3)
    a = O.render_frame(fr, O.OConfig(width=24, height=16))
    b = O.render_frame(fr, cfg)
    np.testing.assert_array_equal(a.coeffs, b.coeffs)
    np.testing.assert_array_equal(a.accum, b.accum)
    # D_p = sum alpha mean(v̂) and out - out_plain = v_tot * w * (blur(bg) - bg)
    D = np.zeros(fr.npix)
    np.add.at(D, fr.pixel, fr.alpha * b.vhat.mean(axis=1))
    np.testing.assert_allclose(b.diffusion, D, atol=1e-14)
    vt = np.exp(-O.total_absorbance_batch(b.coeffs, b.rank))
    img = fr.opaque_color.reshape(16, 24, 3)
    bb = O.blur_image(img, 3).reshape(-1, 3)
    w = np.minimum(1.0, 0.7 * D)[:, None]
    np.testing.assert_allclose(b.output - a.output, vt * w * (bb - fr.opaque_color), atol=1e-13)


def test_oracle_diffusion_band_split_is_identical():
    sf, fr = _plane4()
    cfg = O.OConfig(width=24, height=16, diffusion=0.5, diffusion_radius=2)
    a = O.render_frame(fr, cfg, workers=1)
    b = O.render_frame(fr, cfg, workers=3)
    np.testing.assert_array_equal(a.output, b.output)


@pytest.mark.parametrize("kw", [dict(diffusion=-0.1), dict(diffusion=float("nan")),
                                dict(diffusion=float("inf")), dict(diffusion_radius=0),
                                dict(diffusion_radius=65)])
def test_config_rejects_bad_diffusion(kw):
    with pytest.raises(ValueError):
        RenderConfig(**kw)


def test_config_diffusion_flag():
    assert RenderConfig().flags & _lib.DIFFUSION == 0
    assert RenderConfig(diffusion=0.25).flags & _lib.DIFFUSION


def test_abi_validates_diffusion_without_a_gpu():
    lib = _lib.load()
    p = _lib.Params()
    p.rank, p.aberration_taps, p.flags = 3, 5, _lib.DIFFUSION
    p.diffusion, p.diffusion_radius = -1.0, 4
    f, b = _lib.Frags(), _lib.Bufs()
    assert lib.woit_render_band(f, p, b, None, 0, None) == _lib.EINVAL
    p.diffusion, p.diffusion_radius = 1.0, 0
    assert lib.woit_render_band(f, p, b, None, 0, None) == _lib.EINVAL
    assert lib.woit_resolve_blur(None, 4, 4, 2, None, None, 0, None) == _lib.EINVAL
    buf = (np.zeros(64, np.float32)).ctypes.data
    assert lib.woit_resolve_blur(buf, 4, 4, 0, buf, None, 0, None) == _lib.EINVAL
    assert lib.woit_resolve_blur(buf, 4, 4, 2, buf, None, 0, None) == _lib.EWORKSPACE
    assert lib.woit_blur_workspace_bytes(4, 4) >= 4 * 4 * 3 * 4


# ---------------------------------------------------------------------------
# GPU: the CUDA path against the twin


@pytest.fixture(scope="module")
def W():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2201_00094_b200 as w

    w._lib.load()
    return w


def h(t):
    return t.detach().double().cpu().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("H,Wd,r", [(23, 37, 4), (48, 64, 1), (31, 9, 17), (130, 1030, 5), (8, 6, 64)])
def test_resolve_blur_matches_twin(W, H, Wd, r):
    img = np.random.default_rng(H * Wd + r).random((H, Wd, 3)).astype(np.float32)
    got = h(W.resolve_blur(torch.from_numpy(img).cuda(), r))
    np.testing.assert_allclose(got, O.blur_image(img.astype(np.float64), r), rtol=0, atol=BLUR_TOL)


@pytest.mark.gpu
def test_resolve_blur_unaligned_views(W):
    big = torch.rand(1 + 19 * 21 * 3, device="cuda")
    img = big[1:].view(19, 21, 3)  # 4-B aligned only: the scalar paths
    got = h(W.resolve_blur(img, 3))
    np.testing.assert_allclose(got, O.blur_image(h(img), 3), rtol=0, atol=BLUR_TOL)


def _gpu_render(W, sf, cfg, cam=None, workers=1):
    frame = W.FrameFragments.from_synth(sf)
    rays = W.camera_rays(cam or W.Camera(), cfg.width, cfg.height)
    full = frame.opaque_color.reshape(cfg.height, cfg.width, 3)
    if workers == 1:
        bufs = W.render_band(frame, cfg, rays, full_opaque_image=full, vhat=True)
        torch.cuda.synchronize()
        return bufs
    return W.render_frame(cam or W.Camera(), dataclasses.replace(cfg, workers=workers), frame=frame)


@pytest.mark.gpu
def test_diffusion_zero_is_bit_identical(W):
    sf = synth.generate("smoke", 40, 24, seed=2)
    a = _gpu_render(W, sf, W.RenderConfig(width=40, height=24))
    b = _gpu_render(W, sf, W.RenderConfig(width=40, height=24, diffusion=0.0, diffusion_radius=11))
    for name in ("coeffs", "vhat", "accum", "accum_weight", "output"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name


CASES = [
    ("plane4", dict(), 0.8, 3),
    ("smoke", dict(), 0.3, 6),
    ("ragged", dict(rank=5), 2.0, 2),
]


@pytest.mark.gpu
@pytest.mark.parametrize("workload,over,k,r", CASES)
def test_diffusion_matches_twin(W, workload, over, k, r):
    sf = synth.generate(workload, 32, 20, seed=7)
    cfg = W.RenderConfig(width=32, height=20, diffusion=k, diffusion_radius=r, **over)
    bufs = _gpu_render(W, sf, cfg)
    ref = O.render_frame(O.OFrame.from_synth(sf), O.OConfig(width=32, height=20, diffusion=k,
                                                            diffusion_radius=r, **over))
    assert np.abs(h(bufs.coeffs) - ref.coeffs).max() <= COEF_TOL
    assert np.abs(h(bufs.vhat) - ref.vhat).max() <= VHAT_TOL
    assert np.abs(h(bufs.diffusion) - ref.diffusion).max() <= 1e-5
    assert np.abs(h(bufs.output) - ref.output).max() <= IMG_TOL
    # the feature is visible wherever the background is not flat
    if np.ptp(sf.opaque_color, axis=0).max() > 0.05:
        plain = O.render_frame(O.OFrame.from_synth(sf), O.OConfig(width=32, height=20, **over))
        assert np.abs(ref.output - plain.output).max() > 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["wine33_refr_ca_cube", "glass17_refr"])
def test_diffusion_with_refraction_and_aberration(W, name):
    meta, d = fixtures.load(name)
    sf = fixtures.input_stream(meta, d)
    c = dict(meta["cfg"])
    c.update(diffusion=0.6, diffusion_radius=3)
    cam = meta.get("camera")
    cfg = W.RenderConfig(method="wavelet", **c)
    bufs = _gpu_render(W, sf, cfg, W.Camera(**cam) if cam else None)
    ref = O.render_frame(O.OFrame.from_synth(sf), O.OConfig(**c), O.OCamera(**cam) if cam else O.OCamera())
    assert np.abs(h(bufs.diffusion) - ref.diffusion).max() <= 1e-5
    assert np.abs(h(bufs.output) - ref.output).max() <= IMG_TOL


@pytest.mark.gpu
def test_diffusion_steps_match_fused_and_bands_bitwise(W):
    sf = synth.generate("smoke", 40, 24, seed=4)
    cfg = W.RenderConfig(width=40, height=24, diffusion=0.4, diffusion_radius=4)
    fused = _gpu_render(W, sf, cfg)
    frame = W.FrameFragments.from_synth(sf)
    full = frame.opaque_color.reshape(24, 40, 3)
    bufs = W.FrameBuffers.allocate(frame, cfg.rank)
    W.step1_depth_bounds(frame, bufs)
    W.step2_build(frame, bufs, cfg)
    W.step3_accumulate(None, frame, bufs, cfg)
    W.step4_composite(bufs, cfg, full_opaque_image=full)
    torch.cuda.synchronize()
    assert np.abs(h(bufs.diffusion) - h(fused.diffusion)).max() <= 1e-6
    assert np.abs(h(bufs.output) - h(fused.output)).max() <= 1e-6
    banded = _gpu_render(W, sf, cfg, workers=3)
    assert torch.equal(banded.reshape(-1, 3), fused.output)
