"""Comparison methods (RenderConfig.method = abuffer / wboit / mlab4; baselines.py:135-220;
SURVEY.md §8(f) rank 2): oracle restatement vs the reference's own outputs
(tests/golden/baselines.npz, written by make_golden.py --only-baselines), and the
float64 per-pixel kernels (woit_render_baseline) vs the same fixtures."""

import ast
import os

import numpy as np
import pytest
import torch

from oracle import woit_oracle as O
from paper_2201_00094_b200 import _lib, synth

GOLD = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "baselines.npz"))
CASES = ("ragged", "particles", "smokefire_shuf", "wine")
METHODS = ("abuffer", "wboit", "mlab4")


def stream(name) -> synth.SynthFrame:
    if name == "ragged":
        return synth.generate("ragged", 16, 12, seed=3, layers=40)
    if name == "particles":
        return synth.generate("particles", 8, 6, seed=9, layers=64)
    meta = ast.literal_eval(str(GOLD[f"in_{name}"]))
    g = lambda k: GOLD[f"in_{name}_{k}"]
    return synth.SynthFrame(meta["width"], meta["height"], 0, meta["height"], g("offsets").astype(np.int64),
                            g("depth"), g("alpha"), g("trans"), g("radiance"), g("normal"), g("ior"),
                            g("backface").astype(np.uint8), g("opaque_depth"), g("opaque_color"))


def oracle_method(fr, method, cube):
    bg = fr.opaque_color
    if method == "abuffer":
        return O.abuffer_frame(fr, bg, cube)
    if method == "wboit":
        return O.wboit_frame(fr, bg, cube)
    return O.mlab_frame(fr, bg, 4, cube)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("cube", [False, True])
def test_oracle_matches_reference(name, method, cube):
    fr = O.OFrame.from_synth(stream(name))
    ref = GOLD[f"{method}_{name}_{'cube' if cube else 'plain'}"]
    np.testing.assert_allclose(oracle_method(fr, method, cube), ref, rtol=0, atol=1e-12)


def test_mlab_exact_for_shallow_streams():
    """baselines.py:101-104: streams of <= k fragments reproduce the sorted oracle."""
    sf = synth.generate("ragged", 16, 12, seed=3, layers=4)
    fr = O.OFrame.from_synth(sf)
    np.testing.assert_allclose(O.mlab_frame(fr, fr.opaque_color, 4), O.abuffer_frame(fr, fr.opaque_color),
                               atol=1e-12)


def test_baseline_validation_without_a_gpu():
    lib = _lib.load()
    f = _lib.Frags()
    assert lib.woit_render_baseline(f, 9, 0, None, None, None, 0, None) == _lib.EINVAL
    assert lib.woit_render_baseline(f, 1, 0, None, None, None, 0, None) == _lib.EINVAL  # width 0
    assert lib.woit_baseline_workspace_bytes(7, 1, 1) == 0


@pytest.fixture(scope="module")
def W():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2201_00094_b200 as w

    w._lib.load()
    return w


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("cube", [False, True])
def test_gpu_baseline_matches_reference(W, name, method, cube):
    sf = stream(name)
    frame = W.FrameFragments.from_synth(sf)
    cfg = W.RenderConfig(method=method, width=sf.width, height=sf.height, cube_transmission=cube)
    got = W.render_baseline(frame, cfg).double().cpu().numpy()
    ref = GOLD[f"{method}_{name}_{'cube' if cube else 'plain'}"]
    # float64 in the reference's order, one fp32 rounding at the end (wboit's z^6 is a
    # product instead of libm pow: <= 2 ulp of f64)
    assert np.abs(got - ref).max() <= 1e-6


@pytest.mark.gpu
def test_render_frame_methods(W):
    sf = synth.generate("smoke", 24, 16, seed=5)
    frame = W.FrameFragments.from_synth(sf)
    for method in METHODS:
        img = W.render_frame(None, W.RenderConfig(method=method, width=24, height=16), frame=frame)
        assert img.shape == (16, 24, 3)
        ref = oracle_method(O.OFrame.from_synth(sf), method, False).reshape(16, 24, 3)
        assert np.abs(img.double().cpu().numpy() - ref).max() <= 1e-6


@pytest.mark.gpu
def test_abuffer_is_order_independent_and_close_to_wavelet(W):
    """Acceptance 04 / 07 flavour: the A-buffer ignores arrival order exactly, and the
    wavelet image stays close to it on a smooth volume."""
    sf = synth.generate("smoke", 32, 24, seed=8)
    frame = W.FrameFragments.from_synth(sf)
    cfg = W.RenderConfig(method="abuffer", width=32, height=24)
    a = W.render_baseline(frame, cfg)
    rev = torch.cat([torch.flip(frame.depth[int(s):int(e)], [0]) for s, e in
                     zip(frame.offsets[:-1].tolist(), frame.offsets[1:].tolist())])
    idx = torch.cat([torch.arange(int(e) - 1, int(s) - 1, -1) for s, e in
                     zip(frame.offsets[:-1].tolist(), frame.offsets[1:].tolist())]).cuda()
    flipped = W.FrameFragments(**{**frame.__dict__, "depth": rev.contiguous(), "alpha": frame.alpha[idx],
                                  "trans": frame.trans[idx].contiguous(), "radiance": frame.radiance[idx].contiguous()})
    b = W.render_baseline(flipped, cfg)
    assert torch.equal(a, b)
    wav = W.render_frame(None, W.RenderConfig(width=32, height=24), frame=frame).reshape(-1, 3)
    rmse = float(((wav - a) ** 2).mean().sqrt())
    assert rmse < 0.01  # oracle: 0.0021 on this stream
