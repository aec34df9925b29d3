"""E5B9G9R9 packed coefficient storage as real storage:
``bufs.coeff_words`` [P][S] holds the paper's 4 S bytes per pixel (packing.py:41-43,
PAPER.md:96), written by the fused kernels' epilogue (the fast instance with
``packed_storage`` alone, the general kernel with other flags, the long-pixel
kernel), and every later pass reads the unpacked values (pipeline.py:154-155).

Bit-exact checks:
* the words equal ``pack_rgb9e5`` (the reference's algorithm, packing.py:46-77,
  bit-exact in ``woit_pack_rgb9e5``) of the |coefficients| the same frame yields
  without packing -- packing runs on fp32-valued coefficients, where every step of
  the reference's pack is exact;
* the fp32 coefficients written with packing equal ``unpack(words)`` with the
  positional signs (slot 0 +, others -, packing.py:100-111);
* the fast packed instance and the general kernel agree bit for bit.
Against the float64 oracle (which packs its own f64 coefficients), a word can differ
where a coefficient sits within rounding of a quantisation boundary; those are rare
and one mantissa step apart, and the images agree to RMSE 1e-5.
"""

import numpy as np
import pytest
import torch

from oracle import woit_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def W():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2201_00094_b200 as w

    w._lib.load()
    return w


def words_np(t):
    return t.cpu().numpy().view(np.uint32)


def signed_unpack(W, words):
    out = W.unpack_rgb9e5(words.reshape(-1)).reshape(words.shape + (3,))
    out[:, 1:, :] = -out[:, 1:, :]
    return out


@pytest.mark.parametrize("workload,w,h,layers,rank", [("smoke", 40, 24, 32, 3), ("particles", 24, 16, 128, 2),
                                                      ("ragged", 37, 23, 60, 4), ("plane4", 32, 16, 5, 1),
                                                      ("particles", 12, 8, 256, 3), ("ragged", 16, 12, 300, 3)])
def test_words_are_the_packed_coefficients(W, workload, w, h, layers, rank):
    frame = W.FrameFragments.synthetic(workload, w, h, seed=7, layers=layers)
    exact = W.render_band(frame, W.RenderConfig(rank=rank, width=w, height=h), vhat=True)
    packed = W.render_band(frame, W.RenderConfig(rank=rank, width=w, height=h, packed_storage=True), vhat=True)
    torch.cuda.synchronize()
    words = words_np(packed.coeff_words)
    assert words.shape == (w * h, 2 << rank)
    want = W.pack_rgb9e5(np.abs(exact.coeffs.double().cpu().numpy()).reshape(-1, 3)).reshape(words.shape)
    np.testing.assert_array_equal(words, want)
    np.testing.assert_array_equal(packed.coeffs.double().cpu().numpy(), signed_unpack(W, words))
    # the evaluation read the unpacked coefficients: the oracle's packed render agrees
    sf = frame.to_synth()
    ref = O.render_frame(O.OFrame.from_synth(sf), O.OConfig(rank=rank, width=w, height=h, packed_storage=True))
    ref_words = W.pack_rgb9e5(np.abs(
        O.render_frame(O.OFrame.from_synth(sf), O.OConfig(rank=rank, width=w, height=h)).coeffs).reshape(-1, 3))
    diff = words != ref_words.reshape(words.shape)
    assert diff.mean() < 1e-2, diff.mean()
    if diff.any():  # one mantissa step of the largest channel, same or adjacent exponent
        a, b = words[diff].astype(np.int64), ref_words.reshape(words.shape)[diff].astype(np.int64)
        assert np.all(np.abs((a >> 27) - (b >> 27)) <= 1)
    img = packed.output.double().cpu().numpy()
    assert np.sqrt(np.mean((img - ref.output) ** 2)) < 1e-5
    # packed storage moves the image by at most the quantisation (test_pipeline.py:375-381)
    assert np.sqrt(np.mean((img - exact.output.double().cpu().numpy()) ** 2)) < 2e-3


def test_fast_and_general_packed_agree_bitwise(W):
    """packed_storage alone runs the fast instance; adding cube_transmission (a no-op for
    ior = 1 fragments) sends the same frame through the general kernel."""
    frame = W.FrameFragments.synthetic("particles", 40, 20, seed=3, layers=48)
    a = W.render_band(frame, W.RenderConfig(rank=3, width=40, height=20, packed_storage=True), vhat=True)
    b = W.render_band(frame, W.RenderConfig(rank=3, width=40, height=20, packed_storage=True,
                                            cube_transmission=True), vhat=True)
    torch.cuda.synchronize()
    for name in ("coeff_words", "coeffs", "vhat", "output"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name


def test_step2_packed_writes_words(W):
    frame = W.FrameFragments.synthetic("smoke", 24, 16, seed=5, layers=32)
    cfg = W.RenderConfig(rank=3, width=24, height=16, packed_storage=True)
    fused = W.render_band(frame, cfg)
    bufs = W.FrameBuffers.allocate(frame, 3, packed=True)
    W.step1_depth_bounds(frame, bufs)
    W.step2_build(frame, bufs, cfg)
    torch.cuda.synchronize()
    assert torch.equal(bufs.coeff_words, fused.coeff_words)
    assert torch.equal(bufs.coeffs, fused.coeffs)


def test_empty_pixels_pack_to_zero(W):
    offsets = np.zeros(8 * 4 + 1, np.int64)
    offsets[17:] = 3  # pixel 16 has 3 fragments, the rest none
    rng = np.random.default_rng(0)
    f = W.FrameFragments.from_numpy(8, 4, offsets, rng.uniform(1, 2, 3), rng.uniform(0, 1, 3),
                                    rng.uniform(0, 1, (3, 3)), rng.uniform(0, 1, (3, 3)),
                                    opaque_color=np.full((32, 3), 0.25))
    b = W.render_band(f, W.RenderConfig(rank=3, width=8, height=4, packed_storage=True))
    torch.cuda.synchronize()
    words = words_np(b.coeff_words)
    assert np.all(np.delete(words, 16, axis=0) == 0) and np.any(words[16] != 0)
