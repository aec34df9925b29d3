"""BASELINE configs 4 and 5 at full size on one B200: sampled-row parity against
the oracle plus size-independent properties.

* config 4 (configs[3]): 3840 x 2160 particles, 128 fragments/pixel, rank 3 --
  the plain fast instance (1.06 G fragments);
* config 5 (configs[4]): the 540-row eighth of the 7680 x 4320 x 256 stress frame
  that one GPU of the 8-GPU job renders (1.06 G fragments), at ranks 2 / 3 / 4
  (8 / 16 / 32 coefficients) -- the deep-frame instance (> 160 fragments/pixel)
  that bench.py --config 5 measures.

Rows are drawn at random (fixed seed) from the band; each is regenerated on the
host (the numpy twin of the device generator), rendered by the float64 oracle and
compared with the same rows of the device render: coefficients and v̂ within
1e-5, accumulators and image within 1e-4, near/far bit-exact. The errors are
printed and, with WOIT_PARITY_LOG=<path>, appended there as JSON lines.
"""

import json
import os

import numpy as np
import pytest
import torch

from oracle import woit_oracle as O

pytestmark = pytest.mark.gpu

COEF_TOL, VHAT_TOL, IMG_TOL = 1e-5, 1e-5, 1e-4


@pytest.fixture(scope="module")
def W():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2201_00094_b200 as w

    w._lib.load()
    return w


def h(t):
    return t.detach().double().cpu().numpy()


def _log(rec):
    print(json.dumps(rec))
    path = os.environ.get("WOIT_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def check_rows(W, frame, bufs, workload, width, height, layers, rank, rows, tag):
    host_off = frame.offsets.cpu().numpy()
    worst = dict(coeffs=0.0, vhat=0.0, accum=0.0, output=0.0)
    for r in rows:
        sub = W.synth.generate(workload, width, height, seed=1, layers=layers, row0=int(r), rows=1)
        ref = O.render_frame(O.OFrame.from_synth(sub), O.OConfig(rank=rank, width=width, height=1))
        p0, p1 = int(r) * width, (int(r) + 1) * width
        f0, f1 = int(host_off[p0]), int(host_off[p1])
        np.testing.assert_array_equal(h(bufs.near[p0:p1]), ref.near.astype(np.float32).astype(np.float64))
        np.testing.assert_array_equal(h(bufs.far[p0:p1]), ref.far.astype(np.float32).astype(np.float64))
        errs = dict(coeffs=np.abs(h(bufs.coeffs[p0:p1]) - ref.coeffs).max(),
                    vhat=np.abs(h(bufs.vhat[f0:f1]) - ref.vhat).max(),
                    accum=np.abs(h(bufs.accum[p0:p1]) - ref.accum).max(),
                    output=np.abs(h(bufs.output[p0:p1]) - ref.output).max())
        for k, v in errs.items():
            worst[k] = max(worst[k], float(v))
    _log(dict(test=tag, rank=rank, rows=[int(r) for r in rows], **worst))
    assert worst["coeffs"] <= COEF_TOL, worst
    assert worst["vhat"] <= VHAT_TOL, worst
    assert worst["accum"] <= IMG_TOL and worst["output"] <= IMG_TOL, worst


def properties(bufs, frame):
    assert bool(torch.isfinite(bufs.output).all())
    v = bufs.vhat
    assert bool(((v > 0) & (v <= 1)).all())
    assert bool((bufs.near <= bufs.far).all())
    # c0 >= 0 and every detail coefficient <= 0 (wavelet.py:104-108)
    assert bool((bufs.coeffs[:, 0, :] >= 0).all()) and bool((bufs.coeffs[:, 1:, :] <= 1e-7).all())


def test_config4_full_size(W):
    width, height, layers = 3840, 2160, 128
    frame = W.FrameFragments.synthetic("particles", width, height, seed=1, layers=layers)
    assert frame.nfrag == width * height * layers
    cfg = W.RenderConfig(rank=3, width=width, height=height)
    bufs = W.render_band(frame, cfg, vhat=True)
    torch.cuda.synchronize()
    properties(bufs, frame)
    rows = np.random.default_rng(4).choice(height, 3, replace=False)
    check_rows(W, frame, bufs, "particles", width, height, layers, 3, rows, "config4_full")


@pytest.fixture(scope="module")
def eighth(W):
    width, height, layers = 7680, 4320, 256
    frame = W.FrameFragments.synthetic("particles", width, height, seed=1, layers=layers, row0=0, rows=540)
    assert frame.nfrag == width * 540 * layers
    yield frame
    del frame
    torch.cuda.empty_cache()


@pytest.mark.parametrize("rank", [2, 3, 4])
def test_config5_eighth_full_size(W, eighth, rank):
    width, height, layers = 7680, 4320, 256
    cfg = W.RenderConfig(rank=rank, width=width, height=height)
    bufs = W.render_band(eighth, cfg, vhat=True)
    torch.cuda.synchronize()
    properties(bufs, eighth)
    rows = np.random.default_rng(50 + rank).choice(540, 2, replace=False)
    check_rows(W, eighth, bufs, "particles", width, height, layers, rank, rows, "config5_eighth")
    del bufs
    torch.cuda.empty_cache()
