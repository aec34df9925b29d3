"""The north star's alternative build (fp32 red.global atomics from an unbinned
stream, woit_build_atomic) against the oracle's step2_build (wavelet.py:272-287)."""

import numpy as np
import pytest
import torch

from oracle import woit_oracle as O
from paper_2201_00094_b200 import _lib, synth

COEF_TOL = 1e-5


def test_atomic_build_validation_without_a_gpu():
    lib = _lib.load()
    p = _lib.Params()
    p.rank, p.aberration_taps = 3, 5
    f, b = _lib.Frags(), _lib.Bufs()
    assert lib.woit_build_atomic(f, None, p, b, None, 0, None) == _lib.EINVAL  # no near/far/coeffs
    p.flags = _lib.PACKED_STORAGE
    assert lib.woit_build_atomic(f, None, p, b, None, 0, None) == _lib.EINVAL
    p.rank = 9
    assert lib.woit_build_atomic(f, None, p, b, None, 0, None) == _lib.ERANK
    assert lib.woit_build_atomic_workspace_bytes(10) == 240


@pytest.fixture(scope="module")
def W():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2201_00094_b200 as w

    w._lib.load()
    return w


@pytest.mark.gpu
@pytest.mark.parametrize("workload,rank,layers", [("plane4", 3, 32), ("smoke", 3, 32), ("ragged", 2, 40),
                                                  ("particles", 4, 64), ("smoke", 0, 32)])
def test_atomic_build_matches_oracle(W, workload, rank, layers):
    sf = synth.generate(workload, 24, 16, seed=11, layers=layers)
    frame = W.FrameFragments.from_synth(sf)
    cfg = W.RenderConfig(rank=rank, width=24, height=16)
    bufs = W.FrameBuffers.allocate(frame, rank)
    W.step1_depth_bounds(frame, bufs)
    W.step2_build_atomic(frame, bufs, cfg)
    ofr = O.OFrame.from_synth(sf)
    ob = O.OBuffers.allocate(ofr, rank)
    O.step1_depth_bounds(ofr, ob)
    O.step2_build(ofr, ob, O.OConfig(rank=rank, width=24, height=16))
    got = bufs.coeffs.double().cpu().numpy()
    assert np.abs(got - ob.coeffs).max() <= COEF_TOL


@pytest.mark.gpu
def test_atomic_build_unbinned_order(W):
    """Any fragment order (no binning) gives the same coefficients within tolerance."""
    sf = synth.generate("smoke", 24, 16, seed=3)
    frame = W.FrameFragments.from_synth(sf)
    cfg = W.RenderConfig(width=24, height=16)
    a = W.FrameBuffers.allocate(frame, 3)
    W.step1_depth_bounds(frame, a)
    W.step2_build(frame, a, cfg)
    order = torch.randperm(frame.nfrag, device="cuda")
    pix = W.pixel_ids(frame)[order].contiguous()
    shuffled = W.FrameFragments(**{**frame.__dict__, "depth": frame.depth[order], "alpha": frame.alpha[order],
                                   "trans": frame.trans[order].contiguous()})
    b = W.FrameBuffers.allocate(frame, 3)
    b.near.copy_(a.near)
    b.far.copy_(a.far)
    W.step2_build_atomic(shuffled, b, cfg, pix)
    assert (a.coeffs - b.coeffs).abs().max().item() <= COEF_TOL
