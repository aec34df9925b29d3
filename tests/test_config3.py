"""Config 3 at full size: the reference's wine-bottle frame at
1920x1080 with refraction + aberration (k=5) + cubed transmission, GPU vs the
float64 oracle on the same fp32 inputs. The input (the reference's cast_frame
output) is written by tools/make_config3.py into data/ (git-ignored); without it the
frame comes from the on-device caster (CSR pinned to the reference's by tests/test_cast.py)."""

import os

import numpy as np
import pytest
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DATA = os.path.join(REPO, "data", "config3_wine_1080p.npz")

pytestmark = pytest.mark.gpu


def test_config3_full_frame_matches_oracle():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import sys

    sys.path.insert(0, os.path.join(REPO, "tools"))
    import config3 as C3

    import paper_2201_00094_b200 as W
    from oracle import woit_oracle as O

    sf, cam = C3.load()
    frame = W.FrameFragments.from_synth(sf)
    cfg = W.RenderConfig(width=sf.width, height=sf.height, **C3.CFG)
    rays = W.camera_rays(W.Camera(**cam), sf.width, sf.height)
    bufs = W.render_band(frame, cfg, rays, full_opaque_image=frame.opaque_color.reshape(sf.height, sf.width, 3),
                         vhat=True)
    torch.cuda.synchronize()
    ref = O.render_frame(O.OFrame.from_synth(sf), O.OConfig(width=sf.width, height=sf.height,
                                                             workers=O.default_workers(), **C3.CFG),
                         O.OCamera(**cam))
    h = lambda t: t.detach().double().cpu().numpy()
    np.testing.assert_array_equal(h(bufs.near), ref.near.astype(np.float32).astype(np.float64))
    assert np.abs(h(bufs.coeffs) - ref.coeffs).max() <= 1e-5
    assert np.abs(h(bufs.vhat) - ref.vhat).max() <= 1e-5
    assert np.abs(h(bufs.output) - ref.output).max() <= 1e-4
