"""Every fused-kernel instance against the float64 oracle on the same fp32 inputs.

The library picks a kernel instance per launch: the fast one (plain / thin
sub-tiles / deep-pixel combine, by the frame's average run length) or the general
one (generic, or specialised at rank 3 for the flag sets of config 3 and of
refraction-only scenes). Cast scenes at small random sizes, random ranks and
flag sets drive all of them through the thin and the regular sub-tiles; the
tolerances are the north star's (1e-5 coefficients and v̂, 1e-4 image)."""

import numpy as np
import pytest
import torch

from oracle import woit_oracle as O

pytestmark = pytest.mark.gpu

CASES = [
    # preset, width, height, rank, flags (pipeline.RenderConfig keywords)
    ("wine-bottle", 96, 64, 3, dict(refraction=True, chromatic_aberration=True, cube_transmission=True)),
    ("wine-bottle", 80, 60, 3, dict(refraction=True, chromatic_aberration=True, cube_transmission=True,
                                    diffusion=0.5)),
    ("wine-bottle", 72, 48, 2, dict(refraction=True, chromatic_aberration=True, cube_transmission=True)),
    ("glass-stack", 96, 64, 3, dict(refraction=True)),
    ("glass-stack", 64, 48, 4, dict(refraction=True, normalize=False)),
    ("glass-stack", 64, 40, 3, dict(refraction=True, chromatic_aberration=True, aberration_taps=7)),
    ("car-fog", 64, 48, 3, dict()),
    ("car-fog", 48, 32, 5, dict()),
    ("smoke-fire", 96, 64, 3, dict()),
    ("leaves", 80, 60, 1, dict()),
    ("single-plane", 64, 32, 3, dict(cube_transmission=True)),
]


@pytest.fixture(scope="module")
def W():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2201_00094_b200 as w

    return w


@pytest.mark.parametrize("preset,w,h,rank,flags", CASES)
def test_instance_matches_oracle(W, preset, w, h, rank, flags):
    from paper_2201_00094_b200 import scene as S

    sc = S.preset(preset)
    frame = S.cast_frame(sc, w, h)
    cfg = W.RenderConfig(width=w, height=h, rank=rank, **flags)
    rays = W.camera_rays(sc.camera, w, h)
    full = frame.opaque_color.reshape(h, w, 3)
    bufs = W.render_band(frame, cfg, rays, full_opaque_image=full, vhat=True)
    torch.cuda.synchronize()
    c = sc.camera
    ocfg = O.OConfig(width=w, height=h, rank=rank, **flags)
    ref = O.render_frame(O.OFrame.from_synth(frame.to_synth()), ocfg,
                         O.OCamera(position=tuple(c.position), forward=tuple(c.forward), fov_deg=float(c.fov_deg)))
    hh = lambda t: t.detach().double().cpu().numpy()
    np.testing.assert_array_equal(hh(bufs.near), ref.near.astype(np.float32).astype(np.float64))
    assert np.abs(hh(bufs.coeffs) - ref.coeffs).max() <= 1e-5
    assert np.abs(hh(bufs.vhat) - ref.vhat).max() <= 1e-5
    assert np.abs(hh(bufs.output) - ref.output).max() <= 1e-4
