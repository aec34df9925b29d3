"""Acceptance 07 (SPEC.md criterion 7, the reference's test_acceptance.py:150-176) on the
GPU: the wavelet image is closer to the exact A-buffer than MLAB-4 and WBOIT on the
glass-stack preset (RMSE < 0.02), and within 0.03 on smoke-fire -- at the reference's
256 x 256 and at 1080p, with every method rendered by this package's kernels on the
same device-cast stream (scene.cast_frame). The RMSEs are printed and, with
WOIT_PARITY_LOG=<path>, appended there as a JSON line.
"""

import json
import os

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def W():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2201_00094_b200 as w

    w._lib.load()
    return w


def rmse(a, b):
    return float(((a.double() - b.double()) ** 2).mean().sqrt())


@pytest.mark.parametrize("width,height", [(256, 256), (1920, 1080)])
def test_07_quality_ordering(W, width, height):
    from paper_2201_00094_b200.scene import cast_frame, preset

    res = {}
    for name in ("glass-stack", "smoke-fire"):
        sc = preset(name)
        frame = cast_frame(sc, width, height)
        base = W.RenderConfig(method="abuffer", width=width, height=height)
        imgs = {m: W.render_frame(sc, W.RenderConfig(method=m, rank=3, width=width, height=height), frame=frame)
                for m in ("abuffer", "wavelet", "wboit", "mlab4")}
        ref = imgs["abuffer"]
        res[name] = {m: rmse(imgs[m], ref) for m in ("wavelet", "mlab4", "wboit")}
        del base
    rec = dict(test="acceptance07", width=width, height=height, **{f"{k}_{m}": v for k, d in res.items()
                                                                   for m, v in d.items()})
    print(json.dumps(rec))
    if os.environ.get("WOIT_PARITY_LOG"):
        with open(os.environ["WOIT_PARITY_LOG"], "a") as f:
            f.write(json.dumps(rec) + "\n")
    g, s = res["glass-stack"], res["smoke-fire"]
    assert g["wavelet"] < g["mlab4"] and g["wavelet"] < g["wboit"]
    assert g["wavelet"] < 0.02
    assert s["wavelet"] < 0.03
