"""Build the config-3 input stream: the reference's own
``cast_frame(preset("wine-bottle"), 1920, 1080)``, stored as the device layout
(fp32 SoA, CSR) in data/config3_wine_1080p.npz (git-ignored; it travels to the
GPU box with gpurun). Needs /root/reference, so it runs in the build container:

    PYTHONPATH=/root/reference/pkg/src python tools/make_config3.py
"""
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from woit.scene import cast_frame, preset  # noqa: E402

W, H = 1920, 1080
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data", "config3_wine_1080p.npz")

t0 = time.time()
sc = preset("wine-bottle")
fr = cast_frame(sc, W, H)
print(f"cast_frame {W}x{H}: {int(fr.offsets[-1])} fragments in {time.time() - t0:.1f} s")
f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)
cam = sc.camera
os.makedirs(os.path.dirname(OUT), exist_ok=True)
np.savez_compressed(OUT, width=W, height=H, offsets=fr.offsets.astype(np.int64), depth=f32(fr.depth),
                    alpha=f32(fr.alpha), trans=f32(fr.trans), radiance=f32(fr.radiance), normal=f32(fr.normal),
                    ior=f32(fr.ior), backface=fr.backface.astype(np.uint8), opaque_depth=f32(fr.opaque_depth),
                    opaque_color=f32(fr.opaque_color), cam_position=np.array(cam.position, dtype=np.float64),
                    cam_forward=np.array(cam.forward, dtype=np.float64), cam_fov=np.float64(cam.fov_deg))
print(OUT, os.path.getsize(OUT) / 1e6, "MB")
