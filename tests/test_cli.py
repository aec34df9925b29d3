"""CLI / PPM / scene files (the reference's test_cli.py:79-167)."""

import os
import sys

import numpy as np
import pytest
import torch

from paper_2201_00094_b200 import scene as S
from paper_2201_00094_b200.cli import main
from paper_2201_00094_b200.ppm import decode_u8, encode_u8, read_ppm, write_ppm

gpu = pytest.mark.gpu


def test_ppm_round_trip(tmp_path):
    img = np.random.default_rng(0).random((5, 7, 3))
    p = tmp_path / "x.ppm"
    write_ppm(p, img)
    assert p.read_bytes().startswith(b"P6\n7 5\n255\n")
    np.testing.assert_array_equal(read_ppm(p), encode_u8(img))
    assert np.abs(decode_u8(read_ppm(p)) - img).max() < 0.02


def test_scene_file_matches_preset(tmp_path):
    text = """# the wine bottle as a scene file
    sphere center=0,0,1.5 radius=0.5 alpha=1 transmission=0.96,0.97,0.96 radiance=0.040,0.040,0.045 ior=1.5
    sphere center=0,0,1.5 radius=0.35 alpha=1 transmission=0.74,0.25,0.34 radiance=0.020,0.005,0.008 ior=1.12
    opaque_backdrop d=3 color=0.85,0.80,0.72 checker=0.25,0.22,0.20 cell=0.35
    """
    f = tmp_path / "wine.txt"
    f.write_text(text)
    assert S.resolve_scene(str(f)) == S.preset("wine-bottle")


@pytest.mark.parametrize("text,msg", [("plane alpha=1", "missing required key"), ("cube d=1", "unknown primitive"),
                                      ("plane d=1 bogus=2", "unknown keys"), ("seed 1 2", "seed takes one")])
def test_scene_file_errors(text, msg):
    with pytest.raises(ValueError, match=msg):
        S.parse_scene(text)


def test_usage_errors_exit_two(tmp_path):
    with pytest.raises(SystemExit) as exc:
        main(["render", "--scene", "single-plane", "--method", "magic", "--out", str(tmp_path / "x.ppm")])
    assert exc.value.code == 2
    assert main(["compare", "--scene", "glass-stack", "--methods", "wavelet,magic",
                 "--out", str(tmp_path / "t.csv")]) == 2
    assert main(["render", "--scene", "no-such-preset", "--out", str(tmp_path / "x.ppm")]) == 2


@gpu
def test_render_ppm_deterministic_and_seeded(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    a, b, c = tmp_path / "a.ppm", tmp_path / "b.ppm", tmp_path / "c.ppm"
    args = ["render", "--scene", "smoke-fire", "--width", "32", "--height", "24", "--workers", "1"]
    assert main(args + ["--out", str(a)]) == 0
    assert main(args + ["--out", str(b)]) == 0
    assert a.read_bytes() == b.read_bytes() and a.read_bytes().startswith(b"P6\n32 24\n255\n")
    assert main(args + ["--seed", "1", "--out", str(c)]) == 0
    assert c.read_bytes() != a.read_bytes()
    assert main(["render", "--scene", "single-plane", "--width", "8", "--height", "8",
                 "--out", str(tmp_path / "missing_dir" / "x.ppm")]) == 1


@gpu
def test_render_abuffer_matches_oracle_image(tmp_path):
    """The CLI's A-buffer image of the reference-cast glass stack equals the oracle's
    within one code (cf. test_cli.py:119-127, whose golden PPM is absent here)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from oracle import woit_oracle as O

    gold = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cast.npz"))
    out = tmp_path / "g.ppm"
    assert main(["render", "--scene", "glass-stack", "--method", "abuffer", "--width", "32", "--height", "24",
                 "--out", str(out)]) == 0
    g = lambda k: gold[f"glass_stack_{k}"]
    fr = O.OFrame.from_arrays(32, 24, g("offsets"), g("depth"), g("alpha"), g("trans"), g("radiance"), g("normal"),
                              g("ior"), g("backface"), g("opaque_depth"), g("opaque_color"))
    want = encode_u8(O.abuffer_frame(fr, fr.opaque_color).reshape(24, 32, 3)).astype(np.int16)
    assert np.abs(read_ppm(out).astype(np.int16) - want).max() <= 1


@gpu
@pytest.mark.parametrize("rank,touch,nbytes", [(0, 2, 8), (3, 5, 64), (4, 6, 128)])
def test_bench_accounting(rank, touch, nbytes, capsys):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    assert main(["bench", "--scene", "glass-stack", "--rank", str(rank), "--width", "32", "--height", "32",
                 "--workers", "1"]) == 0
    fields = dict(line.split(": ") for line in capsys.readouterr().out.strip().splitlines())
    assert fields["touches_per_insert"] == str(touch)
    assert fields["touches_per_eval"] == str(touch)
    assert fields["bytes_per_pixel"] == str(nbytes)
    assert int(fields["fragments"]) > 0 and float(fields["wall_time_s"]) >= 0.0


@gpu
def test_compare_table(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    out = tmp_path / "t.csv"
    assert main(["compare", "--scene", "glass-stack", "--methods", "abuffer,wavelet,wboit,mlab4", "--width", "48",
                 "--height", "48", "--normalize", "off", "--out", str(out)]) == 0
    rows = [ln.split(",") for ln in out.read_text().strip().splitlines()]
    assert rows[0] == ["method", "rmse_vs_abuffer", "psnr_db", "curve_l1", "curve_l2", "curve_linf"]
    table = {r[0]: r[1:] for r in rows[1:]}
    assert float(table["abuffer"][0]) == 0.0 and table["abuffer"][1] == "inf"
    assert float(table["wavelet"][0]) < float(table["wboit"][0])
    # curve columns along the centre ray: the A-buffer curve is the truth itself
    assert [float(x) for x in table["abuffer"][2:]] == [0.0, 0.0, 0.0]
    assert all(float(x) >= 0.0 for r in table.values() for x in r[2:])


# ---------------------------------------------------------------------------
# graph (the reference's test_cli.py TestGraph, cli.py:116-131, curves.py:66-111)

TINY_SCENE = """
camera pos=0,0,0 forward=0,0,1 fov=60
plane d=1.0 alpha=0.25 transmission=0,0,0 radiance=0,0,0
opaque_backdrop d=2.0 color=0.85,0.45,0.12
"""


def _rows(path):
    return [ln.split(",") for ln in path.read_text().strip().splitlines()]


@gpu
def test_graph_single_plane_steps(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    out = tmp_path / "curve.csv"
    assert main(["graph", "--scene", "single-plane", "--methods", "wavelet", "--rank", "3", "--samples", "64",
                 "--out", str(out)]) == 0
    rows = _rows(out)
    assert rows[0] == ["z", "truth", "wavelet"]
    body = [tuple(map(float, r)) for r in rows[1:]]
    assert len(body) == 64
    for z, t, w in body:
        expect = 1.0 if z < 0.5 else 0.75
        assert t == pytest.approx(expect, abs=1e-6)
        if abs(z - 0.5) > 1.5 / 16:  # the interpolation ramp at the step
            assert w == pytest.approx(expect, abs=1e-3)
    assert all(len(c.split(".")[1]) == 6 for c in rows[1])  # fixed 6-decimal cells


@gpu
def test_graph_car_fog_truth_shape(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    out = tmp_path / "curve.csv"
    assert main(["graph", "--scene", "car-fog", "--methods", "wavelet,mlab4", "--samples", "256",
                 "--out", str(out)]) == 0
    truth = np.array([float(r[1]) for r in _rows(out)[1:]])
    assert truth[0] > 0.97 and truth[-1] < 0.2
    drops = np.diff(truth)
    assert drops.min() < -0.1 and np.all(drops <= 1e-9)  # a glass step; never increasing


@gpu
def test_graph_empty_pixel_is_one(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    f = tmp_path / "tiny.scene"
    f.write_text(TINY_SCENE.replace("plane d=1.0", "plane extent=0.01,0.01 d=1.0"), encoding="utf-8")
    out = tmp_path / "curve.csv"
    assert main(["graph", "--scene", str(f), "--pixel", "0,0", "--samples", "32", "--out", str(out)]) == 0
    rows = _rows(out)[1:]
    assert len(rows) == 32 and all(float(r[1]) == 1.0 and float(r[2]) == 1.0 for r in rows)


def test_graph_usage_errors(tmp_path, capsys):
    assert main(["graph", "--scene", "nope", "--out", str(tmp_path / "x.csv")]) == 2
    assert "valid presets" in capsys.readouterr().err
    assert main(["graph", "--scene", "single-plane", "--methods", "magic", "--out", str(tmp_path / "x.csv")]) == 2


@gpu
@pytest.mark.parametrize("preset,pixel", [("glass-stack", (32, 32)), ("smoke-fire", (30, 34)),
                                          ("wine-bottle", (32, 32)), ("car-fog", (40, 30))])
def test_curves_match_reference(preset, pixel):
    """Every curve method against the reference's own curves.extract_curves on the same
    pixel (baseline/_ref, when installed): the reference casts with its scalar
    cast_fragments, this repo with the device cast_frame (one fp32 rounding apart)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isfile(os.path.join(ref, "woit", "curves.py")):
        pytest.skip("reference not installed (bash tools/install_ref.sh)")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    ref_mod = pytest.importorskip("woit.curves")
    from woit.scene import cast_fragments as ref_cast
    from woit.scene import preset as ref_preset

    from paper_2201_00094_b200.curves import CURVE_METHODS, extract_curves, pixel_stream

    methods = list(CURVE_METHODS)
    fs, _, _ = ref_cast(ref_preset(preset), pixel[0], pixel[1], 65, 65)
    want = ref_mod.extract_curves(fs, methods, 3, 256)
    got = extract_curves(pixel_stream(S.cast_frame(S.preset(preset), 65, 65), *pixel), methods, 3, 256)
    np.testing.assert_allclose(got.z, want.z, atol=0)
    np.testing.assert_allclose(got.x, want.x, atol=1e-5)
    # the truth is a step function of x: a depth within one fp32 rounding of a sample can
    # flip one step, so compare away from the fragment depths
    far = np.min(np.abs(got.x[:, None] - np.array([f.depth for f in fs])[None, :]), axis=1) > 1e-5 \
        if len(fs) else np.ones(got.x.size, bool)
    np.testing.assert_allclose(got.truth[far], want.truth[far], atol=1e-5)
    for m in methods:
        np.testing.assert_allclose(got.methods[m][far], want.methods[m][far], atol=1e-4, err_msg=m)
