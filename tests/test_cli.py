"""CLI / PPM / scene files (the reference's test_cli.py:79-167)."""

import os

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
