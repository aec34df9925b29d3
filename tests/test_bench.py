"""bench.py's CPU-side contract: the algorithmic byte counts of SURVEY.md §8(d), the
config table and the reference arm's JSON line (run on a tiny band here)."""

import importlib.util
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(REPO, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_algorithmic_bytes_match_survey(bench):
    # config 2: 51.00 B/frag, 3.384 GB per frame
    P, n = 1920 * 1080, 1920 * 1080 * 32
    assert bench.algorithmic_bytes(P, n, 3) == 3_384_115_200
    assert abs(bench.algorithmic_bytes(P, n, 3) / n - 51.0) < 1e-9
    # config 4: 45.75 B/frag, 48.57 GB
    P, n = 3840 * 2160, 3840 * 2160 * 128
    assert abs(bench.algorithmic_bytes(P, n, 3) / n - 45.75) < 1e-9
    assert abs(bench.algorithmic_bytes(P, n, 3) / 1e9 - 48.57) < 0.01
    # config 5: 44.50 / 44.88 / 45.62 B/frag at S = 8 / 16 / 32
    P, n = 7680 * 4320, 7680 * 4320 * 256
    for rank, bpf in ((2, 44.50), (3, 44.875), (4, 45.625)):
        assert abs(bench.algorithmic_bytes(P, n, rank) / n - bpf) < 1e-9


def test_configs_match_baseline(bench):
    c = bench.CONFIGS
    assert (c[2]["width"], c[2]["height"], c[2]["layers"], c[2]["rank"]) == (1920, 1080, 32, 3)
    assert (c[4]["width"], c[4]["height"], c[4]["layers"]) == (3840, 2160, 128) and c[4]["strong"]
    assert (c[5]["width"], c[5]["height"], c[5]["layers"], c[5]["share"]) == (7680, 4320, 256, 8)
    assert c[5]["height"] % c[5]["share"] == 0


def test_reference_arm_line():
    """--impl reference prints one JSON line with the contract's keys (a 4-row band)."""
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--ref-rows", "4"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference" and line["unit"] == "Gfrag/s" and line["value"] > 0
    assert line["metric"] == json.load(open(os.path.join(REPO, "BASELINE.json")))["metric"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == ("reference" if bench_mod().reference_available() else "port")
    assert line["cpu_baseline"]["numpy"] and "cpu_model" in line["cpu_baseline"]
    # the reference arm's config is the GPU arm's, the CPU sample size separate
    assert line["config"] == bench_mod().config_dict(bench_mod().CONFIGS[2], 1)
    assert line["sample_rows"] == 4


def bench_mod():
    spec = importlib.util.spec_from_file_location("bench_t", os.path.join(REPO, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_gpus_relaunch_under_torchrun(bench):
    """--gpus N outside torchrun re-launches N ranks (127.0.0.1 rendezvous)."""
    cmd = bench.relaunch_cmd(["--gpus", "8", "--steps", "5"], 8, 29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-3:] == ["--gpus", "8", "--steps", "5"][-3:] and cmd[-5].endswith("bench.py")


def test_config_dicts(bench):
    c2 = bench.config_dict(bench.CONFIGS[2], 8)
    assert c2["height"] == 8 * 1080 and c2["fragments"] == 8 * 1920 * 1080 * 32
    c4 = bench.config_dict(bench.CONFIGS[4], 8)
    assert c4["height"] == 2160 and c4["fragments"] == 3840 * 2160 * 128
    assert bench.geometry(bench.CONFIGS[4], 8) == (2160, 270)
    assert bench.geometry(bench.CONFIGS[5], 3) == (4320, 540)
