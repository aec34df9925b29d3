"""CPU: pin the oracle against the reference's own outputs and known answers.

The fixtures were produced by running the reference (tests/golden/make_golden.py);
here the numpy restatement in oracle/ must reproduce them to float64 round-off.
The known-answer values are the reference tests' hand-derived numbers
(SURVEY.md §8(c)).
"""

import math

import numpy as np
import pytest

from oracle import woit_oracle as O
from tests import fixtures

PLANE_A = -math.log(0.75)


def oracle_frame(meta, d):
    if meta["kind"] == "synth":
        return O.OFrame.from_synth(fixtures.input_stream(meta, d))
    return O.OFrame.from_arrays(meta["width"], meta["height"], d["f_offsets"], d["f_depth"],
                                d["f_alpha"], d["f_trans"], d["f_radiance"], d["f_normal"],
                                d["f_ior"], d["f_backface"], d["f_opaque_depth"],
                                d["f_opaque_color"])


def oracle_cfg(meta):
    return O.OConfig(**meta["cfg"])


def oracle_cam(meta):
    cam = meta.get("camera")
    return O.OCamera(**cam) if cam else O.OCamera()


@pytest.mark.parametrize("name", fixtures.names())
def test_oracle_matches_reference_fixture(name):
    meta, d = fixtures.load(name)
    out = O.render_frame(oracle_frame(meta, d), oracle_cfg(meta), oracle_cam(meta))
    np.testing.assert_array_equal(out.near, d["near"])
    np.testing.assert_array_equal(out.far, d["far"])
    for key, got in (("coeffs", out.coeffs), ("accum", out.accum), ("weight", out.accum_weight),
                     ("refr", out.refraction_offset), ("output", out.output), ("vhat", out.vhat)):
        np.testing.assert_allclose(got, d[key], rtol=0, atol=1e-12, err_msg=key)


@pytest.mark.parametrize("name", fixtures.names())
def test_oracle_index_restatement(name):
    """z and the slot / cell indices are integer functions of identical inputs."""
    meta, d = fixtures.load(name)
    frame = oracle_frame(meta, d)
    bufs = O.OBuffers.allocate(frame, meta["cfg"]["rank"])
    O.step1_depth_bounds(frame, bufs)
    z = O.fragment_z(frame, bufs)
    np.testing.assert_array_equal(z, d["z"])
    k = O.slot_indices(z, bufs.rank)
    assert k.shape == (z.size, bufs.rank + 1)
    for n in range(bufs.rank + 1):
        assert np.all((k[:, n] >= 0) & (k[:, n] < (1 << n)))


def test_oracle_workers_bitwise():
    """Row bands on threads are bit-identical to one band (test_pipeline.py:361-365)."""
    meta, d = fixtures.load("smokefire24")
    f = oracle_frame(meta, d)
    a = O.render_frame(f, oracle_cfg(meta), workers=1)
    b = O.render_frame(f, oracle_cfg(meta), workers=3)
    assert np.array_equal(a.output, b.output)
    assert np.array_equal(a.coeffs, b.coeffs)


def test_kat_rank0_plane():
    """test_wavelet.py:75-79 and test_pipeline.py:55-64."""
    coeffs = np.zeros((1, 2, 3))
    O.build_into(coeffs, np.zeros(1, np.int64), np.array([0.5]), np.full((1, 3), PLANE_A), 0)
    assert np.allclose(coeffs[0, 0], 0.143841, atol=1e-6)
    assert np.allclose(coeffs[0, 1], -0.143841, atol=1e-6)
    meta, d = fixtures.load("single5_r0")
    assert np.allclose(d["coeffs"][:, 0, :], 0.5 * PLANE_A, atol=1e-6)
    assert np.allclose(d["coeffs"][:, 1, :], -0.5 * PLANE_A, atol=1e-6)


def test_kat_self_inclusive_vhat():
    """test_pipeline.py:174-190: the plane sees half its own absorbance."""
    meta, d = fixtures.load("single5_r3")
    vhat = math.exp(-0.5 * PLANE_A)
    assert np.allclose(d["accum"], np.array([0.18, 0.18, 0.20]) * 0.25 * vhat, atol=1e-9)
    assert np.allclose(d["weight"], 0.25 * vhat, atol=1e-9)


@pytest.mark.parametrize("rank", range(6))
def test_kat_dyadic_staircase(rank):
    """test_wavelet.py:148-160: a step at z=1/2 is exact at every cell centre."""
    M = 1 << (rank + 1)
    coeffs = np.zeros((1, M, 3))
    O.build_into(coeffs, np.zeros(1, np.int64), np.array([0.5]), np.full((1, 3), PLANE_A), rank)
    cells = O.cells_raw_batch(coeffs, np.zeros(M, np.int64), np.arange(M), rank)
    assert np.allclose(cells[: M // 2], 0.0, atol=1e-12)
    assert np.allclose(cells[M // 2:], PLANE_A, atol=1e-12)


def test_kat_total_telescopes(rng):
    """test_wavelet.py:234-247."""
    rank = 5
    M = 1 << (rank + 1)
    coeffs = np.zeros((1, M, 3))
    total = np.zeros(3)
    for _ in range(30):
        z = float(rng.uniform(0, (M - 1) / M))
        a = rng.uniform(0, 1, 3)
        O.build_into(coeffs, np.zeros(1, np.int64), np.array([z]), a[None, :], rank)
        total += a
    assert np.allclose(O.total_absorbance_batch(coeffs, rank)[0], total, atol=1e-9)


def test_kernel_fixture_unbinned():
    """build_into on unbinned pixel ids + the three batch evaluators (wavelet.py:272-337)."""
    d = dict(np.load(fixtures.GOLDEN + "/kernels.npz"))
    rank = int(d["rank"])
    coeffs = np.zeros_like(d["coeffs"])
    O.build_into(coeffs, d["pix"], d["z"], d["a"], rank)
    np.testing.assert_allclose(coeffs, d["coeffs"], atol=1e-12)
    np.testing.assert_allclose(O.interp_absorbance_batch(coeffs, d["qpix"], d["qz"], rank),
                               d["interp"], atol=1e-12)
    np.testing.assert_allclose(O.cells_raw_batch(coeffs, d["qpix"], d["cells"], rank), d["raw"],
                               atol=1e-12)
    np.testing.assert_allclose(O.total_absorbance_batch(coeffs, rank), d["total"], atol=1e-12)
    assert int(d["touches"][0]) == rank + 2


def test_kernel_fixture_packing():
    """E5B9G9R9 words are bit-exact (packing.py:46-88, test_packing.py:19-23)."""
    d = dict(np.load(fixtures.GOLDEN + "/kernels.npz"))
    np.testing.assert_array_equal(O.pack_rgb9e5(d["triples"]), d["words"])
    np.testing.assert_array_equal(O.roundtrip_coeffs(d["coeffs"]), d["packed_rt"])
    exact = O.unpack_rgb9e5(O.pack_rgb9e5([0.5, 0.25, 0.125]))
    assert np.array_equal(exact, [0.5, 0.25, 0.125])


def test_kat_spectral_weights():
    """test_pipeline.py:466-482 / acceptance 09."""
    assert tuple(O.spectral_weight(0, 5)) == (1.0, 0.0, 0.0)
    assert tuple(O.spectral_weight(2, 5)) == (0.0, 1.0, 0.0)
    assert tuple(O.spectral_weight(4, 5)) == (0.0, 0.0, 1.0)
    assert tuple(O.spectral_weight(0, 5, True)) == (0.0, 1.0, 0.0)
    for k in (3, 5, 7, 9):
        for i in range(k):
            assert abs(O.spectral_weight(i, k).sum() - 1.0) < 1e-12
