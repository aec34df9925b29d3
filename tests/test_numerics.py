"""CPU: numerical building blocks of the kernels, emulated bit-for-bit in numpy.

* log_poly (common.cuh): the fp32 natural log the absorbance uses; its exact FMA
  sequence and coefficients are parsed from the CUDA source and emulated here.
* the 32-bit fixed-point z: every slot / cell index derived from it equals the
  reference's floor(2^n z) / floor(z M - 1/2) (wavelet.py:281, :311).
"""

import os
import re

import numpy as np

from oracle import woit_oracle as O

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = open(os.path.join(REPO, "paper_2201_00094_b200", "csrc", "common.cuh")).read()


def _hexf(tok: str) -> np.float32:
    return np.float32(float.fromhex(tok.rstrip("f")))


def _log_poly_coeffs():
    body = SRC[SRC.index("WOIT_D float log_poly"):SRC.index("WOIT_D float absorbance_ch")]
    lead = _hexf(re.search(r"float r = (-?0x[0-9a-f.p+-]+f);", body).group(1))
    steps = [_hexf(t) for t in re.findall(r"r = fmaf\(r, f, (-?0x[0-9a-f.p+-]+f)\);", body)]
    ln2 = _hexf(re.search(r"fmaf\(k, (0x[0-9a-f.p+-]+f), r\)", body).group(1))
    return lead, steps, ln2


def _fma32(a, b, c):
    # a*b is exact in f64 for fp32 operands; one rounding to fp32 like FFMA (the f64
    # addition can double-round only on exact ties, which the ulp bound tolerates)
    return (np.float64(a) * np.float64(b) + np.float64(c)).astype(np.float32)


def log_poly(x):
    lead, steps, ln2 = _log_poly_coeffs()
    x = np.asarray(x, np.float32)
    bits = x.view(np.int32)
    e = (bits - np.int32(0x3F2AAAAB)) & np.int32(-8388608)
    m = (bits - e).view(np.float32)
    k = e.astype(np.float32) * np.float32(2.0 ** -23)
    f = (m - np.float32(1.0)).astype(np.float32)
    s = (f * f).astype(np.float32)
    r = np.full_like(f, lead)
    for c in steps:
        r = _fma32(r, f, c)
    r = _fma32(r, s, f)
    return _fma32(k, ln2, r)


def test_log_poly_accuracy():
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.uniform(1e-6, 1, 1_000_000), rng.uniform(0.5, 1, 1_000_000),
                         np.linspace(1e-6, 1, 500_001), [1e-6, 0.5, 1.0]]).astype(np.float32)
    ref = np.log(xs.astype(np.float64))
    got = log_poly(xs).astype(np.float64)
    ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    nz = ref != 0
    assert (np.abs(got - ref)[nz] / ulp[nz]).max() < 1.0
    assert got[-1] == 0.0  # ln 1 = 0 exactly: no absorbance from a transparent fragment
    # unbiased: mean signed error over uniform t is ~1e-9, far below the 1e-5 bars
    assert abs((got - ref).mean()) < 1e-8


def test_fixed_point_indices_match_reference():
    rng = np.random.default_rng(1)
    z = np.concatenate([rng.uniform(0, 1 - 2 ** -24, 200_000), np.arange(129) / 128.0 * (1 - 2 ** -24),
                        [0.0, 1 - 2 ** -24, 0.5, 0.25 - 2 ** -60, 1.0 / 16]])
    zi = (z * 2.0 ** 32).astype(np.uint64)  # trunc(z 2^32), exact multiply
    for rank in range(7):
        k = O.slot_indices(z, rank)
        for n in range(1, rank + 1):
            np.testing.assert_array_equal(zi >> np.uint64(32 - n), k[:, n])
        c0, c1, _ = O.cell_indices(z, rank)
        sc = 32 - (rank + 1)
        half = np.uint64(1 << (sc - 1))
        M = 2 << rank
        raw = np.where(zi < half, -1, ((zi - half) >> np.uint64(sc)).astype(np.int64))
        np.testing.assert_array_equal(np.clip(raw, 0, M - 1), c0)
