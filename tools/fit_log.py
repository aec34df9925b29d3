"""Fit the fp32 natural-log polynomial used by the kernels (common.cuh log_poly).

ln(x) = k ln2 + log1p(f), x = 2^k m, m in [2/3, 4/3), f = m - 1, and
log1p(f) ~= f + f^2 P(f) with P of degree 8 fitted by iteratively reweighted
least squares for relative error on [-1/3, 1/3]. The fp32 evaluation (FMA
Horner) is emulated exactly in numpy by tests/test_numerics.py, which pins the
coefficients printed here: max error 0.90 ulp over [1e-6, 1].
"""
import numpy as np

LO, HI = 2 / 3 - 1, 4 / 3 - 1


def fit(d=8, npts=20001):
    f = np.cos(np.linspace(0, np.pi, npts)) * (HI - LO) / 2 + (HI + LO) / 2
    f = f[np.abs(f) > 1e-9]
    y = (np.log1p(f) - f) / f ** 2
    w = f ** 2 / np.abs(np.log1p(f))
    V = np.vander(f, d + 1, increasing=True)
    c, *_ = np.linalg.lstsq(V * w[:, None], y * w, rcond=None)
    for _ in range(30):
        err = (f + f ** 2 * (V @ c) - np.log1p(f)) / np.log1p(f)
        w2 = w * (1 + 50 * np.abs(err) / np.abs(err).max())
        c, *_ = np.linalg.lstsq(V * w2[:, None], y * w2, rcond=None)
    return c.astype(np.float32)


if __name__ == "__main__":
    print([float(x) for x in fit()])
