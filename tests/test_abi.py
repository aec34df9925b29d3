"""CPU: the C-ABI library loads, exports every symbol include/woit.h declares, and
the host-side mirror validates like the reference (no kernel launches here)."""

import ctypes
import os
import re

import pytest

from paper_2201_00094_b200 import _lib
from paper_2201_00094_b200.pipeline import RenderConfig

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(REPO, "include", "woit.h")).read()
    return sorted(set(re.findall(r"\b(woit_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_binding():
    assert set(declared_symbols()) == set(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_abi_version_and_status_strings():
    lib = _lib.load()
    assert lib.woit_abi_version() == _lib.ABI_VERSION
    assert lib.woit_status_string(_lib.ERANK) == b"rank must lie in [0, 6]"
    assert lib.woit_status_string(_lib.ETAPS) == b"aberration taps must be odd and >= 3"
    assert lib.woit_status_string(12345) == b"unknown status"


def test_argument_validation_without_a_gpu():
    """Invalid arguments are rejected before any CUDA call."""
    lib = _lib.load()
    p = _lib.Params()
    p.rank, p.aberration_taps = 7, 5
    f = _lib.Frags()
    b = _lib.Bufs()
    assert lib.woit_render_band(f, p, b, None, 0, None) == _lib.ERANK
    p.rank, p.aberration_taps = 3, 4
    assert lib.woit_render_band(f, p, b, None, 0, None) == _lib.ETAPS
    p.aberration_taps = 5
    assert lib.woit_render_band(f, p, b, None, 0, None) == _lib.EINVAL  # width 0
    assert lib.woit_build_into(None, 1, None, None, None, 1, 9, 0, None, 0, None) == _lib.ERANK
    assert lib.woit_build_into(None, 1, None, None, None, 1, 3, 0, None, 0, None) == _lib.EINVAL
    with pytest.raises(ValueError, match="rank must lie"):
        _lib.check(_lib.ERANK, "x")
    with pytest.raises(RuntimeError, match="CUDA error"):
        _lib.check(_lib.ECUDA, "x")


@pytest.mark.parametrize("kw", [dict(method="nope"), dict(rank=7), dict(rank=-1),
                                dict(aberration_taps=4), dict(aberration_taps=1),
                                dict(workers=0)])
def test_config_validation(kw):
    """test_pipeline.py:280-286."""
    base = dict(method="wavelet", rank=3, width=16, height=16, workers=1)
    base.update(kw)
    with pytest.raises(ValueError):
        RenderConfig(**base)


def test_config_flags():
    c = RenderConfig(refraction=True, chromatic_aberration=True, cube_transmission=True,
                     normalize=False, packed_storage=True, literal_spectral_t=True,
                     cube_backface_only=True)
    assert c.flags == 0x77
    assert RenderConfig().flags == _lib.NORMALIZE
