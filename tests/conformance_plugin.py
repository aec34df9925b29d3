"""pytest plugin for the conformance suite (tests/test_conformance.py): loaded with
``-p tests.conformance_plugin`` before the reference's own test modules are
imported, it re-binds the reference's hot-path entry points (woit.pipeline steps,
_wavelet_band, render_frame; woit.wavelet batch kernels) to the B200 binding, and
at the end of the session writes how often each bound function was called to
$WOIT_BINDING_CALLS (proof that the GPU path, not the reference's numpy, ran)."""

import json
import os

from paper_2201_00094_b200 import ref_binding

ref_binding.install()


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("WOIT_BINDING_CALLS")
    if path:
        with open(path, "w") as f:
            json.dump(ref_binding.CALLS, f)
