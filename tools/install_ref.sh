#!/usr/bin/env bash
# Install the UNMODIFIED reference package (woit, pure Python) into baseline/_ref
# for bench.py's reference arm and the conformance suite (tests/test_conformance.py).
# baseline/_ref is git-ignored (not product source) but not gpurun-ignored, so it
# ships to the GPU box with the repo snapshot. Run in the build container, where
# /root/reference exists:  bash tools/install_ref.sh
set -euo pipefail
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
DST="$REPO/baseline/_ref"
[ -d "$SRC" ] || { echo "no $SRC: nothing to install (the GPU box uses the shipped copy)"; exit 0; }
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
# the setuptools build writes egg-info into the source tree: build from a copy
cp -r "$SRC" "$TMP/pkg"
rm -rf "$DST"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$DST" "$TMP/pkg"
# the reference's own test files, run unmodified by tests/test_conformance.py
mkdir -p "$DST/woit_tests"
cp "$SRC"/tests/*.py "$DST/woit_tests/"
echo "installed $(ls "$DST")"
