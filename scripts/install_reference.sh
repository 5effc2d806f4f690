#!/usr/bin/env bash
# Install the unmodified reference package into baseline/_ref (git-ignored, travels to the GPU
# box with gpurun) and stage its own test suite under baseline/_ref/ref_tests for
# tests/test_gpu_scale.py::test_reference_suite_on_dropin (scripts/ref_suite/run.py).
# Needs /root/reference (this container only). numpy/scipy are already in the image, so the
# install runs with --no-deps (the offline wheelhouse has no numpy wheel to resolve against).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no $SRC here" >&2; exit 1; }
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"                      # the build writes into its source tree
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/ref_tests"
rm -rf "$TMP"
echo "reference installed into $ROOT/baseline/_ref (tests in ref_tests/)"
