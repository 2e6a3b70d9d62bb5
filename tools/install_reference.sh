#!/usr/bin/env bash
# Offline install of the reference package (pilothash 0.1.0) into
# baseline/_ref (git-ignored, travels to the GPU box with the snapshot), plus
# a copy of its own test suite (baseline/_ref/reference_tests) so the GPU box
# can run that suite through the compat_kernels shim
# (tests/test_gpu_reference_suite.py) and bench.py --impl reference can time
# pilothash.build itself. Nothing here is committed.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"   # the build writes into its source tree; /root/reference is read-only
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref/reference_tests"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/reference_tests"
rm -rf "$TMP"
echo "installed: $(ls "$ROOT/baseline/_ref")"
