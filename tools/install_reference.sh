#!/bin/bash
# Install the unmodified reference package into baseline/_ref (git-ignored; it travels to the GPU box with the
# working tree): the driver-contract pip install (from a copy -- /root/reference is read-only; --no-deps: numpy
# is not in the offline wheelhouse but is in the image), plus the reference's own unit tests next to it so the
# compat-mode test (tests/test_gpu_compat_reference.py) can run them against this backend on the box.
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg" > /dev/null
mkdir -p "$ROOT/baseline/_ref/ref_tests"
cp "$SRC"/tests/*.py "$ROOT/baseline/_ref/ref_tests/"
rm -rf "$TMP"
echo "installed $(ls "$ROOT/baseline/_ref")"
