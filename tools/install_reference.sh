#!/bin/sh
# Installs the UNMODIFIED reference package (pure Python, /root/reference/pkg)
# into baseline/_ref -- the one offline install the task allows -- plus the
# reference's own test files (they are not part of the wheel) for the GPU
# drop-in run (tests/test_gpu_dropin.py).  baseline/_ref is git-ignored but
# travels to the GPU box with the gpurun snapshot; /root/reference does not.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
[ -d "$SRC" ] || { echo "no reference at $SRC" >&2; exit 1; }
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"   # the build writes egg-info into the source tree: build from a copy
rm -rf "$ROOT/baseline/_ref"
python -m pip install -q --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
mkdir -p "$ROOT/baseline/_ref/tests"
cp "$SRC"/tests/*.py "$ROOT/baseline/_ref/tests/"
echo "installed tomofuse into $ROOT/baseline/_ref"
