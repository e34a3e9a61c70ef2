#!/bin/sh
# Install the UNMODIFIED reference package (terngemm, Python + numba) into baseline/_ref, the
# one offline install the task allows.  baseline/_ref is git-ignored but travels to the GPU box
# with the gpurun snapshot, where bench.py's reference arm / cpu_baseline time it and
# tests/test_gpu_reference_acceptance.py runs its acceptance tests through the B200 backends.
# The reference's own test modules are copied beside it (they are not part of the wheel).
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=${1:-/root/reference/pkg}
[ -d "$SRC" ] || { echo "reference not found at $SRC" >&2; exit 1; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"            # the reference tree is read-only; setuptools writes build files
rm -rf "$HERE/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$HERE/_ref" "$TMP/pkg"
mkdir -p "$HERE/_ref/_reference_tests"
cp "$SRC"/tests/*.py "$HERE/_ref/_reference_tests/"
rm -rf "$TMP"
echo "installed terngemm into $HERE/_ref"
