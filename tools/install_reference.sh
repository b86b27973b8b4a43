#!/bin/bash
# Installs the UNMODIFIED reference package (mpssim, pure Python) under baseline/_ref -- the one
# offline install the task allows -- from a copy under /tmp (its build writes into the source
# tree; /root/reference is read-only), plus its test suite under baseline/_ref_tests so the GPU
# box (which has no /root/reference) can run the reference's own tests with the drop-in shim.
# Both directories are git-ignored and travel to the GPU box with the gpurun snapshot.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
rm -rf /tmp/mpssim_src "$ROOT/baseline/_ref" "$ROOT/baseline/_ref_tests"
cp -r "$SRC" /tmp/mpssim_src
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --target "$ROOT/baseline/_ref" /tmp/mpssim_src
cp -r "$SRC/tests" "$ROOT/baseline/_ref_tests"
echo "installed: $ROOT/baseline/_ref (mpssim), $ROOT/baseline/_ref_tests"
