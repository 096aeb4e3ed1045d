#!/bin/sh
# Installs the UNMODIFIED reference package into baseline/_ref (git-ignored,
# shipped to the GPU box by gpurun): the offline pip install the task
# prescribes (from a /tmp copy: /root/reference is read-only; --no-deps
# because numpy/numba/... are already in the image and not in the wheelhouse
# index), plus a copy of pkg/ (sources + its own tests) for
# tests/test_reference_suite_on_gpu.py and the numba CPU baseline in bench.py.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/boba_ref_src "$ROOT/baseline/_ref"
mkdir -p "$ROOT/baseline/_ref"
cp -r /root/reference/pkg /tmp/boba_ref_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" /tmp/boba_ref_src
cp -r /root/reference/pkg "$ROOT/baseline/_ref/pkg"
find "$ROOT/baseline/_ref" -name __pycache__ -prune -exec rm -rf {} +
