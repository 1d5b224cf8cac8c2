#!/bin/bash
# Install the UNMODIFIED reference package (and its own test modules) under baseline/_ref, the
# git-ignored location that travels to the GPU box with the gpurun snapshot.  Used by
# tests/test_gpu_dropin.py and tests/test_gpu_reference_suite.py; run once in the build container.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/hprop_pkg baseline/_ref
cp -r /root/reference/pkg /tmp/hprop_pkg          # the source tree is read-only: build from a copy
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/hprop_pkg
mkdir -p baseline/_ref/tests
cp /root/reference/pkg/tests/*.py baseline/_ref/tests/
echo "installed: $(ls baseline/_ref)"
