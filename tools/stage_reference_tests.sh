#!/bin/bash
# Stage the reference's own test suites beside its unmodified install in baseline/_ref (git-ignored,
# travels to the GPU box with the snapshot) so tests/test_reference_suites.py can run them against the
# CUDA backend through paper_1404_1831_b200.kernels.install_into.  Run here, where /root/reference exists.
set -e
cd "$(dirname "$0")/.."
test -d baseline/_ref/bilayerpq || python -m pip install --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target baseline/_ref /root/reference/pkg
mkdir -p baseline/_ref/reference_tests
cp /root/reference/pkg/tests/*.py baseline/_ref/reference_tests/
echo "staged $(ls baseline/_ref/reference_tests | wc -l) files"
