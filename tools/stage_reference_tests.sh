#!/bin/bash
# Copy the reference's own test modules next to its install in baseline/_ref
# (git-ignored, shipped to the GPU box by gpurun) so tools/run_reference_suite.py
# can run them against the drop-in there.  Run in the build container, where
# /root/reference exists; nothing is committed.
set -e
mkdir -p baseline/_ref/tests_ref
cp /root/reference/pkg/tests/*.py baseline/_ref/tests_ref/
ls baseline/_ref/tests_ref
