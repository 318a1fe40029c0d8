#!/usr/bin/env bash
# Run the GPU test suite on the box with per-test durations; output under gpurun_out/.
set -o pipefail
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -s --durations=25 ${PYTEST_ARGS:-} 2>&1 | tee gpurun_out/gpu_tests.log | tail -80
