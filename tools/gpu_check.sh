#!/bin/bash
# One gpurun call for an iteration: GPU parity suite + A/B stage times of the
# builds given as arguments (build_ab/*.so). Outputs in gpurun_out/.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
if [ $# -gt 0 ]; then timeout 900 python tools/stage_time.py "$@" > gpurun_out/ab.log 2>&1; fi
