#!/bin/bash
# GPU test files given as arguments (default: all -m gpu tests)
mkdir -p gpurun_out
timeout 2400 python -m pytest ${@:-tests} -m gpu -q -x 2>&1 | tail -25 > gpurun_out/r2_gputests.log
echo "tests rc=${PIPESTATUS[0]}"
tail -5 gpurun_out/r2_gputests.log
