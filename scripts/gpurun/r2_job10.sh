#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/tests.log; echo "tests rc=${PIPESTATUS[0]}"; tail -1 gpurun_out/tests.log
rm -rf gpurun_out/prof; bash scripts/gpurun/r2_prof_pack.sh cfg1
