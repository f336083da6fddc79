#!/bin/bash
# GPU tests + the config-1 bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/tests.log; echo "tests rc=${PIPESTATUS[0]}"; tail -2 gpurun_out/tests.log
timeout 900 python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; echo "bench1 rc=$?"
tail -c 600 gpurun_out/bench_cfg1.json
