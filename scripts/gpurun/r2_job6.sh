#!/bin/bash
# GPU tests, default bench line + config-1 line, bucketed profiles of the config-2 and config-1 kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/tests.log; echo "tests rc=${PIPESTATUS[0]}"; tail -1 gpurun_out/tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; echo "bench1 rc=$?"
rm -rf gpurun_out/prof; bash scripts/gpurun/r2_buckets.sh cfg2
bash scripts/gpurun/r2_prof_pack.sh cfg1
