#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 1 > gpurun_out/bench_try.json 2> gpurun_out/bench_try.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_try.json; tail -5 gpurun_out/bench_try.err
