#!/bin/bash
# GPU tests, then the whole of BASELINE config 4 (2^26 problems) on one GPU in fp64 and fp32 (chunked runner)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/tests.log; echo "tests rc=${PIPESTATUS[0]}"; tail -2 gpurun_out/tests.log
for dt in f64 f32; do
  timeout 1500 python -m paper_2510_15649_b200.runner --config 4 --total 67108864 --chunk 2097152 --dtype $dt \
    > gpurun_out/cfg4_full_$dt.json 2> gpurun_out/cfg4_full_$dt.err; echo "full4 $dt rc=$?"; tail -c 800 gpurun_out/cfg4_full_$dt.json
done
