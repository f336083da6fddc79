#!/bin/bash
# Session-3 re-entry check: GPU tests and the default bench line from a fresh build.
o=gpurun_out/r2s3; mkdir -p $o
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -6 > $o/tests.log; echo "tests rc=${PIPESTATUS[0]}"; tail -2 $o/tests.log
python bench.py > $o/bench_default.json 2> $o/bench_default.err; echo "bench rc=$?"; cat $o/bench_default.json | head -c 600
