#!/bin/bash
# session 3: GPU tests on the working-tree build, same-box A/B against the round-start build, cfg2 line profile
o=gpurun_out/s3; mkdir -p $o
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > $o/tests_ab2.log; echo "tests rc=${PIPESTATUS[0]}"; tail -1 $o/tests_ab2.log
bash scripts/gpurun/ab_cfg.sh 2 65536 2 base new new2 2>&1 | grep -v Warn
bash scripts/gpurun/ab_cfg.sh 3 32768 1 base new2 2>&1 | grep -v Warn
LINES_TOP=300 bash scripts/gpurun/r2_prof_pack.sh cfg2 > $o/prof_cfg2.log 2>&1
cp gpurun_out/prof/lines_cfg2.txt gpurun_out/prof/units_cfg2.json $o/ 2>/dev/null; tail -2 $o/prof_cfg2.log
