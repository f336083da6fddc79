#!/bin/bash
o=gpurun_out/job15; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > $o/tests.log; echo "tests rc=${PIPESTATUS[0]}"; tail -2 $o/tests.log
python bench.py --config 1 --steps 3 --warmup 3 > $o/bench_config1.json 2> $o/bench_config1.err; echo "cfg1 rc=$?"
python -c "import json;d=json.load(open('$o/bench_config1.json'));print('cfg1', round(d['value']), 'e2e', round(d['e2e']['value']), d['parity_sample'])"
LINES_TOP=100 bash scripts/gpurun/r2_prof_pack.sh cfg1
