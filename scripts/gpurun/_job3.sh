#!/bin/bash
o=gpurun_out/job3; mkdir -p $o
bash scripts/gpurun/ab_cfg.sh 1 262144 3 head yield 2>&1 | tee $o/ab_cfg1.log
bash scripts/gpurun/ab_cfg.sh 2 65536 2 head yield 2>&1 | tee $o/ab_cfg2.log
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > $o/tests.log; echo "tests rc=${PIPESTATUS[0]}"; tail -2 $o/tests.log
python bench.py --config 1 --steps 3 --warmup 3 > $o/bench_config1.json 2> $o/bench_config1.err; echo "cfg1 rc=$?"
python -c "import json;d=json.load(open('$o/bench_config1.json'));print('cfg1', round(d['value']), 'e2e', round(d['e2e']['value']), d['parity_sample'])"
python bench.py --warm --steps 3 --warmup 3 > $o/bench_warm.json 2> $o/bench_warm.err; echo "warm rc=$?"
python -c "import json;d=json.load(open('$o/bench_warm.json'));print('warm', round(d['value']), 'e2e', round(d['e2e']['value']), d['parity_sample'])"
