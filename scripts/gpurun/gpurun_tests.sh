#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -4
for c in 0 2; do timeout 600 python bench.py --config $c --steps 3 --warmup 1 --e2e-steps 1 --no-cpu > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "config $c rc=$?"; done
python3 -c "
import json
for c in (0,2):
    try:
        d=json.load(open(f'gpurun_out/bench_c{c}.json'))
        print(c, round(d['value']), 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],4), 'ms/step', round(d['ms_per_step'],1))
    except Exception as e: print(c, 'ERR', e)
"
