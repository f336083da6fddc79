#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -4
for c in 0 1 3 4; do timeout 600 python bench.py --config $c --steps 3 --warmup 1 --e2e-steps 1 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "config $c rc=$?"; done
python3 -c "
import json
for c in (0,1,3,4):
    try:
        d=json.load(open(f'gpurun_out/bench_c{c}.json'))
        print(c, round(d['value']), 'e2e', round(d['e2e']['value']), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value']), 'parity', d['parity_sample'], 'frac', round(d['roofline']['frac'],4), 'S/solve', round(d['roofline']['coord_steps_per_solve']))
    except Exception as e: print(c, 'ERR', e)
"
