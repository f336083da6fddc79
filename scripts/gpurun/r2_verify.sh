#!/bin/bash
# Last check of the shipped binary: smoke, every GPU test, the parity sweep at scale and the default bench line.
o=gpurun_out/verify; mkdir -p $o
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2 | tee $o/tests.log
timeout 1500 python scripts/parity_sweep.py $o/parity_sweep.json > $o/parity_sweep.log 2>&1; echo "sweep rc=$?"
python bench.py > $o/bench_default.json 2> $o/bench_default.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('$o/bench_default.json'));print(round(d['value']), round(d['e2e']['value']), d['parity_sample'], d['clocks'])"
