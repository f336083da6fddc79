#!/bin/bash
o=gpurun_out/job2; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_path.py -m gpu -q -x 2>&1 | tail -5 > $o/tests_path.log; echo "path tests rc=${PIPESTATUS[0]}"; tail -2 $o/tests_path.log
for g in 1 2 4 8; do
  python bench.py --warm --warm-groups $g --steps 3 --warmup 2 --no-cpu > $o/bench_warm_g$g.json 2> $o/bench_warm_g$g.err; echo "warm g$g rc=$?"
  python -c "import json;d=json.load(open('$o/bench_warm_g$g.json'));print('groups $g', round(d['value']), 'e2e', round(d['e2e']['value']), d['step_ms'])"
done
python bench.py --solver brute --steps 10 --warmup 3 > $o/bench_brute.json 2> $o/bench_brute.err; echo "brute rc=$?"
python -c "import json;d=json.load(open('$o/bench_brute.json'));print('brute', round(d['value']), d['step_ms'])"
python bench.py --solver lp --steps 10 --warmup 3 > $o/bench_lp.json 2> $o/bench_lp.err; echo "lp rc=$?"
python -c "import json;d=json.load(open('$o/bench_lp.json'));print('lp', round(d['value']), d['step_ms'])"
bash scripts/gpurun/sanitize.sh
