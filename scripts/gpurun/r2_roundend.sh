#!/bin/bash
# Round-2 evidence (part 1): GPU tests, the default bench line, the reference arm, every config's line,
# the warm lambda path, LP and brute-force lines, and the ncu launch list of the default bench command.
o=gpurun_out/r02final; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4 > $o/tests.log; echo "tests rc=${PIPESTATUS[0]}"; tail -1 $o/tests.log
python bench.py > $o/bench_default.json 2> $o/bench_default.err; echo "bench rc=$?"
python bench.py --impl reference > $o/bench_reference.json 2> $o/bench_reference.err; echo "ref rc=$?"
for v in ternary quadrature; do python bench.py --variant $v --steps 3 --no-cpu > $o/bench_config2_$v.json 2> $o/bench_config2_$v.err; echo "cfg2 $v rc=$?"; done
python bench.py --warm --steps 3 --warmup 3 > $o/bench_config2_warm.json 2> $o/bench_config2_warm.err; echo "warm rc=$?"
for c in 0 1 3 4; do python bench.py --config $c --steps 3 --warmup 3 > $o/bench_config$c.json 2> $o/bench_config$c.err; echo "cfg$c rc=$?"; done
python bench.py --config 4 --dtype f32 --steps 3 --warmup 3 > $o/bench_config4_f32.json 2> $o/bench_config4_f32.err; echo "cfg4 f32 rc=$?"
python bench.py --solver lp --steps 10 --warmup 3 > $o/bench_lp.json 2> $o/bench_lp.err; echo "lp rc=$?"
python bench.py --solver brute --steps 10 --warmup 3 > $o/bench_brute.json 2> $o/bench_brute.err; echo "brute rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > $o/ncu_bench.log 2>&1; echo "launches rc=$?"
