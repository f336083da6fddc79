#!/bin/bash
# Round evidence: default bench line, reference arm, per-config lines, ncu launch list + full capture.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"
for v in ternary quadrature; do python bench.py --variant $v --steps 3 --no-cpu > gpurun_out/bench_config2_$v.json 2> gpurun_out/bench_config2_$v.err; echo "cfg2 $v rc=$?"; done
for c in 0 1 3 4; do python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_config$c.json 2> gpurun_out/bench_config$c.err; echo "cfg$c rc=$?"; done
python bench.py --config 4 --dtype f32 --steps 3 --warmup 3 > gpurun_out/bench_config4_f32.json 2> gpurun_out/bench_config4_f32.err; echo "cfg4 f32 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --block 2048 --no-cpu > gpurun_out/ncu_bench.log 2>&1; echo "launches rc=$?"
python bench.py --solver lp --steps 10 --warmup 3 > gpurun_out/bench_lp.json 2> gpurun_out/bench_lp.err; echo "lp rc=$?"
python bench.py --solver brute --steps 10 --warmup 3 > gpurun_out/bench_brute.json 2> gpurun_out/bench_brute.err; echo "brute rc=$?"
bash scripts/gpurun/gpurun_fullprof.sh
