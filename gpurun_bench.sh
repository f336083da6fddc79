#!/bin/bash
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"
python bench.py --steps 2 --warmup 1 --block 2048 --no-cpu --e2e-steps 1 > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --block 2048 --no-cpu --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
python scripts/prof_locus.py --B 4736 > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:locus -c 1 -o gpurun_out/prof_warp_r1e python scripts/prof_locus.py --B 4736 > gpurun_out/ncu.log 2>&1; echo "full rc=$?"
cat gpurun_out/bench_default.json gpurun_out/bench_reference.json
