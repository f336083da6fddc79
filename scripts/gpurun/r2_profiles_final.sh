#!/bin/bash
# ncu of every library kernel with the final code: --set full (+ source, reduced on the box) for the
# BASELINE-shaped workloads, sections-only for the bench's own full-size config-2 launch and config 1.
rm -rf gpurun_out/prof
bash scripts/gpurun/r2_prof_pack.sh cfg0 cfg2 cfg3 cfg4 cfg4f32 warm2 brute1 brute0 lp2 cert2 gen4 genspec
bash scripts/gpurun/r2_bench2.sh bench2 cfg1
bash scripts/gpurun/r2_buckets.sh cfg2
