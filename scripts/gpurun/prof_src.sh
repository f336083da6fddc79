#!/bin/bash
# ncu --set full (with source) of the config-2 warp kernel and the config-1 thread kernel
mkdir -p gpurun_out
python scripts/prof_locus.py --B 8288 > gpurun_out/plain2.log 2>&1 && \
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:locus -c 1 -o gpurun_out/prof_c2 python scripts/prof_locus.py --B 8288 > gpurun_out/ncu2.log 2>&1; echo "c2 rc=$?"
python scripts/prof_locus.py --config 1 --B 262144 > gpurun_out/plain1.log 2>&1 && \
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:locus -c 1 -o gpurun_out/prof_c1 python scripts/prof_locus.py --config 1 --B 262144 > gpurun_out/ncu1.log 2>&1; echo "c1 rc=$?"
