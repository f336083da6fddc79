#!/bin/bash
# ncu --set full capture of one config-2 locus launch (B = 2 waves of resident warps)
mkdir -p gpurun_out
python scripts/prof_locus.py --B 8288 > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:locus -c 1 -o gpurun_out/prof_cur python scripts/prof_locus.py --B 8288 > gpurun_out/ncu.log 2>&1; echo "full rc=$?"; cat gpurun_out/plain.log
