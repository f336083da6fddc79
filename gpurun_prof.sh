#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
python scripts/prof_locus.py --B 18944 > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:locus_kernel -c 1 -o gpurun_out/prof_locus_r1b python scripts/prof_locus.py --B 18944 > gpurun_out/ncu.log 2>&1
tail -3 gpurun_out/ncu.log
