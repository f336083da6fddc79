#!/bin/bash
# ncu --set full of WORKLOAD (default cfg2) with the in-tree library, reduced on the box to per-source-line
# counts and per-bucket (step phase) instruction counts per coordinate step of locus_warp_kernel<5,30,double>.
w=${1:-cfg2}
mkdir -p gpurun_out/prof
python scripts/prof_kernels.py $w --units gpurun_out/prof/units_$w.json > gpurun_out/prof/plain_$w.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:locus -s 1 -c 1 -f -o gpurun_out/prof/prof_$w \
  python scripts/prof_kernels.py $w > gpurun_out/prof/ncu_$w.log 2>&1
python scripts/ncu_summary.py --db gpurun_out/prof/ncu_r02.json gpurun_out/prof $w > gpurun_out/prof/summary_$w.log 2>&1
units=$(python -c "import json;print(json.load(open('gpurun_out/prof/units_$w.json'))['units'])")
K=$(ncu -i gpurun_out/prof/prof_$w.ncu-rep --page raw --csv --print-kernel-base mangled --metrics gpu__time_duration.sum 2>/dev/null | python -c "
import csv,sys; r=list(csv.reader(sys.stdin)); h=r[0]; print(r[-1][h.index('Kernel Name')])")
B=$(python scripts/warp_buckets.py)
python scripts/ncu_lines.py gpurun_out/prof/prof_$w.ncu-rep paper_2510_15649_b200/libladlasso_b200.so $K --top 150 --sass-top 150 --per $units \
  --buckets "$B" > gpurun_out/prof/buckets_$w.txt 2>&1
rm -f gpurun_out/prof/prof_$w.ncu-rep
