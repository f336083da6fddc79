#!/bin/bash
# ncu --set full of the given workloads (r2_profile_all.sh), then reduce the captures ON THE BOX to
# small summaries (gpurun_out/ returns at most 64 MiB): counters -> gpurun_out/prof/ncu_r02.json,
# per-source-line instruction counts of the locus kernels -> gpurun_out/prof/lines_WORKLOAD.txt.
# Captures above 8 MB are deleted after reduction.  Usage: r2_prof_pack.sh WORKLOAD...
works="$@"
bash scripts/gpurun/r2_profile_all.sh $works
python scripts/ncu_summary.py --db gpurun_out/prof/ncu_r02.json gpurun_out/prof $works > gpurun_out/prof/summary.log 2>&1
for w in $works; do
  rep=gpurun_out/prof/prof_$w.ncu-rep
  [ -f $rep ] || continue
  mangled=$(ncu -i $rep --page raw --csv --print-kernel-base mangled --metrics gpu__time_duration.sum 2>/dev/null | python -c "
import csv,sys; r=list(csv.reader(sys.stdin)); h=r[0]; print(r[-1][h.index('Kernel Name')])")
  units=$(python -c "import json;print(json.load(open('gpurun_out/prof/units_$w.json')).get('units',1))")
  if [ -n "$mangled" ]; then
    python scripts/ncu_lines.py $rep paper_2510_15649_b200/libladlasso_b200.so $mangled --top ${LINES_TOP:-80} --sass-top 120 --per $units \
      > gpurun_out/prof/lines_$w.txt 2>&1
  fi
  sz=$(stat -c %s $rep)
  [ $sz -gt 8000000 ] && rm -f $rep
done
du -sh gpurun_out
