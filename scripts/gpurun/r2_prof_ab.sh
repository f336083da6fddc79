#!/bin/bash
# ncu counters (sections only) of one workload for several builds: r2_prof_ab.sh WORKLOAD TAG...
w=$1; shift
mkdir -p gpurun_out/prof
for t in "$@"; do
  lib=paper_2510_15649_b200/libladlasso_b200_$t.so
  [ "$t" = "cur" ] && lib=paper_2510_15649_b200/libladlasso_b200.so
  LAD_PROF_LIB=$lib python scripts/prof_kernels.py $w --units gpurun_out/prof/units_${w}_$t.json > /dev/null 2>&1 || { echo "$t plain failed"; continue; }
  LAD_PROF_LIB=$lib timeout 900 ncu --section SpeedOfLight --section Occupancy --section WarpStateStats --section SchedulerStats \
    --section InstructionStats --section MemoryWorkloadAnalysis \
    --metrics smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:locus -s 1 -c 1 -f -o gpurun_out/prof/prof_${w}_$t python scripts/prof_kernels.py $w > /dev/null 2>&1
  python scripts/ncu_summary.py --db gpurun_out/prof/ab_$w.json gpurun_out/prof ${w}_$t >> gpurun_out/prof/ab_summary.log 2>&1
  rm -f gpurun_out/prof/prof_${w}_$t.ncu-rep
done
