#!/bin/bash
# The bench's own config-2 launch (16,384 datasets x 16 lambdas, ternary, 262,144 solves) under ncu with
# the sections the summary needs (a --set full replay of this 1 s launch exceeds the time limit), and the
# config-1 thread kernel (B = 262,144) the same way.
mkdir -p gpurun_out/prof
for w in ${@:-bench2 cfg1}; do
  python scripts/prof_kernels.py $w --units gpurun_out/prof/units_$w.json > gpurun_out/prof/plain_$w.log 2>&1 || { echo "$w plain failed"; continue; }
  timeout 1500 ncu --section SpeedOfLight --section LaunchStats --section Occupancy --section WarpStateStats \
    --section SchedulerStats --section MemoryWorkloadAnalysis --section ComputeWorkloadAnalysis --section InstructionStats \
    --metrics smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active \
    --clock-control none -k regex:locus -s 1 -c 1 -f -o gpurun_out/prof/prof_$w python scripts/prof_kernels.py $w > gpurun_out/prof/ncu_$w.log 2>&1
  echo "$w ncu rc=$?"
  python scripts/ncu_summary.py --db gpurun_out/prof/ncu_r02.json gpurun_out/prof $w >> gpurun_out/prof/summary.log 2>&1
  rm -f gpurun_out/prof/prof_$w.ncu-rep
done
