#!/bin/bash
o=gpurun_out/job14; mkdir -p $o
bash scripts/gpurun/ab_cfg.sh 1 262144 2 cmp yf0 yr0 yfr0 2>&1 | tee $o/ab_cfg1.log
for t in ; do
LAD_PROF_LIB=paper_2510_15649_b200/libladlasso_b200_$t.so ncu --metrics l1tex__t_sectors_pipe_lsu_mem_local_op_ld_lookup_hit.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_ld_lookup_miss.sum,launch__shared_mem_config_size,launch__occupancy_limit_shared_mem,launch__registers_per_thread,sm__warps_active.avg.per_cycle_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__inst_executed.sum \
  --clock-control none -k regex:locus_kernel -s 1 -c 1 --csv --log-file $o/m_$t.csv python scripts/prof_kernels.py cfg1 > $o/ncu_$t.log 2>&1
echo "== $t"; awk -F'","' 'NR>1{print $13, $15}' $o/m_$t.csv | tr -d '"' | grep -v "^ *$"
done
