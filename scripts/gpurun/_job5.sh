#!/bin/bash
o=gpurun_out/job5; mkdir -p $o
ncu --metrics l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_ld_lookup_hit.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_ld_lookup_miss.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum,l1tex__t_sector_hit_rate.pct,smsp__inst_executed_op_local_ld.sum,smsp__inst_executed_op_local_st.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,launch__shared_mem_config_size,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,sm__warps_active.avg.per_cycle_active \
  --clock-control none -k regex:locus_kernel -s 1 -c 1 --csv --log-file $o/local_metrics.csv python scripts/prof_kernels.py cfg1 > $o/ncu.log 2>&1
echo "rc=$?"; cat $o/local_metrics.csv | tail -20
