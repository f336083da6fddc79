#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
M=smsp__inst_executed.sum,sm__cycles_elapsed.avg,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warp_latency_per_inst_issued.ratio,launch__registers_per_thread,gpu__time_duration.sum
python scripts/prof_locus.py --B 18944 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none -k regex:locus -c 1 --csv python scripts/prof_locus.py --B 18944 > gpurun_out/metrics.csv 2>&1
cat gpurun_out/plain.log
grep -E "inst_executed.sum|cycles_elapsed|issue_active|warps_active|stalled|latency|registers|duration" gpurun_out/metrics.csv | awk -F'","' '{print $(NF-2)" "$(NF-1)" "$NF}'
timeout 300 python scripts/quick_timing2.py 2>&1 | tail -8
