#!/bin/bash
mkdir -p gpurun_out
bash scripts/gpurun/ab_cfg.sh 2 65536 2 base6 alist rawaw both6 2>&1 | tee gpurun_out/ab7.log
bash scripts/gpurun/ab_cfg.sh 4 16384 1 base6 alist rawaw both6 2>&1 | tee -a gpurun_out/ab7.log
bash scripts/gpurun/ab_cfg.sh 1 262144 2 base6 zdiv 2>&1 | tee -a gpurun_out/ab7.log
