#!/bin/bash
# same-box A/B of warp-kernel builds: config 2 (B = 65,536), config 3 and config 4 (B = 16,384)
mkdir -p gpurun_out
tags=${@:-head v1 v1hq v2 v3}
bash scripts/gpurun/ab_cfg.sh 2 65536 3 $tags 2>&1 | tee gpurun_out/ab2.log
bash scripts/gpurun/ab_cfg.sh 3 32768 1 $tags 2>&1 | tee -a gpurun_out/ab2.log
bash scripts/gpurun/ab_cfg.sh 4 16384 1 $tags 2>&1 | tee -a gpurun_out/ab2.log
