#!/bin/bash
# same-box A/B: config 2 (B = 65,536) and config 4 (B = 16,384) over the given builds, config 1 over head/v2r/goto
mkdir -p gpurun_out
tags=${@:-v2r goto qi hqp walk ddot all4}
bash scripts/gpurun/ab_cfg.sh 2 65536 2 $tags 2>&1 | tee gpurun_out/ab3.log
bash scripts/gpurun/ab_cfg.sh 4 16384 1 $tags 2>&1 | tee -a gpurun_out/ab3.log
bash scripts/gpurun/ab_cfg.sh 1 262144 2 v2r goto 2>&1 | tee -a gpurun_out/ab3.log
