#!/bin/bash
# same-box A/B of thread-kernel builds on config 1 (B = 262,144)
mkdir -p gpurun_out
bash scripts/gpurun/ab_cfg.sh 1 262144 3 ${@:-head base rcp inl rcpinl candrcp} 2>&1 | tee gpurun_out/ab1b.log
