#!/bin/bash
# Round-2 full pass: GPU tests, default bench, reference arm, then ncu of every library kernel.
mkdir -p gpurun_out
bash scripts/gpurun/r2_check.sh
bash scripts/gpurun/r2_profile_all.sh ${PROF_WORKS:-}
