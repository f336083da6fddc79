#!/bin/bash
# Round-2 closing evidence from one box: the bench lines (r2_roundend.sh), the parity sweep at scale, then
# the ncu captures of every library kernel (r2_profiles_final.sh).
bash scripts/gpurun/r2_roundend.sh
timeout 1500 python scripts/parity_sweep.py gpurun_out/r02final/parity_sweep.json > gpurun_out/r02final/parity_sweep.log 2>&1; echo "sweep rc=$?"
bash scripts/gpurun/r2_profiles_final.sh
