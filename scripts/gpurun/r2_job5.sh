mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/tests.log; echo "tests rc=${PIPESTATUS[0]}"; tail -1 gpurun_out/tests.log
bash scripts/gpurun/ab_cfg.sh 2 65536 2 goto ictl ictlh ictlhw idesc 2>&1 | tee gpurun_out/ab5.log
bash scripts/gpurun/ab_cfg.sh 4 16384 1 goto ictl ictlh ictlhw idesc 2>&1 | tee -a gpurun_out/ab5.log
rm -rf gpurun_out/prof; bash scripts/gpurun/r2_buckets.sh cfg2
bash scripts/gpurun/r2_prof_pack.sh cfg1
