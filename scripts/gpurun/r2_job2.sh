mkdir -p gpurun_out/prof
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/tests.log; echo "tests rc=${PIPESTATUS[0]}"; tail -2 gpurun_out/tests.log
bash scripts/gpurun/ab_cfg.sh 1 262144 3 head cand 2>&1 | tee gpurun_out/ab1.log
bash scripts/gpurun/r2_prof_pack.sh cfg1 cfg2 cfg0 cfg3 cfg4 cfg4f32 warm2 brute1 brute0 lp2 cert2 gen4 genspec
