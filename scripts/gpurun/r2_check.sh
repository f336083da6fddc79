mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_gputests.log
echo "tests rc=$?"
tail -3 gpurun_out/r2_gputests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r2_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_ref.json 2>&1; echo "ref rc=$?"
tail -c 600 gpurun_out/r2_ref.json
