#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 1 --block 4096 --no-cpu > gpurun_out/tr1.json 2> gpurun_out/tr1.err; echo "torchrun rc=$?"
tail -c 400 gpurun_out/tr1.json; tail -3 gpurun_out/tr1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/tr_ref.json 2> gpurun_out/tr_ref.err; echo "ref rc=$?"; tail -c 300 gpurun_out/tr_ref.json
