#!/bin/bash
ADASPMV_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err; echo "rc=$?"
cat gpurun_out/bench_gloo2.json | tail -c 1500; grep -E "Error|error" gpurun_out/bench_gloo2.err | head -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --impl reference --gpus 2 --steps 2 --warmup 2 > gpurun_out/bench_ref2.json 2> gpurun_out/bench_ref2.err; echo "rc=$?"; tail -c 300 gpurun_out/bench_ref2.json
