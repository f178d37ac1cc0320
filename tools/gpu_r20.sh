#!/bin/bash
ADASPMV_BENCH_FORCE_MULTI=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/bench_multi1.json; echo "rc=$?"
ls -la gpurun_out/
