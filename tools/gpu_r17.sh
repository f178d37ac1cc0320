#!/bin/bash
timeout 900 python -m pytest tests/ -m gpu -q -p no:cacheprovider -x 2>&1 | grep -E "^E |passed|failed" | head
timeout 900 python tools/bfs_bench.py --scale 22 --reps 5 --out gpurun_out/bfs22.json 2>&1 | tail -12
ADASPMV_BENCH_FORCE_MULTI=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/bench_multi1.json 2> gpurun_out/bench_multi1.err
tail -c 1500 gpurun_out/bench_multi1.json; tail -3 gpurun_out/bench_multi1.err
