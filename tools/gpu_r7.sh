#!/bin/bash
set -x
timeout 600 python -m pytest tests/ -m gpu -q -p no:cacheprovider -x 2>&1 | tail -5
timeout 600 python tools/kernel_sweep.py --inputs rmat22,rmat20,c2 --kernels 0,1 --layouts 0 --reps 5 2>&1 | tail -8
timeout 900 python tools/bfs_bench.py --scale 22 --reps 5 --out gpurun_out/bfs22.json 2>&1 | tail -13
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
