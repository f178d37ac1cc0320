#!/bin/bash
set -x
timeout 600 python -m pytest tests/ -m gpu -q -p no:cacheprovider -x 2>&1 | tail -5
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
timeout 900 python tools/bfs_bench.py --scale 22 --reps 5 --out gpurun_out/bfs22.json 2>&1 | tail -13
timeout 900 python tools/pagerank_bench.py --scale 22 --prune 1e-8 --reps 3 --out gpurun_out/pr22.json 2>&1 | tail -12
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"binned_row_kernel|row_lb_kernel" -c 2 -o gpurun_out/prof_rmat22_spmv python tools/kernel_sweep.py --inputs rmat22 --kernels 0,1 --layouts 0 --reps 1 > /dev/null 2>&1
ls gpurun_out
