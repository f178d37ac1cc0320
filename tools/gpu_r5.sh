#!/bin/bash
set -x
timeout 600 python -m pytest tests/ -m gpu -q -p no:cacheprovider -x 2>&1 | tail -5
python __graft_entry__.py smoke 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
timeout 900 python tools/bfs_bench.py --scale 22 --reps 3 --out gpurun_out/bfs22.json 2>&1 | tail -13
timeout 900 python tools/pagerank_bench.py --scale 22 --prune 1e-8 --reps 2 --out gpurun_out/pr22.json 2>&1 | tail -12
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"col_sort_small_kernel" -c 1 -o gpurun_out/prof_small_sort python tools/kernel_sweep.py --inputs c2 --kernels 5 --densities 0.00001 --reps 1 > /dev/null 2>&1
ls gpurun_out
