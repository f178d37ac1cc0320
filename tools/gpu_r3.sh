#!/bin/bash
set -x
timeout 600 python -m pytest tests/ -m gpu -q -p no:cacheprovider -x 2>&1 | tail -15
timeout 600 python tools/bin_rows_sweep.py 0:0:1,0:0:2,57344:0:1,57344:0:2,0:300000:2,0:200000:2 2>&1 | tail -8
timeout 900 python tools/pagerank_bench.py --scale 20 --prune 1e-8 --reps 2 --out gpurun_out/pr20.json 2>&1 | tail -14
timeout 900 python tools/pagerank_bench.py --scale 20 --prune 1e-8 --reps 2 --dtype f64 --out gpurun_out/pr20_f64.json 2>&1 | tail -14
timeout 600 python tools/kernel_sweep.py --inputs rmat22 --kernels 0,1 --layouts 1,2 --reps 3 2>&1 | tail -8
