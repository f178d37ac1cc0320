#!/bin/bash
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -4
timeout 1500 python tools/c5_bench.py --scale 26 --reps 3 --kernels 0,1 --densities 1.0 --panels -1,16384,32768,49152,98304 --out gpurun_out/c5_panels.json 2>&1 | grep -E "panel|^1.0"
timeout 600 python tools/kernel_sweep.py --inputs c2,rmat22 --kernels 0 --layouts 0 --reps 5 2>&1 | tail -3
