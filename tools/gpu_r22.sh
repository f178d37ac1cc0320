#!/bin/bash
timeout 900 python -m pytest tests/ -m gpu -q -p no:cacheprovider -x 2>&1 | grep -E "^E |passed|failed" | head
python tools/kernel_sweep.py --inputs rmat22,rmat20 --kernels 0,1 --densities 1.0 --reps 9 2>&1 | grep -E "rmat"
timeout 1200 python tools/c5_bench.py --out gpurun_out/c5.json 2>&1 | tail -12
