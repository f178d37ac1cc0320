#!/bin/bash
for h in 4096 2048 1024 512 256 128; do echo "heavy $h"; ADASPMV_HEAVY_MIN=$h python tools/kernel_sweep.py --inputs rmat22,rmat20 --kernels 0 --layouts 2 --densities 1.0 --reps 7 2>&1 | grep -E "rmat"; done
