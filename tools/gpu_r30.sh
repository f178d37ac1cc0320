#!/bin/bash
for h in 4096 2048 1024 512; do echo "heavy $h"; ADASPMV_HEAVY_MIN=$h python tools/kernel_sweep.py --inputs rmat22,rmat20 --kernels 0 --layouts 2 --densities 0.3,0.45,0.6,0.75,0.9,1.0 --reps 5 2>&1 | grep -E "rmat" | awk '{print $1, $2, $7}'; done
