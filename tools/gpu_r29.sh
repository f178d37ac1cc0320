#!/bin/bash
timeout 600 ncu --set full --clock-control none -k regex:"row_direct_kernel" -c 1 -o gpurun_out/prof_c1 python tools/kernel_sweep.py --inputs c1 --kernels 0 --reps 1 > /dev/null 2>&1
ls gpurun_out/
