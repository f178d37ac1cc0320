#!/bin/bash
set -x
timeout 600 python tools/bin_rows_sweep.py 0:0:1,8192:0:1,14336:0:1,20480:0:1,24576:0:1,0:400000:1,0:800000:1,14336:300000:1 2>&1 | tail -9
timeout 600 python tools/kernel_sweep.py --inputs c1 --kernels 0,1 --layouts 1 --lanes 0,1,2,4 --reps 5 2>&1 | tail -8
