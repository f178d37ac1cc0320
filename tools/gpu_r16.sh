#!/bin/bash
python tools/kernel_sweep.py --inputs c2 --kernels 0 --densities 1.0 --reps 9 2>&1 | tail -1
for u in 4 3 2; do echo "GP $u"; ADASPMV_BIN_GP=$u python tools/kernel_sweep.py --inputs c2,c1 --kernels 0,1 --densities 1.0 --layouts 2 --reps 9 2>&1 | grep -E "k=0" ; done
