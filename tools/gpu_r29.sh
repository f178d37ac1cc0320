#!/bin/bash
python tools/kernel_sweep.py --inputs c2 --kernels 4,6 --lanes 0,1,2,8,16,32 --densities 0.00001,0.001,0.01,0.1,0.5 --reps 7 2>&1 | grep c2
