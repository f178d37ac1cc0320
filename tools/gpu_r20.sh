#!/bin/bash
python tools/kernel_sweep.py --inputs c1 --kernels 0,1 --lanes 0,1,2 --densities 1.0 --reps 15 2>&1 | tail -6
