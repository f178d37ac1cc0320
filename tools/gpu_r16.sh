#!/bin/bash
for v in 0 11 12 13; do echo "variant $v"; ADASPMV_BIN_VARIANT=$v python tools/kernel_sweep.py --inputs c2 --kernels 0 --densities 1.0 --reps 9 2>&1 | tail -1; done
