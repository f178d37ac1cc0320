#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k counters 2>&1 | grep -E "^E |passed|failed|Error" | head
timeout 900 python -m pytest tests/ -m gpu -q -p no:cacheprovider -x 2>&1 | grep -E "^E |passed|failed" | head
python tools/kernel_sweep.py --inputs c2 --kernels 0,4 --densities 1.0,0.1 --reps 7 2>&1 | grep c2
