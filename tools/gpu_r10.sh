#!/bin/bash
for g in 1 2 4 8 16 32; do echo "G=$g"; ADASPMV_PULL_LANES=$g timeout 600 python tools/bfs_bench.py --scale 22 --reps 5 2>&1 | grep -E "heuristic|fixed_2 "; done
