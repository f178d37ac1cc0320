#!/bin/bash
set -x
timeout 900 python -m pytest tests/ -m gpu -q -p no:cacheprovider 2>&1 | tail -4
timeout 900 python tools/bfs_bench.py --scale 22 --reps 5 --out gpurun_out/bfs22.json 2>&1 | tail -13
