#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x -k "bfs or BFS or c3" 2>&1 | grep -E "^E |passed|failed" | head
timeout 900 python tools/bfs_bench.py --scale 22 --reps 5 --out gpurun_out/bfs22.json 2>&1 | grep -E "selector |heuristic|fixed|best"
timeout 1200 python tools/c5_bench.py --out gpurun_out/c5.json 2>&1 | grep -E "heuristic|masked|col_lb_atomic [0-9]"
