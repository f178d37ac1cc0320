#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x 2>&1 | grep -E "^E |passed|failed" | head
timeout 900 python tools/pagerank_bench.py --scale 22 --prune 1e-8 --out gpurun_out/pr22.json 2>&1 | grep -E "best"
timeout 1200 python tools/c5_bench.py --out gpurun_out/c5.json 2>&1 | grep -E "^1.0|heuristic"
