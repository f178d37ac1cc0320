#!/bin/bash
timeout 900 python tools/pagerank_bench.py --scale 22 --prune 1e-8 --out gpurun_out/pr22.json 2>&1 | grep -E "selector |heuristic|fixed_0|fixed_6|best"
timeout 900 python tools/pagerank_bench.py --scale 20 --prune 1e-8 --out gpurun_out/pr20.json 2>&1 | grep -E "best"
timeout 900 python -m pytest tests/test_pagerank.py -q -p no:cacheprovider -x 2>&1 | tail -1
