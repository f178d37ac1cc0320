#!/bin/bash
timeout 900 python tools/pagerank_bench.py --scale 22 --prune 1e-8 --out gpurun_out/pr22.json 2>&1 | grep -E "selector|heuristic|fixed_0|fixed_1|best"
