#!/bin/bash
python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1200 python tools/c5_bench.py --out gpurun_out/c5.json 2>&1 | grep -E "^1.0 adaptive|heuristic|masked|col_lb_atomic [0-9]"
