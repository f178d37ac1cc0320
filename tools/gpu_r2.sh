#!/bin/bash
# GPU session: PageRank + C4 + tests.  Outputs in gpurun_out/.
set -x
timeout 600 python -m pytest tests/ -m gpu -q -p no:cacheprovider -x 2>&1 | tail -5
timeout 900 python tools/pagerank_bench.py --scale 22 --prune 1e-8 --reps 3 --out gpurun_out/pr22.json 2>&1 | tail -14
timeout 1200 python tools/c4_bench.py --out gpurun_out/c4.json 2>&1 | tail -40
