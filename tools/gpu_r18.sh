#!/bin/bash
timeout 900 python -m pytest tests/ -m gpu -q -p no:cacheprovider -x 2>&1 | grep -E "^E |passed|failed" | head
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -2 gpurun_out/bench.err; python -c "
import json;d=json.load(open('gpurun_out/bench.json'));print({k:d[k] for k in ('value','ms_per_step','selector_regret','overhead','e2e')})"
timeout 900 python tools/bfs_bench.py --scale 22 --reps 5 --out gpurun_out/bfs22.json 2>&1 | grep -E "selector|heuristic|best"
