#!/bin/bash
timeout 900 python -m pytest tests/ -m gpu -q -p no:cacheprovider -x 2>&1 | grep -E "^E |passed|failed" | head -20
ADASPMV_BATCH_TRACE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --lanes 3 > gpurun_out/bench_trace.json 2> gpurun_out/bench_trace.err
grep run_batch gpurun_out/bench_trace.err | tail -7
for L in 3 4; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --lanes $L > gpurun_out/bench_l$L.json 2> gpurun_out/bench_l$L.err
python -c "import json;d=json.load(open('gpurun_out/bench_l$L.json'));print($L, d['value'], d['e2e'])"; done
timeout 900 python tools/bfs_bench.py --scale 22 --reps 5 --out gpurun_out/bfs22.json 2>&1 | tail -8
