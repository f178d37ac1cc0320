#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_batch.py -q -p no:cacheprovider -x 2>&1 | grep -E "^E |passed|failed" | head -20
for L in 3 5 7; do
ADASPMV_BATCH_TRACE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --lanes $L > gpurun_out/bench_l$L.json 2> gpurun_out/bench_l$L.err
grep run_batch gpurun_out/bench_l$L.err | tail -7
python -c "import json;d=json.load(open('gpurun_out/bench_l$L.json'));print($L, d['value'], d['e2e'])"; done
