#!/bin/bash
for L in 3 4 5; do
ADASPMV_BATCH_TRACE=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --lanes $L > gpurun_out/bench.json 2> gpurun_out/bench.err
grep run_batch gpurun_out/bench.err | tail -7; python -c "
import json;d=json.load(open('gpurun_out/bench.json'));print($L, d['e2e']['value'], d['e2e']['ms_per_step'])"
done
