#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x 2>&1 | grep -E "^E |passed|failed" | head
for i in 1 2; do timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'], d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['sequential_value'])"; done
