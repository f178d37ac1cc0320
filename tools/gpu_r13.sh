#!/bin/bash
set -x
timeout 600 python -m pytest tests/test_gpu_batch.py tests/test_gpu_kernels.py -q -p no:cacheprovider -x 2>&1 | tail -6
for L in 3 2 4; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --lanes $L > gpurun_out/bench_l$L.json 2> gpurun_out/bench_l$L.err
tail -2 gpurun_out/bench_l$L.err
python -c "import json;d=json.load(open('gpurun_out/bench_l$L.json'));print($L, d['value'], d['e2e'])"
done
