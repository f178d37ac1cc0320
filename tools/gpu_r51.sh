#!/bin/bash
python tools/kernel_sweep.py --inputs c2 --kernels 4,5 --densities 0.01,0.1,0.5 --reps 9 2>&1 | grep c2 | awk '{print $2,$3,$7}'
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'], d['ms_per_step'], [p['t_sel_us'] for p in d['points']], d['e2e']['value'])"
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x 2>&1 | tail -1
