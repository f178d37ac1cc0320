#!/bin/bash
timeout 900 python -m pytest tests/ -m gpu -q -p no:cacheprovider -x 2>&1 | grep -E "^E |passed|failed" | head
python __graft_entry__.py smoke 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -2 gpurun_out/bench.err; python -c "
import json;d=json.load(open('gpurun_out/bench.json'));print({k:d[k] for k in ('value','ms_per_step','selector_regret','overhead','e2e','roofline','cpu_baseline','clocks','gpu_launches')})"
