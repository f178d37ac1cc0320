#!/bin/bash
set -x
timeout 600 python -m pytest tests/ -m gpu -q -p no:cacheprovider 2>&1 | tail -5
timeout 900 compute-sanitizer --tool memcheck --print-limit 3 python -m pytest tests/test_cli.py tests/test_pagerank.py -m gpu -q -p no:cacheprovider -k "not large" 2>&1 | grep -E "ERROR SUMMARY|passed|failed|Invalid" | head
timeout 600 python tools/e2e_profile.py 2>&1 | tail -9
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
