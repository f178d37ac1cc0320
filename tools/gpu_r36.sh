#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_multi_capi.py -q -p no:cacheprovider -x 2>&1 | grep -E "^E |passed|failed|Error" | head
timeout 900 python -m pytest tests/ -m gpu -q -p no:cacheprovider -x 2>&1 | grep -E "^E |passed|failed" | head
