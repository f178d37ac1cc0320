#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -x 2>&1 | grep -E "^E |passed|failed" | head
