#!/bin/bash
# One GPU session (gpurun): parity suite, smoke, short bench; outputs in gpurun_out/.
#   tools/gpu_session.sh [pytest-args...]
set -x
free -g | head -2; lscpu | grep -E "Model name|^CPU\(s\)"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/ -m gpu -q -x -p no:cacheprovider "$@" 2>&1 | tail -15
python __graft_entry__.py smoke 2>&1 | tail -2
