#!/bin/bash
# One GPU session: tests, bench (+CPU baseline), BFS C3, launch list and one
# full ncu capture of the bench's dominant kernel.  Outputs in gpurun_out/.
set -x
timeout 900 python -m pytest tests/ -m gpu -q -p no:cacheprovider 2>&1 | tail -5
python __graft_entry__.py smoke 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -2 gpurun_out/bench.err
timeout 900 python tools/bfs_bench.py --scale 22 --reps 3 --out gpurun_out/bfs22.json 2>&1 | tail -13
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"binned_row_kernel" -c 1 -o gpurun_out/prof_c2_spmv python tools/kernel_sweep.py --inputs c2 --kernels 0 --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"col_direct_atomic_kernel" -c 1 -o gpurun_out/prof_c2_colatomic python tools/kernel_sweep.py --inputs c2 --kernels 4 --densities 0.5 --reps 1 > /dev/null 2>&1
ls -la gpurun_out | tail -12
