#!/bin/bash
# Round-1 evidence refresh: bench (+CPU baseline), reference arm, launch list,
# full ncu capture of the dominant kernel, C4 / BFS / PageRank benches.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -2 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"binned_row_kernel" -c 1 -o gpurun_out/prof_c2_spmv python tools/kernel_sweep.py --inputs c2 --kernels 0 --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"col_direct_atomic_kernel" -c 1 -o gpurun_out/prof_c2_colatomic_x10 python tools/kernel_sweep.py --inputs c2 --kernels 4 --densities 0.1 --reps 1 > /dev/null 2>&1
timeout 900 python tools/bfs_bench.py --scale 22 --reps 5 --out gpurun_out/bfs22.json 2>&1 | tail -3
timeout 900 python tools/c4_bench.py --out gpurun_out/c4.json 2>&1 | tail -3
ls -la gpurun_out | tail -12
