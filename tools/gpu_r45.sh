#!/bin/bash
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"binned_row_kernel" -c 1 -o gpurun_out/prof_c2_spmv_final python tools/kernel_sweep.py --inputs c2 --kernels 0 --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"col_lb_kernel" -c 1 -o gpurun_out/prof_bfs_push python tools/bfs_bench.py --scale 20 --reps 1 > /dev/null 2>&1
ls gpurun_out/*final* gpurun_out/*push*
