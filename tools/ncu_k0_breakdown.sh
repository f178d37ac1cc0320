#!/bin/bash
# ncu L1TEX / LTS throughput breakdown of the row-bin K0 on C2 at x = 100 % (profiles/r02_ncu_k0_l1tex_breakdown.txt)
timeout 600 ncu --metrics breakdown:l1tex__throughput.avg.pct_of_peak_sustained_active,breakdown:lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__t_sectors.sum,l1tex__t_requests.sum,l1tex__m_xbar2l1tex_read_sectors.sum,smsp__inst_executed_pipe_lsu.sum,gpu__time_duration.sum --clock-control none -k regex:binned_row_kernel -c 1 --csv python tools/kernel_sweep.py --inputs c2 --kernels 0 --reps 1 > gpurun_out/s3_ncu_k0_breakdown.csv 2> gpurun_out/s3_ncu_k0.err
tail -3 gpurun_out/s3_ncu_k0.err
wc -l gpurun_out/s3_ncu_k0_breakdown.csv
