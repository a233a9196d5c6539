#!/bin/bash
# ncu counters (time, DRAM bytes, fp64 tensor-pipe and fp64-pipe utilisation) of one
# launch of each low-rank / DSA kernel at C4 sizes; outputs gpurun_out/k_*.csv.
set -x
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size"
timeout 200 ncu --clock-control none $M --csv -k regex:gemm_tn_dmma_nt -c 1 tools/gemm_bench 600 40 1048576 3 > gpurun_out/k_tn40.csv 2>&1
timeout 200 ncu --clock-control none $M --csv -k regex:gemm_tn_dmma_nt -c 1 tools/gemm_bench 600 8 1048576 3 > gpurun_out/k_tn8.csv 2>&1
timeout 200 ncu --clock-control none $M --csv -k regex:gemm_nn_dmma_nt -c 1 tools/gemm_bench 1048576 16 600 3 nn > gpurun_out/k_nn16.csv 2>&1
timeout 200 ncu --clock-control none $M --csv -k regex:gemm_nn_dmma_pipe -c 1 tools/gemm_bench 1048576 128 600 3 nn > gpurun_out/k_nn128.csv 2>&1
timeout 200 ncu --clock-control none $M --csv -k regex:lu_trail -s 5 -c 1 tools/lu_bench 600 372 1 > gpurun_out/k_lutrail.csv 2>&1
timeout 300 ncu --clock-control none $M --csv -k regex:"residual_partials|stream_products_kernel|sweep_wave_kernel" -c 6 python tools/run_configs.py C4:lowrank > gpurun_out/k_misc.csv 2>&1
timeout 300 ncu --clock-control none $M --csv -k regex:"pcg_spmv|dg_smooth|l5_smooth|pcg_rz|pcg_update_mg|pcg_direction|dg_first|dg_restrict|dg_prolong" -s 40 -c 14 python tools/run_configs.py C4:full > gpurun_out/k_dsa.csv 2>&1
