#!/bin/bash
# Small-batch Galerkin LU timings (tools/lu_bench) and per-kernel launch
# lists; run on the GPU box from the repo root.  Output: gpurun_out/lu_*.
set -u
NVCC="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo"
$NVCC -I paper_2603_25233_b200/csrc -I include tools/lu_bench.cu -o tools/lu_bench \
  -Lpaper_2603_25233_b200/lib -lrtlr_cu -Xlinker -rpath=$PWD/paper_2603_25233_b200/lib || exit 1
mkdir -p gpurun_out
for cfg in "600 16" "400 16" "300 16" "220 8" "178 8" "128 8" "96 8" "64 8" "48 8" "600 1024"; do
  timeout 60 tools/lu_bench $cfg 20
done 2>&1 | tee gpurun_out/lu_times.txt
for cfg in "600 16" "178 8"; do
  tag=$(echo $cfg | tr ' ' x)
  timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/lu_launch_$tag.csv tools/lu_bench $cfg 3 > /dev/null 2>&1
done
