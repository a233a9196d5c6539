#!/bin/bash
# A/B of the batched Galerkin LU: tools/lu_bench built standalone against two
# dense.cu variants (A = $1, B = $2), timed interleaved, plus warm-L2 launch
# lists (ncu --cache-control none) of B.  Output under gpurun_out/.
set -u
A=${1:-tools/_dense_orig.cu}; B=${2:-paper_2603_25233_b200/csrc/dense.cu}
NVCC="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I paper_2603_25233_b200/csrc -I include"
$NVCC tools/lu_bench.cu $A -o /tmp/lu_A 2>/dev/null || exit 1
$NVCC tools/lu_bench.cu $B -o /tmp/lu_B 2>/dev/null || exit 1
mkdir -p gpurun_out
for cfg in ${CFGS:-"600 16" "400 16" "178 8" "128 8"}; do
  for rep in 1 2; do
    echo "A $(timeout 60 /tmp/lu_A $cfg 20)"
    echo "B $(timeout 60 /tmp/lu_B $cfg 20)"
  done
done 2>&1 | tee gpurun_out/lu_ab.txt
for cfg in "600 16" "178 8"; do
  tag=$(echo $cfg | tr ' ' x)
  for v in A B; do
    timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
      --log-file gpurun_out/lu_warm_${v}_$tag.csv /tmp/lu_$v $cfg 3 > /dev/null 2>&1
  done
done
