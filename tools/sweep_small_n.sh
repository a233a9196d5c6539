#!/bin/bash
# Sweep time for small direction counts (the low-rank solver's p-direction
# batches): scan vs skew kernels.
for g in 256 1024; do
  for d in "2 4" "4 4" "8 4" "8 8" "16 8" "16 16"; do set -- $d
    for impl in scan skew; do
      sel=""; [ "$impl" = skew ] && sel="RTLR_SWEEP=skew"
      out=$(env $sel timeout 60 python bench.py --no-e2e --no-solvers --no-cpu --steps 20 --grid $g --n-theta $1 --n-omega-z $2 |
            python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print("%.4f ms" % d["ms_per_step"])')
      echo "grid $g^2 dirs $(( $1 * $2 )) $impl: $out"
    done
  done
done
