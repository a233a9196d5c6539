#!/bin/bash
# Sweep throughput over a matrix of (grid, CL(n_theta, n_omega_z)) workloads.
# Set SKEW=1 to also time the skewed-wavefront kernel (RTLR_SWEEP=skew).
for g in "256 16 16" "512 32 32" "512 128 32" "2048 16 16" "1024 32 32"; do set -- $g
  for impl in scan ${SKEW:+skew}; do
    sel=""; [ "$impl" = skew ] && sel="RTLR_SWEEP=skew"
    out=$(env $sel timeout 120 python bench.py --no-e2e --no-solvers --no-cpu --steps 10 --grid $1 --n-theta $2 --n-omega-z $3 |
          python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print("%.3e upd/s  frac %.3f  kernel %.3f ms  isolated %.3f ms (frac %.3f)" % (d["value"], d["roofline"]["frac"], d["roofline"]["kernel_ms"], d["roofline"]["kernel_ms_isolated"], d["roofline"]["frac_isolated"]))')
    echo "grid $1^2 CL($2,$3) $impl: $out"
  done
done
