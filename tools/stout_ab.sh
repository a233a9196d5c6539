#!/bin/bash
# A/B of the wide sweep kernel's psi output path (RTLR_SCAN_STOUT = 0 lanes'
# own cells, 1 staged read-back + coalesced stores, 2 TMA stores) at the
# bench workload, interleaved.
for v in ${@:-1 2 1 2}; do
  RTLR_SCAN_STOUT=$v python bench.py --steps 20 --warmup 3 --no-solvers --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('stout $v', round(d['value']/1e9,2), 'G upd/s frac', round(r['frac'],4), 'isolated', round(r['frac_isolated'],4), 'min ms', round(r['kernel_ms_min'],3), d['clocks'])"
done
