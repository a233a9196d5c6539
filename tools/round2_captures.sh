#!/bin/bash
# ncu --set full captures of the round's top kernels (one launch each, one
# GPU), exported to raw CSV for profiles/round2/: the bench's C5 sweep, the
# heterogeneous direction-group sweep (C4 FR), the LR residual kernel, the
# projections' DMMA product, the register LU panel.  Run under gpurun.
set -x
O=gpurun_out/r2cap
mkdir -p $O
F="--set full --import-source on --clock-control none"
timeout 300 ncu $F -k regex:sweep_scan_kernel -s 3 -c 1 -o $O/c5_sweep python bench.py --steps 1 --warmup 3 --no-solvers --no-e2e --no-cpu > $O/c5_sweep.log 2>&1
timeout 300 ncu $F -k regex:sweep_het_kernel -s 1 -c 1 -o $O/het_c4 python tools/het_profile.py C4 5 si > $O/het_c4.log 2>&1
timeout 400 ncu $F -k regex:residual_cells -s 200 -c 1 -o $O/residual_c4 python tools/run_configs.py C4:lowrank > $O/residual_c4.log 2>&1
timeout 300 ncu $F -k regex:gemm_tn_dmma_nt -c 1 -o $O/tn40 tools/gemm_bench 600 40 1048576 2 > $O/tn40.log 2>&1
timeout 300 ncu $F -k regex:lu_panel_reg -s 2 -c 1 -o $O/lu_panel tools/lu_bench 600 16 1 > $O/lu_panel.log 2>&1
for r in c5_sweep het_c4 residual_c4 tn40 lu_panel; do
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null
done
ls -la $O
