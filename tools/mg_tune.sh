#!/bin/bash
# DSA multigrid cycle tuning: PCG iterations and solve time per knob setting
# (RTLR_MG_NU5 / RTLR_MG_NUDG / RTLR_MG_WLEVELS / RTLR_MG_ALPHA, mg.cu).
# Usage (on the GPU box): tools/mg_tune.sh "jobs..." "setting1" "setting2" ...
# where a setting is a space-separated list of VAR=value.
jobs="$1"; shift
for setting in "$@"; do
  echo "=== $setting"
  env $setting timeout 600 python tools/run_configs.py $jobs | python -c '
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    it=d["pcg_iterations"]
    print(d["config"],d["method"],"t=%.3f"%d["time_to_tol_s"],"outer",d["iterations"],"pcg_sum",sum(it),"max",max(it) if it else 0, "conv",d["converged"])'
done
