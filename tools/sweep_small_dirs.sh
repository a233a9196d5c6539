for g in "256 32 8" "512 32 8" "256 64 16"; do set -- $g
for env in "X=1" "RTLR_SWEEP_TMA=1" "RTLR_SWEEP_TMA=0"; do
 out=$(env $env timeout 120 python bench.py --no-e2e --no-solvers --no-cpu --steps 20 --grid $1 --n-theta $2 --n-omega-z $3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print("%.1f G upd/s frac %.3f kernel %.3f ms isolated %.3f" % (d["value"]/1e9, d["roofline"]["frac"], d["roofline"]["kernel_ms"], d["roofline"]["frac_isolated"]))')
 echo "grid $1 CL($2,$3) $env: $out"
done; done
